#!/bin/bash
# DAS kernel bottleneck experiments (dev only): rebuild das.cu with -DDAS_EXP=n into the box's scratch copy of the
# library and time cfg3/cfg4 SRP.  1: epilogue without TMEM loads; 2: loads without squares; 3: no MMA.  Results are
# invalid by construction (timing only).
export PYTHONPATH=$PWD
mkdir -p gpurun_out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude"
cp paper_1811_11785_b200/libsvdphat.so /tmp/lib_prod.so
for e in 0 1 2 3; do
  if [ $e != 0 ]; then
    $NV -DDAS_EXP=$e -c paper_1811_11785_b200/csrc/das.cu -o /tmp/das_exp.o && \
    $NV -shared -o paper_1811_11785_b200/libsvdphat.so build/api.o build/setup.o build/stft_phat.o build/gemm_tc.o \
        build/finalize.o /tmp/das_exp.o -L/usr/local/cuda/lib64 -lcublas -lcusolver -lcudart -Xlinker -rpath,/usr/local/cuda/lib64
  fi
  for c in "3 srp" "4 srp"; do echo "exp $e" >> gpurun_out/exp_stage.log; timeout 300 python tools/stage_time.py $c 10 >> gpurun_out/exp_stage.log 2>&1; done
done
cp /tmp/lib_prod.so paper_1811_11785_b200/libsvdphat.so
timeout 200 python tools/ncu_target.py 3 srp > gpurun_out/ncudas_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"das_kernel" -s 1 -c 1 -f \
    -o gpurun_out/r2_das2_cfg3 python tools/ncu_target.py 3 srp > gpurun_out/r2_ncudas2.log 2>&1
