#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for r in 1 2; do timeout 400 python tools/das_ab.py 3 both >> gpurun_out/ab_both.log 2>&1; done
timeout 400 python tools/das_ab.py 4 both >> gpurun_out/ab_both.log 2>&1
python tools/ncu_target.py 3 svd > gpurun_out/ncusvd_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stft|gemm2" -s 2 -c 2 -f \
    -o gpurun_out/r2_prof_stftproj python tools/ncu_target.py 3 svd > gpurun_out/r2_ncusp.log 2>&1
echo "exit $?" >> gpurun_out/r2_ncusp.log
