#!/bin/bash
# frames-per-tile sweep of the (folded) SRP pair GEMM + ncu of the folded kernel
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for bn in 256 224 192 160; do
  SVDPHAT_PAIR_BN=$bn timeout 300 python tools/quick_time.py 3 10000 srp > gpurun_out/bn_$bn.log 2>&1
done
python tools/ncu_target.py 3 srp > gpurun_out/ncufold_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm2_kernel" -s 1 -c 1 -f -o gpurun_out/prof_fold python tools/ncu_target.py 3 srp > gpurun_out/ncufold.log 2>&1
echo "exit $?" >> gpurun_out/ncufold.log
