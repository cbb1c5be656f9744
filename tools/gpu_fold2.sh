#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fold or cfg1 or srp_svd_streams or topk" > gpurun_out/fold_tests.log 2>&1; echo "exit $?" >> gpurun_out/fold_tests.log
timeout 300 python tools/quick_time.py 3 10000 srp > gpurun_out/bn_256.log 2>&1
python tools/ncu_target.py 3 srp > gpurun_out/ncufold_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm2_kernel" -s 1 -c 1 -f -o gpurun_out/prof_fold python tools/ncu_target.py 3 srp > gpurun_out/ncufold.log 2>&1
echo "exit $?" >> gpurun_out/ncufold.log
