#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fold or cfg1 or srp_svd_streams or topk or small_random" > gpurun_out/fold_tests.log 2>&1; echo "exit $?" >> gpurun_out/fold_tests.log
timeout 300 python tools/quick_time.py 3 10000 srp > gpurun_out/fold1.log 2>&1
SVDPHAT_FOLD=0 timeout 300 python tools/quick_time.py 3 10000 srp > gpurun_out/fold0.log 2>&1
python tools/ncu_target.py 3 srp > gpurun_out/ncufold_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"gemm2_kernel" -s 1 -c 1 python tools/ncu_target.py 3 srp > gpurun_out/ncufold_m.log 2>&1
SVDPHAT_FOLD=0 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"gemm2_kernel" -s 1 -c 1 python tools/ncu_target.py 3 srp > gpurun_out/ncufold0_m.log 2>&1
