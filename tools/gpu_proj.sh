#!/bin/bash
# frames-on-M projection: SVD parity subset, projection timing for tile heights, bench
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "real_v or svd or cfg1 or small_random or srp_svd_streams or mask" > gpurun_out/proj_tests.log 2>&1; echo "exit $?" >> gpurun_out/proj_tests.log
for nt in 0 128 160 192 224 256; do
  SVDPHAT_PROJ_NT=$nt timeout 300 python tools/quick_time.py 3 10000 svd > gpurun_out/proj_nt$nt.log 2>&1
  SVDPHAT_SVD_FOLD=0 SVDPHAT_PROJ_NT=$nt timeout 300 python tools/quick_time.py 3 10000 svd > gpurun_out/proj_c_nt$nt.log 2>&1
done
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/check_b3.jsonl 2>gpurun_out/check_b3.err
