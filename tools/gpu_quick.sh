#!/bin/bash
# quick dev loop: SVD parity subset + contract bench
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "svd or cfg1 or srp_svd_streams or small_random or topk or mask" > gpurun_out/quick_tests.log 2>&1; echo "exit $?" >> gpurun_out/quick_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/quick_b3.jsonl 2>gpurun_out/quick_b3.err
