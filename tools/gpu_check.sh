#!/bin/bash
# Full GPU parity suite + SVD-only timing + contract bench (dev loop)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/check_tests.log 2>&1; echo "exit $?" >> gpurun_out/check_tests.log
timeout 300 python tools/quick_time.py 3 10000 svd,srp > gpurun_out/quick3.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/check_b3.jsonl 2>gpurun_out/check_b3.err
