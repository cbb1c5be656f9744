#!/bin/bash
# antipodal folding: fold tests, full GPU parity suite, contract bench
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fold" > gpurun_out/fold_tests.log 2>&1; echo "exit $?" >> gpurun_out/fold_tests.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/check_tests.log 2>&1; echo "exit $?" >> gpurun_out/check_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/check_b3.jsonl 2>gpurun_out/check_b3.err
