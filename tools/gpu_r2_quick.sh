#!/bin/bash
# quick GPU iteration: parity tests without the headline module, then stage timings
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2_quick_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2_quick_tests.log
for c in "3 svd" "3 srp" "3 both" "4 svd" "5 both" "2 both"; do
  timeout 300 python tools/stage_time.py $c 10 >> gpurun_out/r2_stage.log 2>&1
done
