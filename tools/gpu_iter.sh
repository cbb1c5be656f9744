#!/bin/bash
# quick GPU iteration: selected parity tests ($1, pytest -k expression), stage times, short bench (no cpu baseline)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
K=${1:-"delay_and_sum or headline or power_maps"}
timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/it_tests.log 2>&1; echo "exit $?" >> gpurun_out/it_tests.log
for c in "3 srp" "3 both" "3 svd" "4 both" "4 srp"; do
  timeout 300 python tools/stage_time.py $c 10 >> gpurun_out/it_stage.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/it_bench.jsonl 2> gpurun_out/it_bench.err
