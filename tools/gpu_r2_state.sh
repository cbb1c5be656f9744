#!/bin/bash
# round-2 state check: full GPU suite, contract bench, per-stage times
export PYTHONPATH=$PWD
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/st_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/st_tests.log 2>&1; echo "exit $?" >> gpurun_out/st_tests.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/st_bench.jsonl 2> gpurun_out/st_bench.err
for c in "3 svd" "3 srp" "3 both" "4 both" "5 both"; do
  timeout 300 python tools/stage_time.py $c 10 >> gpurun_out/st_stage.log 2>&1
done
