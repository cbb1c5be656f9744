#!/bin/bash
# A/B of an environment switch on the contract bench: bash tools/gpu_ab.sh VAR
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for v in 0 1 0 1; do
  env $1=$v timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$1_$v.jsonl 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ab_$1_$v.jsonl').read().strip().splitlines()[-1]); print('$1=$v', round(d['value']), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])" >> gpurun_out/ab.log
done
