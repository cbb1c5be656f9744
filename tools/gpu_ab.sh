#!/bin/bash
# A/B of an environment switch: bash tools/gpu_ab.sh VAR "v1 v2 ..." [cfg] [methods]
# (SVD/SRP-only timings via tools/quick_time.py, two rounds)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for r in 1 2; do
  for v in $2; do
    env $1=$v timeout 300 python tools/quick_time.py ${3:-3} 10000 ${4:-svd} 2>&1 | grep -E "^(svd|srp):" | sed "s/^/$1=$v /" >> gpurun_out/ab.log
  done
done
