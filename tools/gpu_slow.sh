#!/bin/bash
# Full-size SVD-PHAT parity against the oracle's own float64 SVD (cfg3, cfg4; minutes of host SVD) + per-config table
export PYTHONPATH=$PWD SVDPHAT_SLOW=1
mkdir -p gpurun_out
timeout 2700 python -m pytest tests/test_gpu_parity.py -x -q -s -k "full_size or full_rank" > gpurun_out/slow.log 2>&1; echo "exit $?" >> gpurun_out/slow.log
timeout 1500 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
