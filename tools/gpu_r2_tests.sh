#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
nproc > gpurun_out/r2_host.txt; lscpu | head -20 >> gpurun_out/r2_host.txt; free -g >> gpurun_out/r2_host.txt
timeout 2400 python -m pytest tests -m gpu -x -q -s --durations=40 > gpurun_out/r2_gpu1.log 2>&1; echo "exit $?" >> gpurun_out/r2_gpu1.log
