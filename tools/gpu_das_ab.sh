#!/bin/bash
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for c in 3 4; do timeout 400 python tools/das_ab.py $c >> gpurun_out/das_ab.log 2>&1; done
