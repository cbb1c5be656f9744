#!/bin/bash
# STFT kernel check: phasor parity tests, then the STFT stage time on cfg3/cfg4 (bench stage events)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "phasors or mask or small_random or odd_strides or cfg1" > gpurun_out/stft_tests.log 2>&1; echo "exit $?" >> gpurun_out/stft_tests.log
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/stft_b3.jsonl 2>gpurun_out/stft_b3.err
