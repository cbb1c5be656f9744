#!/bin/bash
# STFT kernel: phasor/mask parity, then one ncu capture of the cfg3 STFT launch and the bench stage time
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "phasors or mask or odd_strides or cfg1 or small_random or streams" > gpurun_out/stft_tests.log 2>&1; echo "exit $?" >> gpurun_out/stft_tests.log
python tools/ncu_target.py 3 svd > gpurun_out/ncus_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"stft_phat" -s 1 -c 1 python tools/ncu_target.py 3 svd > gpurun_out/ncus.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/stft_b3.jsonl 2>gpurun_out/stft_b3.err
