#!/bin/bash
# STFT kernel: phasor tests, then one full ncu capture of the cfg3 STFT launch (after the same command ran clean)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "phasors or mask or odd_strides" > gpurun_out/stft_tests.log 2>&1; echo "exit $?" >> gpurun_out/stft_tests.log
python tools/ncu_target.py > gpurun_out/ncus_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stft_phat" -s 1 -c 1 -f -o gpurun_out/prof_stft python tools/ncu_target.py > gpurun_out/ncus.log 2>&1
echo "exit $?" >> gpurun_out/ncus.log
