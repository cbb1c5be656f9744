#!/bin/bash
# One GPU session of the r01 evidence: parity tests, the contract bench, the per-config table, an ncu launch list
# of the bench command and a full capture of the hot kernels.  Run with:
#   /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/gpu_suite.sh'
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/tests.log 2>&1; echo "exit $?" >> gpurun_out/tests.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err
timeout 1800 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|stft|finalize|zsplit" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_target.py > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm2_kernel|gemm_kernel|stft_phat|finalize|zsplit" \
    -s 6 -c 7 -o gpurun_out/prof python tools/ncu_target.py > gpurun_out/ncu.log 2>&1
echo "done" >> gpurun_out/ncu.log
