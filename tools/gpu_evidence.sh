#!/bin/bash
# r01 evidence refresh: per-config table, ncu launch list of the bench command, full capture of the SRP GEMM
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1500 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|stft|finalize|zsplit" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_target.py 3 srp > gpurun_out/ncufold_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm2_kernel" -s 1 -c 1 -f -o gpurun_out/prof_fold python tools/ncu_target.py 3 srp > gpurun_out/ncufold.log 2>&1
echo "exit $?" >> gpurun_out/ncufold.log
