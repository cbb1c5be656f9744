#!/bin/bash
# round-2: contract bench (default args), ncu --set full of das_kernel at cfg3, launch list of the bench command
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2_bench.jsonl 2> gpurun_out/r2_bench.err
timeout 200 python tools/ncu_target.py 3 srp > gpurun_out/ncudas_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"das_kernel" -s 1 -c 1 -f \
    -o gpurun_out/r2_das_cfg3 python tools/ncu_target.py 3 srp > gpurun_out/r2_ncudas.log 2>&1
echo "exit $?" >> gpurun_out/r2_ncudas.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "exit $?" >> gpurun_out/r2_ncudas.log
