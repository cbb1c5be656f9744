#!/bin/bash
# ncu --set full of the delay-and-sum SRP kernel at cfg $1 (default 3), report name $2
export PYTHONPATH=$PWD
mkdir -p gpurun_out
C=${1:-3}
N=${2:-das_prof_cfg$C}
timeout 200 python tools/ncu_target.py $C srp > gpurun_out/ncudas_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"das_" -s 2 -c 2 -f \
    -o gpurun_out/$N python tools/ncu_target.py $C srp > gpurun_out/ncudas.log 2>&1
echo "exit $?" >> gpurun_out/ncudas.log
