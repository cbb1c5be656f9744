#!/bin/bash
# ncu --set full of the delay-and-sum SRP kernel (das_kernel) at cfg3 (and cfg4 with argument 4)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
C=${1:-3}
timeout 200 python tools/ncu_target.py $C srp > gpurun_out/ncudas_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"das_kernel" -s 1 -c 1 -f \
    -o gpurun_out/das_prof_cfg$C python tools/ncu_target.py $C srp > gpurun_out/ncudas.log 2>&1
echo "exit $?" >> gpurun_out/ncudas.log
