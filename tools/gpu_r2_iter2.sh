#!/bin/bash
# kernel iteration: stage timings, parity tests (without the headline module), ncu --set full of $1 (kernel regex)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
rm -f gpurun_out/it_stage.log
for c in "3 svd" "3 both" "4 svd" "4 both" "5 svd" "5 both" "2 svd" "1 svd"; do
  timeout 300 python tools/stage_time.py $c 20 >> gpurun_out/it_stage.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/it_tests.log 2>&1; echo "exit $?" >> gpurun_out/it_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${1:-gemm2p}" \
    -s 1 -c 1 -f -o gpurun_out/it_prof python tools/ncu_target.py 3 ${2:-svd} > gpurun_out/it_ncu.log 2>&1
echo "exit $?" >> gpurun_out/it_ncu.log
