#!/bin/bash
# search-epilogue iteration: stage timings, parity tests (without the headline module), ncu --set full of the search
export PYTHONPATH=$PWD
mkdir -p gpurun_out
rm -f gpurun_out/r2s_stage.log
for c in "3 svd" "3 both" "4 svd" "5 svd" "2 svd"; do
  timeout 300 python tools/stage_time.py $c 20 >> gpurun_out/r2s_stage.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/r2s_tests.log 2>&1; echo "exit $?" >> gpurun_out/r2s_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|stft" \
    -s 2 -c 2 -f -o gpurun_out/r2s_prof_search python tools/ncu_target.py 3 svd > gpurun_out/r2s_ncu.log 2>&1
echo "exit $?" >> gpurun_out/r2s_ncu.log
