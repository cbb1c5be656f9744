#!/bin/bash
# round 2: RMSE parity test + Fig. 2a CSV (NEXT-2), ncu --set full of the SVD chain at cfg3
export PYTHONPATH=$PWD
mkdir -p gpurun_out profiles/r02
timeout 900 python -m pytest tests/test_gpu_rmse.py -x -q > gpurun_out/rmse_test.log 2>&1; echo "exit $?" >> gpurun_out/rmse_test.log
timeout 900 python tools/fig2a_rmse.py 300 32 gpurun_out/fig2a_delta_rmse.csv > gpurun_out/fig2a.log 2>&1
python tools/ncu_target.py 3 svd > gpurun_out/ncusvd_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stft|gemm2|gemm_kernel|zsplit|rescore|finalize" \
    -s 8 -c 8 -f -o gpurun_out/r2_prof_svd python tools/ncu_target.py 3 svd > gpurun_out/r2_ncusvd.log 2>&1
echo "exit $?" >> gpurun_out/r2_ncusvd.log
