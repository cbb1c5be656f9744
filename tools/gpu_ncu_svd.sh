#!/bin/bash
# Full ncu capture of the SVD-PHAT chain on cfg3 (method=svd): STFT, projection, zsplit, search, finalize
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python tools/ncu_target.py 3 svd > gpurun_out/ncusvd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^(stft_phat|gemm_kernel|gemm2_kernel|zsplit|finalize)" -s 5 -c 5 -f -o gpurun_out/prof_svd python tools/ncu_target.py 3 svd > gpurun_out/ncusvd.log 2>&1
echo "exit $?" >> gpurun_out/ncusvd.log
