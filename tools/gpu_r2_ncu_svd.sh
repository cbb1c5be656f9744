#!/bin/bash
# ncu --set full of the SVD chain kernels on cfg3 (method=svd): STFT, part projection, zsplit, search, rescore, finalize
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python tools/ncu_target.py 3 svd > gpurun_out/ncusvd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"stft|gemm2p|gemm_kernel|zsplit|rescore|finalize" \
    -s 7 -c 7 -f -o gpurun_out/r2_prof_svd python tools/ncu_target.py 3 svd > gpurun_out/r2_ncusvd.log 2>&1
echo "exit $?" >> gpurun_out/r2_ncusvd.log
