#!/bin/bash
# ncu full capture of the SVD chain's tensor kernels (projection, search) on cfg3, method=svd
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python tools/ncu_target.py 3 svd > gpurun_out/ncusvd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm2f_kernel|gemm_kernel" -s 2 -c 2 -f -o gpurun_out/prof_svd2 python tools/ncu_target.py 3 svd > gpurun_out/ncusvd2.log 2>&1
echo "exit $?" >> gpurun_out/ncusvd2.log
