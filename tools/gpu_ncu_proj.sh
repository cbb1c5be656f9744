#!/bin/bash
# ncu full capture of the SVD projection kernel (cfg3, method=svd)
export PYTHONPATH=$PWD
mkdir -p gpurun_out
python tools/ncu_target.py 3 svd > gpurun_out/ncuproj_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm2f?_kernel" -s 1 -c 1 -f -o gpurun_out/prof_proj python tools/ncu_target.py 3 svd > gpurun_out/ncuproj.log 2>&1
echo "exit $?" >> gpurun_out/ncuproj.log
