export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "last_fold_row" > gpurun_out/lf_tests.log 2>&1; echo "exit $?" >> gpurun_out/lf_tests.log
python tools/ncu_target.py 3 svd > gpurun_out/ncusvd_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm2f_kernel|gemm_kernel" -s 2 -c 2 -f -o gpurun_out/prof_svd2 python tools/ncu_target.py 3 svd > gpurun_out/ncusvd2.log 2>&1
echo "exit $?" >> gpurun_out/ncusvd2.log
