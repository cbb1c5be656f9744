export PYTHONPATH=$PWD
python tools/ncu_target.py > gpurun_out/ncu_plain5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm3_kernel" -s 1 -c 1 -o gpurun_out/prof_ts python tools/ncu_target.py > gpurun_out/ncu5.log 2>&1
echo "exit $?" >> gpurun_out/ncu5.log
