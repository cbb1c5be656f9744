export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t8.log 2>&1; echo "exit $?" >> gpurun_out/t8.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench8.log 2>&1; echo "exit $?" >> gpurun_out/bench8.log
python tools/ncu_target.py > gpurun_out/ncu_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"gemm2_kernel|stft_phat|finalize" -s 3 -c 3 -o gpurun_out/prof_pair2 python tools/ncu_target.py > gpurun_out/ncu4.log 2>&1
echo "exit $?" >> gpurun_out/ncu4.log
