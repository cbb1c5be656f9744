export PYTHONPATH=$PWD
timeout 300 python tools/fig2_rank_gain.py gpurun_out/fig2bc_rank_gain.csv > gpurun_out/fig2.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/t22.log 2>&1; echo "exit $?" >> gpurun_out/t22.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench22.log 2>&1; echo "exit $?" >> gpurun_out/bench22.log
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench22_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|stft|finalize|zsplit|topk" --csv --log-file gpurun_out/launches22.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu22.log 2>&1
echo "exit $?" >> gpurun_out/ncu22.log
