export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg1 or streams or small_random or mask or topk or host or full_rank" > gpurun_out/t28.log 2>&1; echo "exit $?" >> gpurun_out/t28.log
for pp in 1 0 1; do echo "pair_proj=$pp"; SVDPHAT_PAIR_PROJ=$pp timeout 900 python tools/bench_configs.py 3 4 5 2>/dev/null; done > gpurun_out/ab28.log
