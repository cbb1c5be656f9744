export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t25.log 2>&1; echo "exit $?" >> gpurun_out/t25.log
timeout 1200 python tools/bench_configs.py 1 2 5 3 > gpurun_out/configs25.jsonl 2> gpurun_out/configs25.err
