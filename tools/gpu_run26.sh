export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "streams or cfg1 or small_random" > gpurun_out/t26.log 2>&1; echo "exit $?" >> gpurun_out/t26.log
timeout 1200 python tools/bench_configs.py 1 2 5 3 4 > gpurun_out/configs26.jsonl 2> gpurun_out/configs26.err
