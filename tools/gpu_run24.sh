export PYTHONPATH=$PWD
timeout 2400 python tools/bench_configs.py 1 2 3 4 5 > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "exit $?" >> gpurun_out/configs.err
