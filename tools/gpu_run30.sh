export PYTHONPATH=$PWD
timeout 1800 python tools/bench_configs.py 1 2 3 4 5 > gpurun_out/configs30.jsonl 2> gpurun_out/configs30.err; echo "exit $?" >> gpurun_out/configs30.err
