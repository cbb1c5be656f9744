export PYTHONPATH=$PWD
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench16.log 2>&1; echo "exit $?" >> gpurun_out/bench16.log
