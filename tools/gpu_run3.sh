export PYTHONPATH=$PWD
timeout 600 python tools/quick_time.py 3 > gpurun_out/time3.log 2>&1; echo "exit $?" >> gpurun_out/time3.log
