export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -s -k "small_random or cfg4" > gpurun_out/t13.log 2>&1; echo "exit $?" >> gpurun_out/t13.log
