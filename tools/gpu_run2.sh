timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s > gpurun_out/t2.log 2>&1; echo "exit $?" >> gpurun_out/t2.log
timeout 600 python tools/quick_time.py 3 > gpurun_out/time3.log 2>&1; echo "exit $?" >> gpurun_out/time3.log
