export PYTHONPATH=$PWD
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "graph" > gpurun_out/t29.log 2>&1; echo "exit $?" >> gpurun_out/t29.log
