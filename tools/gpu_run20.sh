export PYTHONPATH=$PWD
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -s -k "topk" > gpurun_out/t20.log 2>&1; echo "exit $?" >> gpurun_out/t20.log
