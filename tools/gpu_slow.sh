export PYTHONPATH=$PWD SVDPHAT_SLOW=1
timeout 2700 python -m pytest tests/test_gpu_parity.py -x -q -s -k "full_size or full_rank" > gpurun_out/slow.log 2>&1; echo "exit $?" >> gpurun_out/slow.log
