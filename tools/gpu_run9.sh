export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t9.log 2>&1; echo "exit $?" >> gpurun_out/t9.log
for i in 1 2; do timeout 300 python tools/quick_time.py 3 10000 srp 2>&1 | grep -E "srp:"; done > gpurun_out/ab9.log 2>&1
