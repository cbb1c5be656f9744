export PYTHONPATH=$PWD
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg1_full or streams" > gpurun_out/t31.log 2>&1; echo "exit $?" >> gpurun_out/t31.log
for i in 1 2; do timeout 300 python tools/power_run.py 100 2>&1 | head -1; done > gpurun_out/ab31.log
