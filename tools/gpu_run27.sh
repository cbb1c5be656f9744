export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t27.log 2>&1; echo "exit $?" >> gpurun_out/t27.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench27.log 2>&1; echo "exit $?" >> gpurun_out/bench27.log
