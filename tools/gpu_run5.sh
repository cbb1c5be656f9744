export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t5.log 2>&1; echo "exit $?" >> gpurun_out/t5.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.log 2>&1; echo "exit $?" >> gpurun_out/bench5.log
