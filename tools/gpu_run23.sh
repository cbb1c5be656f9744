export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "streaming or host_buffer" > gpurun_out/t23.log 2>&1; echo "exit $?" >> gpurun_out/t23.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench23.log 2>&1; echo "exit $?" >> gpurun_out/bench23.log
