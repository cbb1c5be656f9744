export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg1 or host_buffer or streams" > gpurun_out/t17.log 2>&1; echo "exit $?" >> gpurun_out/t17.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench17.log 2>&1; echo "exit $?" >> gpurun_out/bench17.log
