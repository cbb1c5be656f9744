export PYTHONPATH=$PWD
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg3 or cfg4_srp or cfg1_full" > gpurun_out/t19.log 2>&1; echo "exit $?" >> gpurun_out/t19.log
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench19.log 2>&1; echo "exit $?" >> gpurun_out/bench19.log
