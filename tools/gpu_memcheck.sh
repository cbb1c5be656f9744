export PYTHONPATH=$PWD
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg1_full or small_random and 2-64 or degenerate" > gpurun_out/memcheck.log 2>&1; echo "exit $?" >> gpurun_out/memcheck.log
