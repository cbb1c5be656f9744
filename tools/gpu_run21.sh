export PYTHONPATH=$PWD
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -s -k "mask or band or cfg1 or streams or topk" > gpurun_out/t21.log 2>&1; echo "exit $?" >> gpurun_out/t21.log
