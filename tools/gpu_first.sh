nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
nproc >> gpurun_out/smi.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "phasors or class or srp_cfg1 or svd_cfg1 or sigma2 or empty" > gpurun_out/t1.log 2>&1
echo "exit $?" >> gpurun_out/t1.log
