export PYTHONPATH=$PWD
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg1 or phasors" > gpurun_out/t14a.log 2>&1; echo "exit $?" >> gpurun_out/t14a.log
if grep -q "exit 0" gpurun_out/t14a.log; then
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t14.log 2>&1; echo "exit $?" >> gpurun_out/t14.log
for ts in 1 0 1 0; do echo "ts=$ts"; SVDPHAT_SRP_TS=$ts timeout 300 python tools/quick_time.py 3 10000 srp 2>&1 | grep -E "srp:"; done > gpurun_out/ab14.log 2>&1
fi
