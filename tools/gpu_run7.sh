export PYTHONPATH=$PWD
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg1 or phasors or streams" > gpurun_out/t7.log 2>&1; echo "exit $?" >> gpurun_out/t7.log
if grep -q "exit 0" gpurun_out/t7.log; then
for ps in 1 0 1; do echo "pair=$ps"; SVDPHAT_PAIR_SRP=$ps timeout 300 python tools/quick_time.py 3 10000 srp 2>&1 | grep -E "srp:"; done > gpurun_out/ab7.log 2>&1
fi
