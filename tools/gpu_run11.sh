export PYTHONPATH=$PWD
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg1 or streams or cfg3" > gpurun_out/t11.log 2>&1; echo "exit $?" >> gpurun_out/t11.log
for cfg in "0 0" "1 0" "0 0" "0 224"; do set -- $cfg; echo "dbg=$1 bn=$2"; SVDPHAT_GEMM_DBG=$1 SVDPHAT_PAIR_BN=$2 timeout 300 python tools/quick_time.py 3 10000 srp 2>&1 | grep -E "srp:"; done > gpurun_out/ab11.log 2>&1
