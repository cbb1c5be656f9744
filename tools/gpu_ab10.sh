export PYTHONPATH=$PWD
for cfg in "0 256" "0 224" "1 256" "2 256" "3 256" "0 256"; do set -- $cfg; echo "dbg=$1 bn=$2"; SVDPHAT_GEMM_DBG=$1 SVDPHAT_PAIR_BN=$2 timeout 300 python tools/quick_time.py 3 10000 srp 2>&1 | grep -E "srp:"; done > gpurun_out/ab10.log 2>&1
