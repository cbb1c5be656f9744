export PYTHONPATH=$PWD
for pf in 0 1 2 0 1 2; do echo "prefetch=$pf"; SVDPHAT_GEMM_PREFETCH=$pf timeout 300 python tools/quick_time.py 3 10000 srp 2>&1 | grep -E "srp:"; done > gpurun_out/ab.log 2>&1
