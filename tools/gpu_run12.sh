export PYTHONPATH=$PWD
timeout 600 python tools/power_run.py 150 > gpurun_out/power.log 2>&1
SVDPHAT_GEMM_DBG=1 timeout 600 python tools/power_run.py 150 > gpurun_out/power_dbg1.log 2>&1
