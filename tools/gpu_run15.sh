export PYTHONPATH=$PWD
SVDPHAT_SRP_TS=1 timeout 600 python tools/power_run.py 150 > gpurun_out/power_ts1.log 2>&1
SVDPHAT_SRP_TS=0 timeout 600 python tools/power_run.py 150 > gpurun_out/power_ts0.log 2>&1
SVDPHAT_SRP_TS=1 timeout 600 python tools/power_run.py 150 > gpurun_out/power_ts1b.log 2>&1
