export PYTHONPATH=$PWD
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench1.log 2>&1; echo "exit $?" >> gpurun_out/bench1.log
