#!/bin/bash
# Round-2 evidence (gpurun --timeout 3300 -- "bash tools/gpu_suite_r2.sh"): GPU test suite, contract bench (with
# cpu_baseline + parity), reference arm, per-config table, ncu launch list of the bench command, ncu --set full of the
# dominant kernel (cfg3 SRP GEMM) and of the delay-and-sum kernel at cfg4.
export PYTHONPATH=$PWD
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/s_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s_smoke.log 2>&1; echo "exit $?" >> gpurun_out/s_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/s_tests.log 2>&1; echo "exit $?" >> gpurun_out/s_tests.log
timeout 900 python bench.py > gpurun_out/s_bench.jsonl 2> gpurun_out/s_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s_ref.jsonl 2> gpurun_out/s_ref.err
timeout 1200 python tools/bench_configs.py > gpurun_out/s_configs.jsonl 2> gpurun_out/s_configs.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/s_ncu_bench.log 2>&1
echo "exit $?" >> gpurun_out/s_ncu_bench.log
python tools/ncu_target.py 3 both > gpurun_out/s_ncu_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm2_kernel" -s 1 -c 1 -f \
    -o gpurun_out/s_prof_srpgemm python tools/ncu_target.py 3 both > gpurun_out/s_ncu_gemm.log 2>&1
echo "exit $?" >> gpurun_out/s_ncu_gemm.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"das_fold_kernel" -s 1 -c 1 -f \
    -o gpurun_out/s_prof_das4 python tools/ncu_target.py 4 srp > gpurun_out/s_ncu_das.log 2>&1
echo "exit $?" >> gpurun_out/s_ncu_das.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"stft|gemm2p|gemm_kernel|zsplit|rescore|finalize" \
    -s 6 -c 6 -f -o gpurun_out/s_prof_svd python tools/ncu_target.py 3 svd > gpurun_out/s_ncu_svd.log 2>&1
echo "exit $?" >> gpurun_out/s_ncu_svd.log
