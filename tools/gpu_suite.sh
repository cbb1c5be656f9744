#!/bin/bash
# Round-end evidence (run: gpurun --timeout 3300 -- "bash tools/gpu_suite.sh"): contract bench (with cpu_baseline), reference arm, per-config table, ncu launch list + captures
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/final_bench.jsonl 2> gpurun_out/final_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.jsonl 2> gpurun_out/final_ref.err
timeout 1500 python tools/bench_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gemm|stft|finalize|zsplit" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_target.py 3 both > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"^(stft_phat|gemm_kernel|gemm2_kernel|gemm2f_kernel|zsplit|finalize)" \
    -s 7 -c 7 -f -o gpurun_out/prof_final python tools/ncu_target.py 3 both > gpurun_out/ncu_final.log 2>&1
echo "exit $?" >> gpurun_out/ncu_final.log
