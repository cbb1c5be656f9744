#!/bin/bash
# Round-2 iteration: f32x2 STFT parity + stage times, L2 -> SM bandwidth microbenchmark, ncu of the SVD chain (cfg3).
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "phasors or cfg1 or odd_strides or tf_mask or empty" \
    > gpurun_out/i1_tests.log 2>&1; echo "exit $?" >> gpurun_out/i1_tests.log
for m in svd srp both; do timeout 300 python tools/stage_time.py 3 $m 20 >> gpurun_out/i1_stage.log 2>&1; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_l2 tools/microbench_l2.cu && timeout 120 /tmp/mb_l2 > gpurun_out/i1_l2.log 2>&1
bash tools/gpu_r2_ncu_svd.sh
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/i1_bench_nocpu.jsonl 2> gpurun_out/i1_bench_nocpu.err
