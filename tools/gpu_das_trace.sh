#!/bin/bash
# dev: rebuild das.cu with -DDAS_TRACE into the box's scratch library copy and print the folded kernel's latency trace
export PYTHONPATH=$PWD
mkdir -p gpurun_out
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude"
$NV -DDAS_TRACE -c paper_1811_11785_b200/csrc/das.cu -o /tmp/das_trace.o && \
$NV -shared -o paper_1811_11785_b200/libsvdphat.so build/api.o build/setup.o build/stft_phat.o build/gemm_tc.o \
    build/finalize.o /tmp/das_trace.o -L/usr/local/cuda/lib64 -lcublas -lcusolver -lcudart -Xlinker -rpath,/usr/local/cuda/lib64
for c in 3 4; do timeout 300 python tools/das_trace.py $c >> gpurun_out/das_trace.log 2>&1; done
