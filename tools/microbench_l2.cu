// microbench_l2.cu — L2 -> SM bandwidth with bulk async copies (cp.async.bulk, the TMA 1-D path) from an L2-resident
// buffer: what a GEMM operand stream fed from L2 can sustain per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_l2 tools/microbench_l2.cu && /tmp/mb_l2
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CHUNK, int STAGES>
__global__ void __launch_bounds__(32) l2_read(const uint8_t* buf, size_t buf_bytes, int iters, long long* cyc) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[STAGES];
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    const size_t nchunks = buf_bytes / CHUNK;
    size_t c = ((size_t)blockIdx.x * 7919) % nchunks;
    long long t0 = clock64();
    for (int it = 0; it < iters + STAGES; ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) {  // wait for the copy issued STAGES iterations ago
            const uint32_t par = ((it / STAGES) - 1) & 1;
            asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                             smem_u32(&bar[s])), "r"(par) : "memory");
        }
        if (it < iters) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(CHUNK)
                         : "memory");
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(sm + s * CHUNK)), "l"(buf + c * CHUNK), "r"(CHUNK), "r"(smem_u32(&bar[s]))
                         : "memory");
            c = (c + 1) % nchunks;
        }
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    uint8_t* buf;
    long long* cyc;
    const size_t MB = 1 << 20;
    cudaMalloc(&buf, 256 * MB);
    cudaMemset(buf, 1, 256 * MB);
    cudaMalloc(&cyc, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    constexpr int CH = 16384, ST = 8;
    cudaFuncSetAttribute(l2_read<CH, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST);
    for (size_t set_mb : {16, 48, 96, 256}) {
        for (int ctas_per_sm : {1, 2}) {
            const int grid = 148 * ctas_per_sm, iters = 4000;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                l2_read<CH, ST><<<grid, 32, CH * ST>>>(buf, set_mb * MB, iters, cyc);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                if (cudaGetLastError() != cudaSuccess) { printf("launch failed\n"); return 1; }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                long long h;
                cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
                const double bytes = (double)grid * iters * CH;
                if (rep == 1)
                    printf("working set %4zu MB, %d CTA/SM: %.2f TB/s chip, %.1f B/clk/SM (cta0 %lld cyc)\n", set_mb,
                           ctas_per_sm, bytes / (ms * 1e-3) / 1e12, bytes / 148 / (double)h * ctas_per_sm / ctas_per_sm,
                           h);
            }
        }
    }
    return 0;
}
