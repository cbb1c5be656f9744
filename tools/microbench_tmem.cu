// microbench_tmem.cu — TMEM read (tcgen05.ld) throughput per SM, with and without an FFMA2 sum-of-squares consumer.
// Decides whether a per-bin |.|^2 epilogue (delay-and-sum-factored SRP) can keep up with the MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb_tmem tools/microbench_tmem.cu && /tmp/mb_tmem
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int X>
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r);

template <>
__device__ __forceinline__ void ld32<32>(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
template <>
__device__ __forceinline__ void ld32<16>(uint32_t taddr, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void ld16x256(uint32_t taddr, uint32_t* r) {  // 16 lanes x 256 bits: 4 regs/thread
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                   "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                   "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                 : "r"(taddr));
}

// mode 0: loads only (xor-fold to keep them live); mode 1: FFMA2 sum of squares of every loaded value; mode 2: 16x256b
template <int MODE>
__global__ void __launch_bounds__(512, 1) tmem_bw(float* out, int iters, long long* cyc) {
    __shared__ uint32_t taddr_s;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&taddr_s))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t base = taddr_s;
    const int nw = blockDim.x >> 5;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const int col0 = (warp >> 2) * 32;  // warps of the same SMSP group read different columns
    float acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = 0.f;
    uint32_t x = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[32];
        const uint32_t col = (uint32_t)((col0 + it * 32 * (nw >> 2)) & 511);
        if (MODE == 2) {
            ld16x256(base + lane_base + col, r);
        } else {
            ld32<32>(base + lane_base + col, r);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 32; i += 2) {
                unsigned long long a, s;
                asm("mov.b64 %0, {%1,%2};" : "=l"(a) : "r"(r[i]), "r"(r[i + 1]));
                asm("mov.b64 %0, {%1,%2};" : "=l"(s) : "f"(acc[i]), "f"(acc[i + 1]));
                asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(s) : "l"(a));
                asm("mov.b64 {%0,%1}, %2;" : "=f"(acc[i]), "=f"(acc[i + 1]) : "l"(s));
            }
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) x ^= r[i];
        }
    }
    long long t1 = clock64();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)x;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}

int main() {
    const int sms = 148, iters = 20000;
    float* out;
    long long* cyc;
    cudaMalloc(&out, sms * 512 * sizeof(float));
    cudaMalloc(&cyc, sms * sizeof(long long));
    long long h[148];
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int mode = 0; mode < 3; ++mode) {
        for (int nw : {4, 8, 16}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) tmem_bw<0><<<sms, nw * 32>>>(out, iters, cyc);
                if (mode == 1) tmem_bw<1><<<sms, nw * 32>>>(out, iters, cyc);
                if (mode == 2) tmem_bw<2><<<sms, nw * 32>>>(out, iters, cyc);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaError_t err = cudaGetLastError();
                if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return 1; }
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
                // bytes per SM: nw warps x iters x (32 lanes x 32 regs x 4 B)
                double bytes = (double)nw * iters * 32 * 32 * 4;
                if (rep == 1)
                    printf("mode %d (%s) warps %2d: %.1f cyc -> %.1f B/clk/SM  (%.3f ms, %.2f TB/s chip)\n", mode,
                           mode == 0 ? "ld 32x32b.x32" : mode == 1 ? "ld + FFMA2 sumsq" : "ld 16x256b.x8", nw,
                           (double)h[0], bytes / (double)h[0], ms, bytes * sms / (ms * 1e-3) / 1e12);
            }
        }
    }
    return 0;
}
