// stft_phat.cu — sine-window STFT + PHAT unit phasors (eq. 3 factorised).
//
// One warp per (frame, channel); a CTA of 8 warps takes 8 consecutive frames of one channel so the phasor records
// it emits (layout P16[c][m][F_pad][bpc*2 halves], internal.h) leave as contiguous 8-frame runs.
// Real N-point FFT = complex N/2-point FFT of z[n] = x[2n] + j x[2n+1] (four-step: R-point DFTs in registers,
// twiddle, 32-point DFTs across lanes with shuffles) + the even/odd split post-pass.  Twiddles come from a table
// computed in float64 at plan creation.  Output e_m[k] = X_m[k]/|X_m[k]| (0 where |X| = 0, reading R4), FP16.
#include <cuda_fp16.h>

#include "internal.h"

namespace svdphat {

constexpr int STFT_WARPS = 8;

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

__device__ __forceinline__ int bitrev5(int x) { return (int)(__brev((unsigned)x) >> 27); }

// Unit phasor of X (0 where |X| = 0).
__device__ __forceinline__ float2 phat(float2 X) {
    const float m2 = X.x * X.x + X.y * X.y;
    if (m2 > 0.f) {
        const float r = rsqrtf(m2);
        return make_float2(X.x * r, X.y * r);
    }
    return make_float2(0.f, 0.f);
}

template <int R>  // N = 64 R, N/2 = 32 R complex points
__global__ void __launch_bounds__(32 * STFT_WARPS)
    stft_phat_kernel(const float* __restrict__ audio, int64_t cs, int64_t fstride, int F, int Mi, int64_t F_pad,
                     const float* __restrict__ win, const float2* __restrict__ twN, uint8_t* __restrict__ P16,
                     int bpc, int n_chunks) {
    constexpr int N = 64 * R;
    constexpr int H = N / 2;
    constexpr int Kb = H + 1;
    extern __shared__ __align__(16) uint8_t sm[];
    float2* zbuf = reinterpret_cast<float2*>(sm);                         // [8][H]
    const int unit_bytes = bpc * 4;
    uint8_t* tile = sm + STFT_WARPS * H * sizeof(float2);                 // [n_chunks][8][unit_bytes]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.y;
    const int f0 = blockIdx.x * STFT_WARPS;
    const int f = f0 + warp;
    float2* z = zbuf + warp * H;

    if (f < F) {
        // ---- load + window: z[n'] for n' = lane + 32 r
        const float* x = audio + (int64_t)m * cs + (int64_t)f * fstride;
        float2 a[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int n2 = 2 * (lane + 32 * r);
            a[r] = make_float2(__ldg(x + n2) * __ldg(win + n2), __ldg(x + n2 + 1) * __ldg(win + n2 + 1));
        }
        // ---- R-point DFT over r (radix-2 DIF, output index bit-reversed)
#pragma unroll
        for (int h = R / 2; h >= 1; h >>= 1) {
#pragma unroll
            for (int s0 = 0; s0 < R; s0 += 2 * h) {
#pragma unroll
                for (int t = 0; t < h; ++t) {
                    const float2 u = a[s0 + t], v = a[s0 + t + h];
                    a[s0 + t] = make_float2(u.x + v.x, u.y + v.y);
                    a[s0 + t + h] = cmul(make_float2(u.x - v.x, u.y - v.y), __ldg(twN + t * (N / (2 * h))));
                }
            }
        }
        // ---- twiddle by W_{N/2}^{lane * k1} = e^{-j 2 pi 2 lane k1 / N}, then 32-point DIF across lanes
        int logR = 0;
        while ((1 << logR) < R) ++logR;
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int k1 = (R == 1) ? 0 : (int)(__brev((unsigned)i) >> (32 - logR));
            a[i] = cmul(a[i], __ldg(twN + ((2 * lane * k1) % N)));
#pragma unroll
            for (int h = 16; h >= 1; h >>= 1) {
                const float ox = __shfl_xor_sync(0xffffffffu, a[i].x, h);
                const float oy = __shfl_xor_sync(0xffffffffu, a[i].y, h);
                if (lane & h) {
                    // (other - mine) * w_{2h}^{lane mod h}
                    a[i] = cmul(make_float2(ox - a[i].x, oy - a[i].y), __ldg(twN + (lane & (h - 1)) * (N / (2 * h))));
                } else {
                    a[i] = make_float2(a[i].x + ox, a[i].y + oy);
                }
            }
            z[k1 + R * bitrev5(lane)] = a[i];
        }
    }
    __syncwarp();

    // ---- real-FFT post pass + PHAT + pack records into the CTA tile
    for (int cc = lane; cc < n_chunks; cc += 32) {
        uint32_t w[4] = {0u, 0u, 0u, 0u};
        if (f < F) {
            float re[4], im[4];
            for (int s = 0; s < bpc; ++s) {
                const int k = cc * bpc + s;
                float2 e = make_float2(0.f, 0.f);
                if (k < Kb) {
                    const float2 Zk = z[k & (H - 1)];
                    const float2 Zm = z[(H - k) & (H - 1)];
                    const float2 Zr = make_float2(Zm.x, -Zm.y);                              // conj(Z[H-k])
                    const float2 E = make_float2(0.5f * (Zk.x + Zr.x), 0.5f * (Zk.y + Zr.y));
                    const float2 Dd = make_float2(0.5f * (Zk.x - Zr.x), 0.5f * (Zk.y - Zr.y));
                    const float2 t = cmul(__ldg(twN + (k % N)), Dd);                        // w^k (Z - Zr)/2
                    e = phat(make_float2(E.x + t.y, E.y - t.x));                            // E - j t
                }
                re[s] = e.x;
                im[s] = e.y;
            }
            if (bpc == 4) {
                __half2 h0 = __floats2half2_rn(re[0], re[1]), h1 = __floats2half2_rn(re[2], re[3]);
                __half2 h2 = __floats2half2_rn(im[0], im[1]), h3 = __floats2half2_rn(im[2], im[3]);
                w[0] = *reinterpret_cast<uint32_t*>(&h0);
                w[1] = *reinterpret_cast<uint32_t*>(&h1);
                w[2] = *reinterpret_cast<uint32_t*>(&h2);
                w[3] = *reinterpret_cast<uint32_t*>(&h3);
            } else {
                __half2 h0 = __floats2half2_rn(re[0], re[1]), h1 = __floats2half2_rn(im[0], im[1]);
                w[0] = *reinterpret_cast<uint32_t*>(&h0);
                w[1] = *reinterpret_cast<uint32_t*>(&h1);
            }
        }
        uint32_t* dst = reinterpret_cast<uint32_t*>(tile + ((int64_t)cc * STFT_WARPS + warp) * unit_bytes);
        for (int q = 0; q < bpc; ++q) dst[q] = w[q];
    }
    __syncthreads();

    // ---- coalesced write-out: per chunk, 8 frames x unit_bytes contiguous at P16[c][m][f0..f0+7]
    const int words_per_chunk = STFT_WARPS * unit_bytes / 4;
    const int total = n_chunks * words_per_chunk;
    const uint32_t* t32 = reinterpret_cast<const uint32_t*>(tile);
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
        const int cc = i / words_per_chunk, wi = i % words_per_chunk;
        uint32_t* out = reinterpret_cast<uint32_t*>(P16 + (((int64_t)cc * Mi + m) * F_pad + f0) * unit_bytes);
        out[wi] = t32[i];
    }
}

// Small-N path (N = 16, 32): direct DFT per lane (test-sized problems only).
__global__ void stft_phat_small_kernel(const float* __restrict__ audio, int64_t cs, int64_t fstride, int F, int Mi,
                                       int64_t F_pad, int N, const float* __restrict__ win,
                                       const float2* __restrict__ twN, uint8_t* __restrict__ P16, int bpc,
                                       int n_chunks) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.y;
    const int f = blockIdx.x * STFT_WARPS + warp;
    if (f >= F) return;
    const int Kb = N / 2 + 1;
    const float* x = audio + (int64_t)m * cs + (int64_t)f * fstride;
    __shared__ float2 e_s[STFT_WARPS][32];
    if (lane < Kb) {
        float2 X = make_float2(0.f, 0.f);
        for (int n = 0; n < N; ++n) {
            const float2 w = __ldg(twN + ((lane * n) % N));
            const float v = __ldg(x + n) * __ldg(win + n);
            X.x += v * w.x;
            X.y += v * w.y;
        }
        e_s[warp][lane] = phat(X);
    }
    __syncwarp();
    const int unit_bytes = bpc * 4;
    for (int cc = lane; cc < n_chunks; cc += 32) {
        float re[4] = {0, 0, 0, 0}, im[4] = {0, 0, 0, 0};
        for (int s = 0; s < bpc; ++s) {
            const int k = cc * bpc + s;
            if (k < Kb) {
                re[s] = e_s[warp][k].x;
                im[s] = e_s[warp][k].y;
            }
        }
        uint32_t* out = reinterpret_cast<uint32_t*>(P16 + (((int64_t)cc * Mi + m) * F_pad + f) * unit_bytes);
        if (bpc == 4) {
            __half2 h[4] = {__floats2half2_rn(re[0], re[1]), __floats2half2_rn(re[2], re[3]),
                            __floats2half2_rn(im[0], im[1]), __floats2half2_rn(im[2], im[3])};
            for (int q = 0; q < 4; ++q) out[q] = *reinterpret_cast<uint32_t*>(&h[q]);
        } else {
            __half2 h[2] = {__floats2half2_rn(re[0], re[1]), __floats2half2_rn(im[0], im[1])};
            for (int q = 0; q < 2; ++q) out[q] = *reinterpret_cast<uint32_t*>(&h[q]);
        }
    }
}

template <int R>
static cudaError_t launch_r(const Plan& p, const float* audio, int64_t cs, int64_t fstride, int F, cudaStream_t s) {
    const int H = 32 * R;
    const size_t smem = STFT_WARPS * H * sizeof(float2) + (size_t)p.L.n_chunks * STFT_WARPS * p.L.unit_bytes;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(stft_phat_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             200 * 1024);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    dim3 grid((F + STFT_WARPS - 1) / STFT_WARPS, p.M);
    stft_phat_kernel<R><<<grid, 32 * STFT_WARPS, smem, s>>>(audio, cs, fstride, F, p.L.Mi, p.F_pad, p.d_window,
                                                            p.d_twN, p.d_P16, p.L.bpc, p.L.n_chunks);
    return cudaGetLastError();
}

cudaError_t launch_stft_phat(const Plan& p, const float* audio, int64_t cs, int64_t fstride, int F,
                             cudaStream_t s) {
    if (F <= 0) return cudaSuccess;
    switch (p.N) {
        case 64: return launch_r<1>(p, audio, cs, fstride, F, s);
        case 128: return launch_r<2>(p, audio, cs, fstride, F, s);
        case 256: return launch_r<4>(p, audio, cs, fstride, F, s);
        case 512: return launch_r<8>(p, audio, cs, fstride, F, s);
        case 1024: return launch_r<16>(p, audio, cs, fstride, F, s);
        case 2048: return launch_r<32>(p, audio, cs, fstride, F, s);
        default: break;
    }
    dim3 grid((F + STFT_WARPS - 1) / STFT_WARPS, p.M);
    stft_phat_small_kernel<<<grid, 32 * STFT_WARPS, 0, s>>>(audio, cs, fstride, F, p.L.Mi, p.F_pad, p.N, p.d_window,
                                                           p.d_twN, p.d_P16, p.L.bpc, p.L.n_chunks);
    return cudaGetLastError();
}

}  // namespace svdphat
