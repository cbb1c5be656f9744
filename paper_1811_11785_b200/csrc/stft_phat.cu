// stft_phat.cu — sine-window STFT + PHAT unit phasors (eq. 3 factorised).
//
// One warp per (frame, channel); a CTA of 8 warps takes 8 consecutive frames of one channel so the phasor records
// it emits (layout P16[c][m][F_pad][bpc*2 halves], internal.h) leave as contiguous 8-frame runs.
// Real N-point FFT = complex N/2-point FFT of z[n] = x[2n] + j x[2n+1] (four-step: R-point DFTs in registers,
// twiddle, 32-point DFTs across lanes with shuffles) + the even/odd split post-pass.  Twiddles come from a table
// computed in float64 at plan creation.  Output e_m[k] = X_m[k]/|X_m[k]| (0 where |X| = 0, reading R4), FP16.
#include <cuda_fp16.h>

#include <type_traits>

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

// e^{-j 2 pi k / 32}, k = 0..31 (float64-rounded literals): the twiddles of every in-register DFT (R <= 32)
struct Tw32 {
    float c, s;
};
constexpr Tw32 kTw32[32] = {
    {1.0f, -0.0f},
    {0.9807852804032304f, -0.19509032201612825f},
    {0.9238795325112867f, -0.3826834323650898f},
    {0.8314696123025452f, -0.5555702330196022f},
    {0.7071067811865476f, -0.7071067811865475f},
    {0.5555702330196023f, -0.8314696123025452f},
    {0.38268343236508984f, -0.9238795325112867f},
    {0.19509032201612833f, -0.9807852804032304f},
    {6.123233995736766e-17f, -1.0f},
    {-0.1950903220161282f, -0.9807852804032304f},
    {-0.3826834323650897f, -0.9238795325112867f},
    {-0.555570233019602f, -0.8314696123025455f},
    {-0.7071067811865475f, -0.7071067811865476f},
    {-0.8314696123025453f, -0.5555702330196022f},
    {-0.9238795325112867f, -0.3826834323650899f},
    {-0.9807852804032304f, -0.1950903220161286f},
    {-1.0f, -1.2246467991473532e-16f},
    {-0.9807852804032304f, 0.19509032201612836f},
    {-0.9238795325112868f, 0.38268343236508967f},
    {-0.8314696123025455f, 0.555570233019602f},
    {-0.7071067811865477f, 0.7071067811865475f},
    {-0.5555702330196022f, 0.8314696123025452f},
    {-0.38268343236509034f, 0.9238795325112865f},
    {-0.19509032201612866f, 0.9807852804032303f},
    {-1.8369701987210297e-16f, 1.0f},
    {0.1950903220161283f, 0.9807852804032304f},
    {0.38268343236509f, 0.9238795325112866f},
    {0.5555702330196018f, 0.8314696123025455f},
    {0.7071067811865474f, 0.7071067811865477f},
    {0.8314696123025452f, 0.5555702330196022f},
    {0.9238795325112865f, 0.3826834323650904f},
    {0.9807852804032303f, 0.19509032201612872f},
};

// twiddle multiply by e^{-j 2 pi K / 32} with K known at compile time (trivial twiddles become swaps)
template <int K>
__device__ __forceinline__ float2 tw32(float2 d) {
    constexpr int k = K & 31;
    if constexpr (k == 0) return d;
    if constexpr (k == 8) return make_float2(d.y, -d.x);           // * (-j)
    if constexpr (k == 16) return make_float2(-d.x, -d.y);         // * (-1)
    if constexpr (k == 24) return make_float2(-d.y, d.x);          // * (+j)
    return make_float2(d.x * kTw32[k].c - d.y * kTw32[k].s, d.x * kTw32[k].s + d.y * kTw32[k].c);
}

// In-register radix-2 DIF DFT of R points; output a[i] = DFT[bitrev_R(i)].  Twiddles are compile-time constants.
template <int R, int H>
struct DifStage {
    template <int S0, int T>
    static __device__ __forceinline__ void bfly(float2 (&a)[R]) {
        if constexpr (T < H) {
            const float2 u = a[S0 + T], v = a[S0 + T + H];
            a[S0 + T] = make_float2(u.x + v.x, u.y + v.y);
            a[S0 + T + H] = tw32<T * (32 / (2 * H))>(make_float2(u.x - v.x, u.y - v.y));
            bfly<S0, T + 1>(a);
        }
    }
    template <int S0>
    static __device__ __forceinline__ void blocks(float2 (&a)[R]) {
        if constexpr (S0 < R) {
            bfly<S0, 0>(a);
            blocks<S0 + 2 * H>(a);
        }
    }
    static __device__ __forceinline__ void run(float2 (&a)[R]) {
        if constexpr (H >= 1) {
            blocks<0>(a);
            DifStage<R, H / 2>::run(a);
        }
    }
};
template <int R>
struct DifStage<R, 0> {
    static __device__ __forceinline__ void run(float2 (&)[R]) {}
};

template <int R>
__device__ __forceinline__ void dft_dif(float2 (&a)[R], const float2* __restrict__, int) {
    DifStage<R, R / 2>::run(a);
}

template <int R>
__device__ __forceinline__ int bitrev_r(int i) {
    int lg = 0;
    while ((1 << lg) < R) ++lg;
    return lg == 0 ? 0 : (int)(__brev((unsigned)i) >> (32 - lg));
}

// Complex H = 32R point FFT of z[n'] = x[2n'] + j x[2n'+1] as 32R = R x 32 (pass 1: R-point DFTs over r in
// registers, twiddle, transpose through padded smem; pass 2: the 32-point DFTs over the lane index split as
// R-point in registers x G = 32/R across lanes).  Then the real-FFT post pass, PHAT, FP16 records.
template <int R, int BPC>
__global__ void __launch_bounds__(32 * STFT_WARPS, R >= 32 ? 1 : 5)
    stft_phat_kernel(const float* __restrict__ audio, int64_t cs, int64_t fstride, int F, int Mi, int64_t F_pad,
                     const float* __restrict__ win, const float2* __restrict__ twN, uint8_t* __restrict__ P16,
                     int n_chunks, int k_lo, int k_hi, const uint8_t* __restrict__ mask, int64_t mask_stride) {
    constexpr int bpc = BPC;
    constexpr int N = 64 * R;
    constexpr int H = N / 2;
    constexpr int Kb = H + 1;
    constexpr int G = 32 / R;                     // lanes per 32-point DFT in pass 2 (R <= 32)
    constexpr int SROW = 34;                      // padded row (float2) of the pass-1 transpose S[k1][l]
    constexpr int WBUF = (R * SROW > H + H / 16 + 2) ? R * SROW : H + H / 16 + 2;   // float2 per warp (even)
    extern __shared__ __align__(16) uint8_t sm[];
    float2* wbuf = reinterpret_cast<float2*>(sm) + (threadIdx.x >> 5) * WBUF;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.y;
    const int f0 = blockIdx.x * STFT_WARPS;
    const int f = f0 + warp;
    const bool live = f < F;

    {   // every warp runs the FFT (a dead warp re-reads frame F-1 and discards it), so the shuffles below are not
        // inside divergent code and compile without WARPSYNC/collective fix-ups
        const float* x = audio + (int64_t)m * cs + (int64_t)(live ? f : F - 1) * fstride;
        float2 a[R];
        const float2* win2 = reinterpret_cast<const float2*>(win);
        if ((reinterpret_cast<uintptr_t>(x) & 7) == 0) {             // 8-byte aligned frame: float2 loads
            const float2* x2 = reinterpret_cast<const float2*>(x);
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float2 v = __ldg(x2 + lane + 32 * r), wv = __ldg(win2 + lane + 32 * r);
                a[r] = make_float2(v.x * wv.x, v.y * wv.y);
            }
        } else {
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const int n2 = 2 * (lane + 32 * r);
                const float2 wv = __ldg(win2 + lane + 32 * r);
                a[r] = make_float2(__ldg(x + n2) * wv.x, __ldg(x + n2 + 1) * wv.y);
            }
        }
        // pass 1: DFT over r, twiddle W_H^{lane k1}, transpose S[k1][lane]
        dft_dif<R>(a, twN, N);
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int k1 = bitrev_r<R>(i);
            wbuf[k1 * SROW + lane] = (k1 == 0) ? a[i] : cmul(a[i], __ldg(twN + ((2 * lane * k1) & (N - 1))));
        }
        __syncwarp();
        // pass 2: lane (k1 = lane / G, h = lane % G) takes l = G j + h, j < R
        const int k1 = lane / G, h = lane % G;
#pragma unroll
        for (int j = 0; j < R; ++j) a[j] = wbuf[k1 * SROW + G * j + h];
        __syncwarp();
        dft_dif<R>(a, twN, N);                                  // a[i] = E_h[bitrev(i)]
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int aa = bitrev_r<R>(i);
            if (h * aa) a[i] = cmul(a[i], __ldg(twN + (((h * aa) * (N / 32)) & (N - 1))));   // W_32^{h a}
#pragma unroll
            for (int hh = G / 2; hh >= 1; hh >>= 1) {           // G-point DIF across the lane group
                const float ox = __shfl_xor_sync(0xffffffffu, a[i].x, hh);
                const float oy = __shfl_xor_sync(0xffffffffu, a[i].y, hh);
                if (h & hh) {
                    const int tw = (h & (hh - 1)) * (N / (2 * hh));
                    const float2 d = make_float2(ox - a[i].x, oy - a[i].y);
                    a[i] = tw ? cmul(d, __ldg(twN + tw)) : d;
                } else {
                    a[i] = make_float2(a[i].x + ox, a[i].y + oy);
                }
            }
        }
        // Z[k1 + R (a + R bitrev_G(h))] -> natural order, padded by two float2 per 32 (keeps 16-byte alignment)
        int bg = 0;
        {
            int lg = 0;
            while ((1 << lg) < G) ++lg;
            bg = lg == 0 ? 0 : (int)(__brev((unsigned)h) >> (32 - lg));
        }
#pragma unroll
        for (int i = 0; i < R; ++i) {
            const int k = k1 + R * (bitrev_r<R>(i) + R * bg);
            wbuf[k + 2 * (k >> 5)] = a[i];
        }
        __syncwarp();
    }

    // ---- real-FFT post pass + PHAT: one lane per record (BPC consecutive bins), 2X = (Z_k + conj Z_{H-k}) -
    // j w^k (Z_k - conj Z_{H-k}) (the factor 1/2 is dropped: PHAT is scale-invariant and 2 is exact), one 16- or
    // 8-byte shared store per record.  Bin H (Nyquist) = Re Z_0 - Im Z_0 is the lone bin of the last record.
    {
        constexpr int NREC = H / BPC;                                   // records of bins 0..H-1
        const bool filter = (k_lo > 0) || (k_hi < Kb) || (mask != nullptr);
        constexpr int NIT = (NREC + 31) / 32;
        using Rec = typename std::conditional<BPC == 4, uint4, uint2>::type;
        Rec recs[NIT];
#pragma unroll
        for (int it = 0; it < NIT; ++it) {
            const int c = lane + 32 * it;
            if (c >= NREC) break;
            float re[BPC], im[BPC];
            if (live) {
                const int k0 = c * BPC;
                const float2* zk = wbuf + k0 + 2 * (k0 >> 5);            // BPC consecutive bins, 16-byte aligned
                float2 Zk[BPC], tw[BPC];
                if constexpr (BPC == 4) {
                    const float4 z01 = *reinterpret_cast<const float4*>(zk);
                    const float4 z23 = *reinterpret_cast<const float4*>(zk + 2);
                    Zk[0] = make_float2(z01.x, z01.y); Zk[1] = make_float2(z01.z, z01.w);
                    Zk[2] = make_float2(z23.x, z23.y); Zk[3] = make_float2(z23.z, z23.w);
                    const float4 t01 = __ldg(reinterpret_cast<const float4*>(twN + k0));
                    const float4 t23 = __ldg(reinterpret_cast<const float4*>(twN + k0 + 2));
                    tw[0] = make_float2(t01.x, t01.y); tw[1] = make_float2(t01.z, t01.w);
                    tw[2] = make_float2(t23.x, t23.y); tw[3] = make_float2(t23.z, t23.w);
                } else {
                    const float4 z01 = *reinterpret_cast<const float4*>(zk);
                    Zk[0] = make_float2(z01.x, z01.y); Zk[1] = make_float2(z01.z, z01.w);
                    const float4 t01 = __ldg(reinterpret_cast<const float4*>(twN + k0));
                    tw[0] = make_float2(t01.x, t01.y); tw[1] = make_float2(t01.z, t01.w);
                }
#pragma unroll
                for (int s2 = 0; s2 < BPC; ++s2) {
                    const int km = (H - k0 - s2) & (H - 1);
                    const float2 Zm = wbuf[km + 2 * (km >> 5)];
                    const float Ex = Zk[s2].x + Zm.x, Ey = Zk[s2].y - Zm.y;              // Z_k + conj Z_{H-k}
                    const float Dx = Zk[s2].x - Zm.x, Dy = Zk[s2].y + Zm.y;              // Z_k - conj Z_{H-k}
                    const float tx = tw[s2].x * Dx - tw[s2].y * Dy, ty = tw[s2].x * Dy + tw[s2].y * Dx;
                    const float2 e = phat(make_float2(Ex + ty, Ey - tx));                   // E - j t
                    re[s2] = e.x;
                    im[s2] = e.y;
                }
                if (filter) {            // bins outside [k_lo, k_hi) or masked out contribute nothing (NEXT-3)
#pragma unroll
                    for (int s2 = 0; s2 < BPC; ++s2) {
                        const int k = k0 + s2;
                        if (k < k_lo || k >= k_hi || (mask && !mask[(int64_t)f * mask_stride + k])) re[s2] = im[s2] = 0.f;
                    }
                }
            } else {
#pragma unroll
                for (int s2 = 0; s2 < BPC; ++s2) re[s2] = im[s2] = 0.f;
            }
            if constexpr (BPC == 4) {
                const __half2 h0 = __floats2half2_rn(re[0], re[1]), h1 = __floats2half2_rn(re[2], re[3]);
                const __half2 h2 = __floats2half2_rn(im[0], im[1]), h3 = __floats2half2_rn(im[2], im[3]);
                recs[it] = make_uint4(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1),
                                      *reinterpret_cast<const uint32_t*>(&h2), *reinterpret_cast<const uint32_t*>(&h3));
            } else {
                const __half2 h0 = __floats2half2_rn(re[0], re[1]), h1 = __floats2half2_rn(im[0], im[1]);
                recs[it] = make_uint2(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1));
            }
        }
        // Nyquist value before the warp's Z area is reused for its records
        const float2 z0 = wbuf[0];
        __syncwarp();
        // the warp's records, in chunk order, over the start of its own (now dead) FFT buffer: no separate tile
        Rec* myrec = reinterpret_cast<Rec*>(wbuf);
#pragma unroll
        for (int it = 0; it < NIT; ++it)
            if (lane + 32 * it < NREC) myrec[lane + 32 * it] = recs[it];
        if (lane == 0) {                                                // record NREC: bin H, zero padding after it
            float e = 0.f;
            if (live && H >= k_lo && H < k_hi && (!mask || mask[(int64_t)f * mask_stride + H])) {
                const float v = z0.x - z0.y;
                e = v > 0.f ? 1.f : (v < 0.f ? -1.f : 0.f);
            }
            __half* rec = reinterpret_cast<__half*>(myrec + NREC);
#pragma unroll
            for (int s2 = 0; s2 < 2 * BPC; ++s2) rec[s2] = __float2half_rn(0.f);
            rec[0] = __float2half_rn(e);
        }
    }
    __syncthreads();

    // ---- coalesced write-out: per chunk, 8 frames x unit_bytes contiguous at P16[c][m][f0..f0+7]
    constexpr int unit_bytes = BPC * 4;
    constexpr int vec_per_chunk = STFT_WARPS * unit_bytes / 16;      // 16-byte stores: 8 (bpc 4) or 4 (bpc 2)
    const int total = n_chunks * vec_per_chunk;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
        const int cc = i / vec_per_chunk, wi = i % vec_per_chunk;
        uint4* out = reinterpret_cast<uint4*>(P16 + (((int64_t)cc * Mi + m) * F_pad + f0) * unit_bytes);
        const uint8_t* base = sm + (size_t)cc * unit_bytes;              // record cc of warp w at w*WBUF float2
        if constexpr (BPC == 4) {
            out[wi] = *reinterpret_cast<const uint4*>(base + (size_t)wi * WBUF * sizeof(float2));
        } else {
            const uint2 lo = *reinterpret_cast<const uint2*>(base + (size_t)(2 * wi) * WBUF * sizeof(float2));
            const uint2 hi = *reinterpret_cast<const uint2*>(base + (size_t)(2 * wi + 1) * WBUF * sizeof(float2));
            out[wi] = make_uint4(lo.x, lo.y, hi.x, hi.y);
        }
    }
}

// Small-N path (N = 16, 32): direct DFT per lane (test-sized problems only).
__global__ void stft_phat_small_kernel(const float* __restrict__ audio, int64_t cs, int64_t fstride, int F, int Mi,
                                       int64_t F_pad, int N, const float* __restrict__ win,
                                       const float2* __restrict__ twN, uint8_t* __restrict__ P16, int bpc,
                                       int n_chunks, int k_lo, int k_hi, const uint8_t* __restrict__ mask,
                                       int64_t mask_stride) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m = blockIdx.y;
    const int f = blockIdx.x * STFT_WARPS + warp;
    if (f >= F) return;
    const int Kb = N / 2 + 1;
    const float* x = audio + (int64_t)m * cs + (int64_t)f * fstride;
    __shared__ float2 e_s[STFT_WARPS][32];
    e_s[warp][lane] = make_float2(0.f, 0.f);
    if (lane < Kb && lane >= k_lo && lane < k_hi && (!mask || mask[(int64_t)f * mask_stride + lane])) {
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

template <int R, int BPC>
static cudaError_t launch_rb(const Plan& p, const Band& b, const float* audio, int64_t cs, int64_t fstride, int F,
                             cudaStream_t s) {
    const int H = 32 * R;
    const int wbuf = (R * 34 > H + H / 16 + 2) ? R * 34 : H + H / 16 + 2;
    const size_t smem = STFT_WARPS * wbuf * sizeof(float2);
    dim3 grid((F + STFT_WARPS - 1) / STFT_WARPS, p.M);
    stft_phat_kernel<R, BPC><<<grid, 32 * STFT_WARPS, smem, s>>>(audio, cs, fstride, F, p.L.Mi, p.F_pad, p.d_window,
                                                                 p.d_twN, p.d_P16, p.L.n_chunks, b.k_lo, b.k_hi,
                                                                 b.mask, b.mask_stride);
    return cudaGetLastError();
}

template <int R>
static cudaError_t launch_r(const Plan& p, const Band& b, const float* audio, int64_t cs, int64_t fstride, int F,
                            cudaStream_t s) {
    return p.L.bpc == 4 ? launch_rb<R, 4>(p, b, audio, cs, fstride, F, s)
                        : launch_rb<R, 2>(p, b, audio, cs, fstride, F, s);
}

// per device: called by plan creation (cudaFuncSetAttribute applies to the current device only)
cudaError_t stft_set_attributes() {
    const int mx = 200 * 1024;
    cudaError_t e = cudaSuccess;
#define SVD_STFT_ATTR(R)                                                                                          \
    if ((e = cudaFuncSetAttribute(stft_phat_kernel<R, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx))) return e; \
    if ((e = cudaFuncSetAttribute(stft_phat_kernel<R, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx))) return e;
    SVD_STFT_ATTR(1)
    SVD_STFT_ATTR(2)
    SVD_STFT_ATTR(4)
    SVD_STFT_ATTR(8)
    SVD_STFT_ATTR(16)
    SVD_STFT_ATTR(32)
#undef SVD_STFT_ATTR
    return e;
}

cudaError_t launch_stft_phat(const Plan& p, const Band& b, const float* audio, int64_t cs, int64_t fstride, int F,
                             cudaStream_t s) {
    if (F <= 0) return cudaSuccess;
    switch (p.N) {
        case 64: return launch_r<1>(p, b, audio, cs, fstride, F, s);
        case 128: return launch_r<2>(p, b, audio, cs, fstride, F, s);
        case 256: return launch_r<4>(p, b, audio, cs, fstride, F, s);
        case 512: return launch_r<8>(p, b, audio, cs, fstride, F, s);
        case 1024: return launch_r<16>(p, b, audio, cs, fstride, F, s);
        case 2048: return launch_r<32>(p, b, audio, cs, fstride, F, s);
        default: break;
    }
    dim3 grid((F + STFT_WARPS - 1) / STFT_WARPS, p.M);
    stft_phat_small_kernel<<<grid, 32 * STFT_WARPS, 0, s>>>(audio, cs, fstride, F, p.L.Mi, p.F_pad, p.N, p.d_window,
                                                           p.d_twN, p.d_P16, p.L.bpc, p.L.n_chunks, b.k_lo, b.k_hi,
                                                           b.mask, b.mask_stride);
    return cudaGetLastError();
}

}  // namespace svdphat
