// finalize.cu — Z normalisation/split for the search GEMM, and the per-frame finalize.
//
// zsplit  : Zhat = Z / ||Z|| (Alg. 1 online step 2), written in FP16 for the search GEMM and in FP32
//           for the exact rescore of its candidates (rescore_kernel).
// finalize: decodes the packed argmax key (class index -> lowest point index of the class), and computes the score
//           Y_q = Re{W_q . X} of eq. 5 for the chosen q (Alg. 1 online step 4) in the
//           exact delay-and-sum form  Y_q = 1/2 sum_k ( |sum_m e_m[k] e^{+j 2 pi k delta_qm / N}|^2 - n_k ),
//           which is eq. 5 rewritten with tau_qij = delta_qi - delta_qj (eqs. 1-2); n_k = #non-zero phasors at k.
//           A frame whose X vector is identically 0 (no bin with two live channels) gets q = -1, score 0 (R4).
#include <cuda_fp16.h>

#include "internal.h"

namespace svdphat {

// sin/cos(pi t): reduce t to [-1, 1] (one period), then the fast hardware sin/cos (|error| < 5e-7 there)
__device__ __forceinline__ void sincospi_fast(float t, float* s, float* c) {
    const float y = t - 2.0f * rintf(0.5f * t);
    __sincosf(3.14159265358979f * y, s, c);
}

__device__ __forceinline__ uint32_t f2o_dev(float v) {   // order-preserving float -> uint32 (as ptx.cuh f2o)
    const uint32_t b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

// Z = sum of the nsplit partial projections (fixed order: deterministic), then Zhat = Z / ||Z||.  One 128-thread CTA
// per frame with the frame's Z row (Z_r | Z_i, zh columns each) held in registers (NV float4 per thread, ldz <= 512 NV):
// every partial is read once with 16-byte loads, all NV x nsplit loads of a thread in flight together.  Columns >= D of
// each half are zero (padding V rows) except the SRP tail rows below; Zhat's first D_h columns of each half are written
// as FP16 Zs16 [Re | Im] (search operand) and FP32 Zn32 (rescore).
constexpr int ZS_THREADS = 128;
// Tail (fold + real V, Plan::tail_n): SRP fold row tail_r0 + r rides in V rows D + 2r (its Re W values) and D + 2r + 1
// (its Im W values), so a = Re W . x_r is column D + 2r of Z_r and b = Im W . x_i is column D + 2r + 1 of Z_i.  Columns
// >= D always leave Z (zeroed before the norm); for a BOTH call (keys != nullptr) the tail rows are scored
// Y_c = a - b, Y_c' = a + b into the SRP keys.
struct ZTail {
    int n, D, r0, fold_rows;
    const int* fold_cls;
    unsigned long long* keys;
};

template <int NV>
__global__ void __launch_bounds__(ZS_THREADS)
    zsplit_cta_kernel(float* __restrict__ Z, int64_t F_pad, int zh, int nsplit, __half* __restrict__ Zs,
                      float* __restrict__ Zn, int Dh, int* __restrict__ zflag, ZTail tail) {
    __shared__ float s_ss[ZS_THREADS / 32];
    __shared__ float s_tail[2][8];
    const int f = blockIdx.x;
    const int t = threadIdx.x;
    const int ldz = 2 * zh, n4 = ldz >> 2;
    float4* z = reinterpret_cast<float4*>(Z + (int64_t)f * ldz);
    const int64_t split4 = F_pad * (int64_t)n4;
    float4 v[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int i = t + ZS_THREADS * j;
        v[j] = i < n4 ? z[i] : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int sp = 1; sp < nsplit; ++sp) {
        float4 w[NV];
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            const int i = t + ZS_THREADS * j;
            w[j] = i < n4 ? z[sp * split4 + i] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            v[j].x += w[j].x;
            v[j].y += w[j].y;
            v[j].z += w[j].z;
            v[j].w += w[j].w;
        }
    }
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int i = t + ZS_THREADS * j;
        if (i < n4) {
            float* e = reinterpret_cast<float*>(&v[j]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int col = 4 * i + q;
                const int part = col < zh ? 0 : 1, c = col - part * zh;
                if (c >= tail.D) {
                    const int r = (c - tail.D - part) >> 1;         // Re rows D + 2r in Z_r, Im rows D + 2r + 1 in Z_i
                    if (r < tail.n && c == tail.D + 2 * r + part) s_tail[part][r] = e[q];
                    e[q] = 0.f;
                }
            }
        }
    }
    float ss = 0.f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int i = t + ZS_THREADS * j;
        if (i < n4) {
            if (nsplit > 1) z[i] = v[j];                  // the summed Z stays readable (debug dump)
            ss += v[j].x * v[j].x + v[j].y * v[j].y + v[j].z * v[j].z + v[j].w * v[j].w;
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((t & 31) == 0) s_ss[t >> 5] = ss;
    __syncthreads();
    ss = 0.f;
#pragma unroll
    for (int w = 0; w < ZS_THREADS / 32; ++w) ss += s_ss[w];   // same order in every thread
    const float inv = ss > 0.f ? rsqrtf(ss) : 0.f;
    if (t == 0) {
        zflag[f] = ss > 0.f ? 0 : 1;
        unsigned long long best = 0ull;
        for (int r = 0; tail.keys && r < tail.n; ++r) {
            const float a = s_tail[0][r], b = s_tail[1][r];
            const int cm = tail.fold_cls[tail.r0 + r], cp = tail.fold_cls[tail.fold_rows + tail.r0 + r];
            const float ym = a - b, yp = a + b;
            const unsigned long long km = ym == ym ? ((unsigned long long)f2o_dev(ym) << 32) | (0xFFFFFFFFull - cm) : 0ull;
            const unsigned long long kp =
                (cp >= 0 && yp == yp) ? ((unsigned long long)f2o_dev(yp) << 32) | (0xFFFFFFFFull - cp) : 0ull;
            best = km > best ? km : best;
            best = kp > best ? kp : best;
        }
        if (best) atomicMax(&tail.keys[f], best);
    }
    uint2* out = reinterpret_cast<uint2*>(Zs + (int64_t)f * 2 * Dh);   // 4 halves per store
    float4* out32 = reinterpret_cast<float4*>(Zn + (int64_t)f * 2 * Dh);
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const int i = t + ZS_THREADS * j;
        const int col = 4 * i;
        const int part = col < zh ? 0 : 1, c = col - part * zh;
        if (i < n4 && c < Dh) {
            const float4 a = make_float4(v[j].x * inv, v[j].y * inv, v[j].z * inv, v[j].w * inv);
            __half h[4] = {__float2half_rn(a.x), __float2half_rn(a.y), __float2half_rn(a.z), __float2half_rn(a.w)};
            const int o4 = (part * Dh + c) >> 2;
            out[o4] = *reinterpret_cast<const uint2*>(h);
            out32[o4] = a;
        }
    }
}

// Exact rescore of the FP16 search (eqs. 14-15 in FP32): warp per frame; the candidates of the search GEMM whose FP16
// score is within SEARCH_TAU of the frame's FP16 maximum are rescored as Re{Dhat_q . Zhat} = R32[q] . Zn32[f] in FP32
// and the best (lowest class on ties) becomes the frame's SVD key.  A frame whose list overflowed (more than
// SEARCH_CAP entries) is rescored over every class.  The key does not depend on the candidates' order.
__global__ void rescore_kernel(const unsigned long long* __restrict__ keys16, const unsigned long long* __restrict__ cand,
                               const int* __restrict__ ccnt, const float* __restrict__ R32,
                               const float* __restrict__ Zn, int K2, int Q, int F,
                               unsigned long long* __restrict__ keys) {
    const int f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (f >= F) return;
    const unsigned long long k16 = keys16[f];
    if (k16 == 0ull) {
        if (lane == 0) keys[f] = 0ull;
        return;
    }
    const float4* zf = reinterpret_cast<const float4*>(Zn + (int64_t)f * K2);
    const int n4 = K2 >> 2;
    auto score = [&](int q) {
        const float4* r = reinterpret_cast<const float4*>(R32 + (int64_t)q * K2);
        float acc = 0.f;
        for (int i = lane; i < n4; i += 32) {
            const float4 a = __ldg(r + i), b = zf[i];
            acc = fmaf(a.x, b.x, acc);
            acc = fmaf(a.y, b.y, acc);
            acc = fmaf(a.z, b.z, acc);
            acc = fmaf(a.w, b.w, acc);
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        return acc;                                   // identical in every lane (butterfly)
    };
    unsigned long long best = 0ull;
    const int n = ccnt[f];
    if (n <= SEARCH_CAP) {
        const uint32_t o16 = (uint32_t)(k16 >> 32);
        const float m16 = __uint_as_float((o16 & 0x80000000u) ? (o16 & 0x7FFFFFFFu) : ~o16);
        for (int c = 0; c < n; ++c) {
            const unsigned long long e = cand[(int64_t)f * SEARCH_CAP + c];
            const uint32_t oe = (uint32_t)(e >> 32);
            const float s16 = __uint_as_float((oe & 0x80000000u) ? (oe & 0x7FFFFFFFu) : ~oe);
            if (s16 < m16 - SEARCH_TAU) continue;
            const int q = (int)(0xFFFFFFFFu - (uint32_t)(e & 0xFFFFFFFFull));
            const float v = score(q);
            const unsigned long long kq = v == v ? ((unsigned long long)f2o_dev(v) << 32) | (0xFFFFFFFFull - q) : 0ull;
            best = kq > best ? kq : best;
        }
    } else {
        for (int q = 0; q < Q; ++q) {
            const float v = score(q);
            const unsigned long long kq = v == v ? ((unsigned long long)f2o_dev(v) << 32) | (0xFFFFFFFFull - q) : 0ull;
            best = kq > best ? kq : best;
        }
    }
    if (lane == 0) keys[f] = best;
}

// CTA = 8 consecutive frames x 8 warps; lane = (chunk sub-slot lane>>3, frame lane&7), so a warp's record loads are
// four coalesced 128-byte rows and the 32 chunk slots of the CTA stride over the bin chunks; partial sums meet in
// shared memory (fixed order: deterministic).  8 frames per CTA keeps ~F/8 CTAs in flight (all SMs busy at 10^4).
constexpr int FIN_WARPS = 8;
constexpr int FIN_FRAMES = 8;
constexpr int FIN_SLOTS = FIN_WARPS * (32 / FIN_FRAMES);
// One or two methods per launch: method slot j in [0, nm) reads keys[j] and writes doa[j]/score[j]; the phasor
// records of the frame are read once for both.
struct FinOut {
    const unsigned long long* keys[4];   // argmax path: keys[j][f]; nullptr -> class-list path
    const int* cls;                      // class-list path: cls[f * cls_stride + j]
    int cls_stride;
    const int* zflag[4];
    int32_t* doa[4];                     // output j of frame f at doa[j][f * out_stride]
    float* score[4];
    int out_stride;
};

template <int NM>
__global__ void __launch_bounds__(32 * FIN_WARPS, NM == 1 ? 4 : 3)
    finalize_kernel(FinOut o, const uint8_t* __restrict__ P16, int F, int64_t F_pad, int M, int Mi, int bpc,
                    int n_chunks, int Kb, int N, const int* __restrict__ rep, const float* __restrict__ delay) {
    static_assert(NM >= 1 && NM <= 4, "1..4 results per frame");
    __shared__ float s_y[NM][FIN_SLOTS][FIN_FRAMES];
    __shared__ int s_p[FIN_SLOTS][FIN_FRAMES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int fl = lane % FIN_FRAMES, slot = warp * (32 / FIN_FRAMES) + lane / FIN_FRAMES;
    const int f = blockIdx.x * FIN_FRAMES + fl;
    const bool valid = f < F;
    int q[NM];
    const float* dq[NM];
#pragma unroll
    for (int j = 0; j < NM; ++j) {
        int cls = -1;
        if (o.keys[j]) {
            const unsigned long long key = valid ? o.keys[j][f] : 0ull;
            cls = key ? (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull)) : -1;
        } else if (valid) {
            cls = o.cls[(int64_t)f * o.cls_stride + j];
        }
        q[j] = cls >= 0 ? rep[cls] : -1;
        dq[j] = delay + (int64_t)(q[j] >= 0 ? q[j] : 0) * M;
    }
    const int ub = bpc * 4;
    const float inv2N = 2.0f / (float)N;
    float ysum[NM];
#pragma unroll
    for (int j = 0; j < NM; ++j) ysum[j] = 0.f;
    int pairs = 0;
    if (valid) {
        for (int cc = slot; cc < n_chunks; cc += FIN_SLOTS) {
            float ar[NM][4], ai[NM][4];
            int nk[4] = {0, 0, 0, 0};
#pragma unroll
            for (int j = 0; j < NM; ++j)
#pragma unroll
                for (int t = 0; t < 4; ++t) ar[j][t] = ai[j][t] = 0.f;
            const int kb0 = cc * bpc;
            // mics in groups of 4: the group's records and delays are loaded before any of them is used
            for (int m0 = 0; m0 < M; m0 += 4) {
                uint4 v[4];
                float dl[NM][4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int m = m0 + u < M ? m0 + u : M - 1;
                    const uint8_t* rec = P16 + (((int64_t)cc * Mi + m) * F_pad + f) * ub;
                    if (bpc == 4) {
                        v[u] = __ldg(reinterpret_cast<const uint4*>(rec));
                    } else {
                        const uint2 w2 = __ldg(reinterpret_cast<const uint2*>(rec));
                        v[u] = make_uint4(w2.x, 0u, w2.y, 0u);      // [re01 | 0 | im01 | 0]: same slots as bpc 4
                    }
#pragma unroll
                    for (int j = 0; j < NM; ++j) dl[j][u] = __ldg(dq[j] + m);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (m0 + u >= M) break;
                    const float2 r01 = __half22float2(*reinterpret_cast<const __half2*>(&v[u].x));
                    const float2 r23 = __half22float2(*reinterpret_cast<const __half2*>(&v[u].y));
                    const float2 i01 = __half22float2(*reinterpret_cast<const __half2*>(&v[u].z));
                    const float2 i23 = __half22float2(*reinterpret_cast<const __half2*>(&v[u].w));
                    const float er[4] = {r01.x, r01.y, r23.x, r23.y}, ei[4] = {i01.x, i01.y, i23.x, i23.y};
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        if (t < bpc && (er[t] != 0.f || ei[t] != 0.f)) nk[t] += 1;
#pragma unroll
                    for (int j = 0; j < NM; ++j) {
                        // e^{+j 2 pi k delta_m / N} for k = kb0 .. kb0+bpc-1: base rotation, then unit steps
                        float bs, bc, ss, sc;
                        sincospi_fast((float)kb0 * dl[j][u] * inv2N, &bs, &bc);
                        sincospi_fast(dl[j][u] * inv2N, &ss, &sc);
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            if (t < bpc) {
                                ar[j][t] += er[t] * bc - ei[t] * bs;
                                ai[j][t] += er[t] * bs + ei[t] * bc;
                            }
                            const float nb = bc * sc - bs * ss;
                            bs = bs * sc + bc * ss;
                            bc = nb;
                        }
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (t < bpc && kb0 + t < Kb) {
#pragma unroll
                    for (int j = 0; j < NM; ++j) ysum[j] += ar[j][t] * ar[j][t] + ai[j][t] * ai[j][t] - (float)nk[t];
                    pairs += nk[t] * (nk[t] - 1) / 2;
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < NM; ++j) s_y[j][slot][fl] = ysum[j];
    s_p[slot][fl] = pairs;
    __syncthreads();
    if (slot == 0 && valid) {
        int pr = 0;
#pragma unroll 8
        for (int w = 0; w < FIN_SLOTS; ++w) pr += s_p[w][fl];
#pragma unroll
        for (int j = 0; j < NM; ++j) {
            float y = 0.f;
#pragma unroll 8
            for (int w = 0; w < FIN_SLOTS; ++w) y += s_y[j][w][fl];
            const bool dead = (pr == 0) || q[j] < 0 || (o.zflag[j] != nullptr && o.zflag[j][f] != 0);
            o.doa[j][(int64_t)f * o.out_stride] = dead ? -1 : q[j];
            o.score[j][(int64_t)f * o.out_stride] = dead ? 0.f : 0.5f * y;
        }
    }
}

// Small-batch SRP: Y[f][q] = sum of the S partial power maps (fixed order: deterministic), argmax over the steering
// classes (lowest index on ties) -> the frame's key.  CTA per frame, 16-byte loads, the 4 x S loads of a thread in
// flight together (a warp per frame with scalar loads left 32 CTAs on the GPU and took 82 us for the 17 MB of a
// 256-frame cfg5 call, ncu r02: as long as the split GEMM it follows).
constexpr int SA_THREADS = 256;
__global__ void __launch_bounds__(SA_THREADS)
    split_argmax_kernel(const float* __restrict__ Yp, int S, int64_t F_pad, int ldq, int Q, int F,
                        unsigned long long* __restrict__ keys) {
    __shared__ unsigned long long s_best[SA_THREADS / 32];
    const int f = blockIdx.x, t = threadIdx.x;
    if (f >= F) return;
    const int n4 = ldq >> 2;                                 // ldq = Q_pad, a multiple of 128
    unsigned long long best = 0ull;
    for (int i0 = 0; i0 < n4; i0 += 4 * SA_THREADS) {
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int sp = 0; sp < S; ++sp) {
            const float4* row = reinterpret_cast<const float4*>(Yp + ((int64_t)sp * F_pad + f) * ldq);
            float4 w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int i = i0 + t + j * SA_THREADS;
                w[j] = i < n4 ? row[i] : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                v[j].x += w[j].x;
                v[j].y += w[j].y;
                v[j].z += w[j].z;
                v[j].w += w[j].w;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int q0 = 4 * (i0 + t + j * SA_THREADS);
            const float e[4] = {v[j].x, v[j].y, v[j].z, v[j].w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int q = q0 + c;
                const unsigned long long k =
                    (q < Q && e[c] == e[c]) ? ((unsigned long long)f2o_dev(e[c]) << 32) | (0xFFFFFFFFull - (uint32_t)q)
                                            : 0ull;
                best = k > best ? k : best;
            }
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
        best = ob > best ? ob : best;
    }
    if ((t & 31) == 0) s_best[t >> 5] = best;
    __syncthreads();
    if (t == 0) {
#pragma unroll
        for (int w = 1; w < SA_THREADS / 32; ++w) best = s_best[w] > best ? s_best[w] : best;
        keys[f] = best;
    }
}

cudaError_t launch_split_argmax(const Plan& p, int F, int S, cudaStream_t s) {
    if (F <= 0) return cudaSuccess;
    split_argmax_kernel<<<F, SA_THREADS, 0, s>>>(p.d_Ypart, S, p.F_pad, p.Q_pad, p.Q_eff, F, p.d_keys);
    return cudaGetLastError();
}

cudaError_t launch_zsplit(const Plan& p, const Band& b, int F, cudaStream_t s, bool both) {
    if (F <= 0) return cudaSuccess;
    const int ldz = 2 * p.Zh, S = proj_shape(p, b, F).ksplit;
    const int nv = (ldz / 4 + ZS_THREADS - 1) / ZS_THREADS;
    // the tail columns always leave Z; their keys are only wanted by a BOTH call (the SRP GEMM then skips them)
    const ZTail tl{p.tail_n, p.D, p.tail_r0, p.fold_rows, p.d_fold_cls, both ? p.d_keys : nullptr};
#define SVD_ZS(NV)                                                                                                  \
    if (nv <= NV) {                                                                                                 \
        zsplit_cta_kernel<NV><<<F, ZS_THREADS, 0, s>>>(p.d_Z32, p.F_pad, p.Zh, S, p.d_Zs16, p.d_Zn32, p.Dh,          \
                                                       p.d_zflag, tl);                                             \
        return cudaGetLastError();                                                                                  \
    }
    SVD_ZS(1)
    SVD_ZS(2)
    SVD_ZS(4)
    SVD_ZS(8)
    SVD_ZS(16)
#undef SVD_ZS
    return cudaErrorInvalidValue;                 // 2*Zh > 8192 columns: excluded at plan creation
}

// Small batches: exact rescore from the stored score map (search GEMM mode 5).  CTA per frame: the frame's FP16-input
// maximum over the classes, then every class within SEARCH_TAU of it is rescored in FP32 (a warp per candidate, lanes
// over K) and the best (lowest class on ties) becomes the frame's SVD key.
constexpr int RM_THREADS = 256;
constexpr int RM_CAND = 512;                          // candidates held in shared memory (more: rescored in passes)
__global__ void __launch_bounds__(RM_THREADS)
    rescore_map_kernel(const float* __restrict__ S, int ldS, int Q, const float* __restrict__ R32,
                       const float* __restrict__ Zn, int K2, int F, unsigned long long* __restrict__ keys) {
    __shared__ float s_red[RM_THREADS / 32];
    __shared__ unsigned long long s_best[RM_THREADS / 32];
    __shared__ int s_cand[RM_CAND];
    __shared__ int s_n;
    const int f = blockIdx.x;
    if (f >= F) return;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const float* row = S + (int64_t)f * ldS;
    float m = -INFINITY;
    for (int q = t; q < Q; q += RM_THREADS) m = fmaxf(m, row[q]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) s_red[warp] = m;
    __syncthreads();
    m = s_red[0];
#pragma unroll
    for (int w = 1; w < RM_THREADS / 32; ++w) m = fmaxf(m, s_red[w]);
    const float thr = m - SEARCH_TAU;
    const float4* zf = reinterpret_cast<const float4*>(Zn + (int64_t)f * K2);
    const int n4 = K2 >> 2;
    unsigned long long best = 0ull;
    for (int q0 = 0; q0 < Q; q0 += RM_CAND * 8) {            // candidate gathering in passes of <= RM_CAND
        if (t == 0) s_n = 0;
        __syncthreads();
        const int q1 = min(Q, q0 + RM_CAND * 8);
        for (int q = q0 + t; q < q1; q += RM_THREADS)
            if (row[q] >= thr) {
                const int i = atomicAdd(&s_n, 1);
                if (i < RM_CAND) s_cand[i] = q;
            }
        __syncthreads();
        const int n = min(s_n, RM_CAND);
        const bool overflow = s_n > RM_CAND;
        // overflow (a flat map): every class of this pass is rescored
        const int cnt = overflow ? q1 - q0 : n;
        for (int c = warp; c < cnt; c += RM_THREADS / 32) {
            const int q = overflow ? q0 + c : s_cand[c];
            const float4* r = reinterpret_cast<const float4*>(R32 + (int64_t)q * K2);
            float acc = 0.f;
            for (int i = lane; i < n4; i += 32) {
                const float4 a = __ldg(r + i), b = zf[i];
                acc = fmaf(a.x, b.x, acc);
                acc = fmaf(a.y, b.y, acc);
                acc = fmaf(a.z, b.z, acc);
                acc = fmaf(a.w, b.w, acc);
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
            const unsigned long long kq =
                acc == acc ? ((unsigned long long)f2o_dev(acc) << 32) | (0xFFFFFFFFull - q) : 0ull;
            best = kq > best ? kq : best;
        }
        __syncthreads();
    }
    if (lane == 0) s_best[warp] = best;
    __syncthreads();
    if (t == 0) {
        unsigned long long b = s_best[0];
        for (int w = 1; w < RM_THREADS / 32; ++w) b = s_best[w] > b ? s_best[w] : b;
        keys[f] = m > -INFINITY ? b : 0ull;
    }
}

cudaError_t launch_rescore(const Plan& p, int F, cudaStream_t s) {
    if (F <= 0) return cudaSuccess;
    if (p.search_map) {
        rescore_map_kernel<<<F, RM_THREADS, 0, s>>>(p.d_Smap, p.Q_pad, p.Q_eff, p.d_R32, p.d_Zn32, p.K2, F,
                                                    p.d_keys + p.F_pad);
        return cudaGetLastError();
    }
    rescore_kernel<<<(F * 32 + 255) / 256, 256, 0, s>>>(p.d_keys + 2 * p.F_pad, p.d_cand, p.d_ccnt, p.d_R32,
                                                        p.d_Zn32, p.K2, p.Q_eff, F, p.d_keys + p.F_pad);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const Plan& p, int method, int F, int32_t* const doa[2], float* const score[2],
                            cudaStream_t s) {
    if (F <= 0) return cudaSuccess;
    FinOut o{};
    o.out_stride = 1;
    int nm = 0;
    if (method & SVDPHAT_METHOD_SRP) {
        o.keys[nm] = p.d_keys;
        o.zflag[nm] = nullptr;
        o.doa[nm] = doa[0];
        o.score[nm] = score[0];
        ++nm;
    }
    if (method & SVDPHAT_METHOD_SVD) {
        o.keys[nm] = p.d_keys + p.F_pad;
        o.zflag[nm] = p.d_zflag;
        o.doa[nm] = doa[1];
        o.score[nm] = score[1];
        ++nm;
    }
    const dim3 grid((F + FIN_FRAMES - 1) / FIN_FRAMES), block(32 * FIN_WARPS);
    if (nm == 2)
        finalize_kernel<2><<<grid, block, 0, s>>>(o, p.d_P16, F, p.F_pad, p.M, p.L.Mi, p.L.bpc, p.L.n_chunks, p.Kb,
                                                  p.N, p.d_rep, p.d_delay);
    else
        finalize_kernel<1><<<grid, block, 0, s>>>(o, p.d_P16, F, p.F_pad, p.M, p.L.Mi, p.L.bpc, p.L.n_chunks, p.Kb,
                                                  p.N, p.d_rep, p.d_delay);
    return cudaGetLastError();
}

cudaError_t launch_finalize_topk(const Plan& p, int F, int k, int32_t* doa, float* score, cudaStream_t s) {
    if (F <= 0) return cudaSuccess;
    FinOut o{};
    o.cls = p.d_cls;
    o.cls_stride = 4;
    o.out_stride = k;
    for (int j = 0; j < k; ++j) {
        o.keys[j] = nullptr;
        o.zflag[j] = nullptr;
        o.doa[j] = doa + j;
        o.score[j] = score + j;
    }
    const dim3 grid((F + FIN_FRAMES - 1) / FIN_FRAMES), block(32 * FIN_WARPS);
#define SVD_FIN(K)                                                                                                 \
    if (k == K) {                                                                                                  \
        finalize_kernel<K><<<grid, block, 0, s>>>(o, p.d_P16, F, p.F_pad, p.M, p.L.Mi, p.L.bpc, p.L.n_chunks, p.Kb,  \
                                                  p.N, p.d_rep, p.d_delay);                                        \
        return cudaGetLastError();                                                                                 \
    }
    SVD_FIN(1)
    SVD_FIN(2)
    SVD_FIN(3)
    SVD_FIN(4)
#undef SVD_FIN
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- multi-source peak picking
// CTA per frame: the frame's power map (one value per steering class) is staged in shared memory; k rounds of a
// block-wide argmax (lowest class on ties) skipping classes within the suppression cone (dot >= cos_sep) of the
// peaks already taken.
__global__ void __launch_bounds__(256)
    topk_kernel(const float* __restrict__ S, int ldS, int Q, int F, const float4* __restrict__ dirs, int k,
                float cos_sep, int* __restrict__ cls_out) {
    extern __shared__ float sc[];
    __shared__ float s_v[8];
    __shared__ int s_i[8];
    __shared__ float4 sel[4];
    const int f = blockIdx.x;
    if (f >= F) return;
    const float* row = S + (int64_t)f * ldS;
    for (int q = threadIdx.x; q < Q; q += blockDim.x) sc[q] = row[q];
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = 0; j < k; ++j) {
        float bv = -INFINITY;
        int bi = 0x7FFFFFFF;
        for (int q = threadIdx.x; q < Q; q += blockDim.x) {
            const float v = sc[q];
            if (!(v > bv || (v == bv && q < bi))) continue;
            const float4 d = __ldg(dirs + q);
            bool sup = false;
            for (int i = 0; i < j; ++i) sup |= (d.x * sel[i].x + d.y * sel[i].y + d.z * sel[i].z) >= cos_sep;
            if (!sup) {
                bv = v;
                bi = q;
            }
        }
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
                bv = ov;
                bi = oi;
            }
        }
        if (lane == 0) {
            s_v[warp] = bv;
            s_i[warp] = bi;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            float v = s_v[0];
            int i = s_i[0];
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
                if (s_v[w] > v || (s_v[w] == v && s_i[w] < i)) {
                    v = s_v[w];
                    i = s_i[w];
                }
            const bool ok = i != 0x7FFFFFFF && v > -INFINITY;
            cls_out[(int64_t)f * 4 + j] = ok ? i : -1;
            if (ok) sc[i] = -INFINITY;            // a taken class is never returned again, whatever the cone test
                                                  // (min_sep 0: an FP32 self-dot may round below 1; a zero direction)
            sel[j] = ok ? dirs[i] : make_float4(0.f, 0.f, 0.f, 0.f);
            if (!ok) sel[j].x = 2.0f;             // no further peak: suppress nothing, later rounds also empty
        }
        __syncthreads();
    }
}

cudaError_t topk_set_attributes() {   // per device, at plan creation
    return cudaFuncSetAttribute(topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152 * (int)sizeof(float));
}

cudaError_t launch_topk(const Plan& p, int F, int k, float cos_sep, cudaStream_t s) {
    if (F <= 0) return cudaSuccess;
    const size_t smem = (size_t)p.Q_eff * sizeof(float);   // <= 192 KB (Q_classes <= 49152, checked by the API)
    topk_kernel<<<F, 256, smem, s>>>(p.d_S, p.Q_pad, p.Q_eff, F, p.d_dirs, k, cos_sep, p.d_cls);
    return cudaGetLastError();
}

}  // namespace svdphat
