// finalize.cu — Z normalisation/split for the search GEMM, and the per-frame finalize.
//
// zsplit  : Zhat = Z / ||Z|| (Alg. 1 online step 2), written as split FP16 [hi | hi | lo] so the
//           search GEMM computes Rhat_hi.Zhat_hi + Rhat_lo.Zhat_hi + Rhat_hi.Zhat_lo (~FP32-accurate scores).
// finalize: decodes the packed argmax key (class index -> lowest point index of the class), and computes the score
//           Y_q = Re{W_q . X} of eq. 5 for the chosen q (Alg. 1 online step 4) in the
//           exact delay-and-sum form  Y_q = 1/2 sum_k ( |sum_m e_m[k] e^{+j 2 pi k delta_qm / N}|^2 - n_k ),
//           which is eq. 5 rewritten with tau_qij = delta_qi - delta_qj (eqs. 1-2); n_k = #non-zero phasors at k.
//           A frame whose X vector is identically 0 (no bin with two live channels) gets q = -1, score 0 (R4).
#include <cuda_fp16.h>

#include "internal.h"

namespace svdphat {

__global__ void zsplit_kernel(const float* __restrict__ Z, int F, int ldz, __half* __restrict__ Zs, int K2,
                              int* __restrict__ zflag) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= F) return;
    const float* z = Z + (int64_t)warp * ldz;
    float ss = 0.f;
    for (int i = lane; i < ldz; i += 32) ss += z[i] * z[i];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    const float inv = ss > 0.f ? rsqrtf(ss) : 0.f;
    if (lane == 0) zflag[warp] = ss > 0.f ? 0 : 1;
    __half* out = Zs + (int64_t)warp * K2;
    for (int i = lane; i < ldz; i += 32) {
        const float v = z[i] * inv;
        const __half hi = __float2half_rn(v);
        const __half lo = __float2half_rn(v - __half2float(hi));
        out[i] = hi;
        out[ldz + i] = hi;
        out[2 * ldz + i] = lo;
    }
}

__global__ void finalize_kernel(const unsigned long long* __restrict__ keys, const uint8_t* __restrict__ P16, int F,
                                int64_t F_pad, int M, int Mi, int bpc, int n_chunks, int Kb, int N,
                                const int* __restrict__ rep, const float* __restrict__ delay,
                                const int* __restrict__ zflag, int32_t* __restrict__ doa, float* __restrict__ score) {
    const int f = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (f >= F) return;
    const unsigned long long key = keys[f];
    const int cls = key ? (int)(0xFFFFFFFFu - (uint32_t)(key & 0xFFFFFFFFull)) : -1;
    const int q = cls >= 0 ? rep[cls] : -1;
    const float* dq = delay + (int64_t)(q >= 0 ? q : 0) * M;
    const int ub = bpc * 4;
    float ysum = 0.f;
    int pairs = 0;
    for (int cc = lane; cc < n_chunks; cc += 32) {
        float ar[4] = {0, 0, 0, 0}, ai[4] = {0, 0, 0, 0};
        int nk[4] = {0, 0, 0, 0};
        for (int m = 0; m < M; ++m) {
            const float dlm = __ldg(dq + m);
            const __half* rec =
                reinterpret_cast<const __half*>(P16 + (((int64_t)cc * Mi + m) * F_pad + f) * ub);
            for (int s = 0; s < bpc; ++s) {
                const float er = __half2float(rec[s]), ei = __half2float(rec[bpc + s]);
                if (er != 0.f || ei != 0.f) {
                    const int k = cc * bpc + s;
                    float sn, cs;
                    sincospif(2.0f * (float)k * dlm / (float)N, &sn, &cs);
                    ar[s] += er * cs - ei * sn;
                    ai[s] += er * sn + ei * cs;
                    nk[s] += 1;
                }
            }
        }
        for (int s = 0; s < bpc; ++s) {
            if (cc * bpc + s < Kb) {
                ysum += ar[s] * ar[s] + ai[s] * ai[s] - (float)nk[s];
                pairs += nk[s] * (nk[s] - 1) / 2;
            }
        }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        ysum += __shfl_xor_sync(0xffffffffu, ysum, o);
        pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
    }
    if (lane == 0) {
        const bool dead = (pairs == 0) || q < 0 || (zflag != nullptr && zflag[f] != 0);
        doa[f] = dead ? -1 : q;
        score[f] = dead ? 0.f : 0.5f * ysum;
    }
}

cudaError_t launch_zsplit(const Plan& p, int F, cudaStream_t s) {
    if (F <= 0) return cudaSuccess;
    const int threads = 256;
    const int blocks = (F * 32 + threads - 1) / threads;
    zsplit_kernel<<<blocks, threads, 0, s>>>(p.d_Z32, F, 2 * p.Dh, p.d_Zs16, p.K2, p.d_zflag);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const Plan& p, int method, int F, int32_t* doa, float* score, cudaStream_t s) {
    if (F <= 0) return cudaSuccess;
    const int threads = 256;
    const int blocks = (F * 32 + threads - 1) / threads;
    finalize_kernel<<<blocks, threads, 0, s>>>(p.d_keys, p.d_P16, F, p.F_pad, p.M, p.L.Mi, p.L.bpc, p.L.n_chunks,
                                               p.Kb, p.N, p.d_rep, p.d_delay,
                                               method == SVDPHAT_METHOD_SVD ? p.d_zflag : nullptr, doa, score);
    return cudaGetLastError();
}

}  // namespace svdphat
