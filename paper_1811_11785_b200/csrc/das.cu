// das.cu — SRP-PHAT through the delay-and-sum form of eq. 5 on the tensor cores.
//
// Eq. 5 with tau_qij = delta_qi - delta_qj (eqs. 1-2: a pair's TDOA is the difference
// of the two microphones' arrival delays) factorises per bin k:
//
//   Y_q = Re sum_{i<j} sum_k e_i[k] conj(e_j[k]) e^{j 2 pi k (delta_qi - delta_qj) / N}
//       = 1/2 sum_k ( |a_q[k]|^2 - n_k ),      a_q[k] = sum_m e_m[k] e^{j 2 pi k delta_qm / N},
//
// e_m the PHAT unit phasors (eq. 3 factorised) and n_k the number of non-zero phasors at bin k, a
// per-frame constant that does not move the argmax of eq. 6.  For one bin, [Re a_q; Im a_q] over all candidates and
// a batch of frames is a real GEMM with a 2M-long contraction:
//
//   row (c, Re) = [ cos phi_cm | -sin phi_cm ],   row (c, Im) = [ sin phi_cm | cos phi_cm ],   phi_cm = 2 pi k delta_cm / N
//   column f    = [ Re e_m[k]  |  Im e_m[k]  ]    (m = 0..ME-1; microphones >= M are zero)
//
// so S_c = sum_k (Re a_c[k])^2 + (Im a_c[k])^2 = 2 Y_c + sum_k n_k is the sum of squares of two accumulator rows.
// Per (candidate, frame, bin) this costs 8 ME flops on the tensor cores against eq. 9's 4 P = 2 M (M - 1): (M-1)/4
// fewer at M = ME (3.75x at M = 16, 7.75x at M = 32).  The price: the squares are taken per bin, so every accumulator
// element is read back from TMEM once per bin (tcgen05.ld + one FFMA2 per two elements).  That epilogue runs at
// ~100 elements/clk/SM (tools/microbench_tmem.cu) against the MMA's 128 (ME = 16) / 64 (ME = 32) elements/clk/SM:
// epilogue-bound at ME = 16, MMA-bound at ME = 32.
//
// Kernel: CTA pairs (cta_group::2), a unit = 256 steering rows (128 classes) x 256 frames, looping over the bins.
// Per bin and CTA: TMA brings 128 steering rows (A16) and 128 frame rows (E16, this CTA's half of the frames), the
// leader issues ME/8 MMAs M = 256, N = 256, K = 16 into one of two TMEM accumulators (256 columns each), and 8
// epilogue warps per CTA fold the squares into 128 running FP32 sums per thread.  After the last bin the two rows of
// a class are added, and per frame the best (S, lowest class) leaves as a packed u64 key (atomicMax) for the
// existing finalize (class -> lowest point index, exact Y_q of eq. 5).
#include <cuda_fp16.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace svdphat {

constexpr int DAS_EW = 16;            // epilogue warps per CTA (4 lane quarters x DAS_EW/4 column slices)
constexpr int DAS_THREADS = 32 * (4 + DAS_EW);   // warpgroup 0: warp 0 TMA, warp 1 MMA issuer; then the epilogue
// registers: each SM sub-partition (warp % 4) has 16384 for its 5 warps (one of warpgroup 0, four epilogue warps).
// Launched at 96 per thread (the pool setmaxnreg redistributes); warpgroup 0 drops to 32 and the epilogue warpgroups
// rise to 112: 32 + 4 x 112 = 480 = 5 x 96 per sub-partition and thread slot.
constexpr int DAS_REGS = 96, DAS_REGS_LO = 32, DAS_REGS_HI = 112;
constexpr int DAS_BN = 256;           // frames per pair unit (128 per CTA)
constexpr int DAS_EC = DAS_BN / (DAS_EW / 4);   // accumulator columns (frames) per epilogue thread
constexpr int DAS_GF = 8;             // frame tiles per raster group (L2 reuse of the units in flight)

template <int ME>
struct DasCfg {
    static constexpr int RB = 4 * ME;                 // bytes per operand row: 2 ME halves
    static constexpr int TILE = 128 * RB;             // one operand tile per CTA per bin
    static constexpr int STAGE = 2 * TILE;            // A tile + B tile
    static constexpr int NST = ME == 32 ? 6 : ME == 16 ? 8 : 12;
    static constexpr int NK = 2 * ME / 16;            // K = 16 MMA steps per bin
    static constexpr uint32_t LAYOUT = ME == 32 ? 2u : ME == 16 ? 4u : 6u;   // SWIZZLE_128B / 64B / 32B
    static constexpr uint32_t HI = ((8u * RB) >> 4) | (1u << 14) | (LAYOUT << 29);  // SBO = 8-row atom, version 1
    static constexpr int SMEM = 1024 + NST * STAGE + 256;
};

struct DasParams {
    int F;                 // valid frames
    int64_t F_pad;
    int R_pad;             // steering rows of A16 (multiple of 256)
    int k_lo, k_hi;        // bins of the call (band limit)
    int n_rt, n_ft;        // 256-row tiles, 256-frame tiles
    int Q_eff;             // classes (rows 2c, 2c+1)
    unsigned long long* keys;
};

__device__ __forceinline__ void das_unit(const DasParams& p, int t, int& rt, int& ft) {
    const int gsize = DAS_GF * p.n_rt;
    const int g = t / gsize, r = t - g * gsize;
    const int nf = min(DAS_GF, p.n_ft - g * DAS_GF);
    rt = r / nf;
    ft = g * DAS_GF + (r - rt * nf);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// s[0..15] += v^2, two lanes per FFMA2
__device__ __forceinline__ void sumsq16(float* s, const uint32_t (&v)[16]) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
        unsigned long long a, acc;
        asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "r"(v[i]), "r"(v[i + 1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(s[i]), "f"(s[i + 1]));
        asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(a));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(s[i]), "=f"(s[i + 1]) : "l"(acc));
    }
}

__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
    return r;
}
__device__ __forceinline__ void wait_u32(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

// One bin of the epilogue: the TMEM buffer at tb (this warp's 32 lanes x DAS_EC columns), its full barrier tf
// (local), its empty barrier te (the leader's, cluster address).  Loads go out in pairs of x16; the buffer is
// released (one elected lane) as soon as the last pair has landed, before the last squares.
__device__ __forceinline__ void das_epi_bin(float* s, uint32_t tb, uint32_t tf, uint32_t te, uint32_t parity) {
    wait_u32(tf, parity);
    tc_fence_after();
#pragma unroll
    for (int c = 0; c < DAS_EC; c += 32) {
        uint32_t ra[16], rb[16];
        tmem_ld16(tb + (uint32_t)c, ra);
        tmem_ld16(tb + (uint32_t)(c + 16), rb);
        tmem_ld_wait();
        if (c + 32 == DAS_EC) {
            tc_fence_before();
            asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e mbarrier.arrive.shared::cluster.b64 _, [%0];\n\t}" ::"r"(te)
                         : "memory");
        }
        sumsq16(s + c, ra);
        sumsq16(s + c + 16, rb);
    }
}

template <int NK>
__device__ __forceinline__ void das_mma(uint32_t tmem_d, uint32_t a_lo, uint32_t b_lo, uint32_t hi, uint32_t idesc) {
    if constexpr (NK == 1) {
        umma_f16_2sm_warp(tmem_d, ((uint64_t)hi << 32) | a_lo, ((uint64_t)hi << 32) | b_lo, idesc, 0u);
    } else {
        umma_f16_2sm_steps<NK>(tmem_d, a_lo, b_lo, hi, idesc, 0u);
    }
}

template <int ME>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(DAS_THREADS, 1)
    das_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmE, DasParams p) {
    using C = DasCfg<ME>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::NST * C::STAGE);
    uint64_t* empty = full + C::NST;
    uint64_t* tfull = empty + C::NST;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int units = p.n_rt * p.n_ft;
    const int nbins = p.k_hi - p.k_lo;

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::NST; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * DAS_EW);    // every epilogue warp of both CTAs arrives on the leader's barrier
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_2sm<512>(tmem_slot);
    if (warp == 1 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmE);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (warp < 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(DAS_REGS_LO));

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = pair; t < units; t += n_pairs) {
                int rt, ft;
                das_unit(p, t, rt, ft);
                const int arow = rt * 256 + (int)rank * 128;
                const int64_t frow = (int64_t)ft * DAS_BN + (int64_t)rank * 128;
                for (int k = p.k_lo; k < p.k_hi; ++k) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE);
                    uint8_t* st = smem + stage * C::STAGE;
                    tma_load_2d_2sm(st, &tmA, 0, k * p.R_pad + arow, &full[stage]);
                    tma_load_2d_2sm(st + C::TILE, &tmE, 0, (int32_t)(k * p.F_pad + frow), &full[stage]);
                    if (++stage == C::NST) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            const uint32_t idesc = umma_idesc_f16(256, DAS_BN);
            const uint32_t a_lo0 = umma_desc_lo(smem_u32(smem)), b_lo0 = umma_desc_lo(smem_u32(smem + C::TILE));
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int t = pair; t < units; t += n_pairs) {
                for (int k = 0; k < nbins; ++k) {
                    mbar_wait(&tempty[acc], acc_phase ^ 1);
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t so = (uint32_t)(stage * (C::STAGE >> 4));
                    das_mma<C::NK>(tmem_base + (uint32_t)(acc * DAS_BN), a_lo0 + so, b_lo0 + so, C::HI, idesc);
                    umma_commit_2sm_warp(&empty[stage], 0x3);
                    umma_commit_2sm_warp(&tfull[acc], 0x3);
                    if (++stage == C::NST) {
                        stage = 0;
                        phase ^= 1;
                    }
                    if (++acc == 2) {
                        acc = 0;
                        acc_phase ^= 1;
                    }
                }
            }
        }
    } else if (warp >= 4) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(DAS_REGS_HI));
        // epilogue: lane quarter g (TMEM lanes 32g..32g+31 = rows), column slice h (frames DAS_EC h .. + DAS_EC).
        // Everything a bin needs besides the data is fixed per warp: both buffers' TMEM addresses, both tfull
        // barriers, both tempty barriers of the leader (mapa once); the bin loop is unrolled by the buffer pair so
        // the buffer index is a constant.
        const int g = warp & 3, h = (warp - 4) >> 2;
        const uint32_t tb0 = tmem_base + ((uint32_t)(g * 32) << 16) + (uint32_t)(h * DAS_EC);
        const uint32_t tf0 = smem_u32(&tfull[0]), tf1 = smem_u32(&tfull[1]);
        const uint32_t te0 = mapa_u32(smem_u32(&tempty[0]), 0), te1 = mapa_u32(smem_u32(&tempty[1]), 0);
        int acc = 0;
        uint32_t ph = 0;
        float s[DAS_EC];
        for (int t = pair; t < units; t += n_pairs) {
            int rt, ft;
            das_unit(p, t, rt, ft);
#pragma unroll
            for (int i = 0; i < DAS_EC; ++i) s[i] = 0.f;
            int k = 0;
            if (acc == 1 && k < nbins) {
                das_epi_bin(s, tb0 + DAS_BN, tf1, te1, ph);
                ph ^= 1;
                acc = 0;
                ++k;
            }
            for (; k + 1 < nbins; k += 2) {
                das_epi_bin(s, tb0, tf0, te0, ph);
                das_epi_bin(s, tb0 + DAS_BN, tf1, te1, ph);
                ph ^= 1;
            }
            if (k < nbins) {
                das_epi_bin(s, tb0, tf0, te0, ph);
                acc = 1;
            }
            // S_c = (sum of squares of row 2c) + (row 2c + 1), adjacent lanes; both lanes then hold S_c, so the even
            // lane keeps frames 0..31 of the slice and the odd lane frames 32..63, and a 4-step transpose-max over
            // lanes of equal parity leaves each lane the best (S, lowest class) of two frames.
            const int row = rt * 256 + (int)rank * 128 + g * 32 + lane;
            const int cls = row >> 1;
            const bool ok = cls < p.Q_eff;
            const int par = lane & 1;
            unsigned long long key[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const float lo = s[j] + __shfl_xor_sync(0xffffffffu, s[j], 1);
                const float hi = s[32 + j] + __shfl_xor_sync(0xffffffffu, s[32 + j], 1);
                key[j] = ok ? make_key(par ? hi : lo, (uint32_t)cls) : 0ull;
            }
#pragma unroll
            for (int hh = 16; hh >= 2; hh >>= 1) {
                const bool upper = (lane & hh) != 0;
#pragma unroll
                for (int c = 0; c < hh; ++c) {
                    const unsigned long long send = upper ? key[c] : key[c + hh];
                    const unsigned long long mine = upper ? key[c + hh] : key[c];
                    const unsigned long long recv = __shfl_xor_sync(0xffffffffu, send, hh);
                    key[c] = mine > recv ? mine : recv;
                }
            }
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int f = ft * DAS_BN + h * DAS_EC + 32 * par + (lane & 0x1E) + b;
                if (f < p.F && key[b] != 0ull) atomicMax(&p.keys[f], key[b]);
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc_2sm<512>(tmem_base);
    }
}

// ---------------------------------------------------------------- frame operand: P16 records -> E16 bin rows
// E16[k][f] = [Re e_0 .. Re e_{ME-1} | Im e_0 .. Im e_{ME-1}] (FP16, microphones >= M zero): one 4 ME-byte row per
// (bin, frame), the K-major B operand of das_kernel.  Thread per (bin chunk, frame): reads the frame's M records of
// the chunk (coalesced across frames), writes its BPC rows (contiguous across frames).
template <int ME, int BPC>
__global__ void __launch_bounds__(128) das_bins_kernel(const uint8_t* __restrict__ P16, int F, int64_t F_pad, int Mi,
                                                       int M, int Kb, int c_lo, __half* __restrict__ E16) {
    const int f = blockIdx.x * blockDim.x + threadIdx.x;
    const int c = c_lo + (int)blockIdx.y;
    if (f >= F) return;
    constexpr int UB = BPC * 4;                       // record bytes: [Re k0..k_{BPC-1} | Im k0..]
    uint32_t re[BPC][ME / 2], im[BPC][ME / 2];
#pragma unroll
    for (int m = 0; m < ME; m += 2) {
        uint32_t w0[4] = {0u, 0u, 0u, 0u}, w1[4] = {0u, 0u, 0u, 0u};   // words of mics m, m+1: [Re | Im]
        const uint8_t* r0 = P16 + (((int64_t)c * Mi + m) * F_pad + f) * UB;
        const uint8_t* r1 = r0 + F_pad * UB;
        if constexpr (BPC == 4) {
            if (m < M) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(r0));
                w0[0] = v.x, w0[1] = v.y, w0[2] = v.z, w0[3] = v.w;
            }
            if (m + 1 < M) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(r1));
                w1[0] = v.x, w1[1] = v.y, w1[2] = v.z, w1[3] = v.w;
            }
        } else {
            if (m < M) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(r0));
                w0[0] = v.x, w0[1] = v.y;
            }
            if (m + 1 < M) {
                const uint2 v = __ldg(reinterpret_cast<const uint2*>(r1));
                w1[0] = v.x, w1[1] = v.y;
            }
        }
#pragma unroll
        for (int t = 0; t < BPC; ++t) {
            const uint32_t sel = (t & 1) ? 0x7632u : 0x5410u;   // high / low halves of both words
            re[t][m / 2] = __byte_perm(w0[t / 2], w1[t / 2], sel);
            im[t][m / 2] = __byte_perm(w0[BPC / 2 + t / 2], w1[BPC / 2 + t / 2], sel);
        }
    }
#pragma unroll
    for (int t = 0; t < BPC; ++t) {
        const int k = c * BPC + t;
        if (k >= Kb) break;
        uint4* row = reinterpret_cast<uint4*>(E16 + ((int64_t)k * F_pad + f) * (2 * ME));
#pragma unroll
        for (int i = 0; i < ME / 8; ++i) {
            row[i] = make_uint4(re[t][4 * i], re[t][4 * i + 1], re[t][4 * i + 2], re[t][4 * i + 3]);
            row[ME / 8 + i] = make_uint4(im[t][4 * i], im[t][4 * i + 1], im[t][4 * i + 2], im[t][4 * i + 3]);
        }
    }
}

// ---------------------------------------------------------------- steering operand (setup, float64)
// A16[k][r][0..2ME): row r = 2c (Re a_c) = [cos phi_cm | -sin phi_cm], r = 2c + 1 (Im a_c) = [sin phi_cm | cos phi_cm],
// phi_cm = 2 pi k delta_cm / N in float64 (delta_cm: class c's arrival delays in samples, relative to the earliest
// microphone); rows >= 2 Q_eff and microphones >= M are zero.  Thread per (row, bin).
__global__ void das_steer_kernel(const double* __restrict__ delay, int Q_eff, int M, int ME, int N, int R_pad,
                                 __half* __restrict__ A16) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (r >= R_pad) return;
    __half* row = A16 + ((int64_t)k * R_pad + r) * (2 * ME);
    const int c = r >> 1, v = r & 1;
    for (int m = 0; m < ME; ++m) {
        double sn = 0.0, cs = 0.0;
        if (c < Q_eff && m < M) sincospi(2.0 * (double)k * delay[(int64_t)c * M + m] / (double)N, &sn, &cs);
        row[m] = __double2half(v == 0 ? cs : sn);
        row[ME + m] = __double2half(v == 0 ? -sn : cs);
    }
}

int das_me(int M) { return M <= 8 ? 8 : M <= 16 ? 16 : 32; }

svdphat_status setup_das_operand(Plan& p, const double* h_delay_cls) {
    p.das_me = das_me(p.M);
    p.das_rows = (2 * p.Q_eff + 255) / 256 * 256;
    const int64_t bytes = (int64_t)p.Kb * p.das_rows * 2 * p.das_me * (int64_t)sizeof(__half);
    double* d_delay = nullptr;
    SVD_CUDA_TRY(cudaMalloc(&d_delay, (size_t)p.Q_eff * p.M * sizeof(double)));
    cudaError_t e = cudaMemcpy(d_delay, h_delay_cls, (size_t)p.Q_eff * p.M * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&p.d_A16, bytes);
    if (e == cudaSuccess) {
        das_steer_kernel<<<dim3((p.das_rows + 127) / 128, p.Kb), 128>>>(d_delay, p.Q_eff, p.M, p.das_me, p.N,
                                                                       p.das_rows, p.d_A16);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(d_delay);
    SVD_CUDA_TRY(e);
    p.bytes_A = bytes;
    return SVDPHAT_OK;
}

cudaError_t das_set_attributes() {
    cudaError_t e = cudaFuncSetAttribute(das_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, DasCfg<8>::SMEM);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(das_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, DasCfg<16>::SMEM);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(das_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, DasCfg<32>::SMEM);
    return e;
}

bool das_active(const Plan& p, int F) {
    // enough 256 x 256 units to give every CTA pair work (small batches keep the split-K W GEMM), or forced
    if (!p.d_A16 || !p.d_E16) return false;
    if (p.options & SVDPHAT_OPT_DAS) return true;
    const int64_t units = (int64_t)(p.das_rows / 256) * ((F + DAS_BN - 1) / DAS_BN);
    return units >= p.num_sms / 2;
}

cudaError_t launch_das_bins(const Plan& p, const Band& b, int F, cudaStream_t s) {
    if (F <= 0 || b.c_hi <= b.c_lo) return cudaSuccess;
    const dim3 grid((F + 127) / 128, b.c_hi - b.c_lo);
    const int Mi = p.L.Mi;
    switch (p.das_me) {
        case 8:
            if (p.L.bpc != 4) return cudaErrorInvalidValue;
            das_bins_kernel<8, 4><<<grid, 128, 0, s>>>(p.d_P16, F, p.F_pad, Mi, p.M, p.Kb, b.c_lo, p.d_E16);
            break;
        case 16:
            if (p.L.bpc != 4) return cudaErrorInvalidValue;
            das_bins_kernel<16, 4><<<grid, 128, 0, s>>>(p.d_P16, F, p.F_pad, Mi, p.M, p.Kb, b.c_lo, p.d_E16);
            break;
        default:
            if (p.L.bpc != 2) return cudaErrorInvalidValue;
            das_bins_kernel<32, 2><<<grid, 128, 0, s>>>(p.d_P16, F, p.F_pad, Mi, p.M, p.Kb, b.c_lo, p.d_E16);
    }
    return cudaGetLastError();
}

cudaError_t launch_das(const Plan& p, const Band& b, int F, cudaStream_t s) {
    if (F <= 0 || b.k_hi <= b.k_lo) return cudaSuccess;
    DasParams dp;
    dp.F = F;
    dp.F_pad = p.F_pad;
    dp.R_pad = p.das_rows;
    dp.k_lo = b.k_lo;
    dp.k_hi = b.k_hi;
    dp.n_rt = p.das_rows / 256;
    dp.n_ft = (F + DAS_BN - 1) / DAS_BN;
    dp.Q_eff = p.Q_eff;
    dp.keys = p.d_keys;
    const int units = dp.n_rt * dp.n_ft;
    const int grid = 2 * std::min(units, p.num_sms / 2);
    switch (p.das_me) {
        case 8:
            das_kernel<8><<<grid, DAS_THREADS, DasCfg<8>::SMEM, s>>>(p.tm_A, p.tm_E, dp);
            break;
        case 16:
            das_kernel<16><<<grid, DAS_THREADS, DasCfg<16>::SMEM, s>>>(p.tm_A, p.tm_E, dp);
            break;
        default:
            das_kernel<32><<<grid, DAS_THREADS, DasCfg<32>::SMEM, s>>>(p.tm_A, p.tm_E, dp);
    }
    return cudaGetLastError();
}

}  // namespace svdphat
