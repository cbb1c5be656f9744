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
// Per bin and CTA: TMA brings 128 steering rows (A16) and 128 frame rows (E16, this CTA's half of the frames); the
// leader issues, per frame half, ME/8 MMAs M = 256, N = 128, K = 16 into one of four 128-column TMEM regions (two
// bins in flight), and 16 epilogue warps per CTA load each region (tcgen05.ld 16x256b: Re and Im of a class reach
// the same thread), release it, and fold |a|^2 into 32 running FP32 sums per thread.  After the last bin, per frame
// the best (S, lowest class) leaves as a packed u64 key (atomicMax) for the existing finalize (class -> lowest point
// index, exact Y_q of eq. 5).
#include <cuda_fp16.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"

namespace svdphat {

constexpr int DAS_EW = 16;            // epilogue warps per CTA (4 lane quarters x DAS_EW/4 column slices)
// warp 0 TMA producer, warp 1 MMA issuer, warps 2..17 the epilogue (warp w reads TMEM lanes 32 (w % 4) ..).  576
// threads leave 112 registers per thread (65536 / 576), enough for the epilogue's 64 running sums + 32 loaded values.
constexpr int DAS_THREADS = 32 * (2 + DAS_EW);
constexpr int DAS_BN = 256;           // frames per pair unit (128 per CTA)
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
    static constexpr int SMEM = 1024 + NST * STAGE;
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

// TMEM: two bin buffers x two frame halves = four 128-column regions.  Bin k's MMA is issued as two N = 128 halves
// (B rows 0..63 and 64..127 of each CTA's frame tile) into regions 2 (k & 1) and 2 (k & 1) + 1, each with its own
// full / empty barrier, so an epilogue warp loads its piece of a region, releases the region, and squares the values
// from registers while the MMA refills it: a region is held for the load latency, not for the squares.
constexpr int DAS_RCOLS = 128;                     // columns (frames) per region
constexpr int DAS_WC = DAS_RCOLS / (DAS_EW / 4);   // columns of a region per epilogue warp (32)

// 16 TMEM lanes x 4 x 256 bits: thread t gets, for column chunk j = 0..3, lane (t / 4) columns 8 j + 2 (t % 4) + {0, 1}
// in r[4j], r[4j+1] and lane (t / 4) + 8, same columns, in r[4j+2], r[4j+3].  The steering rows are laid out so that
// lanes i and i + 8 of every 16-lane group hold Re a_c and Im a_c of one class (das_steer_kernel): each thread gets
// whole complex values.
__device__ __forceinline__ void tmem_ld16x256_x4(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.16x256b.x4.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// s[2j + e] += |a|^2 = Re^2 + Im^2 for the 8 (frame) columns of one 16-lane load, two FFMA2 per column pair
__device__ __forceinline__ void sumsq_c8(float* s, const uint32_t (&v)[16]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        unsigned long long re, im, acc;
        asm("mov.b64 %0, {%1, %2};" : "=l"(re) : "r"(v[4 * j]), "r"(v[4 * j + 1]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(im) : "r"(v[4 * j + 2]), "r"(v[4 * j + 3]));
        asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(s[2 * j]), "f"(s[2 * j + 1]));
        asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(re));
        asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc) : "l"(im));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(s[2 * j]), "=f"(s[2 * j + 1]) : "l"(acc));
    }
}

// One region of one bin: wait until its MMA half has landed (tf, local), load this warp's 32 lanes (two 16-lane
// groups: classes u = 0, 1 of the thread) x 32 columns, release the region on the leader's empty barrier (te, cluster
// address), then add |a|^2 into s[u * 8 + 2 j + e].
__device__ __forceinline__ void das_epi_region(float* s, uint32_t taddr, uint32_t tf, uint32_t te, uint32_t parity) {
    wait_u32(tf, parity);
    tc_fence_after();
    uint32_t va[16], vb[16];
    tmem_ld16x256_x4(taddr, va);
    tmem_ld16x256_x4(taddr + (16u << 16), vb);
    tmem_ld_wait();
    tc_fence_before();
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e mbarrier.arrive.shared::cluster.b64 _, [%0];\n\t}" ::"r"(te)
                 : "memory");
    sumsq_c8(s, va);
    sumsq_c8(s + 8, vb);
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
    // barriers in static shared memory: their addresses are constants (no registers held across the bin loop)
    __shared__ uint64_t full[C::NST], empty[C::NST], tfull[4], tempty[4];
    __shared__ uint32_t tmem_slot;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

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
        for (int a = 0; a < 4; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * DAS_EW);    // every epilogue warp of both CTAs arrives on the leader's barrier
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_2sm<512>(&tmem_slot);
    if (warp == 1 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmE);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = tmem_slot;

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
            const uint32_t idesc = umma_idesc_f16(256, DAS_RCOLS);
            const uint32_t a_lo0 = umma_desc_lo(smem_u32(smem)), b_lo0 = umma_desc_lo(smem_u32(smem + C::TILE));
            constexpr uint32_t HALF_B = (uint32_t)((64 * C::RB) >> 4);   // B rows 64..127 of the frame tile
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int t = pair; t < units; t += n_pairs) {
                for (int k = 0; k < nbins; ++k) {
                    mbar_wait(&full[stage], phase);
                    const uint32_t so = (uint32_t)(stage * (C::STAGE >> 4));
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        const int r = 2 * acc + hf;
                        mbar_wait(&tempty[r], acc_phase ^ 1);
                        tc_fence_after();
                        das_mma<C::NK>(tmem_base + (uint32_t)(r * DAS_RCOLS), a_lo0 + so, b_lo0 + so + hf * HALF_B,
                                       C::HI, idesc);
                        umma_commit_2sm_warp(&tfull[r], 0x3);
                    }
                    umma_commit_2sm_warp(&empty[stage], 0x3);
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
    } else {
        // epilogue: lane quarter g (TMEM lanes 32g..32g+31: classes 16 g' .. of the CTA's 128 rows), column slice h
        // (columns 32h..32h+31 of every region).  s[16 hf + 8 u + 2 j + e]: frame half hf, class u of the thread,
        // column 8 j + 2 (t % 4) + e of the slice.
        const int g = warp & 3, h = (warp - 2) >> 2;
        const uint32_t tb = tmem_base + ((uint32_t)(g * 32) << 16) + (uint32_t)(h * DAS_WC);
        const uint32_t te = mapa_u32(smem_u32(&tempty[0]), 0);
        const uint32_t tf = smem_u32(&tfull[0]);
        int acc = 0;
        uint32_t ph = 0;
        float s[32];
        for (int t = pair; t < units; t += n_pairs) {
            int rt, ft;
            das_unit(p, t, rt, ft);
#pragma unroll
            for (int i = 0; i < 32; ++i) s[i] = 0.f;
            int k = 0;
            if (acc == 1 && k < nbins) {
                das_epi_region(s, tb + 2 * DAS_RCOLS, tf + 16, te + 16, ph);
                das_epi_region(s + 16, tb + 3 * DAS_RCOLS, tf + 24, te + 24, ph);
                ph ^= 1;
                acc = 0;
                ++k;
            }
            for (; k + 1 < nbins; k += 2) {
                das_epi_region(s, tb, tf, te, ph);
                das_epi_region(s + 16, tb + DAS_RCOLS, tf + 8, te + 8, ph);
                das_epi_region(s, tb + 2 * DAS_RCOLS, tf + 16, te + 16, ph);
                das_epi_region(s + 16, tb + 3 * DAS_RCOLS, tf + 24, te + 24, ph);
                ph ^= 1;
            }
            if (k < nbins) {
                das_epi_region(s, tb, tf, te, ph);
                das_epi_region(s + 16, tb + DAS_RCOLS, tf + 8, te + 8, ph);
                acc = 1;
            }
            // per column: the best of the thread's two classes, then of the 8 threads sharing the column (lane % 4
            // equal: xor 4, 8, 16), lowest class on ties (packed keys)
            const int cls0 = (rt * 256 + (int)rank * 128 + g * 32) / 2 + (lane >> 2);
            const bool ok0 = cls0 < p.Q_eff, ok1 = cls0 + 8 < p.Q_eff;
            unsigned long long key[16];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const unsigned long long k0 = ok0 ? make_key(s[16 * hf + i], (uint32_t)cls0) : 0ull;
                    const unsigned long long k1 = ok1 ? make_key(s[16 * hf + 8 + i], (uint32_t)(cls0 + 8)) : 0ull;
                    key[8 * hf + i] = k0 > k1 ? k0 : k1;
                }
            }
#pragma unroll
            for (int x = 4; x <= 16; x <<= 1) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, key[i], x);
                    key[i] = key[i] > o ? key[i] : o;
                }
            }
            // column 32 h + 8 j + 2 (lane % 4) + e of region half hf is frame (h & 1) 32 + (h >> 1) 128 + 64 hf +
            // 8 j + 2 (lane % 4) + e of the pair's 256 (the N = 128 MMA takes B rows 64 hf .. 64 hf + 63 of each
            // CTA: columns 0..63 leader, 64..127 peer); key i = 8 hf + 2 j + e, written by the thread with lane / 4
            // == i / 2
            const int fbase = ft * DAS_BN + (h & 1) * 32 + (h >> 1) * 128 + 2 * (lane & 3);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if ((i >> 1) == (lane >> 2)) {
                    const int f = fbase + 64 * (i >> 3) + 8 * ((i >> 1) & 3) + (i & 1);
                    if (f < p.F && key[i] != 0ull) atomicMax(&p.keys[f], key[i]);
                }
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

// ---------------------------------------------------------------- folded form (centrally symmetric grids)
// For an antipodal class pair (q, q') the arrival delays satisfy delta_q'm = -delta_qm + const (tau_q' = -tau_q, the
// condition of reading R22), so |a_q'[k]| = |sum_m e_m e^{-j phi_qm}|.  With e_m = x_m + j y_m, c = cos phi_qm,
// s = sin phi_qm and the four real dot products A = x.c, B = y.s, C = x.s, D = y.c over the microphones:
//
//   a_q = (A - B) + j (C + D),     a_q' ~ (A + B) + j (D - C),
//
// so a (cos, sin) row pair per class pair against a (Re e, Im e) column pair per frame (K = ME per bin) yields both
// classes: half the MMA work and half the accumulator traffic of the unfolded kernel per class.  The epilogue thread
// gets A, D (cos lane) and C, B (sin lane) of one (pair, frame) in one 16x256b load and accumulates
// (|a_q|^2, |a_q'|^2) with two FADD2 and two FFMA2 (fold_acc4).  Operand rows hold a whole bin chunk (bpc bins x ME halves = 128 bytes, SWIZZLE_128B):
// one TMA row serves bpc bins, and bin b of the chunk is the K offset b * ME of the row.
template <int ME>
struct DasFCfg {
    static constexpr int BPR = 64 / ME;                 // bins per operand row (= the phasor records' bpc)
    static constexpr int TILE = 128 * 128;              // 128 rows x 128 bytes
    static constexpr int STAGE = 2 * TILE;
    static constexpr int NST = 6;
    static constexpr int NK = ME / 16;                  // K = 16 MMA steps per bin
    static constexpr uint32_t HI = (1024u >> 4) | (1u << 14) | (2u << 29);   // SBO 1024, version 1, SWIZZLE_128B
    static constexpr int SMEM = 1024 + NST * STAGE;
};
constexpr int DASF_BF = 128;          // frames per pair unit (2 columns each: N = 128 per region, 2 regions per bin)
// 18 warps: warp 0 TMA, warp 1 MMA, warps 2..17 the epilogue (lane quarter warp % 4, column quarter (warp - 2) / 4):
// four epilogue warps per SM sub-partition hide the TMEM load latency of a region behind each other's arithmetic.
constexpr int DASF_EW = 16;
constexpr int DASF_THREADS = 32 * (2 + DASF_EW);

#ifdef DAS_TRACE   // dev-only latency trace (tools/das_trace.py): [0] MMA issue, [1] epilogue wake, [2] epilogue release
__device__ long long g_das_trace[3][8192];
extern "C" int svdphat_dev_das_trace(long long* out, int n) {
    return (int)cudaMemcpyFromSymbol(out, g_das_trace, (size_t)n * sizeof(long long));
}
#define DAS_TRACE_REC(i, s) \
    if ((s) < 8192) g_das_trace[i][s] = clock64();
#else
#define DAS_TRACE_REC(i, s)
#endif

struct DasFParams {
    int F;
    int64_t F_pad;
    int R_pad;                  // operand rows of A16 (multiple of 256)
    int k_lo, k_hi, c_lo, c_hi;
    int n_rt, n_ft;             // 256-row (128 class-pair) tiles, 128-frame tiles
    int fold_rows;
    const int* fold_cls;        // [2][fold_rows]: class of a_q, class of a_q' (-1: none)
    unsigned long long* keys;
};

__device__ __forceinline__ void das_unit_f(const DasFParams& p, int t, int& rt, int& ft) {
    const int gsize = DAS_GF * p.n_rt;
    const int g = t / gsize, r = t - g * gsize;
    const int nf = min(DAS_GF, p.n_ft - g * DAS_GF);
    rt = r / nf;
    ft = g * DAS_GF + (r - rt * nf);
}

// The frame operand's rows come in blocks of 16 per 8 frames (8 Re rows, then the 8 Im rows of the same frames), so
// in one 16-lane x 32-column load (four 8-column chunks) a thread gets, for two frames f, f' of a block, the packed
// pairs PA = (A_f, A_f') and PC = (C_f, C_f') from the Re chunk (cos lane, sin lane) and PD, PB from the Im chunk.
// Per block: T = PA - PB, U = PC + PD (class q), T' = PA + PB, U' = PD - PC (class q'), four FADD2, and
// (S_q, S_q') += T^2 + U^2, T'^2 + U'^2, four FFMA2, each over the frame pair (all operands aligned register pairs:
// no moves, no swaps).
__device__ __forceinline__ void fold_acc_load(float2* w, const uint32_t (&v)[16]) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        const uint32_t* r = v + 8 * b;
        const float2 PA = make_float2(__uint_as_float(r[0]), __uint_as_float(r[1]));
        const float2 PC = make_float2(__uint_as_float(r[2]), __uint_as_float(r[3]));
        const float2 PD = make_float2(__uint_as_float(r[4]), __uint_as_float(r[5]));
        const float2 PB = make_float2(__uint_as_float(r[6]), __uint_as_float(r[7]));
        const float2 t = __fadd2_rn(PA, make_float2(-PB.x, -PB.y));
        const float2 u = __fadd2_rn(PC, PD);
        const float2 t2 = __fadd2_rn(PA, PB);
        const float2 u2 = __fadd2_rn(PD, make_float2(-PC.x, -PC.y));
        w[2 * b] = __ffma2_rn(u, u, __ffma2_rn(t, t, w[2 * b]));
        w[2 * b + 1] = __ffma2_rn(u2, u2, __ffma2_rn(t2, t2, w[2 * b + 1]));
    }
}

// one region of one bin: w[4 u + 2 b + {q, q'}] for class pair u of the thread (lanes 16 u + {i, i + 8} of the warp's
// quarter) and frame block b of the warp's 32 columns: two loads, the region released once both have landed, then
// the sums.
__device__ __forceinline__ void dasf_epi_region(float2* w, uint32_t taddr, uint32_t tf, uint32_t te,
                                                uint32_t parity, int& dbg) {
    wait_u32(tf, parity);
    tc_fence_after();
    const bool rec = blockIdx.x == 0 && threadIdx.x == 64;
    if (rec) { DAS_TRACE_REC(1, dbg) }
    uint32_t va[16], vb[16];
    tmem_ld16x256_x4(taddr, va);
    tmem_ld16x256_x4(taddr + (16u << 16), vb);
    tmem_ld_wait();
    tc_fence_before();
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e mbarrier.arrive.shared::cluster.b64 _, [%0];\n\t}" ::"r"(te)
                 : "memory");
    if (rec) { DAS_TRACE_REC(2, dbg) }
    ++dbg;
    fold_acc_load(w, va);
    fold_acc_load(w + 4, vb);
}

template <int ME>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(DASF_THREADS, 1)
    das_fold_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmE, DasFParams p) {
    using C = DasFCfg<ME>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t full[C::NST], empty[C::NST], tfull[4], tempty[4];
    __shared__ uint32_t tmem_slot;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));

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
        for (int a = 0; a < 4; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 2 * DASF_EW);
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_2sm<512>(&tmem_slot);
    if (warp == 1 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmE);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = pair; t < units; t += n_pairs) {
                int rt, ft;
                das_unit_f(p, t, rt, ft);
                const int arow = rt * 256 + (int)rank * 128;
                const int64_t erow = 2 * ((int64_t)ft * DASF_BF + (int64_t)rank * 64);   // 2 rows per frame
                for (int c = p.c_lo; c < p.c_hi; ++c) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE);
                    uint8_t* st = smem + stage * C::STAGE;
                    tma_load_2d_2sm(st, &tmA, 0, (int32_t)((int64_t)c * p.R_pad + arow), &full[stage]);
                    tma_load_2d_2sm(st + C::TILE, &tmE, 0, (int32_t)((int64_t)c * 2 * p.F_pad + erow), &full[stage]);
                    if (++stage == C::NST) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {
            const uint32_t idesc = umma_idesc_f16(256, DAS_RCOLS);
            const uint32_t a_lo0 = umma_desc_lo(smem_u32(smem)), b_lo0 = umma_desc_lo(smem_u32(smem + C::TILE));
            constexpr uint32_t HALF_B = (uint32_t)((64 * 128) >> 4);   // B rows 64..127 (frames 32..63 of the CTA)
            int stage = 0, acc = 0, dbg_step = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int t = pair; t < units; t += n_pairs) {
                for (int c = p.c_lo; c < p.c_hi; ++c) {
                    mbar_wait(&full[stage], phase);
                    const uint32_t so = (uint32_t)(stage * (C::STAGE >> 4));
                    const int kb0 = max(p.k_lo, c * C::BPR), kb1 = min(p.k_hi, c * C::BPR + C::BPR);
                    for (int k = kb0; k < kb1; ++k) {
                        const uint32_t ko = (uint32_t)((k - c * C::BPR) * (2 * ME / 16));   // bin's K offset
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf) {
                            const int r = 2 * acc + hf;
                            mbar_wait(&tempty[r], acc_phase ^ 1);
                            tc_fence_after();
                            if (blockIdx.x == 0 && lane == 0) { DAS_TRACE_REC(0, dbg_step) }
                            ++dbg_step;
                            das_mma<C::NK>(tmem_base + (uint32_t)(r * DAS_RCOLS), a_lo0 + so + ko,
                                           b_lo0 + so + hf * HALF_B + ko, C::HI, idesc);
                            umma_commit_2sm_warp(&tfull[r], 0x3);
                        }
                        if (++acc == 2) {
                            acc = 0;
                            acc_phase ^= 1;
                        }
                    }
                    umma_commit_2sm_warp(&empty[stage], 0x3);
                    if (++stage == C::NST) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else {
        // lane quarter g, column quarter h: class pairs u = 0, 1 (lanes 32 g + 16 u + {i, i + 8}), columns 32 h .. 32 h + 31
        // of each region (two blocks of 8 frames)
        const int g = warp & 3, h = (warp - 2) >> 2;
        const uint32_t tb = tmem_base + ((uint32_t)(g * 32) << 16) + (uint32_t)(h * 32);
        const uint32_t te = mapa_u32(smem_u32(&tempty[0]), 0);
        const uint32_t tf = smem_u32(&tfull[0]);
        int acc = 0, dbg = 0;
        uint32_t ph = 0;
        float2 w[16];                      // [hf][u][b][q, q']: partial sums over a frame pair
        for (int t = pair; t < units; t += n_pairs) {
            int rt, ft;
            das_unit_f(p, t, rt, ft);
#pragma unroll
            for (int i = 0; i < 16; ++i) w[i] = make_float2(0.f, 0.f);
            int k = 0;
            if (acc == 1 && k < nbins) {
                dasf_epi_region(w, tb + 2 * DAS_RCOLS, tf + 16, te + 16, ph, dbg);
                dasf_epi_region(w + 8, tb + 3 * DAS_RCOLS, tf + 24, te + 24, ph, dbg);
                ph ^= 1;
                acc = 0;
                ++k;
            }
            for (; k + 1 < nbins; k += 2) {
                dasf_epi_region(w, tb, tf, te, ph, dbg);
                dasf_epi_region(w + 8, tb + DAS_RCOLS, tf + 8, te + 8, ph, dbg);
                dasf_epi_region(w, tb + 2 * DAS_RCOLS, tf + 16, te + 16, ph, dbg);
                dasf_epi_region(w + 8, tb + 3 * DAS_RCOLS, tf + 24, te + 24, ph, dbg);
                ph ^= 1;
            }
            if (k < nbins) {
                dasf_epi_region(w, tb, tf, te, ph, dbg);
                dasf_epi_region(w + 8, tb + DAS_RCOLS, tf + 8, te + 8, ph, dbg);
                acc = 1;
            }
            // classes of the thread's two class pairs
            int cq_[2], cp_[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int pr = rt * 128 + (int)rank * 64 + 8 * (2 * g + u) + (lane >> 2);
                cq_[u] = pr < p.fold_rows ? __ldg(p.fold_cls + pr) : -1;
                cp_[u] = pr < p.fold_rows ? __ldg(p.fold_cls + p.fold_rows + pr) : -1;
            }
            // per frame i = 4 hf + 2 b + e: best of the 4 candidates (class pairs u, classes q / q'), then of the 8
            // threads sharing lane % 4
            unsigned long long key[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int hf = i >> 2, bb = (i >> 1) & 1, e = i & 1;
                unsigned long long best = 0ull;
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const float2 sq = w[8 * hf + 4 * u + 2 * bb];
                    const float2 sp = w[8 * hf + 4 * u + 2 * bb + 1];
                    const unsigned long long kq = cq_[u] >= 0 ? make_key(e ? sq.y : sq.x, (uint32_t)cq_[u]) : 0ull;
                    const unsigned long long kp = cp_[u] >= 0 ? make_key(e ? sp.y : sp.x, (uint32_t)cp_[u]) : 0ull;
                    best = kq > best ? kq : best;
                    best = kp > best ? kp : best;
                }
                key[i] = best;
            }
#pragma unroll
            for (int xx = 4; xx <= 16; xx <<= 1) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const unsigned long long o = __shfl_xor_sync(0xffffffffu, key[i], xx);
                    key[i] = key[i] > o ? key[i] : o;
                }
            }
            // region hf column 32 h + 8 j + 2 (lane % 4) + e is B row 64 hf + 32 (h & 1) + ... of the leader (h < 2) or
            // peer (h >= 2): frame 64 (h >> 1) + 32 hf + 16 (h & 1) + 8 (j / 2) + 2 (lane % 4) + e of the unit's 128
            // (16-row blocks: 8 Re rows, 8 Im rows per 8 frames); key i is written by the thread with lane / 4 == i
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (i == (lane >> 2)) {
                    const int f = ft * DASF_BF + 64 * (h >> 1) + 32 * (i >> 2) + 16 * (h & 1) + 8 * ((i >> 1) & 1) +
                                  2 * (lane & 3) + (i & 1);
                    if (f < p.F && key[i] != 0ull) atomicMax(&p.keys[f], key[i]);
                }
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
template <int ME, int BPC, bool FOLD>
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
    if constexpr (FOLD) {
        // E16[c][16 (f / 8) + (f % 8)] = Re e of the chunk's bins, row + 8 = Im e: 128-byte rows [bin t: mics
        // 0..ME-1]; blocks of 16 rows per 8 frames (das_fold_kernel's epilogue pairs frames, not Re / Im)
        uint4* rre = reinterpret_cast<uint4*>(E16 + ((int64_t)c * 2 * F_pad + 16 * (int64_t)(f >> 3) + (f & 7)) * 64);
        uint4* rim = rre + 8 * 8;
#pragma unroll
        for (int t = 0; t < BPC; ++t) {
#pragma unroll
            for (int i = 0; i < ME / 8; ++i) {
                rre[t * (ME / 8) + i] = make_uint4(re[t][4 * i], re[t][4 * i + 1], re[t][4 * i + 2], re[t][4 * i + 3]);
                rim[t * (ME / 8) + i] = make_uint4(im[t][4 * i], im[t][4 * i + 1], im[t][4 * i + 2], im[t][4 * i + 3]);
            }
        }
    } else {
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
}

// ---------------------------------------------------------------- steering operand (setup, float64)
// A16[k][r][0..2ME): rows in groups of 16, 8 classes per group: row r = 16 G + i holds, for class c = 8 G + (i % 8),
// Re a_c = [cos phi_cm | -sin phi_cm] if i < 8 and Im a_c = [sin phi_cm | cos phi_cm] if i >= 8 (TMEM lanes i and
// i + 8 reach the same epilogue thread, see tmem_ld16x256_x4); phi_cm = 2 pi k delta_cm / N in float64 (delta_cm:
// class c's arrival delays in samples, relative to the earliest microphone); classes >= Q_eff and microphones >= M
// are zero.  Thread per (row, bin).
__global__ void das_steer_kernel(const double* __restrict__ delay, int Q_eff, int M, int ME, int N, int R_pad,
                                 __half* __restrict__ A16) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = blockIdx.y;
    if (r >= R_pad) return;
    __half* row = A16 + ((int64_t)k * R_pad + r) * (2 * ME);
    const int c = 8 * (r >> 4) + (r & 7), v = (r >> 3) & 1;   // 16-row groups: Re a of 8 classes, then their Im a
    for (int m = 0; m < ME; ++m) {
        double sn = 0.0, cs = 0.0;
        if (c < Q_eff && m < M) sincospi(2.0 * (double)k * delay[(int64_t)c * M + m] / (double)N, &sn, &cs);
        row[m] = __double2half(v == 0 ? cs : sn);
        row[ME + m] = __double2half(v == 0 ? -sn : cs);
    }
}

// folded steering operand A16[c][r][BPC * ME] (setup, float64): row r = 16 G + i is, for class pair
// p = 8 G + (i % 8), cos phi_pm (i < 8) or sin phi_pm (i >= 8) for the chunk's bins t = 0..BPC-1 at halves
// t * ME + m, phi_pm = 2 pi k delta_pm / N with delta_pm the delays of the pair's first class (d_fold_cls[0][p]);
// pairs >= fold_rows, microphones >= M and bins >= Kb are zero.  Thread per (row, chunk).
__global__ void das_fold_steer_kernel(const double* __restrict__ delay, int fold_rows, int M, int ME, int BPC, int N,
                                      int Kb, int R_pad, __half* __restrict__ A16) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    const int c = blockIdx.y;
    if (r >= R_pad) return;
    __half* row = A16 + ((int64_t)c * R_pad + r) * 64;
    const int pr = 8 * (r >> 4) + (r & 7), v = (r >> 3) & 1;
    for (int t = 0; t < BPC; ++t) {
        const int k = c * BPC + t;
        for (int m = 0; m < ME; ++m) {
            double sn = 0.0, cs = 0.0;
            if (pr < fold_rows && m < M && k < Kb) sincospi(2.0 * (double)k * delay[(int64_t)pr * M + m] / (double)N, &sn, &cs);
            row[t * ME + m] = __double2half(v == 0 ? cs : sn);
        }
    }
}

svdphat_status setup_das_fold_operand(Plan& p, const double* h_delay_fold) {
    p.das_me = das_me(p.M);
    if (p.das_me < 16 || p.das_me != p.L.Mi || 2 * p.das_me * p.L.bpc != 128) {
        set_error("folded delay-and-sum needs 128-byte chunk rows (das_me >= 16)");
        return SVDPHAT_UNSUPPORTED;
    }
    p.das_rows = (2 * p.fold_rows + 255) / 256 * 256;
    const int64_t bytes = (int64_t)p.L.n_chunks * p.das_rows * 128;
    double* d_delay = nullptr;
    SVD_CUDA_TRY(cudaMalloc(&d_delay, (size_t)p.fold_rows * p.M * sizeof(double)));
    cudaError_t e = cudaMemcpy(d_delay, h_delay_fold, (size_t)p.fold_rows * p.M * sizeof(double), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&p.d_A16, bytes);
    if (e == cudaSuccess) {
        das_fold_steer_kernel<<<dim3((p.das_rows + 127) / 128, p.L.n_chunks), 128>>>(
            d_delay, p.fold_rows, p.M, p.das_me, p.L.bpc, p.N, p.Kb, p.das_rows, p.d_A16);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(d_delay);
    SVD_CUDA_TRY(e);
    p.bytes_A = bytes;
    return SVDPHAT_OK;
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
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(das_fold_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, DasFCfg<16>::SMEM);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(das_fold_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, DasFCfg<32>::SMEM);
    return e;
}

bool das_active(const Plan& p, int F) {
    // enough 256 x 256 units to give every CTA pair work (small batches keep the split-K W GEMM), or forced
    if (!p.d_A16 || !p.d_E16) return false;
    if (p.options & SVDPHAT_OPT_DAS) return true;
    const int bf = p.das_fold ? DASF_BF : DAS_BN;
    const int64_t units = (int64_t)(p.das_rows / 256) * ((F + bf - 1) / bf);
    return units >= p.num_sms / 2;
}

cudaError_t launch_das_bins(const Plan& p, const Band& b, int F, cudaStream_t s) {
    if (F <= 0 || b.c_hi <= b.c_lo) return cudaSuccess;
    const dim3 grid((F + 127) / 128, b.c_hi - b.c_lo);
    const int Mi = p.L.Mi;
    if (p.das_fold) {
        if (p.das_me == 16)
            das_bins_kernel<16, 4, true><<<grid, 128, 0, s>>>(p.d_P16, F, p.F_pad, Mi, p.M, p.Kb, b.c_lo, p.d_E16);
        else
            das_bins_kernel<32, 2, true><<<grid, 128, 0, s>>>(p.d_P16, F, p.F_pad, Mi, p.M, p.Kb, b.c_lo, p.d_E16);
        return cudaGetLastError();
    }
    switch (p.das_me) {
        case 8:
            if (p.L.bpc != 4) return cudaErrorInvalidValue;
            das_bins_kernel<8, 4, false><<<grid, 128, 0, s>>>(p.d_P16, F, p.F_pad, Mi, p.M, p.Kb, b.c_lo, p.d_E16);
            break;
        case 16:
            if (p.L.bpc != 4) return cudaErrorInvalidValue;
            das_bins_kernel<16, 4, false><<<grid, 128, 0, s>>>(p.d_P16, F, p.F_pad, Mi, p.M, p.Kb, b.c_lo, p.d_E16);
            break;
        default:
            if (p.L.bpc != 2) return cudaErrorInvalidValue;
            das_bins_kernel<32, 2, false><<<grid, 128, 0, s>>>(p.d_P16, F, p.F_pad, Mi, p.M, p.Kb, b.c_lo, p.d_E16);
    }
    return cudaGetLastError();
}

cudaError_t launch_das(const Plan& p, const Band& b, int F, cudaStream_t s) {
    if (F <= 0 || b.k_hi <= b.k_lo) return cudaSuccess;
    if (p.das_fold) {
        DasFParams dp;
        dp.F = F;
        dp.F_pad = p.F_pad;
        dp.R_pad = p.das_rows;
        dp.k_lo = b.k_lo;
        dp.k_hi = b.k_hi;
        dp.c_lo = b.c_lo;
        dp.c_hi = b.c_hi;
        dp.n_rt = p.das_rows / 256;
        dp.n_ft = (F + DASF_BF - 1) / DASF_BF;
        dp.fold_rows = p.fold_rows;
        dp.fold_cls = p.d_fold_cls;
        dp.keys = p.d_keys;
        const int units = dp.n_rt * dp.n_ft;
        const int grid = 2 * std::min(units, p.num_sms / 2);
        if (p.das_me == 16)
            das_fold_kernel<16><<<grid, DASF_THREADS, DasFCfg<16>::SMEM, s>>>(p.tm_A, p.tm_E, dp);
        else
            das_fold_kernel<32><<<grid, DASF_THREADS, DasFCfg<32>::SMEM, s>>>(p.tm_A, p.tm_E, dp);
        return cudaGetLastError();
    }
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
