// gemm_tc.cu — the projection GEMMs of SRP-PHAT and SVD-PHAT on the 5th-generation tensor cores (tcgen05).
//
//   mode 0 (SRP, eq. 9):   Y[q,f] = Re{W_q . X_f} = sum_kappa W16[q,kappa] * x16[f,kappa]
//                                        + fused argmax over q (eq. 6), lowest index on ties.
//   mode 1 (SVD, eq. 12):  [Z_r; Z_i][d,f] = sum_kappa V16[d,kappa] * x16[f,kappa]   -> Z32
//   mode 2 (SVD, eqs. 14-15): s[q,f] = Re{Dhat_q . Zhat_f} over split-FP16 operands
//                                        + fused argmax over q.
//
// A operand (M side, 128 rows per tile) = W16 / V16 / R16 streamed by TMA (SWIZZLE_128B, K-major).
// B operand (N side, 256 frames per tile) = in modes 0/1 the PHAT cross-spectrum X (eqs. 3, 7) built in shared
// memory by 8 producer warps from the per-channel unit phasors (it never exists in HBM); in mode 2 Zhat via TMA.
// Accumulators: FP32 in TMEM, two 256-column buffers so the epilogue of tile t overlaps the MMAs of tile t+1.
// Warp roles: 0 TMA, 1 MMA issuer (one thread), 2..5 epilogue (TMEM lane groups 2,3,0,1), 6..13 producer.
#include <cuda_fp16.h>

#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace svdphat {

constexpr int BM = 128;                    // tile rows (A)
constexpr int BN = 256;                    // tile frames (B)
constexpr int BK = 64;                     // fp16 per slab row = 128 B = one swizzle atom row
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;       // 16 KB
constexpr int B_BYTES = BN * BK * 2;       // 32 KB
constexpr int NUM_PRODUCER_WARPS = 8;
constexpr int SMEM_BYTES = 1024 + STAGES * (A_BYTES + B_BYTES) + 256;

struct GemmParams {
    const uint8_t* P16;                    // phasors (modes 0/1)
    int F;                                 // valid frames
    int F_pad;
    int n_chunks;
    int n_slabs;                           // K / 64
    int m_tiles, n_tiles;
    int rows_valid;                        // rows of A that are real (mask for the argmax / store)
    unsigned long long* keys;              // argmax keys [F]
    float* Z;                              // mode 1 output [ksplit][F_pad][ldz] (partial sums per K split)
    int ldz;
    int ksplit;                            // K splits (mode 1 only; splits fall on chunk boundaries)
    int spc;                               // slabs per chunk
    int prefetch;                          // 0 none, 1 L2 prefetch of the next chunk's phasors, 2 same evict_last
    int bn;                                // frames per tile of the CTA-pair kernel (multiple of 32, <= 256)
    int c_lo, c_hi;                        // active bin-chunk range (band limit, NEXT-3); producer modes only
    const int* fold_cls;                   // folded SRP (FOLD kernels): [2][fold_rows] classes of a - b / a + b
    int fold_rows;
    // part projection (gemm2p_kernel): ring stages, stage bytes, MMAs per K step and their N, Z_i column offset
    int stages, stage_bytes, n_mma, nmma, zh;
    // FP16 search (mode 2): candidate lists (FP16 score, class) of rows within SEARCH_TAU of the running maximum
    unsigned long long* cand;
    int* ccnt;
};

// Work unit t -> output tile (m, n) and the slab / chunk range of its K split.
struct Unit {
    int m, n, s, c0, c1, k0, k1;
};
__device__ __forceinline__ Unit unit_of(const GemmParams& p, int t) {
    Unit u;
    u.s = t % p.ksplit;
    const int tile = t / p.ksplit;
    u.m = tile / p.n_tiles;
    u.n = tile % p.n_tiles;
    if (p.c_hi <= p.c_lo) {                // TMA-B modes: the whole contraction
        u.c0 = u.c1 = 0;
        u.k0 = 0;
        u.k1 = p.n_slabs;
    } else {                               // producer modes: chunk range [c_lo, c_hi) split ksplit ways
        const int nc = p.c_hi - p.c_lo;
        u.c0 = p.c_lo + (int)((int64_t)u.s * nc / p.ksplit);
        u.c1 = p.c_lo + (int)((int64_t)(u.s + 1) * nc / p.ksplit);
        u.k0 = u.c0 * p.spc;
        u.k1 = u.c1 * p.spc;
    }
    return u;
}

// Work-unit order of the frames-on-M projection (gemm2f_kernel): split slowest, then V tile, frame tile fastest, so
// the pairs in flight share one V slab range and the split's phasor records stay L2-resident across the V tiles.
__device__ __forceinline__ Unit unit_of_f(const GemmParams& p, int t) {
    Unit u;
    const int per_s = p.m_tiles * p.n_tiles;
    u.s = t / per_s;
    const int r = t - u.s * per_s;
    u.n = r / p.m_tiles;
    u.m = r - u.n * p.m_tiles;
    const int nc = p.c_hi - p.c_lo;
    u.c0 = p.c_lo + (int)((int64_t)u.s * nc / p.ksplit);
    u.c1 = p.c_lo + (int)((int64_t)(u.s + 1) * nc / p.ksplit);
    u.k0 = u.c0 * p.spc;
    u.k1 = u.c1 * p.spc;
    return u;
}

// ---------------------------------------------------------------- compile-time pair enumeration over Mi mics
template <int Mi>
struct PairTab {
    int i[Mi * (Mi - 1) / 2 + 1];
    int j[Mi * (Mi - 1) / 2 + 1];
    int last[Mi];                          // last pair index that uses mic m (its record is dead after it)
    constexpr PairTab() : i(), j(), last() {
        int p = 0;
        for (int a = 0; a < Mi; ++a)
            for (int b = a + 1; b < Mi; ++b) {
                i[p] = a;
                j[p] = b;
                last[a] = p;
                last[b] = p;
                ++p;
            }
    }
};

__device__ __forceinline__ uint32_t h2mul(uint32_t a, uint32_t b) {
    __half2 r = __hmul2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t h2fma(uint32_t a, uint32_t b, uint32_t c) {
    __half2 r = __hfma2(*reinterpret_cast<__half2*>(&a), *reinterpret_cast<__half2*>(&b),
                        *reinterpret_cast<__half2*>(&c));
    return *reinterpret_cast<uint32_t*>(&r);
}


template <int Mi, int BPC, int MODE>
__global__ void __launch_bounds__(32 * (6 + NUM_PRODUCER_WARPS), 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmParams p) {
    // MODE 0: producer B + argmax, 1: producer B + store, 2: TMA B + argmax, 3: TMA B + store
    constexpr bool kProducer = (MODE == 0 || MODE == 1);
    // TMA-B modes have no producer warps: warps 6-9 join the epilogue (frames [128, 256) of the tile), warps 2-5 take
    // frames [0, 128) (each lane group of TMEM is read by two warps: warp w may access lanes 32 (w % 4) ..)
    constexpr int kEpiWarps = kProducer ? 4 : 8;
    constexpr int kPairs = Mi * (Mi - 1) / 2;
    constexpr int kUnitsRaw = (BPC == 4) ? kPairs : (kPairs + 1) / 2;
    constexpr int kU = (kUnitsRaw + 7) / 8 * 8;        // units per chunk
    constexpr uint32_t kIdesc = umma_idesc_f16(BM, BN);

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int n_tiles_total = p.m_tiles * p.n_tiles * p.ksplit;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], kProducer ? 1 + NUM_PRODUCER_WARPS : 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], kEpiWarps);
        }
        fence_mbar_init();
    }
    if (warp == 0) {
        tmem_alloc<512>(tmem_slot);
    }
    if (warp == 1 && lane == 0) {
        tma_prefetch_desc(&tmA);
        if (!kProducer) tma_prefetch_desc(&tmB);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ============================================================ TMA producer (A, and B in mode 2)
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t bytes = kProducer ? A_BYTES : (A_BYTES + B_BYTES);
            for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
                const Unit w = unit_of(p, t);
                for (int ks = w.k0; ks < w.k1; ++ks) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_arrive_expect_tx(&full[stage], bytes);
                    tma_load_2d(sA + stage * A_BYTES, &tmA, ks * BK, w.m * BM, &full[stage]);
                    if (!kProducer) tma_load_2d(sB + stage * B_BYTES, &tmB, ks * BK, w.n * BN, &full[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ============================================================ MMA issuer (converged warp, elect.sync in the asm)
        const uint64_t adesc0 = umma_desc_sw128(smem_u32(sA)), bdesc0 = umma_desc_sw128(smem_u32(sB));
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
            mbar_wait(&tempty[acc], acc_phase ^ 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            const Unit w = unit_of(p, t);
            for (int ks = w.k0; ks < w.k1; ++ks) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                const uint64_t ad = adesc0 + (uint64_t)(stage * (A_BYTES >> 4));
                const uint64_t bd = bdesc0 + (uint64_t)(stage * (B_BYTES >> 4));
                const uint32_t acc0 = ks != w.k0;
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                    umma_f16_warp(d_tmem, ad + 2 * kk, bd + 2 * kk, kIdesc, kk ? 1u : acc0);
                umma_commit_warp(&empty[stage]);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            umma_commit_warp(&tfull[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp < 2 + kEpiWarps) {
        // ============================================================ epilogue: TMEM -> registers -> argmax / Z
        const int g = warp & 3;                                    // TMEM lane group this warp may access
        const int jbeg = (warp < 6) ? 0 : BN / 2, jend = (kEpiWarps == 4 || warp >= 6) ? BN : BN / 2;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
            const Unit w = unit_of(p, t);
            const int m = w.m, n = w.n;
            float* Zs = p.Z + (int64_t)w.s * p.F_pad * p.ldz;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int row = m * BM + g * 32 + lane;
            const bool row_ok = row < p.rows_valid;
#pragma unroll 1
            for (int j0 = jbeg; j0 < jend; j0 += 32) {
                uint32_t r[32];
                const int f0 = n * BN + j0;
                const bool fok = f0 + lane < p.F;
                // the frame's running maximum (a possibly stale read is a lower bound: more candidates, never fewer)
                const unsigned long long prev = (MODE == 2 && fok) ? __ldcg(&p.keys[f0 + lane]) : 0ull;
                tmem_ld_32x32b_x32(tmem_base + (uint32_t(g * 32) << 16) + acc * BN + j0, r);
                tmem_ld_wait();
                if (MODE == 1 || MODE == 3) {
                    if (row_ok) {
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            if (f0 + jj < p.F) Zs[(int64_t)(f0 + jj) * p.ldz + row] = __uint_as_float(r[jj]);
                        }
                    }
                } else if (MODE == 2) {
                    // FP16 search: only the frame's running FP16 maximum (the base of the candidate threshold) and the
                    // candidate rows leave the tile; the class of that maximum is never used (rescore_kernel decides
                    // among the candidates in FP32), so the column maximum over the warp's 32 rows is one
                    // redux.sync.max.f32 per frame instead of a u64 key transpose (ncu r02: the key epilogue issued
                    // ~3500 instructions per warp and tile, 21k cycles per tile against 5k of MMA; NaN inputs are
                    // ignored by the reduction and fail the >= below).
                    float mx = -INFINITY;
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) {
                        const float v = row_ok ? __uint_as_float(r[jj]) : -INFINITY;
                        const float m = warp_max_f32(v);
                        mx = lane == jj ? m : mx;
                    }
                    const float prev_f = prev ? o2f((uint32_t)(prev >> 32)) : -INFINITY;
                    // candidates of the exact rescore: rows within SEARCH_TAU of the running FP16 maximum.  The exact
                    // argmax q* has s16(q*) >= max16 - 2e >= running - SEARCH_TAU (e: FP16 error bound).
                    const float thr = fmaxf(prev_f, mx) - SEARCH_TAU;
                    const bool any = fok && mx > -INFINITY && mx >= thr;
                    if (any && mx > prev_f) atomicMax(&p.keys[f0 + lane], make_key(mx, 0u));
                    const uint32_t mask = __ballot_sync(0xffffffffu, any);
                    if (mask) {
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            if (mask & (1u << jj)) {
                                const float tj = __shfl_sync(0xffffffffu, thr, jj);
                                const float v = __uint_as_float(r[jj]);
                                if (row_ok && v >= tj) {
                                    const int idx = atomicAdd(&p.ccnt[f0 + jj], 1);
                                    if (idx < SEARCH_CAP)
                                        p.cand[(int64_t)(f0 + jj) * SEARCH_CAP + idx] = make_key(v, (uint32_t)row);
                                }
                            }
                        }
                    }
                } else {
                    unsigned long long k[32];
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) {
                        const float v = __uint_as_float(r[jj]);
                        k[jj] = (row_ok && v == v) ? make_key(v, (uint32_t)row) : 0ull;
                    }
                    const unsigned long long best = transpose_max32(k, lane);
                    if (fok && best != 0ull) atomicMax(&p.keys[f0 + lane], best);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (kProducer) {
        // ============================================================ B producer: X (eqs. 3, 7) from phasors
        constexpr PairTab<Mi> PT{};
        const int tp = (warp - 6) * 32 + lane;                    // frame row of the B tile: 0..255
        const uint32_t row_off = (uint32_t)((tp >> 3) * 1024 + (tp & 7) * 128);
        const uint32_t xr = (uint32_t)(tp & 7);
        int stage = 0;
        uint32_t phase = 0;
        constexpr int kUB = BPC * 4;                               // bytes per phasor record: bpc*2 halves
        for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
            const Unit w = unit_of(p, t);
            const int f = w.n * BN + tp;
            const bool valid = f < p.F;
#pragma unroll 1
            for (int c = w.c0; c < w.c1; ++c) {
                // e[m][w]: BPC=4 -> {Re k0k1, Re k2k3, Im k0k1, Im k2k3}; BPC=2 -> {Re k0k1, Im k0k1}
                uint32_t e[Mi][BPC];
                const uint8_t* src = p.P16 + ((int64_t)c * Mi * p.F_pad + f) * kUB;
#pragma unroll
                for (int m = 0; m < Mi; ++m) {
                    if (BPC == 4) {
                        uint4 v = valid ? __ldg(reinterpret_cast<const uint4*>(src + (int64_t)m * p.F_pad * kUB))
                                        : make_uint4(0, 0, 0, 0);
                        e[m][0] = v.x;
                        e[m][1] = v.y;
                        e[m][2 % BPC] = v.z;
                        e[m][3 % BPC] = v.w;
                    } else {
                        uint2 v = valid ? __ldg(reinterpret_cast<const uint2*>(src + (int64_t)m * p.F_pad * kUB))
                                        : make_uint2(0, 0);
                        e[m][0] = v.x;
                        e[m][1] = v.y;
                    }
                }
                // L2 prefetch of the next chunk's phasor records: the chunk-boundary reload then hits L2, well inside
                // the STAGES-deep smem buffer (ncu r01: chunk-boundary HBM latency starved the MMA warp).
                if (p.prefetch && valid && c + 1 < w.c1) {
                    const uint8_t* nsrc = src + (int64_t)Mi * p.F_pad * kUB;
                    if (p.prefetch == 2) {
#pragma unroll
                        for (int m = 0; m < Mi; ++m)
                            asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(nsrc + (int64_t)m * p.F_pad * kUB));
                    } else {
#pragma unroll
                        for (int m = 0; m < Mi; ++m)
                            asm volatile("prefetch.global.L2 [%0];" ::"l"(nsrc + (int64_t)m * p.F_pad * kUB));
                    }
                }
                uint32_t outw[4];
#pragma unroll
                for (int u = 0; u < kU; ++u) {
                    if ((u & 7) == 0) mbar_wait(&empty[stage], phase ^ 1);
                    if (BPC == 4) {
                        if (u < kPairs) {
                            const int a = PT.i[u], b = PT.j[u];
                            // x = e_a conj(e_b): Re = ra rb + ia ib, Im = ia rb - ra ib   (eq. 3)
                            const uint32_t nra01 = e[a][0] ^ 0x80008000u, nra23 = e[a][1 % BPC] ^ 0x80008000u;
                            outw[0] = h2fma(e[a][0], e[b][0], h2mul(e[a][2 % BPC], e[b][2 % BPC]));
                            outw[1] = h2fma(e[a][1 % BPC], e[b][1 % BPC], h2mul(e[a][3 % BPC], e[b][3 % BPC]));
                            outw[2] = h2fma(e[a][2 % BPC], e[b][0], h2mul(nra01, e[b][2 % BPC]));
                            outw[3] = h2fma(e[a][3 % BPC], e[b][1 % BPC], h2mul(nra23, e[b][3 % BPC]));
                        } else {
                            outw[0] = outw[1] = outw[2] = outw[3] = 0u;
                        }
                    } else {
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const int pp = 2 * u + h;
                            if (pp < kPairs) {
                                const int a = PT.i[pp], b = PT.j[pp];
                                const uint32_t nra = e[a][0] ^ 0x80008000u;
                                outw[2 * h + 0] = h2fma(e[a][0], e[b][0], h2mul(e[a][1], e[b][1]));
                                outw[2 * h + 1] = h2fma(e[a][1], e[b][0], h2mul(nra, e[b][1]));
                            } else {
                                outw[2 * h + 0] = outw[2 * h + 1] = 0u;
                            }
                        }
                    }
                    const uint32_t dst = smem_u32(sB + stage * B_BYTES) + row_off + ((((uint32_t)u & 7u) ^ xr) << 4);
                    st_shared_v4(dst, outw[0], outw[1], outw[2], outw[3]);
                    if ((u & 7) == 7) {
                        fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&full[stage]);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    }

    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

// ================================================================================================================
// CTA-pair variant (cta_group::2): one MMA computes a 256-row x 256-frame tile on two SMs.  CTA r of the pair
// TMA-loads rows [m*256 + 128r, +128) of A and its 4 producer warps build frames [n*256 + 128r, +128) of B; the
// even (leader) CTA issues tcgen05.mma.cta_group::2 for both.  Per SM this halves the shared-memory operand
// traffic of the 1-CTA kernel (ncu r01: ~192 B/clk/SM needed at full MMA rate), the reason for the pair.
// Warps: 0 TMA (+TMEM alloc), 1 MMA (leader), 2-5 epilogue (lane groups 2,3,0,1), 6-9 producer (produce_x_pair).
// ================================================================================================================
constexpr int STAGES2 = 6;
constexpr int A2_BYTES = 128 * BK * 2;                 // 16 KB: this CTA's half of the 256 A rows
constexpr int B2_BYTES = 128 * BK * 2;                 // 16 KB: this CTA's half of the 256 frames
constexpr int NPW2 = 4;                                // producer warps per CTA (128 frames)
constexpr int THREADS2 = 32 * (6 + NPW2);
constexpr int SMEM2_BYTES = 1024 + STAGES2 * (A2_BYTES + B2_BYTES) + 256;

// Producer warps of the CTA-pair kernels: this thread's frame row of the cross-spectrum X (eqs. 3, 7, PAPER.md:66,
// 99) for the bin chunks [w.c0, w.c1) of a work unit, written into the SW128 K-major operand ring sX (stage stride
// XB bytes, 8 units = one 64-element slab per stage).  The frame's phasors of the current chunk stay in registers.
// (Register double-buffering of the next chunk was tried and removed: the apparent 'load cost' was power - zeroed
// operands keep the clock high under the cap.)
// FOLD (antipodal folding, internal.h): a stage holds slab pair u/16 - its Re slab at offset 0 and its Im slab at
// SLAB - and unit u's Re / Im words go to byte 8*(u%16) of the swizzled row of each.
template <int Mi, int BPC, int NSTAGES, int XB, bool FOLD = false, int SLAB = XB>
__device__ __forceinline__ void produce_x_pair(const GemmParams& p, const Unit& w, int f, bool valid, uint8_t* sX,
                                               uint64_t* full, uint64_t* empty, int& stage, uint32_t& phase,
                                               uint32_t row_off, uint32_t xr) {
    static_assert(!FOLD || XB == 2 * SLAB, "a fold stage holds a Re slab and an Im slab");
    constexpr PairTab<Mi> PT{};
    constexpr int kPairs = Mi * (Mi - 1) / 2;
    constexpr int kUnitsRaw = (BPC == 4) ? kPairs : (kPairs + 1) / 2;
    constexpr int kU = (kUnitsRaw + 7) / 8 * 8;
    constexpr int kUB = BPC * 4;
    const int lane = threadIdx.x & 31;
    // e[m] = this frame's record of mic m for the current chunk.  Record m of chunk c+1 is loaded into e[m] right
    // after the last unit of chunk c that uses mic m, so the reloads are spread over the chunk and mostly complete
    // before the next chunk needs them (a chunk-start reload stalled the producer for a full memory round trip).
    uint32_t e[Mi][BPC];
    auto load_rec = [&](int m, const uint8_t* base) {
        if constexpr (BPC == 4) {
            const uint4 v = valid ? __ldg(reinterpret_cast<const uint4*>(base + (int64_t)m * p.F_pad * kUB))
                                  : make_uint4(0, 0, 0, 0);
            e[m][0] = v.x;
            e[m][1] = v.y;
            e[m][2] = v.z;
            e[m][3] = v.w;
        } else {
            const uint2 v = valid ? __ldg(reinterpret_cast<const uint2*>(base + (int64_t)m * p.F_pad * kUB))
                                  : make_uint2(0, 0);
            e[m][0] = v.x;
            e[m][1] = v.y;
        }
    };
    if (w.c0 < w.c1) {
        const uint8_t* src0 = p.P16 + ((int64_t)w.c0 * Mi * p.F_pad + f) * kUB;
#pragma unroll
        for (int m = 0; m < Mi; ++m) load_rec(m, src0);
    }
#pragma unroll 1
    for (int c = w.c0; c < w.c1; ++c) {
        const uint8_t* src = p.P16 + ((int64_t)c * Mi * p.F_pad + f) * kUB;
        const uint8_t* nxt = src + (int64_t)Mi * p.F_pad * kUB;
        const bool more = c + 1 < w.c1;
        if constexpr (BPC != 4) {          // M' = 32 (248 units): reload at the chunk start (a 32 x 248 unrolled
            if (c != w.c0) {               // schedule of progressive loads sends e[][] to local memory)
#pragma unroll
                for (int m = 0; m < Mi; ++m) load_rec(m, src);
            }
        }
        // L2 prefetch of the next chunk's records: the chunk-boundary reload then hits L2 (with N = 160 V rows the
        // 3-deep ring of slab pairs holds ~2k MMA cycles, less than an HBM round trip)
        if (p.prefetch && valid && c + 1 < w.c1) {
            const uint8_t* nsrc = src + (int64_t)Mi * p.F_pad * kUB;
#pragma unroll
            for (int m = 0; m < Mi; ++m)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(nsrc + (int64_t)m * p.F_pad * kUB));
        }
        uint32_t outw[4], pend[4];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if constexpr (FOLD) {
                if ((u & 15) == 0) mbar_wait(&empty[stage], phase ^ 1);
            } else {
                if ((u & 7) == 0) mbar_wait(&empty[stage], phase ^ 1);
            }
            if constexpr (BPC == 4) {
                if (u < kPairs) {
                    const int a = PT.i[u], b = PT.j[u];
                    const uint32_t nra01 = e[a][0] ^ 0x80008000u, nra23 = e[a][1] ^ 0x80008000u;
                    outw[0] = h2fma(e[a][0], e[b][0], h2mul(e[a][2], e[b][2]));
                    outw[1] = h2fma(e[a][1], e[b][1], h2mul(e[a][3], e[b][3]));
                    outw[2] = h2fma(e[a][2], e[b][0], h2mul(nra01, e[b][2]));
                    outw[3] = h2fma(e[a][3], e[b][1], h2mul(nra23, e[b][3]));
                } else {
                    outw[0] = outw[1] = outw[2] = outw[3] = 0u;
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int pp = 2 * u + h;
                    if (pp < kPairs) {
                        const int a = PT.i[pp], b = PT.j[pp];
                        const uint32_t nra = e[a][0] ^ 0x80008000u;
                        outw[2 * h + 0] = h2fma(e[a][0], e[b][0], h2mul(e[a][1], e[b][1]));
                        outw[2 * h + 1] = h2fma(e[a][1], e[b][0], h2mul(nra, e[b][1]));
                    } else {
                        outw[2 * h + 0] = outw[2 * h + 1] = 0u;
                    }
                }
            }
            // records whose last use in this chunk was this unit: load the next chunk's (compile-time tests)
            if constexpr (BPC == 4) {
#pragma unroll
                for (int m = 0; m < Mi; ++m)
                    if (PT.last[m] == u && more) load_rec(m, nxt);
            }
            if constexpr (FOLD) {
                // Re words: BPC 4 {Re k0k1, Re k2k3} = outw[0..1]; BPC 2 {Re p0, Re p1} = outw[0], outw[2].
                // Units 2j and 2j+1 share the 16-byte chunk j of a slab row: one STS.128 per slab per unit pair
                // (two STS.64 per unit were 4-way bank-conflicted: 505M conflicts, tensor pipe 59%).
                const uint32_t re0 = outw[0], re1 = (BPC == 4) ? outw[1] : outw[2];
                const uint32_t im0 = (BPC == 4) ? outw[2] : outw[1], im1 = outw[3];
                if ((u & 1) == 0) {
                    pend[0] = re0;
                    pend[1] = re1;
                    pend[2] = im0;
                    pend[3] = im1;
                } else {
                    const uint32_t pos = row_off + (((((uint32_t)u & 15u) >> 1) ^ xr) << 4);
                    st_shared_v4(smem_u32(sX + stage * XB) + pos, pend[0], pend[1], re0, re1);
                    st_shared_v4(smem_u32(sX + stage * XB + SLAB) + pos, pend[2], pend[3], im0, im1);
                }
                if ((u & 15) == 15 || u == kU - 1) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(&full[stage], 0);
                    if (++stage == NSTAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            } else {
                const uint32_t dst = smem_u32(sX + stage * XB) + row_off + ((((uint32_t)u & 7u) ^ xr) << 4);
                st_shared_v4(dst, outw[0], outw[1], outw[2], outw[3]);
                if ((u & 7) == 7) {
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(&full[stage], 0);   // the leader's barrier
                    if (++stage == NSTAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    }
}

// FOLD (SRP with antipodal folding): A = fold rows, slabs alternate Re (accumulator a, TMEM columns [0,256)) and Im
// (accumulator b, [256,512)); the epilogue scores a - b for class fold_cls[row] and a + b for fold_cls[R + row].
// Both accumulators are live for the whole tile, so the epilogue of tile t is not overlapped with tile t+1 (~2 us
// per ~0.5 ms tile at cfg3).
template <int Mi, int BPC, int MODE, bool FOLD = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS2, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmParams p) {
    constexpr bool kProducer = (MODE != 2);
    static_assert(!FOLD || kProducer, "folding applies to the producer (SRP) modes");
    constexpr int kUnitsRaw = (BPC == 4) ? Mi * (Mi - 1) / 2 : (Mi * (Mi - 1) / 2 + 1) / 2;
    constexpr int kU = (kUnitsRaw + 7) / 8 * 8;
    constexpr bool kHalfPair = FOLD && (kU % 16 == 8);      // last slab pair of a chunk holds 8 units: 2 MMAs
    // FOLD stages hold a slab pair (Re, Im of the same 16 units): one barrier round trip per 8 MMAs, same ring bytes
    constexpr int kSt = FOLD ? STAGES2 / 2 : STAGES2;
    constexpr int kSP = FOLD ? 2 : 1;                       // slabs per stage
    constexpr int kAS = kSP * A2_BYTES, kBS = kSP * B2_BYTES;

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + kSt * kAS;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + kSt * kBS);
    uint64_t* empty = full + kSt;
    uint64_t* tfull = empty + kSt;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int units = p.m_tiles * p.n_tiles * p.ksplit;   // m_tiles counts 256-row pair tiles
    const int bn = p.bn, hb = p.bn / 2;                    // frames per pair tile / per CTA
    const uint32_t idesc = umma_idesc_f16(256, (uint32_t)bn);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kSt; ++s) {
            // leader: its TMA (expect_tx) + the producer warps of both CTAs (peer ones arrive remotely)
            mbar_init(&full[s], kProducer ? 1 + 2 * NPW2 : 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8);
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_2sm<512>(tmem_slot);
    if (warp == 1 && lane == 0) {
        tma_prefetch_desc(&tmA);
        if (!kProducer) tma_prefetch_desc(&tmB);
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t bytes = kSP * (kProducer ? 2 * A2_BYTES : 2 * (A2_BYTES + B2_BYTES));
            for (int t = pair; t < units; t += n_pairs) {
                const Unit w = unit_of(p, t);
                for (int ks = w.k0; ks < w.k1; ks += kSP) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
#pragma unroll
                    for (int j = 0; j < kSP; ++j) {
                        tma_load_2d_2sm(sA + stage * kAS + j * A2_BYTES, &tmA, (ks + j) * BK,
                                        w.m * 256 + (int)rank * 128, &full[stage]);
                        if (!kProducer)
                            tma_load_2d_2sm(sB + stage * kBS + j * B2_BYTES, &tmB, (ks + j) * BK,
                                            w.n * bn + (int)rank * hb, &full[stage]);
                    }
                    if (++stage == kSt) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // MMA issuer: the whole warp, converged; elect.sync inside the issue asm picks one lane.  Descriptors advance by constant offsets (stage: bytes >> 4; K step of 16 halves:
        // 32 B >> 4 = 2) and the fold's slab parity / half-pair test use counters, so the per-slab issue cost stays
        // well under the 512 MMA cycles of a slab (ncu r01: an integer modulo here left the tensor pipe 40% idle).
        if (leader) {
            const uint64_t adesc0 = umma_desc_sw128(smem_u32(sA)), bdesc0 = umma_desc_sw128(smem_u32(sB));
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = pair; t < units; t += n_pairs) {
                const Unit w = unit_of(p, t);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                int lp = 0;                                         // slab pair within the bin chunk (FOLD)
                const int n_lp = p.spc / 2;
                for (int ks = w.k0; ks < w.k1; ks += kSP) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t ad = adesc0 + (uint64_t)(stage * (kAS >> 4));
                    const uint64_t bd = bdesc0 + (uint64_t)(stage * (kBS >> 4));
                    if constexpr (FOLD) {
                        const bool half = kHalfPair && lp == n_lp - 1;
                        const uint32_t acc0 = ks != w.k0;
#pragma unroll
                        for (int part = 0; part < 2; ++part) {          // Re slab -> a, Im slab -> b
                            const uint32_t d_tmem = tmem_base + (uint32_t)part * BN;
                            const uint64_t pa = ad + part * (A2_BYTES >> 4), pb = bd + part * (B2_BYTES >> 4);
                            umma_f16_2sm_warp(d_tmem, pa, pb, idesc, acc0);
                            umma_f16_2sm_warp(d_tmem, pa + 2, pb + 2, idesc, 1u);
                            if (!half) {
                                umma_f16_2sm_warp(d_tmem, pa + 4, pb + 4, idesc, 1u);
                                umma_f16_2sm_warp(d_tmem, pa + 6, pb + 6, idesc, 1u);
                            }
                        }
                        if (++lp == n_lp) lp = 0;
                    } else {
                        const uint32_t d_tmem = tmem_base + acc * BN;
                        const uint32_t acc0 = ks != w.k0;
#pragma unroll
                        for (int kk = 0; kk < BK / 16; ++kk)
                            umma_f16_2sm_warp(d_tmem, ad + 2 * kk, bd + 2 * kk, idesc, kk ? 1u : acc0);
                    }
                    umma_commit_2sm_warp(&empty[stage], 0x3);
                    if (++stage == kSt) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_2sm_warp(&tfull[acc], 0x3);
                if (FOLD) {
                    acc_phase ^= 1;                                     // one accumulator pair, reused per tile
                } else if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 2 && warp < 6) {
        const int g = warp & 3;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = pair; t < units; t += n_pairs) {
            const Unit w = unit_of(p, t);
            float* Zs = p.Z + (int64_t)w.s * p.F_pad * p.ldz;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int row = w.m * 256 + (int)rank * 128 + g * 32 + lane;
            const bool row_ok = row < p.rows_valid;
            int cls_m = row, cls_p = -1;                            // classes scored by this accumulator row
            if (FOLD && row_ok) {
                cls_m = p.fold_cls[row];
                cls_p = p.fold_cls[p.fold_rows + row];
            }
#pragma unroll 1
            for (int j0 = 0; j0 < bn; j0 += 32) {
                uint32_t r[32], rb[32];
                tmem_ld_32x32b_x32(tmem_base + (uint32_t(g * 32) << 16) + acc * BN + j0, r);
                if (FOLD) tmem_ld_32x32b_x32(tmem_base + (uint32_t(g * 32) << 16) + BN + j0, rb);
                tmem_ld_wait();
                const int f0 = w.n * bn + j0;
                if (MODE == 1) {
                    if (row_ok) {
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            if (f0 + jj >= p.F) continue;
                            float* zf = Zs + (int64_t)(f0 + jj) * p.ldz;
                            if (FOLD) {
                                const float a = __uint_as_float(r[jj]), b = __uint_as_float(rb[jj]);
                                zf[cls_m] = a - b;
                                if (cls_p >= 0) zf[cls_p] = a + b;
                            } else {
                                zf[row] = __uint_as_float(r[jj]);
                            }
                        }
                    }
                } else {
                    unsigned long long k[32];
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj) {
                        if (FOLD) {
                            const float a = __uint_as_float(r[jj]), b = __uint_as_float(rb[jj]);
                            const unsigned long long km = row_ok ? make_key(a - b, (uint32_t)cls_m) : 0ull;
                            const unsigned long long kp = cls_p >= 0 ? make_key(a + b, (uint32_t)cls_p) : 0ull;
                            k[jj] = km > kp ? km : kp;
                        } else {
                            k[jj] = row_ok ? make_key(__uint_as_float(r[jj]), (uint32_t)row) : 0ull;
                        }
                    }
                    const unsigned long long best = transpose_max32(k, lane);
                    if (f0 + lane < p.F && best != 0ull) atomicMax(&p.keys[f0 + lane], best);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
            if (FOLD) {
                acc_phase ^= 1;
            } else if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 6 && kProducer) {
        const int tp = (warp - 6) * 32 + lane;                    // frame row of this CTA's half tile: 0..127
        const uint32_t row_off = (uint32_t)((tp >> 3) * 1024 + (tp & 7) * 128);
        const uint32_t xr = (uint32_t)(tp & 7);
        int stage = 0;
        uint32_t phase = 0;
        for (int t = pair; t < units; t += n_pairs) {
            const Unit w = unit_of(p, t);
            const int f = w.n * bn + (int)rank * hb + tp;
            const bool valid = f < p.F && tp < hb;
            produce_x_pair<Mi, BPC, kSt, kBS, FOLD, B2_BYTES>(p, w, f, valid, sB, full, empty, stage, phase, row_off,
                                                              xr);
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

// ================================================================================================================
// SVD projection with a complex V on CTA pairs, frames on M (eq. 12): Z[f, r] = sum_kappa x16[f,kappa]
// V16[r,kappa] (rows r < D_h -> Z_r, rows D_h + d -> Z_i, real-split [Re V | Im V] / [-Im V | Re V]).  A = this CTA's
// 128 frames of X from the producer warps (produce_x_pair), B = proj_nt rows of V16 per pair tile (proj_nt/2 per CTA,
// 2-SM TMA), N = proj_nt chosen at plan creation to cover the V rows tightly (cfg5: 2 x D_h = 384 -> 2 x 192).  The
// accumulator lane is a frame and its columns are V rows, so each thread writes a contiguous segment of its frame's Z
// row.  Warps as gemm2_kernel; work units in unit_of_f order.  (Real V plans use gemm2p_kernel.)
// ================================================================================================================
template <int Mi, int BPC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS2, 1)
    gemm2f_kernel(const __grid_constant__ CUtensorMap tmV, GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sX = smem;                                     // A: 128 frames x 64 K per slab
    uint8_t* sV = smem + STAGES2 * A2_BYTES;                // B: nt/2 V rows x 64 K per slab (<= 16 KB)
    uint64_t* full = reinterpret_cast<uint64_t*>(sV + STAGES2 * B2_BYTES);
    uint64_t* empty = full + STAGES2;
    uint64_t* tfull = empty + STAGES2;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int units = p.m_tiles * p.n_tiles * p.ksplit;
    const int nt = p.bn, hn = p.bn / 2;                     // V rows per pair tile / per CTA
    const uint32_t idesc = umma_idesc_f16(256, (uint32_t)nt);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES2; ++s) {
            mbar_init(&full[s], 1 + 2 * NPW2);              // leader's TMA (expect_tx) + producers of both CTAs
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], 8);
        }
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_2sm<512>(tmem_slot);
    if (warp == 1 && lane == 0) tma_prefetch_desc(&tmV);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t bytes = 2u * (uint32_t)hn * BK * 2;
            for (int t = pair; t < units; t += n_pairs) {
                const Unit w = unit_of_f(p, t);
                for (int ks = w.k0; ks < w.k1; ++ks) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
                    tma_load_2d_2sm(sV + stage * B2_BYTES, &tmV, ks * BK, w.n * nt + (int)rank * hn, &full[stage]);
                    if (++stage == STAGES2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {                                       // converged-warp MMA issue (see gemm2_kernel)
            const uint64_t adesc0 = umma_desc_sw128(smem_u32(sX)), bdesc0 = umma_desc_sw128(smem_u32(sV));
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int t = pair; t < units; t += n_pairs) {
                const Unit w = unit_of_f(p, t);
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                for (int ks = w.k0; ks < w.k1; ++ks) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint64_t ad = adesc0 + (uint64_t)(stage * (A2_BYTES >> 4));
                    const uint64_t bd = bdesc0 + (uint64_t)(stage * (B2_BYTES >> 4));
                    const uint32_t d_tmem = tmem_base + acc * BN;
                    const uint32_t acc0 = ks != w.k0;
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        umma_f16_2sm_warp(d_tmem, ad + 2 * kk, bd + 2 * kk, idesc, kk ? 1u : acc0);
                    umma_commit_2sm_warp(&empty[stage], 0x3);
                    if (++stage == STAGES2) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_2sm_warp(&tfull[acc], 0x3);
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else if (warp < 6) {
        // epilogue: TMEM lane = frame, columns = V rows [n*nt, n*nt + nt) -> Z[s][f][row] (row < 2*D_h)
        const int g = warp & 3;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int t = pair; t < units; t += n_pairs) {
            const Unit w = unit_of_f(p, t);
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const int f = w.m * 256 + (int)rank * 128 + g * 32 + lane;
            float* zrow = p.Z + ((int64_t)w.s * p.F_pad + f) * p.ldz;
#pragma unroll 1
            for (int j0 = 0; j0 < nt; j0 += 32) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + (uint32_t(g * 32) << 16) + acc * BN + j0, r);
                tmem_ld_wait();
                const int r0 = w.n * nt + j0;               // first V row of these 32 columns
                if (f < p.F && r0 < p.ldz) {
                    float4* z = reinterpret_cast<float4*>(zrow + r0);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        z[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                           __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(&tempty[acc], 0);
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else {
        const int tp = (warp - 6) * 32 + lane;              // frame row of this CTA's half tile: 0..127
        const uint32_t row_off = (uint32_t)((tp >> 3) * 1024 + (tp & 7) * 128);
        const uint32_t xr = (uint32_t)(tp & 7);
        int stage = 0;
        uint32_t phase = 0;
        for (int t = pair; t < units; t += n_pairs) {
            const Unit w = unit_of_f(p, t);
            const int f = w.m * 256 + (int)rank * 128 + tp;
            produce_x_pair<Mi, BPC, STAGES2, A2_BYTES>(p, w, f, f < p.F, sX, full, empty, stage, phase, row_off, xr);
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

// ================================================================================================================
// SVD projection with a real V (R22) on CTA pairs, "part rows" (eq. 12): Z_r = V^T x_r and
// Z_i = V^T x_i share V, so the A operand carries the two parts of a frame as two rows — CTA r of the pair: rows
// [0,64) = Re x of frames [m*128 + 64r, +64), rows [64,128) = Im x of the same frames — and B = V16 in the part layout
// (one copy of V per K position, Plan::K_P) holds all nt <= 512 V rows of the tile in one accumulator of nt TMEM
// columns (n_mma = ceil(nt/256) MMAs of nmma columns per K step).  X is produced once per frame tile for all V rows
// (gemm2f_kernel, 256-column tiles, produced it once per V tile and was producer-bound at N = 160), and each V slab
// is staged once.  One accumulator (<= 512 columns): the epilogue is not overlapped with the next tile's MMAs.
// Warps: 0 TMA (+TMEM alloc), 1 MMA (leader), 2-5 epilogue (lane groups 2,3,0,1), 6-7 producers of the Re rows,
// 8-9 producers of the Im rows (one instruction stream for both, produce_x_part).  Work units in unit_of_f order (split slowest, V tile, frame tile fastest).
// ================================================================================================================
constexpr int P_A_BYTES = 128 * BK * 2;                // 16 KB: this CTA's 128 A rows (64 frames x {Re, Im})
constexpr int P_MAX_STAGES = 8;

// Producer warps of gemm2p_kernel: this thread's A row (part 0: Re x, part 1: Im x of frame f, eqs. 3, 7) for the bin
// chunks [w.c0, w.c1), one 16-unit slab per stage (the last slab of a chunk holds kU % 16 units when that is 8).
// `part` is a run-time (warp-uniform) value so that the Re and the Im producer warps run ONE copy of the unrolled
// chunk body: with a copy per part the producers' code was 44 KB, past the 32 KB L1.5 instruction cache, and half of
// their stall samples were instruction fetches (ncu r02: no_instruction on every 128-byte line, tensor pipe 40%).
// Both parts are x = av . (r_b, i_b) with the first microphone's record viewed as av = (r_a, i_a) for Re x and
// (i_a, -r_a) for Im x; the pairs are enumerated a-major, so av is rebuilt once per run of pairs (a, *).
template <int Mi, int BPC, int STG>
__device__ __forceinline__ void produce_x_part(const GemmParams& p, const Unit& w, int f, bool valid, uint8_t* smem,
                                               uint64_t* full, uint64_t* empty, int& stage, uint32_t& phase,
                                               uint32_t row_off, uint32_t xr, const bool part) {
    constexpr PairTab<Mi> PT{};
    constexpr int kPairs = Mi * (Mi - 1) / 2;
    constexpr int kUnitsRaw = (BPC == 4) ? kPairs : (kPairs + 1) / 2;
    constexpr int kU = (kUnitsRaw + 7) / 8 * 8;
    constexpr int kUB = BPC * 4;
    const int lane = threadIdx.x & 31;
    uint32_t e[Mi][BPC];
    auto load_rec = [&](int m, const uint8_t* base) {
        if constexpr (BPC == 4) {
            const uint4 v = valid ? __ldg(reinterpret_cast<const uint4*>(base + (int64_t)m * p.F_pad * kUB))
                                  : make_uint4(0, 0, 0, 0);
            e[m][0] = v.x;
            e[m][1] = v.y;
            e[m][2] = v.z;
            e[m][3] = v.w;
        } else {
            const uint2 v = valid ? __ldg(reinterpret_cast<const uint2*>(base + (int64_t)m * p.F_pad * kUB))
                                  : make_uint2(0, 0);
            e[m][0] = v.x;
            e[m][1] = v.y;
        }
    };
    if (w.c0 < w.c1) {
        const uint8_t* src0 = p.P16 + ((int64_t)w.c0 * Mi * p.F_pad + f) * kUB;
#pragma unroll
        for (int m = 0; m < Mi; ++m) load_rec(m, src0);
    }
#pragma unroll 1
    for (int c = w.c0; c < w.c1; ++c) {
        const uint8_t* src = p.P16 + ((int64_t)c * Mi * p.F_pad + f) * kUB;
        const uint8_t* nxt = src + (int64_t)Mi * p.F_pad * kUB;
        const bool more = c + 1 < w.c1;
        if constexpr (BPC != 4) {
            if (c != w.c0) {
#pragma unroll
                for (int m = 0; m < Mi; ++m) load_rec(m, src);
            }
        }
        if (p.prefetch && valid && more) {
#pragma unroll
            for (int m = 0; m < Mi; ++m)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(nxt + (int64_t)m * p.F_pad * kUB));
        }
        uint32_t pend0 = 0u, pend1 = 0u;
        uint32_t av[BPC] = {};                 // the a-side view of the current run of pairs (a, *)
        const uint32_t neg = part ? 0x80008000u : 0u;
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            if ((u & 15) == 0) mbar_wait(&empty[stage], phase ^ 1);
            // this part's two words of unit u: BPC 4 -> bins k0k1, k2k3 of pair u; BPC 2 -> bins k0k1 of pairs 2u, 2u+1
            uint32_t w0 = 0u, w1 = 0u;
            if constexpr (BPC == 4) {
                if (u < kPairs) {
                    const int a = PT.i[u], b = PT.j[u];
                    if (b == a + 1) {          // Re x = ra rb + ia ib, Im x = ia rb - ra ib   (eq. 3)
                        av[0] = part ? e[a][2] : e[a][0];
                        av[1] = part ? e[a][3] : e[a][1];
                        av[2] = (part ? e[a][0] : e[a][2]) ^ neg;
                        av[3] = (part ? e[a][1] : e[a][3]) ^ neg;
                    }
                    w0 = h2fma(av[0], e[b][0], h2mul(av[2], e[b][2]));
                    w1 = h2fma(av[1], e[b][1], h2mul(av[3], e[b][3]));
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int pp = 2 * u + h;
                    uint32_t v = 0u;
                    if (pp < kPairs) {
                        const int a = PT.i[pp], b = PT.j[pp];
                        if (b == a + 1) {
                            av[0] = part ? e[a][1] : e[a][0];
                            av[1] = (part ? e[a][0] : e[a][1]) ^ neg;
                        }
                        v = h2fma(av[0], e[b][0], h2mul(av[1], e[b][1]));
                    }
                    if (h == 0) w0 = v; else w1 = v;
                }
            }
            if constexpr (BPC == 4) {
#pragma unroll
                for (int m = 0; m < Mi; ++m)
                    if (PT.last[m] == u && more) load_rec(m, nxt);
            }
            if ((u & 1) == 0) {
                pend0 = w0;
                pend1 = w1;
            } else {                           // units 2j, 2j+1 -> 16-byte chunk j of the slab row (swizzled)
                const uint32_t pos = row_off + (((((uint32_t)u & 15u) >> 1) ^ xr) << 4);
                st_shared_v4(smem_u32(smem + stage * p.stage_bytes) + pos, pend0, pend1, w0, w1);
            }
            if ((u & 15) == 15 || u == kU - 1) {
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(&full[stage], 0);   // the leader's barrier
                if (++stage == STG) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    }
}

// NMMA: MMAs per K step (tile rows nt = NMMA * nmma); STG: ring stages (6 for nt <= 320, 4 up to 512).  The MMA issue
// loop is unrolled over the SP slabs of a bin chunk with compile-time stage/half-slab logic (ncu r02: a runtime n_mma
// loop, half-slab test and stage multiply cost ~185 issue instructions per slab and left the tensor pipe 45% active).
template <int Mi, int BPC, int NMMA, int STG>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS2, 1)
    gemm2p_kernel(const __grid_constant__ CUtensorMap tmV, GemmParams p) {
    constexpr int kUnitsRaw = (BPC == 4) ? Mi * (Mi - 1) / 2 : (Mi * (Mi - 1) / 2 + 1) / 2;
    constexpr int kU = (kUnitsRaw + 7) / 8 * 8;
    constexpr int kSP = (kU + 15) / 16;                     // slabs per bin chunk
    constexpr bool kHalf = (kU % 16 == 8);                  // the last slab of a chunk holds 8 units: K = 32
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // stage s: [A: 128 rows x 128 B][B: nt/2 V rows x 128 B, as n_mma blocks of nmma/2 rows]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STG * p.stage_bytes);
    uint64_t* empty = full + P_MAX_STAGES;
    uint64_t* tfull = empty + P_MAX_STAGES;
    uint64_t* tempty = tfull + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
    const int units = p.m_tiles * p.n_tiles * p.ksplit;
    const int nt = p.bn, hm = p.nmma / 2;                  // V rows per tile / per CTA per MMA
    const uint32_t idesc = umma_idesc_f16(256, (uint32_t)p.nmma);

    if (threadIdx.x == 0) {
        for (int s = 0; s < STG; ++s) {
            mbar_init(&full[s], 1 + 2 * NPW2);              // leader's TMA (expect_tx) + producers of both CTAs
            mbar_init(&empty[s], 1);
        }
        mbar_init(tfull, 1);
        mbar_init(tempty, 8);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc_2sm<512>(tmem_slot);
    if (warp == 1 && lane == 0) tma_prefetch_desc(&tmV);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t bytes = (uint32_t)nt * BK * 2;     // both CTAs' nt/2 rows x 128 B
            for (int t = pair; t < units; t += n_pairs) {
                const Unit w = unit_of_f(p, t);
                for (int ks = w.k0; ks < w.k1; ++ks) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_arrive_expect_tx(&full[stage], bytes);
                    uint8_t* sB = smem + stage * p.stage_bytes + P_A_BYTES;
#pragma unroll
                    for (int j = 0; j < NMMA; ++j)
                        tma_load_2d_2sm(sB + j * hm * (BK * 2), &tmV, ks * BK, w.n * nt + j * p.nmma + (int)rank * hm,
                                        &full[stage]);
                    if (++stage == STG) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader) {                                       // converged-warp MMA issue (see gemm2_kernel)
            const uint32_t lo0 = umma_desc_lo(smem_u32(smem)), hi = umma_desc_hi_sw128();
            const uint32_t sdesc = (uint32_t)(p.stage_bytes >> 4);
            const uint32_t bdesc = (uint32_t)(P_A_BYTES >> 4), jdesc = (uint32_t)((hm * BK * 2) >> 4);
            int stage = 0;
            uint32_t phase = 0, acc_phase = 0;
            uint32_t alo = lo0;                             // A descriptor low word of the current stage
            for (int t = pair; t < units; t += n_pairs) {
                const Unit w = unit_of_f(p, t);
                mbar_wait(tempty, acc_phase ^ 1);
                tc_fence_after();
                uint32_t acc0 = 0u;
                for (int c = w.c0; c < w.c1; ++c) {
#pragma unroll
                    for (int sl = 0; sl < kSP; ++sl) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
#pragma unroll
                        for (int j = 0; j < NMMA; ++j) {
                            const uint32_t d_tmem = tmem_base + (uint32_t)(j * p.nmma);
                            if (kHalf && sl == kSP - 1)   // compile-time after unrolling: 8 units = K 32
                                umma_f16_2sm_steps<2>(d_tmem, alo, alo + bdesc + j * jdesc, hi, idesc, acc0);
                            else
                                umma_f16_2sm_steps<4>(d_tmem, alo, alo + bdesc + j * jdesc, hi, idesc, acc0);
                        }
                        acc0 = 1u;
                        umma_commit_2sm_warp(&empty[stage], 0x3);
                        if (++stage == STG) {
                            stage = 0;
                            phase ^= 1;
                            alo = lo0;
                        } else {
                            alo += sdesc;
                        }
                    }
                }
                umma_commit_2sm_warp(tfull, 0x3);
                acc_phase ^= 1;
            }
        }
    } else if (warp < 6) {
        // epilogue: TMEM lane = A row (part g/2, frame (g&1)*32 + lane), columns = V rows [n*nt, n*nt + nt) -> Z
        const int g = warp & 3;
        const int part = g >> 1;
        uint32_t acc_phase = 0;
        for (int t = pair; t < units; t += n_pairs) {
            const Unit w = unit_of_f(p, t);
            mbar_wait(tfull, acc_phase);
            tc_fence_after();
            const int f = w.m * 128 + (int)rank * 64 + (g & 1) * 32 + lane;
            float* zrow = p.Z + ((int64_t)w.s * p.F_pad + f) * p.ldz + part * p.zh + w.n * nt;
#pragma unroll 1
            for (int j0 = 0; j0 < nt; j0 += 32) {
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + (uint32_t(g * 32) << 16) + j0, r);
                tmem_ld_wait();
                if (f < p.F) {
                    float4* z = reinterpret_cast<float4*>(zrow + j0);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        z[q] = make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]),
                                           __uint_as_float(r[4 * q + 2]), __uint_as_float(r[4 * q + 3]));
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty, 0);
            acc_phase ^= 1;
        }
    } else {
        const int tp = (warp - 6) * 32 + lane;              // A row of this CTA: 0..63 Re part, 64..127 Im part
        const uint32_t row_off = (uint32_t)((tp >> 3) * 1024 + (tp & 7) * 128);
        const uint32_t xr = (uint32_t)(tp & 7);
        int stage = 0;
        uint32_t phase = 0;
        for (int t = pair; t < units; t += n_pairs) {
            const Unit w = unit_of_f(p, t);
            const int f = w.m * 128 + (int)rank * 64 + (tp & 63);
            produce_x_part<Mi, BPC, STG>(p, w, f, f < p.F, smem, full, empty, stage, phase, row_off, xr, tp >= 64);
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

// ---------------------------------------------------------------- host side
template <int Mi, int BPC, int MODE>
static cudaError_t set_attr_one() {
    return cudaFuncSetAttribute(gemm_kernel<Mi, BPC, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                SMEM_BYTES);
}

template <int Mi, int BPC>
static cudaError_t set_attr_pair() {
    cudaError_t e = cudaSuccess;
    const int sm = SMEM2_BYTES;
    const auto attr = cudaFuncAttributeMaxDynamicSharedMemorySize;
    if ((e = cudaFuncSetAttribute(gemm2_kernel<Mi, BPC, 0, false>, attr, sm))) return e;
    if ((e = cudaFuncSetAttribute(gemm2_kernel<Mi, BPC, 1, false>, attr, sm))) return e;
    if ((e = cudaFuncSetAttribute(gemm2_kernel<Mi, BPC, 0, true>, attr, sm))) return e;
    if ((e = cudaFuncSetAttribute(gemm2_kernel<Mi, BPC, 1, true>, attr, sm))) return e;
    if ((e = cudaFuncSetAttribute(gemm2f_kernel<Mi, BPC>, attr, sm))) return e;
    if ((e = cudaFuncSetAttribute(gemm2p_kernel<Mi, BPC, 1, 6>, attr, 227 * 1024))) return e;
    if ((e = cudaFuncSetAttribute(gemm2p_kernel<Mi, BPC, 2, 6>, attr, 227 * 1024))) return e;
    return cudaFuncSetAttribute(gemm2p_kernel<Mi, BPC, 2, 4>, attr, 227 * 1024);
}

cudaError_t gemm_set_attributes() {
    cudaError_t e = cudaSuccess;
    if ((e = set_attr_pair<4, 4>()) != cudaSuccess) return e;
    if ((e = set_attr_pair<8, 4>()) != cudaSuccess) return e;
    if ((e = set_attr_pair<16, 4>()) != cudaSuccess) return e;
    if ((e = set_attr_pair<32, 2>()) != cudaSuccess) return e;
#define SVD_ATTR(MI, B)                                        \
    if ((e = set_attr_one<MI, B, 0>()) != cudaSuccess) return e; \
    if ((e = set_attr_one<MI, B, 1>()) != cudaSuccess) return e;
    SVD_ATTR(4, 4)
    SVD_ATTR(8, 4)
    SVD_ATTR(16, 4)
    SVD_ATTR(32, 2)
#undef SVD_ATTR
    if ((e = set_attr_one<4, 4, 3>()) != cudaSuccess) return e;
    return set_attr_one<4, 4, 2>();
}

// CTA-pair launch over the instantiated mic counts; MODE 0 argmax / 1 store, FOLD = antipodally folded W
template <int MODE>
static cudaError_t launch_pair(const Plan& p, const CUtensorMap& A, const CUtensorMap& B, const GemmParams& gp,
                               int pairs, bool fold, cudaStream_t s) {
#define SVD_PAIR(MI, BP)                                                                                  \
    if (p.L.Mi == MI) {                                                                                  \
        if (fold)                                                                                        \
            gemm2_kernel<MI, BP, MODE, true><<<2 * pairs, THREADS2, SMEM2_BYTES, s>>>(A, B, gp);        \
        else                                                                                             \
            gemm2_kernel<MI, BP, MODE, false><<<2 * pairs, THREADS2, SMEM2_BYTES, s>>>(A, B, gp);       \
        return cudaGetLastError();                                                                       \
    }
    SVD_PAIR(4, 4)
    SVD_PAIR(8, 4)
    SVD_PAIR(16, 4)
    SVD_PAIR(32, 2)
#undef SVD_PAIR
    return cudaErrorInvalidValue;
}

template <int Mi, int BPC, int MODE>
static cudaError_t launch_one(const CUtensorMap& A, const CUtensorMap& B, const GemmParams& gp, int grid,
                              cudaStream_t s) {
    gemm_kernel<Mi, BPC, MODE><<<grid, 32 * (6 + NUM_PRODUCER_WARPS), SMEM_BYTES, s>>>(A, B, gp);
    return cudaGetLastError();
}

// SVD projection launch shape: CTA-pair tiles of 256 V rows (p.pair_proj) or 1-CTA tiles of 128, and its K splits
ProjShape proj_shape(const Plan& p, const Band& b, int F) {
    ProjShape sh;
    sh.pair = p.pair_proj;
    const int f_tiles = p.svd_fold && p.pair_proj ? (F + 127) / 128 : (F + BN - 1) / BN;   // part kernel: 128 frames
    sh.m_tiles = sh.pair ? f_tiles : (2 * p.Dh) / BM;
    sh.n_tiles = sh.pair ? p.proj_ntiles : f_tiles;
    const int units = sh.m_tiles * sh.n_tiles;
    const int slots = sh.pair ? p.num_sms / 2 : p.num_sms;
    const int nc = b.c_hi - b.c_lo;
    const double slabs = (double)nc * (p.svd_fold ? p.spc_P : p.L.U / 8) * (p.svd_fold ? p.proj_nmma : 1);
    double best_t = 1e300;
    sh.ksplit = 1;
    constexpr double fixed = 24.0;            // per-unit fixed cost in slabs (pipeline fill + epilogue), r01 fit
    for (int S = 1; S <= p.zsplit_max && S <= nc; ++S) {
        const double waves = (double)((units * S + slots - 1) / slots);
        const double t = waves * (slabs / S + fixed);
        if (t < best_t - 1e-9) {
            best_t = t;
            sh.ksplit = S;
        }
    }
    return sh;
}

Band make_band(const Plan& p, int k_lo, int k_hi, const uint8_t* mask, int64_t mask_stride) {
    Band b;
    b.k_lo = k_lo;
    b.k_hi = k_hi;
    b.c_lo = k_lo / p.L.bpc;
    b.c_hi = (k_hi + p.L.bpc - 1) / p.L.bpc;
    b.mask = mask;
    b.mask_stride = mask_stride;
    return b;
}

// K splits of the small-batch SRP path (fewer 256 x 256 units than half the CTA pairs), 1 = the argmax GEMM path
int srp_split_ways(const Plan& p, const Band& b, int F) {
    if (!p.pair_srp || p.srp_split_max <= 1) return 1;
    const int npairs = p.num_sms / 2;
    const int units = (p.W_rows / 256) * ((F + 255) / 256);
    int S = units > 0 ? npairs / units : 1;
    S = S < p.srp_split_max ? S : p.srp_split_max;
    S = S < b.c_hi - b.c_lo ? S : b.c_hi - b.c_lo;
    return (units * 2 <= npairs && S > 1) ? S : 1;
}

cudaError_t launch_gemm(const Plan& p, const Band& b, int mode, int F, cudaStream_t s, bool both) {
    GemmParams gp{};
    const bool srp_mode = (mode == 0 || mode == 3);             // W16 operand (folded when p.fold)
    const bool producer_mode = srp_mode || mode == 1;
    gp.c_lo = producer_mode ? b.c_lo : 0;
    gp.c_hi = producer_mode ? b.c_hi : 0;
    gp.P16 = p.d_P16;
    gp.F = F;
    gp.F_pad = (int)p.F_pad;
    gp.n_chunks = p.L.n_chunks;
    gp.n_tiles = (F + BN - 1) / BN;
    gp.keys = p.d_keys;
    gp.Z = p.d_Z32;
    gp.ldz = 2 * p.Zh;
    gp.ksplit = 1;
    gp.spc = srp_mode ? p.spc_W : p.L.U / 8;
    gp.bn = BN;
    gp.fold_cls = p.d_fold_cls;
    gp.fold_rows = p.fold_rows;
    gp.prefetch = 1;                   // L2 prefetch of the next chunk's phasor records (r01: +2% at cfg3)
    const CUtensorMap* A = nullptr;
    const CUtensorMap* B = &p.tm_W;  // unused placeholder for producer modes
    const int npairs = p.num_sms / 2;
    if (srp_mode) {
        A = &p.tm_W;
        gp.n_slabs = (int)(p.K_W / BK);
        gp.rows_valid = p.fold ? p.fold_rows : p.Q_eff;
        gp.m_tiles = p.W_rows / (p.pair_srp ? 256 : BM);
    } else if (mode == 1) {
        A = &p.tm_V;                   // complex V (the real-V part kernel sets its own shape below)
        gp.n_slabs = (int)(p.L.K_total / BK);
        gp.rows_valid = 2 * p.Dh;
        gp.m_tiles = (2 * p.Dh) / BM;
    } else {                           // 2: SVD search + argmax; 4/5: its score map Re{Dhat Zhat}[f][class] -> S / Smap
        A = &p.tm_R;
        B = &p.tm_Zs;
        gp.n_slabs = p.K2 / BK;
        gp.m_tiles = p.Q_pad / BM;
        gp.rows_valid = p.Q_eff;
        if (mode == 2) {
            gp.keys = p.d_keys + 2 * p.F_pad;                 // FP16 keys; the rescore writes the SVD keys
            gp.cand = p.d_cand;
            gp.ccnt = p.d_ccnt;
        } else {
            gp.Z = mode == 5 ? p.d_Smap : p.d_S;
            gp.ldz = p.Q_pad;
        }
    }
    if (mode == 3) {                   // SRP power map Y[f][class] -> S (multi-source search); pair kernel, store
        gp.m_tiles = p.W_rows / 256;
        gp.Z = p.d_S;
        gp.ldz = p.Q_pad;
        const int units = gp.m_tiles * gp.n_tiles;
        if (units == 0) return cudaSuccess;
        return launch_pair<1>(p, *A, *B, gp, units < npairs ? units : npairs, p.fold, s);
    }
    int tiles = gp.m_tiles * gp.n_tiles;
    if (mode == 1) {
        // split K (at chunk boundaries) to fill the SMs, deterministic partial buffers
        const ProjShape sh = proj_shape(p, b, F);
        gp.ksplit = sh.ksplit;
        if (sh.pair && p.svd_fold) {   // real V: part rows (gemm2p_kernel), all V rows of a tile in one accumulator
            gp.m_tiles = sh.m_tiles;
            gp.n_tiles = sh.n_tiles;
            gp.bn = p.proj_nt;
            gp.spc = p.spc_P;
            gp.n_slabs = (int)(p.K_P / BK);
            gp.n_mma = p.proj_nmma;
            gp.nmma = p.proj_nt / p.proj_nmma;
            gp.ldz = 2 * p.Zh;
            gp.zh = p.Zh;
            gp.stage_bytes = P_A_BYTES + (p.proj_nt / 2) * BK * 2;
            gp.stages = 1024 + 6 * gp.stage_bytes + 256 <= 227 * 1024 ? 6 : 4;
            const int units = gp.m_tiles * gp.n_tiles * gp.ksplit;
            if (units == 0) return cudaSuccess;
            const int pairs = units < npairs ? units : npairs;
            const size_t smem = 1024 + (size_t)gp.stages * gp.stage_bytes + 256;
#define SVD_PROJP(MI, BP)                                                                                        \
    if (p.L.Mi == MI) {                                                                                         \
        if (gp.n_mma == 1)                                                                                      \
            gemm2p_kernel<MI, BP, 1, 6><<<2 * pairs, THREADS2, smem, s>>>(*A, gp);                              \
        else if (gp.stages == 6)                                                                                \
            gemm2p_kernel<MI, BP, 2, 6><<<2 * pairs, THREADS2, smem, s>>>(*A, gp);                              \
        else                                                                                                    \
            gemm2p_kernel<MI, BP, 2, 4><<<2 * pairs, THREADS2, smem, s>>>(*A, gp);                              \
        return cudaGetLastError();                                                                              \
    }
            SVD_PROJP(4, 4)
            SVD_PROJP(8, 4)
            SVD_PROJP(16, 4)
            SVD_PROJP(32, 2)
#undef SVD_PROJP
            return cudaErrorInvalidValue;
        }
        if (sh.pair) {                 // complex V: frames on M, V rows on N (gemm2f_kernel)
            gp.m_tiles = sh.m_tiles;
            gp.n_tiles = sh.n_tiles;
            gp.bn = p.proj_nt;
            const int units = gp.m_tiles * gp.n_tiles * gp.ksplit;
            if (units == 0) return cudaSuccess;
            const int pairs = units < npairs ? units : npairs;
#define SVD_PROJ(MI, BP)                                                                                         \
    if (p.L.Mi == MI) {                                                                                         \
        gemm2f_kernel<MI, BP><<<2 * pairs, THREADS2, SMEM2_BYTES, s>>>(*A, gp);                                 \
        return cudaGetLastError();                                                                              \
    }
            SVD_PROJ(4, 4)
            SVD_PROJ(8, 4)
            SVD_PROJ(16, 4)
            SVD_PROJ(32, 2)
#undef SVD_PROJ
            return cudaErrorInvalidValue;
        }
        tiles *= gp.ksplit;
    }
    const int grid = tiles < p.num_sms ? tiles : p.num_sms;
    if (tiles == 0) return cudaSuccess;
    if (mode == 2) return launch_one<4, 4, 2>(*A, *B, gp, grid, s);
    if (mode == 4 || mode == 5) return launch_one<4, 4, 3>(*A, *B, gp, grid, s);
    if (mode == 0 && srp_split_ways(p, b, F) > 1) {
        // small batch: fewer units than half the CTA pairs -> split K into chunk ranges with partial power maps
        const int S = srp_split_ways(p, b, F);
        const int units = gp.m_tiles * gp.n_tiles;
        gp.ksplit = S;
        gp.Z = p.d_Ypart;
        gp.ldz = p.Q_pad;
        const cudaError_t e = launch_pair<1>(p, *A, *B, gp, units * S < npairs ? units * S : npairs, p.fold, s);
        return e != cudaSuccess ? e : launch_split_argmax(p, F, S, s);
    }
    if (mode == 0 && p.pair_srp) {
        gp.bn = 256;                   // r01: 224 (the wave-quantisation optimum) was slower under the power cap
        gp.n_tiles = (F + gp.bn - 1) / gp.bn;
        if (both && p.tail_n > 0) gp.m_tiles = p.tail_r0 / 256;   // the tail rows are scored by the projection
        // (a BOTH call reaches here only on the argmax path: srp_split_ways(p, b, F) == 1, see localize_impl)
        const int units = gp.m_tiles * gp.n_tiles;
        return launch_pair<0>(p, *A, *B, gp, units < npairs ? units : npairs, p.fold, s);
    }
#define SVD_DISPATCH(MI, BP)                                                                      \
    if (p.L.Mi == MI) {                                                                          \
        return mode == 0 ? launch_one<MI, BP, 0>(*A, *B, gp, grid, s) : launch_one<MI, BP, 1>(*A, *B, gp, grid, s); \
    }
    SVD_DISPATCH(4, 4)
    SVD_DISPATCH(8, 4)
    SVD_DISPATCH(16, 4)
    SVD_DISPATCH(32, 2)
#undef SVD_DISPATCH
    return cudaErrorInvalidValue;
}

}  // namespace svdphat
