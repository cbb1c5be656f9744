// ptx.cuh — inline-PTX wrappers for sm_100a: mbarrier, TMA, tcgen05 (UMMA / TMEM), proxy fences.
// Descriptor bit layouts follow the sm_100 UMMA encodings (shared-memory matrix descriptor and the kind::f16
// instruction descriptor); see DESIGN.md "GEMM kernel" for the fields used.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace svdphat {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
                     smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// ------------------------------------------------------------------------------------------------ fences
// generic-proxy smem writes -> visible to the async proxy (tcgen05.mma operand reads, TMA)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ------------------------------------------------------------------------------------------------ TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
// 2-D tiled load: box lands at smem_dst (swizzle per the tensor map), completes tx bytes on bar.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

// ------------------------------------------------------------------------------------------------ tcgen05
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst) {  // whole warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {  // whole warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}

// Shared-memory matrix descriptor: K-major operand tile, SWIZZLE_128B (rows of 128 B, 8-row atoms of 1024 B).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t smem_addr) {
    uint64_t d = 0;
    d |= (uint64_t)((smem_addr >> 4) & 0x3FFFu);        // [0,14)  start address >> 4
    d |= (uint64_t)(16u >> 4) << 16;                     // [16,30) leading byte offset (unused for SW128 K-major)
    d |= (uint64_t)(1024u >> 4) << 32;                   // [32,46) stride byte offset: 8-row atom pitch
    d |= (uint64_t)1u << 46;                             // [46,48) descriptor version (sm_100)
    d |= (uint64_t)2u << 61;                             // [61,64) layout: SWIZZLE_128B
    return d;
}

// Instruction descriptor, kind::f16: A,B = FP16, D = FP32, both K-major, shape M x N.
__host__ __device__ constexpr uint32_t umma_idesc_f16(uint32_t M, uint32_t N) {
    return (1u << 4)            // [4,6)   D format: F32
           | (0u << 7)          // [7,10)  A format: F16
           | (0u << 10)         // [10,13) B format: F16
           | (0u << 15)         // A K-major
           | (0u << 16)         // B K-major
           | ((N >> 3) << 17)   // [17,23) N >> 3
           | ((M >> 4) << 24);  // [24,29) M >> 4
}

// One tcgen05.mma (cta_group::1), issued by the converged warp: every lane executes the asm with identical operands
// and elect.sync picks the issuing lane, so ptxas keeps the operands in uniform registers (a single-thread issue
// under `if (lane == 0)` costs an ELECT / R2UR.BROADCAST / BRA.U.ANY sequence per MMA).
__device__ __forceinline__ void umma_f16_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Arrive (once) on an mbarrier when all previously issued tcgen05.mma of the warp have completed.
__device__ __forceinline__ void umma_commit_warp(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
        : "memory");
}

// TMEM -> registers: 32 lanes x 32 consecutive 32-bit columns (thread t of the warp gets lane base+t).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------------------------------------ CTA pair (2-SM)
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Arrive on the mbarrier at the same smem offset in CTA `cta` of the cluster (default .release semantics; the
// cluster-scope variant costs a MEMBAR.ALL.GPU + ERRBAR per arrival, ncu r01 pair profile).
__device__ __forceinline__ void mbar_arrive_cluster(uint64_t* bar, uint32_t cta) {
    asm volatile(
        "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, %1;\n\t"
        "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
        "r"(cta)
        : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait_cluster(bar, parity)) {
    }
}
// 2-SM TMA load: the box lands in THIS CTA's smem, completion bytes go to the even (leader) CTA's barrier.
__device__ __forceinline__ void tma_load_2d_2sm(void* smem_dst, const void* tmap, int32_t x, int32_t y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];" ::"r"(smem_u32(smem_dst)),
        "l"(reinterpret_cast<uint64_t>(tmap)), "r"(x), "r"(y), "r"(smem_u32(bar) & 0xFEFFFFFFu)
        : "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc_2sm(uint32_t* smem_dst) {  // same warp in both CTAs
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)),
                 "n"(kCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_dealloc_2sm(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(kCols) : "memory");
}
// CTA-pair MMA / commit from the converged warp (see umma_f16_warp); the leader CTA issues for both.
__device__ __forceinline__ void umma_f16_2sm_warp(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                  uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit_2sm_warp(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
        ::"r"(smem_u32(bar)), "h"(mask)
        : "memory");
}
// Descriptor words of umma_desc_sw128: lo = (smem address >> 4) | LBO field, hi = SBO | version | layout.  Smem
// addresses stay below 256 KB, so advancing the start address never carries out of the low word.
__device__ __forceinline__ uint32_t umma_desc_lo(uint32_t smem_addr) {
    return ((smem_addr >> 4) & 0x3FFFu) | ((16u >> 4) << 16);
}
__host__ __device__ constexpr uint32_t umma_desc_hi_sw128() { return (1024u >> 4) | (1u << 14) | (2u << 29); }

// NK consecutive K = 16 steps of a CTA-pair MMA (one 32-byte K step = +2 in both descriptors' low words) in ONE asm
// block with one elect.sync: ptxas then moves the two base words into uniform registers once and advances them in the
// uniform datapath, instead of an ELECT / R2UR.BROADCAST / VOTEU sequence per MMA (ncu r02: ~23 issue instructions per
// MMA, a dependent chain that starved the tensor pipe at N = 160).  accumulate applies to the first step only.
template <int NK>
__device__ __forceinline__ void umma_f16_2sm_steps(uint32_t tmem_d, uint32_t a_lo, uint32_t b_lo, uint32_t hi,
                                                   uint32_t idesc, uint32_t accumulate) {
    static_assert(NK == 2 || NK == 4, "2 or 4 K steps");
    if constexpr (NK == 4) {
        asm volatile(
            "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a0, b0, a1, b1, a2, b2, a3, b3;\n\t.reg .b32 x, y;\n\t"
            "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
            "mov.b64 a0, {%1, %3};\n\tmov.b64 b0, {%2, %3};\n\t"
            "add.u32 x, %1, 2;\n\tadd.u32 y, %2, 2;\n\tmov.b64 a1, {x, %3};\n\tmov.b64 b1, {y, %3};\n\t"
            "add.u32 x, %1, 4;\n\tadd.u32 y, %2, 4;\n\tmov.b64 a2, {x, %3};\n\tmov.b64 b2, {y, %3};\n\t"
            "add.u32 x, %1, 6;\n\tadd.u32 y, %2, 6;\n\tmov.b64 a3, {x, %3};\n\tmov.b64 b3, {y, %3};\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %4, p;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %4, t;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a2, b2, %4, t;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a3, b3, %4, t;\n\t}" ::"r"(tmem_d),
            "r"(a_lo), "r"(b_lo), "r"(hi), "r"(idesc), "r"(accumulate)
            : "memory");
    } else {
        asm volatile(
            "{\n\t.reg .pred e, p, t;\n\t.reg .b64 a0, b0, a1, b1;\n\t.reg .b32 x, y;\n\t"
            "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %5, 0;\n\tsetp.eq.b32 t, 1, 1;\n\t"
            "mov.b64 a0, {%1, %3};\n\tmov.b64 b0, {%2, %3};\n\t"
            "add.u32 x, %1, 2;\n\tadd.u32 y, %2, 2;\n\tmov.b64 a1, {x, %3};\n\tmov.b64 b1, {y, %3};\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a0, b0, %4, p;\n\t"
            "@e tcgen05.mma.cta_group::2.kind::f16 [%0], a1, b1, %4, t;\n\t}" ::"r"(tmem_d),
            "r"(a_lo), "r"(b_lo), "r"(hi), "r"(idesc), "r"(accumulate)
            : "memory");
    }
}

// A operand from TMEM ("TS" form): [a_tmem] is the TMEM address of this CTA's 128 rows x 16 K (8 columns).
__device__ __forceinline__ void umma_f16_2sm_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
        "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// registers -> TMEM: 32 lanes x 32 consecutive 32-bit columns (thread t of the warp writes lane base+t)
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
        "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]),
        "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),
        "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Arrive once on the barrier at this smem offset in every CTA of `mask` when the issued MMAs complete.
__device__ __forceinline__ void umma_commit_2sm(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}

// ------------------------------------------------------------------------------------------------ misc
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

// Order-preserving map float -> uint32 (larger float -> larger uint); NaN never wins over a finite value.
__device__ __forceinline__ uint32_t f2o(float v) {
    if (v != v) return 0u;
    uint32_t b = __float_as_uint(v);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float o2f(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}
// Packed argmax key: larger score first, then LOWER index (0xFFFFFFFF - idx larger).
__device__ __forceinline__ unsigned long long make_key(float v, uint32_t idx) {
    return ((unsigned long long)f2o(v) << 32) | (unsigned long long)(0xFFFFFFFFu - idx);
}

// maximum of v over the 32 lanes of the (converged) warp, in every lane: one CREDUX.MAX.F32 (sm_100a); NaN inputs are
// ignored unless every lane holds one
__device__ __forceinline__ float warp_max_f32(float v) {
    float m;
    asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(m) : "f"(v));
    return m;
}

// u64 max-reduce of 32 columns across the 32 lanes of a warp; afterwards lane l holds column l's maximum.
__device__ __forceinline__ unsigned long long transpose_max32(unsigned long long (&k)[32], int lane) {
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) {
        const bool upper = (lane & h) != 0;
#pragma unroll
        for (int c = 0; c < h; ++c) {
            unsigned long long send = upper ? k[c] : k[c + h];
            unsigned long long mine = upper ? k[c + h] : k[c];
            unsigned long long recv = __shfl_xor_sync(0xffffffffu, send, h);
            k[c] = mine > recv ? mine : recv;
        }
    }
    return k[0];
}

}  // namespace svdphat
