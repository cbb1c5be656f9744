// setup.cu — Alg. 1 offline in float64, run once per plan on the device.
//
//  * W16 : W_{q,i,j}[k] = exp(+j 2 pi k tau_{q,i,j} / N) (eq. 4) packed real-split FP16 as
//          [Re W | -Im W] in the GEMM contraction order (internal.h), one row per steering class; or folded (one
//          row per antipodal class pair, Re and Im in separate slabs, R22).
//  * SVD : sigma^2 and U from the Hermitian Gram G = W W^H (same singular values / left vectors as eq. 10),
//          with G built in closed form: G_ab = sum_p sum_{k<Kb} e^{j 2 pi k (tau_ap - tau_bp)/N}
//          = sum_p e^{j pi (Kb-1) x} sin(pi Kb x) / sin(pi x),  x = (tau_ap - tau_bp)/N  (geometric series).
//          Twin classes (bitwise-identical rows, R11) enter with multiplicity n_c:  G' = N^1/2 G_r N^1/2
//          has the spectrum of the full W W^H.  Rank D by eq. 11 with Tr{W W^H} = Q P Kb exactly.
//          V_D = W^H U_D S_D^{-1} (eq. 10) formed column-chunk-wise with cuBLAS ZGEMM on generated W chunks.
//          Dictionary rows D_q = (U S)_q (eq. 13) normalised -> FP16 [Re | -Im] for the search GEMM
//          and FP32 for the exact rescore of its candidates.
#include <cublas_v2.h>
#include <cuComplex.h>
#include <cuda_fp16.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <string>
#include <vector>

#include "internal.h"

namespace svdphat {

// kappa index of (instantiated pair pi, bin k, imaginary?) in the GEMM contraction order
__host__ __device__ __forceinline__ int64_t kappa_of(int pi, int k, int im, int bpc, int U) {
    const int c = k / bpc, s = k % bpc;
    if (bpc == 4) return ((int64_t)c * U + pi) * 8 + (im ? 4 : 0) + s;
    return ((int64_t)c * U + (pi >> 1)) * 8 + (pi & 1) * 4 + (im ? 2 : 0) + s;
}

// instantiated pair index of real pair (i, j) in the lexicographic enumeration over Mi mics
__host__ __device__ __forceinline__ int pair_index(int i, int j, int Mi) {
    return i * (2 * Mi - i - 1) / 2 + (j - i - 1);
}

// one thread per (class row, real pair): all bins of that pair
__global__ void pack_w16_kernel(const double* __restrict__ tau, int Q_eff, int P, int M, int Mi, int N, int Kb,
                                int bpc, int U, int64_t K_total, __half* __restrict__ W16) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= (int64_t)Q_eff * P) return;
    const int row = (int)(tid / P), p = (int)(tid % P);
    // real pair p -> (i, j) over M mics
    int i = 0, rem = p;
    while (rem >= M - 1 - i) {
        rem -= M - 1 - i;
        ++i;
    }
    const int j = i + 1 + rem;
    const int pi = pair_index(i, j, Mi);
    const double t = tau[(int64_t)row * P + p];
    __half* dst = W16 + (int64_t)row * K_total;
    for (int k = 0; k < Kb; ++k) {
        double s, c;
        sincospi(2.0 * (double)k * t / (double)N, &s, &c);  // e^{j 2 pi k tau / N}
        dst[kappa_of(pi, k, 0, bpc, U)] = __double2half(c);
        dst[kappa_of(pi, k, 1, bpc, U)] = __double2half(-s);
    }
}

// Folded W (antipodal folding, internal.h / DESIGN.md R22): fold row r carries class fold_m[r]'s Re W in the Re slabs
// and its Im W (sign +: b = Im W . x_i, Y = a - b, Y_antipode = a + b) in the Im slabs.  Unit u of chunk c, value s
// (BPC 4: bin 4c+s; BPC 2: pair 2u + s/2, bin 2c + s%2) sits at ((c*SP + u/16)*2 + im)*64 + (u%16)*4 + s.
__host__ __device__ __forceinline__ int64_t kappa_fold(int pi, int k, int im, int bpc, int SP) {
    const int c = k / bpc;
    const int u = (bpc == 4) ? pi : (pi >> 1);
    const int s = (bpc == 4) ? (k % 4) : ((pi & 1) * 2 + k % 2);
    return (((int64_t)c * SP + u / 16) * 2 + im) * 64 + (u % 16) * 4 + s;
}

__global__ void pack_w16f_kernel(const double* __restrict__ tau, const int* __restrict__ fold_m, int rows, int P,
                                 int M, int Mi, int N, int Kb, int bpc, int SP, int64_t K_W,
                                 __half* __restrict__ W16) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= (int64_t)rows * P) return;
    const int row = (int)(tid / P), p = (int)(tid % P);
    int i = 0, rem = p;
    while (rem >= M - 1 - i) {
        rem -= M - 1 - i;
        ++i;
    }
    const int pi = pair_index(i, i + 1 + rem, Mi);
    const double t = tau[(int64_t)fold_m[row] * P + p];
    __half* dst = W16 + (int64_t)row * K_W;
    for (int k = 0; k < Kb; ++k) {
        double sn, cs;
        sincospi(2.0 * (double)k * t / (double)N, &sn, &cs);  // e^{j 2 pi k tau / N}
        dst[kappa_fold(pi, k, 0, bpc, SP)] = __double2half(cs);
        dst[kappa_fold(pi, k, 1, bpc, SP)] = __double2half(sn);
    }
}

// lower triangle (column-major) of G' = diag(sqrt n) G_r diag(sqrt n), G_r[a][b] = sum_p Dirichlet(tau_a - tau_b)
__global__ void gram_kernel(const double* __restrict__ tau, const int* __restrict__ cnt, int n, int P, int N, int Kb,
                            cuDoubleComplex* __restrict__ G) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int b = blockIdx.y;
    if (a >= n || a < b) return;
    double re = 0.0, im = 0.0;
    const double* ta = tau + (int64_t)a * P;
    const double* tb = tau + (int64_t)b * P;
    for (int p = 0; p < P; ++p) {
        const double x = (ta[p] - tb[p]) / (double)N;
        if (x == 0.0) {
            re += (double)Kb;
        } else {
            const double amp = sinpi((double)Kb * x) / sinpi(x);
            double s, c;
            sincospi((double)(Kb - 1) * x, &s, &c);
            re += amp * c;
            im += amp * s;
        }
    }
    const double w = sqrt((double)cnt[a] * (double)cnt[b]);
    G[(int64_t)b * n + a] = make_cuDoubleComplex(w * re, w * im);
}

// Bmat[a][d] (column-major n x D) = sqrt(n_a) U'[a][jd] / sqrt(lambda_d), jd = n-1-d (eigenvalues ascending)
__global__ void bmat_kernel(const cuDoubleComplex* __restrict__ Uv, const double* __restrict__ lam,
                            const int* __restrict__ cnt, int n, int D, cuDoubleComplex* __restrict__ B) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int d = blockIdx.y;
    if (a >= n) return;
    const int jd = n - 1 - d;
    const double s = sqrt((double)cnt[a] / lam[jd]);
    const cuDoubleComplex u = Uv[(int64_t)jd * n + a];
    B[(int64_t)d * n + a] = make_cuDoubleComplex(s * u.x, s * u.y);
}

// W chunk, column-major n x C: columns c0..c0+C-1 of eq. 8 (pair-major, bins inner), rows = classes
__global__ void wchunk_kernel(const double* __restrict__ tau, int n, int P, int N, int Kb, int64_t c0, int C,
                              cuDoubleComplex* __restrict__ Wc) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int cc = blockIdx.y;
    if (a >= n) return;
    const int64_t col = c0 + cc;
    const int p = (int)(col / Kb), k = (int)(col % Kb);
    double s, c;
    sincospi(2.0 * (double)k * tau[(int64_t)a * P + p] / (double)N, &s, &c);
    Wc[(int64_t)cc * n + a] = make_cuDoubleComplex(c, s);
}

// V chunk (column-major C x D) -> V16 rows: d -> [V_r | V_i] (Z_r), Dh + d -> [-V_i | V_r] (Z_i), scaled by sqrt(PK)
__global__ void pack_v16_kernel(const cuDoubleComplex* __restrict__ Vc, int C, int D, int Dh, int64_t c0, int M,
                                int Mi, int Kb, int bpc, int U, int64_t K_total, double scale,
                                __half* __restrict__ V16) {
    const int cc = blockIdx.x * blockDim.x + threadIdx.x;
    const int d = blockIdx.y;
    if (cc >= C) return;
    const int64_t col = c0 + cc;
    const int p = (int)(col / Kb), k = (int)(col % Kb);
    int i = 0, rem = p;
    while (rem >= M - 1 - i) {
        rem -= M - 1 - i;
        ++i;
    }
    const int j = i + 1 + rem;
    const int pi = pair_index(i, j, Mi);
    const cuDoubleComplex v = Vc[(int64_t)d * C + cc];
    const int64_t kr = kappa_of(pi, k, 0, bpc, U), ki = kappa_of(pi, k, 1, bpc, U);
    __half* zr = V16 + (int64_t)d * K_total;
    __half* zi = V16 + (int64_t)(Dh + d) * K_total;
    zr[kr] = __double2half(scale * v.x);
    zr[ki] = __double2half(scale * v.y);
    zi[kr] = __double2half(-scale * v.y);
    zi[ki] = __double2half(scale * v.x);
}

// ---------------------------------------------------------------- real-basis SVD (svd_fold, R22)
// Real basis row i = sum over its class rows x of coef_i[x] W'_x: kind 0 (W_c + W_c')/sqrt2 = sqrt2 Re W_c, kind 1
// (W_c - W_c')/(sqrt2 j) = sqrt2 Im W_c, kind 2 W_c (real row).  T with these rows is unitary and T W' is real.
__device__ __forceinline__ int rb_terms(int kind, int c, int cp, int* cls, cuDoubleComplex* coef) {
    const double h = 0.70710678118654752440;
    if (kind == 2) {
        cls[0] = c;
        coef[0] = make_cuDoubleComplex(1.0, 0.0);
        return 1;
    }
    cls[0] = c;
    cls[1] = cp;
    coef[0] = kind == 0 ? make_cuDoubleComplex(h, 0.0) : make_cuDoubleComplex(0.0, -h);
    coef[1] = kind == 0 ? make_cuDoubleComplex(h, 0.0) : make_cuDoubleComplex(0.0, h);
    return 2;
}

// G~ = T G' T^H (real symmetric), lower triangle column-major, from the Hermitian G' (lower triangle column-major)
__global__ void rgram_kernel(const cuDoubleComplex* __restrict__ G, int n, const int* __restrict__ rb_cls,
                             const int* __restrict__ rb_partner, const int* __restrict__ rb_kind, double* __restrict__ Gr) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= n || i < j) return;
    int ci[2], cj[2];
    cuDoubleComplex ai[2], aj[2];
    const int ni = rb_terms(rb_kind[i], rb_cls[i], rb_partner[i], ci, ai);
    const int nj = rb_terms(rb_kind[j], rb_cls[j], rb_partner[j], cj, aj);
    double acc = 0.0;
    for (int x = 0; x < ni; ++x)
        for (int y = 0; y < nj; ++y) {
            const int a = ci[x], b = cj[y];
            const cuDoubleComplex g = a >= b ? G[(int64_t)b * n + a] : cuConj(G[(int64_t)a * n + b]);
            // Re{ ai conj(aj) g }
            acc += cuCreal(cuCmul(cuCmul(ai[x], cuConj(aj[y])), g));
        }
    Gr[(int64_t)j * n + i] = acc;
}

// B~[i][d] (column-major n x D) = sqrt(n_i) U~[i][jd] / sqrt(lambda_jd)
__global__ void rbmat_kernel(const double* __restrict__ Ur, const double* __restrict__ lam, const int* __restrict__ cnt,
                             const int* __restrict__ rb_cls, int n, int D, double* __restrict__ B) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int d = blockIdx.y;
    if (i >= n) return;
    const int jd = n - 1 - d;
    B[(int64_t)d * n + i] = sqrt((double)cnt[rb_cls[i]] / lam[jd]) * Ur[(int64_t)jd * n + i];
}

// W~ chunk, column-major n x C (real): columns c0..c0+C-1 of eq. 8 in the real basis
__global__ void rwchunk_kernel(const double* __restrict__ tau, const int* __restrict__ rb_cls,
                               const int* __restrict__ rb_kind, int n, int P, int N, int Kb, int64_t c0, int C,
                               double* __restrict__ Wc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int cc = blockIdx.y;
    if (i >= n) return;
    const int64_t col = c0 + cc;
    const int p = (int)(col / Kb), k = (int)(col % Kb);
    double sn, cs;
    sincospi(2.0 * (double)k * tau[(int64_t)rb_cls[i] * P + p] / (double)N, &sn, &cs);
    const int kind = rb_kind[i];
    const double r2 = 1.41421356237309504880;
    Wc[(int64_t)cc * n + i] = kind == 0 ? r2 * cs : (kind == 1 ? r2 * sn : cs);
}

// real V chunk -> "part" V16 row d (svd_part: the projection's A rows carry Re x and Im x of a frame separately, so V is
// stored once per K position): unit u of chunk c, value s at (c*SP + u/16)*64 + (u%16)*4 + s
__global__ void pack_v16p_kernel(const double* __restrict__ Vc, int C, int64_t c0, int M, int Mi, int Kb, int bpc,
                                 int SP, int64_t K_P, double scale, __half* __restrict__ V16) {
    const int cc = blockIdx.x * blockDim.x + threadIdx.x;
    const int d = blockIdx.y;
    if (cc >= C) return;
    const int64_t col = c0 + cc;
    const int p = (int)(col / Kb), k = (int)(col % Kb);
    int i = 0, rem = p;
    while (rem >= M - 1 - i) {
        rem -= M - 1 - i;
        ++i;
    }
    const int pi = pair_index(i, i + 1 + rem, Mi);
    const int c = k / bpc;
    const int u = (bpc == 4) ? pi : (pi >> 1);
    const int sl = (bpc == 4) ? (k % 4) : ((pi & 1) * 2 + k % 2);
    V16[(int64_t)d * K_P + ((int64_t)c * SP + u / 16) * 64 + (u % 16) * 4 + sl] =
        __double2half(scale * Vc[(int64_t)d * C + cc]);
}

// class-basis eigenvectors U' = T^H U~ (columns jd >= n - D) into the complex n x n buffer read by pack_r16_kernel:
// pair rows (ip, im): U'_c = (U~_ip + j U~_im)/sqrt2, U'_c' = (U~_ip - j U~_im)/sqrt2; a real row: U'_c = U~_ip
__global__ void ucplx_kernel(const double* __restrict__ Ur, const int* __restrict__ cls_ip,
                             const int* __restrict__ cls_im, const int* __restrict__ cls_sign, int n, int D,
                             cuDoubleComplex* __restrict__ Uc) {
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    const int d = blockIdx.y;
    if (a >= n) return;
    const int jd = n - 1 - d;
    const double up = Ur[(int64_t)jd * n + cls_ip[a]];
    if (cls_im[a] < 0) {
        Uc[(int64_t)jd * n + a] = make_cuDoubleComplex(up, 0.0);
    } else {
        const double h = 0.70710678118654752440;
        const double um = Ur[(int64_t)jd * n + cls_im[a]];
        Uc[(int64_t)jd * n + a] = make_cuDoubleComplex(h * up, h * cls_sign[a] * um);
    }
}

// Row a of the dictionary: Rhat_a = normalise(U'[a][jd] sqrt(lambda_d)) -> R16 FP16 [Re | -Im] (search GEMM) and R32
// FP32 [Re | -Im] (exact rescore of the search candidates)
__global__ void pack_r16_kernel(const cuDoubleComplex* __restrict__ Uv, const double* __restrict__ lam, int n, int D,
                                int Dh, int K2, __half* __restrict__ R16, float* __restrict__ R32) {
    const int a = blockIdx.x;
    __shared__ double red[32];
    double ss = 0.0;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        const int jd = n - 1 - d;
        const cuDoubleComplex u = Uv[(int64_t)jd * n + a];
        ss += (u.x * u.x + u.y * u.y) * lam[jd];
    }
    for (int o = 16; o >= 1; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) red[0] = v;
    }
    __syncthreads();
    const double inv = 1.0 / sqrt(red[0]);
    __half* row = R16 + (int64_t)a * K2;
    float* row32 = R32 + (int64_t)a * K2;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
        const int jd = n - 1 - d;
        const cuDoubleComplex u = Uv[(int64_t)jd * n + a];
        const double sl = sqrt(lam[jd]) * inv;
        const float vr = (float)(u.x * sl), vi = (float)(-u.y * sl);  // [Re R | -Im R]
        row[d] = __float2half_rn(vr);
        row[Dh + d] = __float2half_rn(vi);
        row32[d] = vr;
        row32[Dh + d] = vi;
    }
}

static inline unsigned cdiv(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

svdphat_status setup_srp_operand(Plan& p, const double* d_tau_cls) {
    p.bytes_W = (int64_t)p.W_rows * p.K_W * 2;
    SVD_CUDA_TRY(cudaMalloc(&p.d_W16, p.bytes_W));
    SVD_CUDA_TRY(cudaMemset(p.d_W16, 0, p.bytes_W));
    if (p.fold) {
        const int64_t n = (int64_t)p.fold_rows * p.P;
        pack_w16f_kernel<<<cdiv(n, 256), 256>>>(d_tau_cls, p.d_fold_cls, p.fold_rows, p.P, p.M, p.L.Mi, p.N, p.Kb,
                                                p.L.bpc, p.spc_W / 2, p.K_W, p.d_W16);
    } else {
        const int64_t n = (int64_t)p.Q_eff * p.P;
        pack_w16_kernel<<<cdiv(n, 256), 256>>>(d_tau_cls, p.Q_eff, p.P, p.M, p.L.Mi, p.N, p.Kb, p.L.bpc, p.L.U,
                                               p.K_W, p.d_W16);
    }
    SVD_CUDA_TRY(cudaGetLastError());
    SVD_CUDA_TRY(cudaDeviceSynchronize());
    return SVDPHAT_OK;
}

// V row tiling of the frames-on-M pair projections: the fewest tiles covering `rows`, each a multiple of 32 rows and at
// most 256 (complex V, gemm2f: one MMA of N <= 256 per K step) or 512 (real V "part" kernel gemm2p: one accumulator of
// <= 512 TMEM columns, ceil(nt/256) MMAs per K step).  cfg3: real V, D = 318 (+2 SRP tail rows) -> 1 x 320; complex
// V, 2*D_h = 640 -> 3 x 224.
static void choose_proj_tiles(Plan& p, int rows) {
    if (!p.pair_proj) {
        p.V_rows = rows;
        return;
    }
    const int cap = p.svd_fold ? 512 : 256;
    p.proj_ntiles = (rows + cap - 1) / cap;
    p.proj_nt = ((rows + p.proj_ntiles - 1) / p.proj_ntiles + 31) / 32 * 32;
    p.V_rows = p.proj_ntiles * p.proj_nt;
    p.proj_nmma = p.proj_nt > 256 ? 2 : 1;
}

namespace {
struct DevBuf {
    void* ptr = nullptr;
    ~DevBuf() {
        if (ptr) cudaFree(ptr);
    }
};
}  // namespace

// svd_fold: V_D = W~^T N^1/2 U~ Lambda^{-1/2} (real; DGEMM on generated W~ chunks) packed as fold rows, and the
// class-basis eigenvectors U' = T^H U~ written into Uc for the dictionary rows.
static svdphat_status setup_real_v(Plan& p, const double* d_tau_cls, int n, int D, const double* Ur, const double* lam,
                                   const int* cnt, const int* d_rb, cuDoubleComplex* Uc) {
    DevBuf B, Wc, Vc, maps, pc;
    SVD_CUDA_TRY(cudaMalloc(&B.ptr, (size_t)n * D * sizeof(double)));
    {
        dim3 grid(cdiv(n, 128), D);
        rbmat_kernel<<<grid, 128>>>(Ur, lam, cnt, d_rb, n, D, (double*)B.ptr);
        SVD_CUDA_TRY(cudaGetLastError());
    }
    choose_proj_tiles(p, D + 2 * p.tail_n);                 // + the SRP tail rows (a Re row and an Im row each)
    p.bytes_V = (int64_t)p.V_rows * p.K_P * 2;
    SVD_CUDA_TRY(cudaMalloc(&p.d_V16, p.bytes_V));
    SVD_CUDA_TRY(cudaMemset(p.d_V16, 0, p.bytes_V));
    int64_t CH = std::max<int64_t>(256, std::min<int64_t>(p.PK, (int64_t)(1ll << 30) / ((int64_t)n * 8)));
    CH = std::min<int64_t>(CH, 16384);
    SVD_CUDA_TRY(cudaMalloc(&Wc.ptr, (size_t)n * CH * sizeof(double)));
    SVD_CUDA_TRY(cudaMalloc(&Vc.ptr, (size_t)CH * D * sizeof(double)));
    cublasHandle_t bh = nullptr;
    if (cublasCreate(&bh) != CUBLAS_STATUS_SUCCESS) {
        set_error("cublasCreate failed");
        return SVDPHAT_CUDA;
    }
    const double one = 1.0, zero = 0.0;
    const double scale = std::sqrt((double)p.PK);
    for (int64_t c0 = 0; c0 < p.PK; c0 += CH) {
        const int C = (int)std::min<int64_t>(CH, p.PK - c0);
        dim3 g1(cdiv(n, 128), C);
        rwchunk_kernel<<<g1, 128>>>(d_tau_cls, d_rb, d_rb + 2 * n, n, p.P, p.N, p.Kb, c0, C, (double*)Wc.ptr);
        cublasStatus_t bs = cublasDgemm(bh, CUBLAS_OP_T, CUBLAS_OP_N, C, D, n, &one, (const double*)Wc.ptr, n,
                                        (const double*)B.ptr, n, &zero, (double*)Vc.ptr, C);
        if (bs != CUBLAS_STATUS_SUCCESS) {
            cublasDestroy(bh);
            set_error("cublasDgemm failed: " + std::to_string((int)bs));
            return SVDPHAT_CUDA;
        }
        dim3 g2(cdiv(C, 128), D);
        pack_v16p_kernel<<<g2, 128>>>((const double*)Vc.ptr, C, c0, p.M, p.L.Mi, p.Kb, p.L.bpc, p.spc_P, p.K_P,
                                      scale, p.d_V16);
    }
    cublasDestroy(bh);
    SVD_CUDA_TRY(cudaGetLastError());
    // class -> its real rows: Re row, Im row (-1 for a real row), sign of the Im part (+ for c, - for the antipode)
    std::vector<int> ip(n, -1), im(n, -1), sg(n, 1);
    for (int i = 0; i < n; ++i) {
        const int c = p.rb_cls[i], cp = p.rb_partner[i];
        if (p.rb_kind[i] == 2) {
            ip[c] = i;
        } else if (p.rb_kind[i] == 0) {
            ip[c] = ip[cp] = i;
            sg[cp] = -1;
        } else {
            im[c] = im[cp] = i;
        }
    }
    SVD_CUDA_TRY(cudaMalloc(&maps.ptr, (size_t)3 * n * sizeof(int)));
    int* d_maps = (int*)maps.ptr;
    SVD_CUDA_TRY(cudaMemcpy(d_maps, ip.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice));
    SVD_CUDA_TRY(cudaMemcpy(d_maps + n, im.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice));
    SVD_CUDA_TRY(cudaMemcpy(d_maps + 2 * n, sg.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice));
    {
        dim3 grid(cdiv(n, 128), D);
        ucplx_kernel<<<grid, 128>>>(Ur, d_maps, d_maps + n, d_maps + 2 * n, n, D, Uc);
        SVD_CUDA_TRY(cudaGetLastError());
    }
    SVD_CUDA_TRY(cudaDeviceSynchronize());
    return SVDPHAT_OK;
}

svdphat_status setup_svd_operands(Plan& p, const double* d_tau_cls, int rank_D) {
    const int n = p.Q_eff;
    DevBuf G, lam, cnt, work, info, B, Wc, Vc;
    SVD_CUDA_TRY(cudaMalloc(&G.ptr, (size_t)n * n * sizeof(cuDoubleComplex)));
    SVD_CUDA_TRY(cudaMalloc(&lam.ptr, (size_t)n * sizeof(double)));
    SVD_CUDA_TRY(cudaMalloc(&cnt.ptr, (size_t)n * sizeof(int)));
    SVD_CUDA_TRY(cudaMalloc(&info.ptr, sizeof(int)));
    SVD_CUDA_TRY(cudaMemcpy(cnt.ptr, p.cls_count.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice));
    {
        dim3 grid(cdiv(n, 128), n);
        gram_kernel<<<grid, 128>>>(d_tau_cls, (const int*)cnt.ptr, n, p.P, p.N, p.Kb, (cuDoubleComplex*)G.ptr);
        SVD_CUDA_TRY(cudaGetLastError());
    }
    // ---- eigendecomposition (float64, cuSOLVER): Hermitian G', or (svd_fold) the real symmetric G~ = T G' T^H
    DevBuf Gr, rb;
    int* d_rb = nullptr;                                     // [3][n] real basis: class, partner, kind
    if (p.svd_fold) {
        SVD_CUDA_TRY(cudaMalloc(&Gr.ptr, (size_t)n * n * sizeof(double)));
        SVD_CUDA_TRY(cudaMalloc(&rb.ptr, (size_t)3 * n * sizeof(int)));
        d_rb = (int*)rb.ptr;
        SVD_CUDA_TRY(cudaMemcpy(d_rb, p.rb_cls.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice));
        SVD_CUDA_TRY(cudaMemcpy(d_rb + n, p.rb_partner.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice));
        SVD_CUDA_TRY(cudaMemcpy(d_rb + 2 * n, p.rb_kind.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice));
        dim3 grid(cdiv(n, 128), n);
        rgram_kernel<<<grid, 128>>>((const cuDoubleComplex*)G.ptr, n, d_rb, d_rb + n, d_rb + 2 * n, (double*)Gr.ptr);
        SVD_CUDA_TRY(cudaGetLastError());
    }
    cusolverDnHandle_t sh = nullptr;
    if (cusolverDnCreate(&sh) != CUSOLVER_STATUS_SUCCESS) {
        set_error("cusolverDnCreate failed");
        return SVDPHAT_CUDA;
    }
    int lwork = 0;
    cusolverStatus_t cs =
        p.svd_fold ? cusolverDnDsyevd_bufferSize(sh, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                                 (double*)Gr.ptr, n, (double*)lam.ptr, &lwork)
                   : cusolverDnZheevd_bufferSize(sh, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                                 (cuDoubleComplex*)G.ptr, n, (double*)lam.ptr, &lwork);
    if (cs != CUSOLVER_STATUS_SUCCESS) {
        cusolverDnDestroy(sh);
        set_error("cusolver eigensolver bufferSize failed: " + std::to_string((int)cs));
        return SVDPHAT_CUDA;
    }
    {
        cudaError_t e = cudaMalloc(&work.ptr, (size_t)lwork * (p.svd_fold ? sizeof(double) : sizeof(cuDoubleComplex)));
        if (e != cudaSuccess) {
            cusolverDnDestroy(sh);
            set_error("eigensolver workspace allocation failed");
            return SVDPHAT_ALLOC;
        }
    }
    cs = p.svd_fold ? cusolverDnDsyevd(sh, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n, (double*)Gr.ptr, n,
                                       (double*)lam.ptr, (double*)work.ptr, lwork, (int*)info.ptr)
                    : cusolverDnZheevd(sh, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n,
                                       (cuDoubleComplex*)G.ptr, n, (double*)lam.ptr, (cuDoubleComplex*)work.ptr,
                                       lwork, (int*)info.ptr);
    cudaError_t se = cudaDeviceSynchronize();
    cusolverDnDestroy(sh);
    int hinfo = 0;
    cudaMemcpy(&hinfo, info.ptr, sizeof(int), cudaMemcpyDeviceToHost);
    if (cs != CUSOLVER_STATUS_SUCCESS || se != cudaSuccess || hinfo != 0) {
        set_error("cusolver eigensolver failed: status " + std::to_string((int)cs) + " info " + std::to_string(hinfo));
        return SVDPHAT_NUMERIC;
    }
    cudaFree(work.ptr);
    work.ptr = nullptr;
    std::vector<double> hl(n);
    SVD_CUDA_TRY(cudaMemcpy(hl.data(), lam.ptr, (size_t)n * sizeof(double), cudaMemcpyDeviceToHost));
    p.sigma2.resize(n);
    for (int i = 0; i < n; ++i) p.sigma2[i] = std::max(0.0, hl[n - 1 - i]);
    for (double v : p.sigma2)
        if (!std::isfinite(v)) {
            set_error("non-finite eigenvalue");
            return SVDPHAT_NUMERIC;
        }
    // ---- rank rule (eq. 11): smallest D with sum_{d<=D} sigma^2 >= (1 - delta) Q P Kb
    int numrank = 0;
    for (int i = 0; i < n; ++i)
        if (p.sigma2[i] > 1e-12 * p.sigma2[0]) numrank = i + 1;
    int D = 0;
    if (rank_D > 0) {
        D = std::min(rank_D, numrank);
    } else {
        double acc = 0.0;
        D = numrank;
        for (int i = 0; i < n; ++i) {
            acc += p.sigma2[i];
            if (acc >= (1.0 - p.delta) * p.trace) {
                D = i + 1;
                break;
            }
        }
        D = std::min(D, numrank);
    }
    if (D < 1) D = 1;
    p.D = D;
    double kept = 0.0;
    for (int i = 0; i < D; ++i) kept += p.sigma2[i];
    p.energy_kept = kept / p.trace;
    p.Dh = (D + 63) / 64 * 64;
    p.K2 = 2 * p.Dh;

    if (p.svd_fold) {
        svdphat_status st = setup_real_v(p, d_tau_cls, n, D, (const double*)Gr.ptr, (const double*)lam.ptr,
                                         (const int*)cnt.ptr, d_rb, (cuDoubleComplex*)G.ptr);
        if (st != SVDPHAT_OK) return st;
    } else {
        // ---- V_D = W^H N^1/2 U' Lambda^{-1/2}, column chunks of W, ZGEMM (float64)
        SVD_CUDA_TRY(cudaMalloc(&B.ptr, (size_t)n * D * sizeof(cuDoubleComplex)));
        {
            dim3 grid(cdiv(n, 128), D);
            bmat_kernel<<<grid, 128>>>((const cuDoubleComplex*)G.ptr, (const double*)lam.ptr, (const int*)cnt.ptr, n, D,
                                       (cuDoubleComplex*)B.ptr);
            SVD_CUDA_TRY(cudaGetLastError());
        }
        choose_proj_tiles(p, 2 * p.Dh);
        p.bytes_V = (int64_t)p.V_rows * p.L.K_total * 2;
        SVD_CUDA_TRY(cudaMalloc(&p.d_V16, p.bytes_V));
        SVD_CUDA_TRY(cudaMemset(p.d_V16, 0, p.bytes_V));
        int64_t CH = std::max<int64_t>(256, std::min<int64_t>(p.PK, (int64_t)(1ll << 30) / ((int64_t)n * 16)));
        CH = std::min<int64_t>(CH, 16384);
        SVD_CUDA_TRY(cudaMalloc(&Wc.ptr, (size_t)n * CH * sizeof(cuDoubleComplex)));
        SVD_CUDA_TRY(cudaMalloc(&Vc.ptr, (size_t)CH * D * sizeof(cuDoubleComplex)));
        cublasHandle_t bh = nullptr;
        if (cublasCreate(&bh) != CUBLAS_STATUS_SUCCESS) {
            set_error("cublasCreate failed");
            return SVDPHAT_CUDA;
        }
        const cuDoubleComplex one = make_cuDoubleComplex(1, 0), zero = make_cuDoubleComplex(0, 0);
        const double scale = std::sqrt((double)p.PK);
        for (int64_t c0 = 0; c0 < p.PK; c0 += CH) {
            const int C = (int)std::min<int64_t>(CH, p.PK - c0);
            dim3 g1(cdiv(n, 128), C);
            wchunk_kernel<<<g1, 128>>>(d_tau_cls, n, p.P, p.N, p.Kb, c0, C, (cuDoubleComplex*)Wc.ptr);
            cublasStatus_t bs = cublasZgemm(bh, CUBLAS_OP_C, CUBLAS_OP_N, C, D, n, &one, (cuDoubleComplex*)Wc.ptr, n,
                                            (cuDoubleComplex*)B.ptr, n, &zero, (cuDoubleComplex*)Vc.ptr, C);
            if (bs != CUBLAS_STATUS_SUCCESS) {
                cublasDestroy(bh);
                set_error("cublasZgemm failed: " + std::to_string((int)bs));
                return SVDPHAT_CUDA;
            }
            dim3 g2(cdiv(C, 128), D);
            pack_v16_kernel<<<g2, 128>>>((const cuDoubleComplex*)Vc.ptr, C, D, p.Dh, c0, p.M, p.L.Mi, p.Kb, p.L.bpc,
                                         p.L.U, p.L.K_total, scale, p.d_V16);
        }
        cublasDestroy(bh);
        SVD_CUDA_TRY(cudaGetLastError());
    }
    // ---- normalised dictionary rows (split FP16)
    p.bytes_R = (int64_t)p.Q_pad * p.K2 * 2 + (int64_t)n * p.K2 * 4;
    SVD_CUDA_TRY(cudaMalloc(&p.d_R16, (size_t)p.Q_pad * p.K2 * 2));
    SVD_CUDA_TRY(cudaMemset(p.d_R16, 0, (size_t)p.Q_pad * p.K2 * 2));
    SVD_CUDA_TRY(cudaMalloc(&p.d_R32, (size_t)n * p.K2 * 4));
    SVD_CUDA_TRY(cudaMemset(p.d_R32, 0, (size_t)n * p.K2 * 4));
    pack_r16_kernel<<<n, 256>>>((const cuDoubleComplex*)G.ptr, (const double*)lam.ptr, n, D, p.Dh, p.K2, p.d_R16,
                                p.d_R32);
    SVD_CUDA_TRY(cudaGetLastError());
    SVD_CUDA_TRY(cudaDeviceSynchronize());
    return SVDPHAT_OK;
}

}  // namespace svdphat
