// api.cu — the C-ABI of libsvdphat (include/svdphat.h): validation, float64 geometry, steering classes, plan
// assembly and the per-call orchestration of the hot path kernels.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <new>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "internal.h"

namespace svdphat {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }

static svdphat_status fail(svdphat_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

// No C++ exception crosses the C ABI: a host allocation failure (std::bad_alloc) becomes ALLOC, anything else CUDA.
template <class Fn>
static svdphat_status guarded(Fn&& fn) {
    try {
        return fn();
    } catch (const std::bad_alloc&) {
        return fail(SVDPHAT_ALLOC, "host allocation failed");
    } catch (const std::exception& e) {
        return fail(SVDPHAT_CUDA, std::string("internal error: ") + e.what());
    } catch (...) {
        return fail(SVDPHAT_CUDA, "internal error");
    }
}

// Every entry point runs on the plan's device and restores the caller's current device on return.
struct DeviceGuard {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        if (prev != dev) err = cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
    }
};
#define SVD_DEVICE_GUARD(dev)                                                                            \
    DeviceGuard _dg(dev);                                                                                \
    if (_dg.err != cudaSuccess)                                                                          \
        return fail(SVDPHAT_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(_dg.err));

// Allocates a pair of per-plan buffers that are used together: both or neither (a partial failure frees the first
// and clears the runtime's sticky last-error so a later launch check does not report it).
static bool alloc_pair(void** a, size_t na, void** b, size_t nb) {
    if (*a && *b) return true;
    if (*a) cudaFree(*a);
    if (*b) cudaFree(*b);
    *a = *b = nullptr;
    if (cudaMalloc(a, na) != cudaSuccess) {
        *a = nullptr;
        cudaGetLastError();
        return false;
    }
    if (cudaMalloc(b, nb) != cudaSuccess) {
        cudaFree(*a);
        *a = *b = nullptr;
        cudaGetLastError();
        return false;
    }
    return true;
}

// ---------------------------------------------------------------- TMA descriptor encoding (driver entry point)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}

// 2-D FP16 row-major [rows][cols] tensor, box = 64 cols (128 B) x box_rows, 128-byte swizzle
static bool encode_2d(CUtensorMap* tm, const void* base, int64_t rows, int64_t cols, int box_rows) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// 2-D FP16 row-major [rows][cols] tensor, box = cols x box_rows with cols * 2 bytes in {32, 64, 128} and the
// matching swizzle (the K-major operand rows of das_kernel: one bin's 2 ME halves per row)
static bool encode_2d_rows(CUtensorMap* tm, const void* base, int64_t rows, int cols, int box_rows) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    const CUtensorMapSwizzle sw = cols == 64   ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : cols == 32 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : cols == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                               : CU_TENSOR_MAP_SWIZZLE_NONE;
    if (sw == CU_TENSOR_MAP_SWIZZLE_NONE) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {(cuuint32_t)cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static Layout make_layout(int M, int N) {
    Layout L;
    L.M = M;
    L.Mi = M <= 4 ? 4 : M <= 8 ? 8 : M <= 16 ? 16 : 32;
    L.P = M * (M - 1) / 2;
    L.Pi = L.Mi * (L.Mi - 1) / 2;
    L.N = N;
    L.Kb = N / 2 + 1;
    L.bpc = L.Mi <= 16 ? 4 : 2;
    L.n_chunks = (L.Kb + L.bpc - 1) / L.bpc;
    const int units = L.bpc == 4 ? L.Pi : (L.Pi + 1) / 2;
    L.U = (units + 7) / 8 * 8;
    L.K_total = (int64_t)L.n_chunks * L.U * 8;
    L.unit_bytes = L.bpc * 4;
    return L;
}

static svdphat_status validate(const svdphat_plan_desc* d) {
    if (!d) return fail(SVDPHAT_INVALID_ARG, "desc is NULL");
    if (d->M < 2 || d->M > 32) return fail(SVDPHAT_INVALID_ARG, "M must be in [2, 32]");
    if (!d->mic_xyz || !d->points_xyz) return fail(SVDPHAT_INVALID_ARG, "mic_xyz / points_xyz is NULL");
    if (!(d->fs > 0) || !std::isfinite(d->fs)) return fail(SVDPHAT_INVALID_ARG, "fs must be > 0");
    if (!(d->c > 0) || !std::isfinite(d->c)) return fail(SVDPHAT_INVALID_ARG, "c must be > 0");
    if (d->N < 16 || d->N > 2048 || (d->N & (d->N - 1)))
        return fail(SVDPHAT_INVALID_ARG, "N must be a power of two in [16, 2048]");
    if (d->hop <= 0 || d->hop > d->N) return fail(SVDPHAT_INVALID_ARG, "hop must be in (0, N]");
    if (d->field != SVDPHAT_FIELD_FAR && d->field != SVDPHAT_FIELD_NEAR)
        return fail(SVDPHAT_INVALID_ARG, "field must be FAR or NEAR");
    if (d->Q < 1 || d->Q > (1 << 24)) return fail(SVDPHAT_INVALID_ARG, "Q must be in [1, 2^24]");
    if (d->methods <= 0 || (d->methods & ~(SVDPHAT_METHOD_SRP | SVDPHAT_METHOD_SVD)))
        return fail(SVDPHAT_INVALID_ARG, "methods must be a non-empty subset of SRP|SVD");
    if ((d->methods & SVDPHAT_METHOD_SVD) && d->rank_D <= 0 && !(d->delta > 0 && d->delta < 1))
        return fail(SVDPHAT_INVALID_ARG, "delta must be in (0, 1)");
    if (d->rank_D < 0) return fail(SVDPHAT_INVALID_ARG, "rank_D must be >= 0");
    if (d->max_frames < 0 || d->max_frames > (1ll << 26)) return fail(SVDPHAT_INVALID_ARG, "max_frames out of range");
    if (d->options & ~(SVDPHAT_OPT_NO_SRP_FOLD | SVDPHAT_OPT_NO_SVD_FOLD | SVDPHAT_OPT_ONE_CTA_SRP |
                       SVDPHAT_OPT_ONE_CTA_PROJ | SVDPHAT_OPT_NO_DAS | SVDPHAT_OPT_DAS | SVDPHAT_OPT_DAS_FOLD))
        return fail(SVDPHAT_INVALID_ARG, "unknown option bits");
    for (int i = 0; i < 3 * d->M; ++i)
        if (!std::isfinite(d->mic_xyz[i])) return fail(SVDPHAT_INVALID_ARG, "non-finite microphone coordinate");
    for (int64_t q = 0; q < d->Q; ++q) {
        const double* s = d->points_xyz + 3 * q;
        if (!std::isfinite(s[0]) || !std::isfinite(s[1]) || !std::isfinite(s[2]))
            return fail(SVDPHAT_INVALID_ARG, "non-finite candidate point " + std::to_string(q));
        if (d->field == SVDPHAT_FIELD_FAR && s[0] == 0 && s[1] == 0 && s[2] == 0)
            return fail(SVDPHAT_INVALID_ARG, "zero far-field direction at " + std::to_string(q));
    }
    return SVDPHAT_OK;
}

// Records a start/end event pair around one kernel launch when profiling is on.
template <class Fn>
cudaError_t staged(Plan& p, int stage, cudaStream_t s, Fn&& fn) {
    const bool rec = p.prof_on && p.prof_n < p.prof_cap;
    if (rec) cudaEventRecord(p.prof_ev[2 * p.prof_n], s);
    cudaError_t e = fn();
    if (rec) {
        cudaEventRecord(p.prof_ev[2 * p.prof_n + 1], s);
        p.prof_stage[p.prof_n++] = stage;
    }
    return e;
}

}  // namespace svdphat

using namespace svdphat;

struct svdphat_plan_s {
    Plan p;
    ~svdphat_plan_s() {
        for (cudaEvent_t e : p.prof_ev) cudaEventDestroy(e);
        for (int i = 0; i < 2; ++i) {
            if (p.ev_copied[i]) cudaEventDestroy(p.ev_copied[i]);
            if (p.ev_done[i]) cudaEventDestroy(p.ev_done[i]);
        }
        if (p.copy_stream) cudaStreamDestroy(p.copy_stream);
        for (auto& sl : p.slots) {
            if (sl.d_audio) cudaFree(sl.d_audio);
            if (sl.d_doa) cudaFree(sl.d_doa);
            if (sl.d_score) cudaFree(sl.d_score);
            if (sl.h2d) cudaEventDestroy(sl.h2d);
            if (sl.comp) cudaEventDestroy(sl.comp);
            if (sl.d2h) cudaEventDestroy(sl.d2h);
        }
        if (p.up_stream) cudaStreamDestroy(p.up_stream);
        if (p.down_stream) cudaStreamDestroy(p.down_stream);
        if (p.ev_fork) cudaEventDestroy(p.ev_fork);
        if (p.ev_join) cudaEventDestroy(p.ev_join);
        if (p.svd_stream) cudaStreamDestroy(p.svd_stream);
        if (p.srp_stream) cudaStreamDestroy(p.srp_stream);
        if (p.ev_join2) cudaEventDestroy(p.ev_join2);
        if (p.ev_z) cudaEventDestroy(p.ev_z);
        void* bufs[] = {p.d_W16,   p.d_V16,   p.d_R16,   p.d_rep,   p.d_delay,     p.d_window,      p.d_twN,
                        p.d_P16,   p.d_keys,  p.d_Z32,   p.d_Zs16,  p.d_zflag,     p.d_stage,       p.d_doa_stage,
                        p.d_R32,   p.d_Zn32,  p.d_cand,  p.d_ccnt,  p.d_Smap,
                        p.d_score_stage, p.d_S, p.d_cls, p.d_dirs, p.d_Ypart, p.d_fold_cls, p.d_A16, p.d_E16};
        for (void* b : bufs)
            if (b) cudaFree(b);
    }
};

extern "C" {

const char* svdphat_status_str(svdphat_status s) {
    switch (s) {
        case SVDPHAT_OK: return "OK";
        case SVDPHAT_INVALID_ARG: return "INVALID_ARG";
        case SVDPHAT_ALLOC: return "ALLOC";
        case SVDPHAT_CUDA: return "CUDA";
        case SVDPHAT_NUMERIC: return "NUMERIC";
        case SVDPHAT_UNSUPPORTED: return "UNSUPPORTED";
        case SVDPHAT_TOO_LARGE: return "TOO_LARGE";
    }
    return "UNKNOWN";
}

const char* svdphat_last_error(void) { return g_err.c_str(); }

int64_t svdphat_frame_count(int64_t L, int32_t N, int32_t hop) {
    if (N <= 0 || hop <= 0 || L < N) return 0;
    return 1 + (L - N) / hop;
}

void svdphat_plan_destroy(svdphat_plan_t plan) {
    if (!plan) return;
    DeviceGuard g(plan->p.device);
    try {
        delete plan;
    } catch (...) {
    }
}

static svdphat_status plan_create_impl(const svdphat_plan_desc* d, svdphat_plan_t* out) {
    if (!out) return fail(SVDPHAT_INVALID_ARG, "out is NULL");
    *out = nullptr;
    svdphat_status st = validate(d);
    if (st != SVDPHAT_OK) return st;
    const auto t0 = std::chrono::steady_clock::now();

    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(SVDPHAT_UNSUPPORTED, "no CUDA device");
    }
    if (d->device < 0 || d->device >= ndev) return fail(SVDPHAT_INVALID_ARG, "device ordinal out of range");
    SVD_DEVICE_GUARD(d->device);
    cudaDeviceProp prop;
    SVD_CUDA_TRY(cudaGetDeviceProperties(&prop, d->device));
    if (prop.major != 10 || prop.minor != 0)
        return fail(SVDPHAT_UNSUPPORTED, "libsvdphat is built for sm_100a; device is sm_" +
                                             std::to_string(prop.major) + std::to_string(prop.minor));

    std::unique_ptr<svdphat_plan_s> h(new svdphat_plan_s());
    Plan& p = h->p;
    p.M = d->M;
    p.N = d->N;
    p.hop = d->hop;
    p.Kb = d->N / 2 + 1;
    p.P = d->M * (d->M - 1) / 2;
    p.PK = (int64_t)p.P * p.Kb;
    p.Q = d->Q;
    p.field = d->field;
    p.methods = d->methods;
    p.device = d->device;
    p.fs = d->fs;
    p.c = d->c;
    p.delta = d->delta;
    p.max_frames = d->max_frames;
    p.F_pad = std::max<int64_t>(256, (d->max_frames + 255) / 256 * 256);
    p.L = make_layout(d->M, d->N);
    p.options = d->options;
    p.trace = (double)p.Q * (double)p.P * (double)p.Kb;  // Tr{W W^H}, every |W| = 1 (eq. 4)
    p.num_sms = prop.multiProcessorCount;

    // ---- TDOAs in samples (float64): eq. 2 (FAR) or eq. 1 (NEAR); arrival delays
    const int M = p.M, P = p.P, Q = p.Q;
    const double k = p.fs / p.c;
    if ((double)Q * P * 8.0 > (double)(48ll << 30))                   // host float64 TDOA table
        return fail(SVDPHAT_TOO_LARGE, "Q * P TDOA table exceeds 48 GB of host memory");
    std::vector<double> tau((size_t)Q * P), delay((size_t)Q * M);
    const double* r = d->mic_xyz;
    for (int q = 0; q < Q; ++q) {
        const double* s = d->points_xyz + 3 * (size_t)q;
        double* dl = &delay[(size_t)q * M];
        if (p.field == SVDPHAT_FIELD_FAR) {
            const double nrm = std::sqrt(s[0] * s[0] + s[1] * s[1] + s[2] * s[2]);
            const double u[3] = {s[0] / nrm, s[1] / nrm, s[2] / nrm};
            int pp = 0;
            for (int i = 0; i < M; ++i)
                for (int j = i + 1; j < M; ++j) {
                    const double dx = r[3 * j] - r[3 * i], dy = r[3 * j + 1] - r[3 * i + 1],
                                 dz = r[3 * j + 2] - r[3 * i + 2];
                    tau[(size_t)q * P + pp++] = k * (dx * u[0] + dy * u[1] + dz * u[2]) + 0.0;  // +0.0: no -0 rows
                }
            for (int m = 0; m < M; ++m) dl[m] = -k * (r[3 * m] * u[0] + r[3 * m + 1] * u[1] + r[3 * m + 2] * u[2]);
        } else {
            std::vector<double> dist(M);
            for (int m = 0; m < M; ++m) {
                const double dx = s[0] - r[3 * m], dy = s[1] - r[3 * m + 1], dz = s[2] - r[3 * m + 2];
                dist[m] = std::sqrt(dx * dx + dy * dy + dz * dz);
                dl[m] = k * dist[m];
            }
            int pp = 0;
            for (int i = 0; i < M; ++i)
                for (int j = i + 1; j < M; ++j) tau[(size_t)q * P + pp++] = k * (dist[i] - dist[j]) + 0.0;
        }
        const double mn = *std::min_element(dl, dl + M);
        for (int m = 0; m < M; ++m) dl[m] -= mn;
    }

    // ---- steering classes: bitwise-identical tau rows share one W row (R11); rep = lowest index
    {
        std::unordered_map<uint64_t, std::vector<int>> buckets;
        std::vector<int> cls_of(Q, -1);
        for (int q = 0; q < Q; ++q) {
            const unsigned char* b = reinterpret_cast<const unsigned char*>(&tau[(size_t)q * P]);
            uint64_t hsh = 1469598103934665603ull;
            for (size_t i = 0; i < (size_t)P * 8; ++i) hsh = (hsh ^ b[i]) * 1099511628211ull;
            auto& v = buckets[hsh];
            int found = -1;
            for (int c : v)
                if (std::memcmp(&tau[(size_t)p.rep_q[c] * P], &tau[(size_t)q * P], (size_t)P * 8) == 0) {
                    found = c;
                    break;
                }
            if (found < 0) {
                found = (int)p.rep_q.size();
                p.rep_q.push_back(q);
                p.cls_count.push_back(0);
                v.push_back(found);
            }
            p.cls_count[found]++;
            cls_of[q] = found;
        }
    }
    p.Q_eff = (int)p.rep_q.size();
    p.pair_srp = !(p.options & SVDPHAT_OPT_ONE_CTA_SRP);
    p.Q_pad = p.pair_srp ? (p.Q_eff + 255) / 256 * 256 : (p.Q_eff + 127) / 128 * 128;

    p.pair_proj = !(p.options & SVDPHAT_OPT_ONE_CTA_PROJ);
    // ---- antipodal class pairs (R22): class c' is the antipode of class c when its tau row is the bitwise
    // negation of c's (far field on a centrally symmetric grid: eq. 2 is odd in s_q, so every product and sum
    // negates exactly).  Then W_c' = conj W_c (eq. 4): one SRP fold row gives both scores, and W^H W is real, so
    // the SVD's V can be taken real (the projection then folds the same way).  A class whose tau row is all zeros is
    // its own antipode (a real W row).
    std::vector<int> fold_m, fold_p;
    bool all_paired = true;
    {
        auto row_hash = [&](const double* t) {
            const unsigned char* b = reinterpret_cast<const unsigned char*>(t);
            uint64_t hsh = 1469598103934665603ull;
            for (size_t i = 0; i < (size_t)P * 8; ++i) hsh = (hsh ^ b[i]) * 1099511628211ull;
            return hsh;
        };
        std::unordered_map<uint64_t, std::vector<int>> by_hash;
        for (int c = 0; c < p.Q_eff; ++c) by_hash[row_hash(&tau[(size_t)p.rep_q[c] * P])].push_back(c);
        std::vector<double> neg(P);
        std::vector<char> used(p.Q_eff, 0);
        for (int c = 0; c < p.Q_eff; ++c) {
            if (used[c]) continue;
            const double* t = &tau[(size_t)p.rep_q[c] * P];
            bool zero = true;
            for (int i = 0; i < P; ++i) {
                neg[i] = -t[i] + 0.0;                                  // +0.0: rows never hold -0
                zero = zero && t[i] == 0.0;
            }
            int partner = -1;
            auto it = by_hash.find(row_hash(neg.data()));
            if (it != by_hash.end())
                for (int c2 : it->second)
                    if (c2 != c && !used[c2] &&
                        std::memcmp(&tau[(size_t)p.rep_q[c2] * P], neg.data(), (size_t)P * 8) == 0) {
                        partner = c2;
                        break;
                    }
            used[c] = 1;
            if (partner >= 0) used[partner] = 1;
            all_paired = all_paired && (partner >= 0 || zero);
            fold_m.push_back(c);
            fold_p.push_back(partner);
        }
    }
    const bool few_rows = 4 * (int64_t)fold_m.size() <= 3 * (int64_t)p.Q_eff;   // folding removes >= 1/4 of rows
    p.fold = !(p.options & SVDPHAT_OPT_NO_SRP_FOLD) && p.pair_srp && (p.methods & SVDPHAT_METHOD_SRP) && few_rows;
    p.svd_fold = !(p.options & SVDPHAT_OPT_NO_SVD_FOLD) && p.pair_proj && (p.methods & SVDPHAT_METHOD_SVD) &&
                 few_rows && all_paired;
    p.fold_rows = (int)fold_m.size();
    // delay-and-sum SRP (das.cu) for M >= 17, where its (M-1)/4-fold saving in MMA work beats eq. 9's GEMM (cfg4
    // BOTH: 24.3 vs 50.2 ms); at 16 microphones the two SRP paths are within 3% alone and eq. 9's GEMM wins the BOTH
    // call (cfg3: 10.2-10.5 vs 11.0-11.1 ms, profiles/r02/ab_both_das_vs_eq9.log) because the SVD chain overlaps it.  Folded on
    // centrally symmetric grids (antipodal class pairs, reading R22) for 17..32 microphones (cfg4 SRP 13.0 -> 11.0
    // ms), or when forced
    const bool use_das = (p.methods & SVDPHAT_METHOD_SRP) &&
                         ((p.options & SVDPHAT_OPT_DAS) || (!(p.options & SVDPHAT_OPT_NO_DAS) && p.M >= 17));
    p.das_fold = use_das && few_rows && !(p.options & SVDPHAT_OPT_NO_SRP_FOLD) &&
                 (das_me(p.M) == 32 || (das_me(p.M) == 16 && (p.options & SVDPHAT_OPT_DAS_FOLD)));
    p.spc_F = 2 * ((p.L.U + 15) / 16);
    p.K_F = (int64_t)p.L.n_chunks * p.spc_F * 64;
    p.spc_P = (p.L.U + 15) / 16;
    p.K_P = (int64_t)p.L.n_chunks * p.spc_P * 64;
    // BOTH with fold + real V: the few SRP fold rows past the last full 256-row tile ride in the projection's spare V
    // rows (a Re row and an Im row each), so the SRP GEMM skips that tile (cfg3/cfg4: 5121 = 20 x 256 + 1 rows)
    {
        const int nr = p.fold_rows % 256;
        if (p.fold && p.svd_fold && p.fold_rows > 256 && nr > 0 && nr <= 8) {
            p.tail_r0 = p.fold_rows - nr;
            p.tail_n = nr;
        }
    }
    if (p.fold) {
        p.W_rows = (p.fold_rows + 255) / 256 * 256;
        p.spc_W = p.spc_F;
        p.K_W = p.K_F;
    } else {
        p.W_rows = (p.Q_eff + 255) / 256 * 256;
        p.spc_W = p.L.U / 8;
        p.K_W = p.L.K_total;
    }
    if (p.svd_fold) {
        // real basis of the class rows: a pair (c, c') -> sqrt2 Re W_c, sqrt2 Im W_c; a self-antipodal c -> W_c
        for (size_t r = 0; r < fold_m.size(); ++r) {
            p.rb_cls.push_back(fold_m[r]);
            p.rb_partner.push_back(fold_p[r]);
            p.rb_kind.push_back(fold_p[r] >= 0 ? 0 : 2);
            if (fold_p[r] >= 0) {
                p.rb_cls.push_back(fold_m[r]);
                p.rb_partner.push_back(fold_p[r]);
                p.rb_kind.push_back(1);
            }
        }
    }

    // ---- size limits (TOO_LARGE before any large allocation): the SVD setup holds a Q_classes^2 float64 Gram matrix
    // (complex, plus its real form with a real V) and launches grids with Q_classes rows in gridDim.y
    {
        size_t free_b = 0, total_b = 0;
        SVD_CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
        const double n = p.Q_eff;
        if (p.methods & SVDPHAT_METHOD_SVD) {
            if (p.Q_eff > 65535) return fail(SVDPHAT_TOO_LARGE, "SVD setup needs Q_classes <= 65535");
            const double gram = n * n * (16.0 + (p.svd_fold ? 8.0 : 0.0)) * 1.1;
            if (gram > (double)free_b)
                return fail(SVDPHAT_TOO_LARGE, "the Q_classes^2 float64 Gram matrix of the SVD setup (" +
                                                   std::to_string((int64_t)(gram / 1e6)) + " MB) exceeds free memory");
        }
        if (p.methods & SVDPHAT_METHOD_SRP) {
            const double wbytes = (double)p.W_rows * (double)p.K_W * 2.0;
            if (wbytes > 0.9 * (double)free_b)
                return fail(SVDPHAT_TOO_LARGE, "the FP16 steering matrix (" + std::to_string((int64_t)(wbytes / 1e6)) +
                                                   " MB) exceeds free device memory");
        }
    }

    // ---- device tables
    std::vector<double> tau_cls((size_t)p.Q_eff * P);
    for (int c = 0; c < p.Q_eff; ++c)
        std::memcpy(&tau_cls[(size_t)c * P], &tau[(size_t)p.rep_q[c] * P], (size_t)P * 8);
    double* d_tau = nullptr;
    SVD_CUDA_TRY(cudaMalloc(&d_tau, tau_cls.size() * 8));
    std::unique_ptr<double, decltype(&cudaFree)> tau_guard(d_tau, &cudaFree);
    SVD_CUDA_TRY(cudaMemcpy(d_tau, tau_cls.data(), tau_cls.size() * 8, cudaMemcpyHostToDevice));
    if (p.fold || p.das_fold) {
        std::vector<int> fc(fold_m);
        fc.insert(fc.end(), fold_p.begin(), fold_p.end());
        SVD_CUDA_TRY(cudaMalloc(&p.d_fold_cls, fc.size() * sizeof(int)));
        SVD_CUDA_TRY(cudaMemcpy(p.d_fold_cls, fc.data(), fc.size() * sizeof(int), cudaMemcpyHostToDevice));
    }
    SVD_CUDA_TRY(cudaMalloc(&p.d_rep, (size_t)p.Q_eff * sizeof(int)));
    SVD_CUDA_TRY(cudaMemcpy(p.d_rep, p.rep_q.data(), (size_t)p.Q_eff * sizeof(int), cudaMemcpyHostToDevice));
    {
        std::vector<float> df(delay.begin(), delay.end());
        SVD_CUDA_TRY(cudaMalloc(&p.d_delay, df.size() * sizeof(float)));
        SVD_CUDA_TRY(cudaMemcpy(p.d_delay, df.data(), df.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    {
        // unit direction of each class representative as seen from the array centroid (multi-source suppression)
        double cx = 0, cy = 0, cz = 0;
        for (int m = 0; m < M; ++m) {
            cx += r[3 * m] / M;
            cy += r[3 * m + 1] / M;
            cz += r[3 * m + 2] / M;
        }
        std::vector<float4> dirs(p.Q_eff);
        for (int c = 0; c < p.Q_eff; ++c) {
            const double* s = d->points_xyz + 3 * (size_t)p.rep_q[c];
            double v[3] = {s[0], s[1], s[2]};
            if (p.field == SVDPHAT_FIELD_NEAR) {
                v[0] -= cx;
                v[1] -= cy;
                v[2] -= cz;
            }
            const double n = std::sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]);
            dirs[c] = n > 0 ? make_float4((float)(v[0] / n), (float)(v[1] / n), (float)(v[2] / n), 0.f)
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        SVD_CUDA_TRY(cudaMalloc(&p.d_dirs, dirs.size() * sizeof(float4)));
        SVD_CUDA_TRY(cudaMemcpy(p.d_dirs, dirs.data(), dirs.size() * sizeof(float4), cudaMemcpyHostToDevice));
    }
    {
        std::vector<float> w(p.N);
        std::vector<float2> tw(p.N);
        const double pi = 3.14159265358979323846;
        for (int n = 0; n < p.N; ++n) {
            w[n] = (float)std::sin(pi * (n + 0.5) / p.N);  // sine window (reading R1)
            tw[n] = make_float2((float)std::cos(2 * pi * n / p.N), (float)-std::sin(2 * pi * n / p.N));
        }
        SVD_CUDA_TRY(cudaMalloc(&p.d_window, p.N * sizeof(float)));
        SVD_CUDA_TRY(cudaMemcpy(p.d_window, w.data(), p.N * sizeof(float), cudaMemcpyHostToDevice));
        SVD_CUDA_TRY(cudaMalloc(&p.d_twN, p.N * sizeof(float2)));
        SVD_CUDA_TRY(cudaMemcpy(p.d_twN, tw.data(), p.N * sizeof(float2), cudaMemcpyHostToDevice));
    }

    // ---- operands
    if (p.methods & SVDPHAT_METHOD_SRP) {
        st = setup_srp_operand(p, d_tau);
        if (st != SVDPHAT_OK) return st;
        if (!encode_2d(&p.tm_W, p.d_W16, p.W_rows, p.K_W, 128))
            return fail(SVDPHAT_CUDA, "cuTensorMapEncodeTiled(W) failed");
        if (p.das_fold) {
            std::vector<double> dfold((size_t)p.fold_rows * M);
            for (int r = 0; r < p.fold_rows; ++r)
                std::memcpy(&dfold[(size_t)r * M], &delay[(size_t)p.rep_q[fold_m[r]] * M], (size_t)M * 8);
            st = setup_das_fold_operand(p, dfold.data());
            if (st != SVDPHAT_OK) return st;
            if (!encode_2d_rows(&p.tm_A, p.d_A16, (int64_t)p.L.n_chunks * p.das_rows, 64, 128))
                return fail(SVDPHAT_CUDA, "cuTensorMapEncodeTiled(A16) failed");
        } else if (use_das) {
            std::vector<double> dcls((size_t)p.Q_eff * M);
            for (int c = 0; c < p.Q_eff; ++c)
                std::memcpy(&dcls[(size_t)c * M], &delay[(size_t)p.rep_q[c] * M], (size_t)M * 8);
            st = setup_das_operand(p, dcls.data());
            if (st != SVDPHAT_OK) return st;
            if (!encode_2d_rows(&p.tm_A, p.d_A16, (int64_t)p.Kb * p.das_rows, 2 * p.das_me, 128))
                return fail(SVDPHAT_CUDA, "cuTensorMapEncodeTiled(A16) failed");
        }
    }
    if (p.methods & SVDPHAT_METHOD_SVD) {
        st = setup_svd_operands(p, d_tau, d->rank_D);
        if (st != SVDPHAT_OK) return st;
        // the SRP tail rows' W values: Re slabs of fold row tail_r0 + r -> V row D + 2r, Im slabs -> V row D + 2r + 1
        for (int r = 0; r < p.tail_n; ++r)
            for (int im = 0; im < 2; ++im)
                SVD_CUDA_TRY(cudaMemcpy2D(p.d_V16 + (int64_t)(p.D + 2 * r + im) * p.K_P, 64 * sizeof(__half),
                                          p.d_W16 + (int64_t)(p.tail_r0 + r) * p.K_W + 64 * im, 128 * sizeof(__half),
                                          64 * sizeof(__half), (size_t)p.L.n_chunks * p.spc_P,
                                          cudaMemcpyDeviceToDevice));
        p.Zh = p.svd_fold ? std::max(p.Dh, p.V_rows) : p.Dh;
        if (2 * p.Zh > 8192) return fail(SVDPHAT_TOO_LARGE, "SVD rank too large for the Z normalisation (D <= 4000)");
        const int v_box = !p.pair_proj ? 128 : p.svd_fold ? p.proj_nt / (2 * p.proj_nmma) : p.proj_nt / 2;
        if (!encode_2d(&p.tm_V, p.d_V16, p.V_rows, p.svd_fold ? p.K_P : p.L.K_total, v_box))
            return fail(SVDPHAT_CUDA, "cuTensorMapEncodeTiled(V) failed");
        if (!encode_2d(&p.tm_R, p.d_R16, p.Q_pad, p.K2, 128))
            return fail(SVDPHAT_CUDA, "cuTensorMapEncodeTiled(R) failed");
    }

    // ---- workspace for max_frames
    const int64_t Fp = p.F_pad;
    const int64_t bytes_P16 = (int64_t)p.L.n_chunks * p.L.Mi * Fp * p.L.unit_bytes;
    SVD_CUDA_TRY(cudaMalloc(&p.d_P16, bytes_P16));
    SVD_CUDA_TRY(cudaMemset(p.d_P16, 0, bytes_P16));
    SVD_CUDA_TRY(cudaMalloc(&p.d_keys, 3 * Fp * sizeof(unsigned long long)));
    p.bytes_ws = bytes_P16 + 3 * Fp * 8;
    if (p.d_A16) {
        // folded: [n_chunks][2 F_pad][64 halves] (Re row, Im row per frame); else [Kb][F_pad][2 das_me]
        const int64_t e_rows = p.das_fold ? (int64_t)p.L.n_chunks * 2 * Fp : (int64_t)p.Kb * Fp;
        const int e_cols = p.das_fold ? 64 : 2 * p.das_me;
        const int64_t bytes_E16 = e_rows * e_cols * 2;
        SVD_CUDA_TRY(cudaMalloc(&p.d_E16, bytes_E16));
        SVD_CUDA_TRY(cudaMemset(p.d_E16, 0, bytes_E16));
        if (!encode_2d_rows(&p.tm_E, p.d_E16, e_rows, e_cols, 128))
            return fail(SVDPHAT_CUDA, "cuTensorMapEncodeTiled(E16) failed");
        p.bytes_ws += bytes_E16;
    }
    if (p.methods & SVDPHAT_METHOD_SVD) {
        // split-K partial buffers: as many splits (<= MAX_KSPLIT) as fit in ~256 MB
        const int64_t zbytes = Fp * 2 * p.Zh * (int64_t)sizeof(float);
        p.zsplit_max = (int)std::max<int64_t>(1, std::min<int64_t>(MAX_KSPLIT, (256ll << 20) / zbytes));
        SVD_CUDA_TRY(cudaMalloc(&p.d_Z32, p.zsplit_max * zbytes));
        SVD_CUDA_TRY(cudaMemset(p.d_Z32, 0, p.zsplit_max * zbytes));
        SVD_CUDA_TRY(cudaMalloc(&p.d_Zs16, Fp * p.K2 * 2));
        SVD_CUDA_TRY(cudaMemset(p.d_Zs16, 0, Fp * p.K2 * 2));
        SVD_CUDA_TRY(cudaMalloc(&p.d_zflag, Fp * sizeof(int)));
        SVD_CUDA_TRY(cudaMemset(p.d_zflag, 0, Fp * sizeof(int)));
        SVD_CUDA_TRY(cudaMalloc(&p.d_Zn32, Fp * p.K2 * sizeof(float)));
        SVD_CUDA_TRY(cudaMemset(p.d_Zn32, 0, Fp * p.K2 * sizeof(float)));
        SVD_CUDA_TRY(cudaMalloc(&p.d_cand, Fp * SEARCH_CAP * sizeof(unsigned long long)));
        SVD_CUDA_TRY(cudaMalloc(&p.d_ccnt, Fp * sizeof(int)));
        const int64_t map_bytes = Fp * (int64_t)p.Q_pad * (int64_t)sizeof(float);
        if (map_bytes <= (64ll << 20)) {        // small batches: score map + per-frame rescore (see internal.h)
            SVD_CUDA_TRY(cudaMalloc(&p.d_Smap, map_bytes));
            p.search_map = true;
            p.bytes_ws += map_bytes;
        }
        p.bytes_ws += zbytes * p.zsplit_max + Fp * p.K2 * 6 + Fp * 8 + Fp * SEARCH_CAP * 8;
        if (!encode_2d(&p.tm_Zs, p.d_Zs16, Fp, p.K2, 256))
            return fail(SVDPHAT_CUDA, "cuTensorMapEncodeTiled(Zs) failed");
    }
    // small batches (fewer SRP tile units than half the CTA pairs): split-K partial power maps, <= 64 MB
    if ((p.methods & SVDPHAT_METHOD_SRP) && p.pair_srp) {
        const int64_t units = (int64_t)(p.W_rows / 256) * ((p.max_frames + 255) / 256);
        if (units * 2 <= p.num_sms / 2) {
            const int64_t ybytes = Fp * (int64_t)p.Q_pad * (int64_t)sizeof(float);
            p.srp_split_max = (int)std::min<int64_t>(8, std::max<int64_t>(1, (64ll << 20) / ybytes));
            if (p.srp_split_max > 1) {
                SVD_CUDA_TRY(cudaMalloc(&p.d_Ypart, p.srp_split_max * ybytes));
                p.bytes_ws += p.srp_split_max * ybytes;
            } else {
                p.srp_split_max = 0;
            }
        }
    }
    SVD_CUDA_TRY(gemm_set_attributes());
    SVD_CUDA_TRY(das_set_attributes());
    SVD_CUDA_TRY(stft_set_attributes());
    SVD_CUDA_TRY(topk_set_attributes());
    if ((p.methods & SVDPHAT_METHOD_BOTH) == SVDPHAT_METHOD_BOTH) {
        int lo = 0, hi = 0;
        SVD_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        // the SRP GEMM gets the SMs first after the STFT; the SVD chain fills its last wave (r01 A/B: the reverse
        // order was 3% slower)
        SVD_CUDA_TRY(cudaStreamCreateWithPriority(&p.svd_stream, cudaStreamNonBlocking, lo));
        SVD_CUDA_TRY(cudaStreamCreateWithPriority(&p.srp_stream, cudaStreamNonBlocking, hi));
        SVD_CUDA_TRY(cudaEventCreateWithFlags(&p.ev_fork, cudaEventDisableTiming));
        SVD_CUDA_TRY(cudaEventCreateWithFlags(&p.ev_join, cudaEventDisableTiming));
        SVD_CUDA_TRY(cudaEventCreateWithFlags(&p.ev_join2, cudaEventDisableTiming));
        SVD_CUDA_TRY(cudaEventCreateWithFlags(&p.ev_z, cudaEventDisableTiming));
    }
    SVD_CUDA_TRY(cudaDeviceSynchronize());
    p.setup_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = h.release();
    return SVDPHAT_OK;
}

svdphat_status svdphat_plan_create(const svdphat_plan_desc* d, svdphat_plan_t* out) {
    return guarded([&] { return plan_create_impl(d, out); });
}

svdphat_status svdphat_plan_info(svdphat_plan_t plan, svdphat_plan_info_t* out) {
    if (!plan || !out) return fail(SVDPHAT_INVALID_ARG, "NULL argument");
    const Plan& p = plan->p;
    std::memset(out, 0, sizeof(*out));
    out->M = p.M;
    out->P = p.P;
    out->N = p.N;
    out->K_bins = p.Kb;
    out->PK = p.PK;
    out->Q = p.Q;
    out->Q_classes = p.Q_eff;
    out->D = p.D;
    out->energy_kept = p.energy_kept;
    out->trace_WWH = p.trace;
    out->methods = p.methods;
    out->gemm_k = (int32_t)p.L.K_total;
    out->max_frames = p.max_frames;
    out->bytes_W = p.bytes_W;
    out->bytes_V = p.bytes_V;
    out->bytes_R = p.bytes_R;
    out->bytes_workspace = p.bytes_ws;
    out->setup_seconds = p.setup_seconds;
    out->srp_rows = (p.methods & SVDPHAT_METHOD_SRP) ? (p.fold ? p.fold_rows : p.Q_eff) : 0;
    out->svd_rows = (p.methods & SVDPHAT_METHOD_SVD) ? (p.svd_fold ? p.D : 2 * p.D) : 0;
    out->das_rows = p.d_A16 ? p.das_rows : 0;
    out->das_me = p.d_A16 ? p.das_me : 0;
    out->srp_gemm_k = (p.methods & SVDPHAT_METHOD_SRP) ? p.K_W : 0;
    out->srp_gemm_rows = (p.methods & SVDPHAT_METHOD_SRP) ? p.W_rows : 0;
    out->srp_tail_rows = p.tail_n;
    return SVDPHAT_OK;
}

svdphat_status svdphat_plan_sigma2(svdphat_plan_t plan, double* out, int32_t n) {
    if (!plan || !out || n < 0) return fail(SVDPHAT_INVALID_ARG, "NULL argument");
    const Plan& p = plan->p;
    if (!(p.methods & SVDPHAT_METHOD_SVD)) return fail(SVDPHAT_INVALID_ARG, "SVD was not planned");
    const int m = std::min<int>(n, (int)p.sigma2.size());
    std::memcpy(out, p.sigma2.data(), (size_t)m * sizeof(double));
    return SVDPHAT_OK;
}

static svdphat_status localize_impl(Plan& p, const Band& b, int32_t method, const float* d_audio, int F,
                                    int64_t channel_stride, int64_t frame_stride, int32_t* doa_srp, float* sc_srp,
                                    int32_t* doa_svd, float* sc_svd, cudaStream_t s) {
    // BOTH: after the STFT the SRP GEMM (high-priority stream) and the SVD chain (low-priority stream) run
    // concurrently: the SRP CTAs take every SM first and the SVD kernels fill the SMs its last wave releases.
    // Stage events are recorded on each kernel's own stream (an SVD stage's time may include waiting for SMs).
    const bool fork = method == SVDPHAT_METHOD_BOTH && p.svd_stream;
    cudaStream_t sr = fork ? p.srp_stream : s, sv = fork ? p.svd_stream : s;
    SVD_CUDA_TRY(cudaMemsetAsync(p.d_keys, 0, (size_t)3 * p.F_pad * 8, s));
    if (method & SVDPHAT_METHOD_SVD) SVD_CUDA_TRY(cudaMemsetAsync(p.d_ccnt, 0, (size_t)F * sizeof(int), s));
    SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_STFT, s,
                        [&] { return launch_stft_phat(p, b, d_audio, channel_stride, frame_stride, F, s); }));
    if (fork) {
        SVD_CUDA_TRY(cudaEventRecord(p.ev_fork, s));
        SVD_CUDA_TRY(cudaStreamWaitEvent(sr, p.ev_fork, 0));
        SVD_CUDA_TRY(cudaStreamWaitEvent(sv, p.ev_fork, 0));
    }
    int32_t* const doas[2] = {doa_srp, doa_svd};
    float* const scores[2] = {sc_srp, sc_svd};
    // SRP: the delay-and-sum GEMM (das.cu) when the plan has it and the batch fills the CTA pairs, else eq. 9's GEMM
    const bool das = (method & SVDPHAT_METHOD_SRP) && das_active(p, F);
    // SRP tail rows scored through the projection: BOTH calls on the argmax GEMM path (not the small-batch split)
    const bool both = method == SVDPHAT_METHOD_BOTH && !das && p.tail_n > 0 && srp_split_ways(p, b, F) == 1;
    auto run_srp = [&]() -> svdphat_status {
        if (das) {
            SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_SRP_BINS, sr, [&] { return launch_das_bins(p, b, F, sr); }));
            SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_SRP_DAS, sr, [&] { return launch_das(p, b, F, sr); }));
        } else if (method & SVDPHAT_METHOD_SRP) {
            SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_SRP_GEMM, sr, [&] { return launch_gemm(p, b, 0, F, sr, both); }));
        }
        return SVDPHAT_OK;
    };
    auto run_proj = [&]() -> svdphat_status {
        if (method & SVDPHAT_METHOD_SVD) {
            SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_SVD_PROJ, sv, [&] { return launch_gemm(p, b, 1, F, sv); }));
            SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_SVD_NORM, sv, [&] { return launch_zsplit(p, b, F, sv, both); }));
        }
        return SVDPHAT_OK;
    };
    // Small batches (the split-K SRP path, cfg5's 256-frame calls): both GEMMs want whole SMs and neither fills the GPU
    // for long, so the short projection (26 us at cfg5) goes first and the rest of the SVD chain runs beside the SRP
    // GEMM (102 us); SRP first left the whole SVD chain (84 us) behind it (ncu r02).  Large batches: SRP first (r01 A/B).
    const bool svd_first = fork && !das && (method & SVDPHAT_METHOD_SRP) && srp_split_ways(p, b, F) > 1;
    svdphat_status st_l = svd_first ? run_proj() : run_srp();
    if (st_l != SVDPHAT_OK) return st_l;
    st_l = svd_first ? run_srp() : run_proj();
    if (st_l != SVDPHAT_OK) return st_l;
    // forked: the SRP half of the finalize runs on the SRP stream while the SVD search is still busy (after zsplit
    // when the SRP tail rows' keys come from it)
    if (fork && (method & SVDPHAT_METHOD_SRP)) {
        if (both) {
            SVD_CUDA_TRY(cudaEventRecord(p.ev_z, sv));
            SVD_CUDA_TRY(cudaStreamWaitEvent(sr, p.ev_z, 0));
        }
        SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_FINALIZE, sr,
                            [&] { return launch_finalize(p, SVDPHAT_METHOD_SRP, F, doas, scores, sr); }));
    }
    if (method & SVDPHAT_METHOD_SVD) {
        SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_SVD_SEARCH, sv,
                            [&] { return launch_gemm(p, b, p.search_map ? 5 : 2, F, sv); }));
        SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_SVD_RESCORE, sv, [&] { return launch_rescore(p, F, sv); }));
        if (fork)
            SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_FINALIZE, sv,
                                [&] { return launch_finalize(p, SVDPHAT_METHOD_SVD, F, doas, scores, sv); }));
    }
    if (fork) {
        SVD_CUDA_TRY(cudaEventRecord(p.ev_join, sr));
        SVD_CUDA_TRY(cudaEventRecord(p.ev_join2, sv));
        SVD_CUDA_TRY(cudaStreamWaitEvent(s, p.ev_join, 0));
        SVD_CUDA_TRY(cudaStreamWaitEvent(s, p.ev_join2, 0));
    } else {
        SVD_CUDA_TRY(
            staged(p, SVDPHAT_STAGE_FINALIZE, s, [&] { return launch_finalize(p, method, F, doas, scores, s); }));
    }
    p.last_frames = F;
    p.last_method = method;
    return SVDPHAT_OK;
}

static svdphat_status check_localize_args(Plan& p, int32_t method, int64_t n_frames, int64_t cs, int64_t fs) {
    if (method < SVDPHAT_METHOD_SRP || method > SVDPHAT_METHOD_BOTH)
        return fail(SVDPHAT_INVALID_ARG, "method must be SRP, SVD or BOTH");
    if ((p.methods & method) != method) return fail(SVDPHAT_INVALID_ARG, "method was not planned");
    if (n_frames < 0 || n_frames > p.max_frames) return fail(SVDPHAT_INVALID_ARG, "n_frames out of [0, max_frames]");
    if (cs < 0 || fs < 0) return fail(SVDPHAT_INVALID_ARG, "negative stride");
    return SVDPHAT_OK;
}

// svdphat_localize and svdphat_localize_masked: validation, then the hot path on the caller's stream
static svdphat_status localize_device(svdphat_plan_t plan, const Band& b, int32_t method, const float* d_audio,
                                      int64_t n_frames, int64_t channel_stride, int64_t frame_stride, int32_t* d_doa,
                                      float* d_score, void* stream) {
    Plan& p = plan->p;
    svdphat_status st = check_localize_args(p, method, n_frames, channel_stride, frame_stride);
    if (st != SVDPHAT_OK) return st;
    if (n_frames == 0) return SVDPHAT_OK;
    if (!d_audio || !d_doa || !d_score) return fail(SVDPHAT_INVALID_ARG, "NULL buffer");
    if (reinterpret_cast<uintptr_t>(d_audio) & 3) return fail(SVDPHAT_INVALID_ARG, "d_audio not 4-byte aligned");
    SVD_DEVICE_GUARD(p.device);
    const int F = (int)n_frames;
    const bool both = method == SVDPHAT_METHOD_BOTH;
    return localize_impl(p, b, method, d_audio, F, channel_stride, frame_stride, d_doa, d_score,
                         both ? d_doa + F : d_doa, both ? d_score + F : d_score, reinterpret_cast<cudaStream_t>(stream));
}

svdphat_status svdphat_localize(svdphat_plan_t plan, int32_t method, const float* d_audio, int64_t n_frames,
                                int64_t channel_stride, int64_t frame_stride, int32_t* d_doa, float* d_score,
                                void* stream) {
    if (!plan) return fail(SVDPHAT_INVALID_ARG, "plan is NULL");
    return guarded([&] {
        return localize_device(plan, full_band(plan->p), method, d_audio, n_frames, channel_stride, frame_stride,
                               d_doa, d_score, stream);
    });
}

svdphat_status svdphat_localize_masked(svdphat_plan_t plan, int32_t method, const float* d_audio, int64_t n_frames,
                                       int64_t channel_stride, int64_t frame_stride, int32_t k_lo, int32_t k_hi,
                                       const uint8_t* d_mask, int64_t mask_stride, int32_t* d_doa, float* d_score,
                                       void* stream) {
    if (!plan) return fail(SVDPHAT_INVALID_ARG, "plan is NULL");
    const Plan& p = plan->p;
    if (k_lo < 0 || k_hi > p.Kb || k_lo >= k_hi) return fail(SVDPHAT_INVALID_ARG, "need 0 <= k_lo < k_hi <= N/2+1");
    if (mask_stride < 0) return fail(SVDPHAT_INVALID_ARG, "negative mask_stride");
    const Band b = make_band(p, k_lo, k_hi, d_mask, mask_stride);     // per call; the plan is not modified
    return guarded([&] {
        return localize_device(plan, b, method, d_audio, n_frames, channel_stride, frame_stride, d_doa, d_score,
                               stream);
    });
}

static svdphat_status localize_topk_impl(svdphat_plan_t plan, int32_t method, const float* d_audio,
                                         int64_t n_frames, int64_t channel_stride, int64_t frame_stride, int32_t k,
                                         double min_sep_deg, int32_t* d_doa, float* d_score, void* stream) {
    Plan& p = plan->p;
    if (method != SVDPHAT_METHOD_SRP && method != SVDPHAT_METHOD_SVD)
        return fail(SVDPHAT_INVALID_ARG, "top-k: method must be SRP or SVD");
    svdphat_status st = check_localize_args(p, method, n_frames, channel_stride, frame_stride);
    if (st != SVDPHAT_OK) return st;
    if (k < 1 || k > 4) return fail(SVDPHAT_INVALID_ARG, "k must be in [1, 4]");
    if (!(min_sep_deg >= 0.0 && min_sep_deg <= 180.0)) return fail(SVDPHAT_INVALID_ARG, "min_sep_deg in [0, 180]");
    if (p.Q_eff > 49152) return fail(SVDPHAT_INVALID_ARG, "top-k needs Q_classes <= 49152");
    if (n_frames == 0) return SVDPHAT_OK;
    if (!d_audio || !d_doa || !d_score) return fail(SVDPHAT_INVALID_ARG, "NULL buffer");
    SVD_DEVICE_GUARD(p.device);
    if (!alloc_pair(reinterpret_cast<void**>(&p.d_S), (size_t)p.F_pad * p.Q_pad * sizeof(float),
                    reinterpret_cast<void**>(&p.d_cls), (size_t)p.F_pad * 4 * sizeof(int)))
        return fail(SVDPHAT_ALLOC, "top-k workspace allocation failed");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int F = (int)n_frames;
    const Band b = full_band(p);
    SVD_CUDA_TRY(staged(p, SVDPHAT_STAGE_STFT, s,
                        [&] { return launch_stft_phat(p, b, d_audio, channel_stride, frame_stride, F, s); }));
    if (method == SVDPHAT_METHOD_SRP) {
        SVD_CUDA_TRY(launch_gemm(p, b, 3, F, s));
    } else {
        SVD_CUDA_TRY(launch_gemm(p, b, 1, F, s));
        SVD_CUDA_TRY(launch_zsplit(p, b, F, s));
        SVD_CUDA_TRY(launch_gemm(p, b, 4, F, s));
    }
    const double kPi = 3.14159265358979323846;
    SVD_CUDA_TRY(launch_topk(p, F, k, (float)std::cos(min_sep_deg * kPi / 180.0), s));
    SVD_CUDA_TRY(launch_finalize_topk(p, F, k, d_doa, d_score, s));
    p.last_frames = F;
    p.last_method = method;
    return SVDPHAT_OK;
}

svdphat_status svdphat_localize_topk(svdphat_plan_t plan, int32_t method, const float* d_audio, int64_t n_frames,
                                     int64_t channel_stride, int64_t frame_stride, int32_t k, double min_sep_deg,
                                     int32_t* d_doa, float* d_score, void* stream) {
    if (!plan) return fail(SVDPHAT_INVALID_ARG, "plan is NULL");
    return guarded([&] {
        return localize_topk_impl(plan, method, d_audio, n_frames, channel_stride, frame_stride, k, min_sep_deg,
                                  d_doa, d_score, stream);
    });
}

static svdphat_status profile_begin_impl(Plan& p, int32_t capacity) {
    SVD_DEVICE_GUARD(p.device);
    for (cudaEvent_t e : p.prof_ev) cudaEventDestroy(e);
    p.prof_ev.assign(2 * (size_t)capacity, nullptr);
    p.prof_on = false;
    p.prof_cap = p.prof_n = 0;
    for (auto& e : p.prof_ev) SVD_CUDA_TRY(cudaEventCreate(&e));
    p.prof_stage.assign(capacity, 0);
    p.prof_cap = capacity;
    p.prof_n = 0;
    p.prof_on = true;
    return SVDPHAT_OK;
}

svdphat_status svdphat_profile_begin(svdphat_plan_t plan, int32_t capacity) {
    if (!plan || capacity < 0) return fail(SVDPHAT_INVALID_ARG, "bad argument");
    return guarded([&] { return profile_begin_impl(plan->p, capacity); });
}

int32_t svdphat_profile_end(svdphat_plan_t plan, int32_t* stage_ids, float* ms, int32_t max) {
    if (!plan) return -(int32_t)fail(SVDPHAT_INVALID_ARG, "plan is NULL");
    Plan& p = plan->p;
    DeviceGuard g(p.device);
    int n = std::min(p.prof_n, std::max(0, max));
    int32_t ret = n;
    for (int i = 0; i < n; ++i) {
        if (cudaEventSynchronize(p.prof_ev[2 * i + 1]) != cudaSuccess) {
            ret = -(int32_t)SVDPHAT_CUDA;
            break;
        }
        float t = 0.f;
        cudaEventElapsedTime(&t, p.prof_ev[2 * i], p.prof_ev[2 * i + 1]);
        if (stage_ids) stage_ids[i] = p.prof_stage[i];
        if (ms) ms[i] = t;
    }
    for (cudaEvent_t e : p.prof_ev) cudaEventDestroy(e);
    p.prof_ev.clear();
    p.prof_stage.clear();
    p.prof_on = false;
    p.prof_cap = p.prof_n = 0;
    return ret;
}

static svdphat_status localize_host_impl(Plan& p, int32_t method, const float* h_audio, int64_t audio_elems,
                                         int64_t n_frames, int64_t channel_stride, int64_t frame_stride,
                                         int32_t* h_doa, float* h_score, void* stream) {
    svdphat_status st = check_localize_args(p, method, n_frames, channel_stride, frame_stride);
    if (st != SVDPHAT_OK) return st;
    if (n_frames == 0) return SVDPHAT_OK;
    if (!h_audio || !h_doa || !h_score || audio_elems <= 0) return fail(SVDPHAT_INVALID_ARG, "NULL/empty buffer");
    const int64_t M1 = p.M - 1;
    const int64_t need = M1 * channel_stride + (n_frames - 1) * frame_stride + p.N;
    if (need > audio_elems) return fail(SVDPHAT_INVALID_ARG, "audio buffer smaller than the addressed frames");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    SVD_DEVICE_GUARD(p.device);
    const int F = (int)n_frames;
    const Band b = full_band(p);
    // Frame-major buffers (each frame's samples inside its own frame_stride span) are pipelined in chunks of
    // whole 256-frame tiles: the H2D of chunk i+1 (copy stream) overlaps the kernels of chunk i (caller stream).
    const int64_t span1 = M1 * channel_stride + p.N;            // elements touched by one frame
    const bool frame_major = frame_stride >= span1;
    int chunk = F;
    if (frame_major && F >= 2048) chunk = (int)std::min<int64_t>(F, ((F + 3) / 4 + 255) / 256 * 256);
    const int nchunks = (F + chunk - 1) / chunk;
    const int64_t slot_elems = nchunks == 1 ? need : (int64_t)(chunk - 1) * frame_stride + span1;
    if (slot_elems > p.stage_elems) {
        if (p.d_stage) cudaFree(p.d_stage);
        p.d_stage = nullptr;
        p.stage_elems = 0;
        if (cudaMalloc(&p.d_stage, 2 * slot_elems * sizeof(float)) != cudaSuccess) {
            p.d_stage = nullptr;
            cudaGetLastError();
            return fail(SVDPHAT_ALLOC, "staging buffer allocation failed");
        }
        p.stage_elems = slot_elems;
    }
    if (!alloc_pair(reinterpret_cast<void**>(&p.d_doa_stage), 2 * p.F_pad * sizeof(int32_t),
                    reinterpret_cast<void**>(&p.d_score_stage), 2 * p.F_pad * sizeof(float)))
        return fail(SVDPHAT_ALLOC, "result staging allocation failed");
    if (!p.copy_stream) {
        SVD_CUDA_TRY(cudaStreamCreateWithFlags(&p.copy_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            SVD_CUDA_TRY(cudaEventCreateWithFlags(&p.ev_copied[i], cudaEventDisableTiming));
            SVD_CUDA_TRY(cudaEventCreateWithFlags(&p.ev_done[i], cudaEventDisableTiming));
        }
    }
    const bool both = method == SVDPHAT_METHOD_BOTH;
    SVD_CUDA_TRY(cudaEventRecord(p.ev_done[0], s));            // copy stream starts after prior work on s
    SVD_CUDA_TRY(cudaEventRecord(p.ev_done[1], s));
    for (int i = 0; i < nchunks; ++i) {
        const int slot = i & 1;
        const int f0 = i * chunk, n = std::min(chunk, F - f0);
        const int64_t off = (int64_t)f0 * frame_stride;
        const int64_t elems = nchunks == 1 ? need : (int64_t)(n - 1) * frame_stride + span1;
        float* dst = p.d_stage + slot * p.stage_elems;
        SVD_CUDA_TRY(cudaStreamWaitEvent(p.copy_stream, p.ev_done[slot], 0));
        SVD_CUDA_TRY(cudaMemcpyAsync(dst, h_audio + off, elems * sizeof(float), cudaMemcpyHostToDevice, p.copy_stream));
        SVD_CUDA_TRY(cudaEventRecord(p.ev_copied[slot], p.copy_stream));
        SVD_CUDA_TRY(cudaStreamWaitEvent(s, p.ev_copied[slot], 0));
        st = localize_impl(p, b, method, dst, n, channel_stride, frame_stride, p.d_doa_stage + f0,
                           p.d_score_stage + f0, p.d_doa_stage + (both ? F : 0) + f0,
                           p.d_score_stage + (both ? F : 0) + f0, s);
        if (st != SVDPHAT_OK) return st;
        SVD_CUDA_TRY(cudaEventRecord(p.ev_done[slot], s));
    }
    const int64_t nout = (both ? 2 : 1) * (int64_t)F;
    SVD_CUDA_TRY(cudaMemcpyAsync(h_doa, p.d_doa_stage, nout * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SVD_CUDA_TRY(cudaMemcpyAsync(h_score, p.d_score_stage, nout * sizeof(float), cudaMemcpyDeviceToHost, s));
    SVD_CUDA_TRY(cudaStreamSynchronize(s));
    p.last_frames = F;
    return SVDPHAT_OK;
}

svdphat_status svdphat_localize_host(svdphat_plan_t plan, int32_t method, const float* h_audio, int64_t audio_elems,
                                     int64_t n_frames, int64_t channel_stride, int64_t frame_stride, int32_t* h_doa,
                                     float* h_score, void* stream) {
    if (!plan) return fail(SVDPHAT_INVALID_ARG, "plan is NULL");
    return guarded([&] {
        return localize_host_impl(plan->p, method, h_audio, audio_elems, n_frames, channel_stride, frame_stride,
                                  h_doa, h_score, stream);
    });
}

static svdphat_status submit_host_impl(Plan& p, int32_t method, const float* h_audio, int64_t audio_elems,
                                       int64_t n_frames, int64_t channel_stride, int64_t frame_stride, int32_t* h_doa,
                                       float* h_score, void* stream, int64_t* ticket) {
    svdphat_status st = check_localize_args(p, method, n_frames, channel_stride, frame_stride);
    if (st != SVDPHAT_OK) return st;
    if (n_frames == 0) return fail(SVDPHAT_INVALID_ARG, "n_frames must be > 0");
    if (!h_audio || !h_doa || !h_score || audio_elems <= 0) return fail(SVDPHAT_INVALID_ARG, "NULL/empty buffer");
    const int64_t need = (int64_t)(p.M - 1) * channel_stride + (n_frames - 1) * frame_stride + p.N;
    if (need > audio_elems) return fail(SVDPHAT_INVALID_ARG, "audio buffer smaller than the addressed frames");
    SVD_DEVICE_GUARD(p.device);
    if (!p.up_stream) {
        SVD_CUDA_TRY(cudaStreamCreateWithFlags(&p.up_stream, cudaStreamNonBlocking));
        SVD_CUDA_TRY(cudaStreamCreateWithFlags(&p.down_stream, cudaStreamNonBlocking));
        for (auto& sl : p.slots) {
            SVD_CUDA_TRY(cudaEventCreateWithFlags(&sl.h2d, cudaEventDisableTiming));
            SVD_CUDA_TRY(cudaEventCreateWithFlags(&sl.comp, cudaEventDisableTiming));
            SVD_CUDA_TRY(cudaEventCreateWithFlags(&sl.d2h, cudaEventDisableTiming));
        }
    }
    Plan::HostSlot& sl = p.slots[p.next_ticket & 1];
    if (sl.ticket >= 0) SVD_CUDA_TRY(cudaEventSynchronize(sl.d2h));     // the slot's previous batch is done
    if (need > sl.elems) {
        if (sl.d_audio) cudaFree(sl.d_audio);
        sl.d_audio = nullptr;
        sl.elems = 0;
        if (cudaMalloc(&sl.d_audio, need * sizeof(float)) != cudaSuccess) {
            sl.d_audio = nullptr;
            cudaGetLastError();
            return fail(SVDPHAT_ALLOC, "streaming staging allocation failed");
        }
        sl.elems = need;
    }
    if (!alloc_pair(reinterpret_cast<void**>(&sl.d_doa), 2 * p.F_pad * sizeof(int32_t),
                    reinterpret_cast<void**>(&sl.d_score), 2 * p.F_pad * sizeof(float)))
        return fail(SVDPHAT_ALLOC, "streaming result allocation failed");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int F = (int)n_frames;
    const bool both = method == SVDPHAT_METHOD_BOTH;
    SVD_CUDA_TRY(cudaMemcpyAsync(sl.d_audio, h_audio, need * sizeof(float), cudaMemcpyHostToDevice, p.up_stream));
    SVD_CUDA_TRY(cudaEventRecord(sl.h2d, p.up_stream));
    SVD_CUDA_TRY(cudaStreamWaitEvent(s, sl.h2d, 0));
    st = localize_impl(p, full_band(p), method, sl.d_audio, F, channel_stride, frame_stride, sl.d_doa, sl.d_score,
                       sl.d_doa + (both ? F : 0), sl.d_score + (both ? F : 0), s);
    if (st != SVDPHAT_OK) return st;
    SVD_CUDA_TRY(cudaEventRecord(sl.comp, s));
    SVD_CUDA_TRY(cudaStreamWaitEvent(p.down_stream, sl.comp, 0));
    const int64_t nout = (both ? 2 : 1) * (int64_t)F;
    SVD_CUDA_TRY(cudaMemcpyAsync(h_doa, sl.d_doa, nout * sizeof(int32_t), cudaMemcpyDeviceToHost, p.down_stream));
    SVD_CUDA_TRY(cudaMemcpyAsync(h_score, sl.d_score, nout * sizeof(float), cudaMemcpyDeviceToHost, p.down_stream));
    SVD_CUDA_TRY(cudaEventRecord(sl.d2h, p.down_stream));
    sl.ticket = p.next_ticket;
    *ticket = p.next_ticket++;
    return SVDPHAT_OK;
}

svdphat_status svdphat_submit_host(svdphat_plan_t plan, int32_t method, const float* h_audio, int64_t audio_elems,
                                   int64_t n_frames, int64_t channel_stride, int64_t frame_stride, int32_t* h_doa,
                                   float* h_score, void* stream, int64_t* ticket) {
    if (!plan || !ticket) return fail(SVDPHAT_INVALID_ARG, "NULL argument");
    return guarded([&] {
        return submit_host_impl(plan->p, method, h_audio, audio_elems, n_frames, channel_stride, frame_stride, h_doa,
                                h_score, stream, ticket);
    });
}

svdphat_status svdphat_wait(svdphat_plan_t plan, int64_t ticket) {
    if (!plan) return fail(SVDPHAT_INVALID_ARG, "plan is NULL");
    Plan& p = plan->p;
    if (ticket < 0 || ticket >= p.next_ticket) return fail(SVDPHAT_INVALID_ARG, "unknown ticket");
    const Plan::HostSlot& sl = p.slots[ticket & 1];
    if (sl.ticket != ticket) return SVDPHAT_OK;                          // slot reused: that batch completed
    SVD_DEVICE_GUARD(p.device);
    SVD_CUDA_TRY(cudaEventSynchronize(sl.d2h));
    return SVDPHAT_OK;
}

static svdphat_status debug_dump_impl(Plan& p, int32_t what, int64_t n_frames, void* host_out, int64_t bytes) {
    SVD_DEVICE_GUARD(p.device);
    SVD_CUDA_TRY(cudaDeviceSynchronize());
    if (n_frames < 0 || n_frames > p.last_frames) return fail(SVDPHAT_INVALID_ARG, "n_frames > frames of last call");
    const int F = (int)n_frames;
    if (what == SVDPHAT_DUMP_CLASS_REP) {
        if (bytes < (int64_t)p.Q_eff * 4) return fail(SVDPHAT_INVALID_ARG, "buffer too small");
        std::memcpy(host_out, p.rep_q.data(), (size_t)p.Q_eff * 4);
        return SVDPHAT_OK;
    }
    if (what == SVDPHAT_DUMP_KEYS) {
        if (bytes < (int64_t)F * 8) return fail(SVDPHAT_INVALID_ARG, "buffer too small");
        SVD_CUDA_TRY(cudaMemcpy(host_out, p.d_keys + (p.last_method == SVDPHAT_METHOD_SVD ? p.F_pad : 0),
                                (size_t)F * 8, cudaMemcpyDeviceToHost));
        return SVDPHAT_OK;
    }
    if (what == SVDPHAT_DUMP_POWER) {
        if (!p.d_S) return fail(SVDPHAT_INVALID_ARG, "no svdphat_localize_topk call yet");
        if (bytes < (int64_t)F * p.Q_eff * 4) return fail(SVDPHAT_INVALID_ARG, "buffer too small");
        SVD_CUDA_TRY(cudaMemcpy2D(host_out, (size_t)p.Q_eff * 4, p.d_S, (size_t)p.Q_pad * 4, (size_t)p.Q_eff * 4, F,
                                  cudaMemcpyDeviceToHost));
        return SVDPHAT_OK;
    }
    if (what == SVDPHAT_DUMP_Z) {
        if (!p.d_Z32) return fail(SVDPHAT_INVALID_ARG, "SVD not planned");
        if (bytes < (int64_t)F * 2 * p.D * 4) return fail(SVDPHAT_INVALID_ARG, "buffer too small");
        std::vector<float> z((size_t)F * 2 * p.Zh);
        SVD_CUDA_TRY(cudaMemcpy(z.data(), p.d_Z32, z.size() * 4, cudaMemcpyDeviceToHost));
        float* o = static_cast<float*>(host_out);
        for (int f = 0; f < F; ++f)
            for (int d = 0; d < p.D; ++d) {
                o[((size_t)f * 2 * p.D) + d] = z[(size_t)f * 2 * p.Zh + d];
                o[((size_t)f * 2 * p.D) + p.D + d] = z[(size_t)f * 2 * p.Zh + p.Zh + d];
            }
        return SVDPHAT_OK;
    }
    if (what == SVDPHAT_DUMP_PHASORS) {
        if (bytes < (int64_t)F * p.M * p.Kb * 2 * 4) return fail(SVDPHAT_INVALID_ARG, "buffer too small");
        const int64_t nb = (int64_t)p.L.n_chunks * p.L.Mi * p.F_pad * p.L.unit_bytes;
        std::vector<__half> h((size_t)nb / 2);
        SVD_CUDA_TRY(cudaMemcpy(h.data(), p.d_P16, nb, cudaMemcpyDeviceToHost));
        float* o = static_cast<float*>(host_out);
        const int bpc = p.L.bpc;
        for (int f = 0; f < F; ++f)
            for (int m = 0; m < p.M; ++m)
                for (int kb = 0; kb < p.Kb; ++kb) {
                    const int c = kb / bpc, s = kb % bpc;
                    const size_t rec = (((size_t)c * p.L.Mi + m) * p.F_pad + f) * (size_t)(bpc * 2);
                    o[(((size_t)f * p.M + m) * p.Kb + kb) * 2 + 0] = __half2float(h[rec + s]);
                    o[(((size_t)f * p.M + m) * p.Kb + kb) * 2 + 1] = __half2float(h[rec + bpc + s]);
                }
        return SVDPHAT_OK;
    }
    return fail(SVDPHAT_INVALID_ARG, "unknown dump id");
}

svdphat_status svdphat_debug_dump(svdphat_plan_t plan, int32_t what, int64_t n_frames, void* host_out, int64_t bytes) {
    if (!plan || !host_out) return fail(SVDPHAT_INVALID_ARG, "NULL argument");
    return guarded([&] { return debug_dump_impl(plan->p, what, n_frames, host_out, bytes); });
}

}  // extern "C"
