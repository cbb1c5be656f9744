// internal.h — plan structure and kernel launchers of libsvdphat (not part of the public ABI).
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/svdphat.h"

namespace svdphat {

// ---------------------------------------------------------------- device data layout
// The GEMM contraction index kappa runs over (chunk c, unit u, slot s):  kappa = ((c*U + u)*8 + s).
//   bpc = 4 (M' <= 16): unit = one pair p = u; slots 0..3 = Re of bins 4c..4c+3, 4..7 = Im of the same bins.
//   bpc = 2 (M' = 32) : unit = pairs 2u, 2u+1; slots {0,1} Re p=2u bins 2c,2c+1; {2,3} Im p=2u; {4,5} Re p=2u+1;
//                       {6,7} Im p=2u+1.
// Pairs are enumerated lexicographically over M' >= M "instantiated" mics; pairs touching a mic >= M, bins
// >= N/2+1 and units >= pairs are zero.  Phasors live in P16[c][m][F_pad][bpc*2 halves] (Re bins | Im bins).
struct Layout {
    int M = 0, Mi = 0;        // real mics, instantiated mics (kernel template)
    int P = 0, Pi = 0;        // real pairs, instantiated pairs
    int N = 0, Kb = 0;        // frame size, bins N/2+1
    int bpc = 4;              // bins per chunk
    int n_chunks = 0;         // ceil(Kb / bpc)
    int U = 0;                // units per chunk (multiple of 8)
    int64_t K_total = 0;      // n_chunks * U * 8  (multiple of 64)
    int unit_bytes = 16;      // bytes of one phasor record (bpc*2 halves)
};

struct Plan {
    // description
    int M = 0, P = 0, N = 0, hop = 0, Kb = 0, field = 0, Q = 0, methods = 0, device = 0;
    int64_t PK = 0, max_frames = 0, F_pad = 0;
    double fs = 0, c = 0, delta = 0;
    Layout L;
    // steering classes (bitwise-identical tau rows; R11)
    int Q_eff = 0, Q_pad = 0;
    std::vector<int> rep_q;       // [Q_eff] lowest point index of each class
    std::vector<int> cls_count;   // [Q_eff]
    // SVD
    int D = 0, Dh = 0, K2 = 0;    // rank, rank padded to 64, search contraction length 3*2*Dh
    double energy_kept = 0, trace = 0;
    std::vector<double> sigma2;   // descending
    double setup_seconds = 0;
    // device operands (owned)
    __half* d_W16 = nullptr;      // [W_rows][K_W]: class rows (standard kappa) or fold rows (fold kappa)
    // antipodal folding of the SRP GEMM (R22): class c' with tau_c' = -tau_c bitwise has W_c' = conj W_c,
    // so one fold row carrying (Re W_c, Im W_c) yields Y_c = a - b and Y_c' = a + b with a = Re W_c . x_r and
    // b = Im W_c . x_i: half the rows, same K.  Fold kappa: per chunk, SP = ceil(U/16) slab pairs (Re slab, Im slab);
    // unit u's 4 Re values sit at 4*(u%16) of Re slab u/16, its 4 Im values likewise in the Im slab.
    bool fold = false;
    int fold_rows = 0;            // rows of the folded W (classes paired with their antipode, or alone)
    int* d_fold_cls = nullptr;    // [2][fold_rows]: class of a - b, class of a + b (-1: none)
    int W_rows = 0;               // rows of W16 (multiple of 256 for the pair kernel)
    int64_t K_F = 0;              // fold contraction length (n_chunks * spc_F * 64)
    int spc_F = 0;                // fold slabs per bin chunk (2 * ceil(U/16))
    // SVD with a real V (R22): when every class has its antipode (or a zero tau row), W^H W is real; the
    // SVD is taken of the real W~ = T W (rows sqrt2 Re W_c, sqrt2 Im W_c per pair, W_c for a real row), so V is real
    // and Z_r = V^T x_r, Z_i = V^T x_i: the projection runs as a fold GEMM on D rows (a -> Z_r, b -> Z_i).
    bool svd_fold = false;
    // BOTH with fold + real V: the few fold rows past the last full 256-row SRP tile ride in spare rows [D, D+tail_n)
    // of the projection's last V tile (W values copied there); zsplit turns their (a, b) into SRP keys, so the SRP
    // GEMM skips that tile (cfg3/cfg4: 5121 = 20 x 256 + 1 rows -> one wave fewer).
    int tail_r0 = -1, tail_n = 0;
    std::vector<int> rb_cls, rb_partner, rb_kind;   // real basis row i: class, antipode (-1), kind 0 Re / 1 Im / 2 real
    int64_t K_W = 0;              // contraction length of W16
    int spc_W = 0;                // W16 slabs per bin chunk
    __half* d_V16 = nullptr;      // [V_rows][K_total] (complex V), or [V_rows][K_P] part layout (svd_fold)
    // part layout (real V, gemm2p): the projection's A rows carry Re x and Im x of a frame separately, so V is stored
    // once per K position: per chunk SP = ceil(U/16) slabs, unit u's 4 values at (c*SP + u/16)*64 + (u%16)*4
    int64_t K_P = 0;
    int spc_P = 0;
    __half* d_R16 = nullptr;      // [Q_pad][K2]   FP16 normalised dictionary rows [Re | -Im] (search GEMM)
    float* d_R32 = nullptr;       // [Q_eff][K2]   the same in FP32 (exact rescore of the search candidates)
    int* d_rep = nullptr;         // [Q_eff]
    float* d_delay = nullptr;     // [Q][M]  relative arrival delays (samples)
    float* d_window = nullptr;    // [N]
    float2* d_twN = nullptr;      // [N]     e^{-j 2 pi k / N}
    // workspace
    uint8_t* d_P16 = nullptr;     // phasors
    unsigned long long* d_keys = nullptr;  // [3][F_pad]: SRP keys, SVD keys (rescored), SVD FP16 search keys
    float* d_Z32 = nullptr;       // [zsplit_max][F_pad][2*Zh] partial Z of the split-K projection (Z_r | Z_i)
    int Zh = 0;                   // half width of a Z32 row: >= D_h and >= the projection's V rows
    float* d_Zn32 = nullptr;      // [F_pad][K2] FP32 Zhat = Z/||Z|| [Re | Im] (rescore)
    unsigned long long* d_cand = nullptr;  // [F_pad][SEARCH_CAP] search candidates (FP16 score, class)
    int* d_ccnt = nullptr;        // [F_pad] candidates per frame
    // small batches (F_pad x Q_pad FP32 <= 64 MB): the search GEMM stores its FP16-input score map and the rescore
    // scans it per frame (all row tiles of a frame run concurrently there, so running-maximum lists would overflow)
    float* d_Smap = nullptr;      // [F_pad][Q_pad]
    bool search_map = false;
    int V_rows = 0;               // rows of V16: proj_ntiles * proj_nt (pair projection) or 2*Dh (1-CTA)
    int proj_nt = 0;              // V rows per pair tile of the frames-on-M projection (multiple of 32, <= 256)
    int proj_ntiles = 0;          // V row tiles
    int proj_nmma = 1;            // MMAs per K step of a part-kernel tile (proj_nt > 256 -> 2 of proj_nt/2 columns)
    bool pair_proj = true;
    int zsplit_max = 1;
    // small batches: SRP as split-K partial power maps + sum/argmax (the argmax epilogue cannot split K)
    float* d_Ypart = nullptr;     // [srp_split_max][F_pad][Q_pad]
    int srp_split_max = 0;
    __half* d_Zs16 = nullptr;     // [F_pad][K2] FP16 Zhat [Re | Im] (search GEMM operand)
    int* d_zflag = nullptr;       // [F_pad]
    // multi-source (top-k) workspace, allocated on first use: power map S[F_pad][Q_pad], class lists [F_pad][4]
    float* d_S = nullptr;
    int* d_cls = nullptr;
    float4* d_dirs = nullptr;     // [Q_eff] unit direction of each class representative (from the array centroid)
    // delay-and-sum SRP (das.cu, NEXT-4): per-bin steering rows A16[Kb][das_rows][2 das_me] (Re / Im rows of each
    // class) and the frames' phasors re-laid per bin, E16[Kb][F_pad][2 das_me]
    int das_me = 0;               // microphones per K block (8, 16, 32): K = 2 das_me per bin
    int das_rows = 0;             // 2 Q_eff rounded up to 256 (folded: 2 fold_rows rounded up to 256)
    // folded delay-and-sum (centrally symmetric grids, das_me >= 16): one (cos, sin) row pair per antipodal class
    // pair, K = das_me per bin, frames as (Re e, Im e) column pairs; operands per bin chunk, one 128-byte row holding
    // the chunk's bins: A16[n_chunks][das_rows][bpc * das_me], E16[n_chunks][2 F_pad][bpc * das_me]
    bool das_fold = false;
    __half* d_A16 = nullptr;
    __half* d_E16 = nullptr;
    int64_t bytes_W = 0, bytes_V = 0, bytes_R = 0, bytes_ws = 0, bytes_A = 0;
    // TMA descriptors
    alignas(64) CUtensorMap tm_W;
    alignas(64) CUtensorMap tm_V;
    alignas(64) CUtensorMap tm_R;
    alignas(64) CUtensorMap tm_Zs;
    alignas(64) CUtensorMap tm_A;     // A16 as [Kb * das_rows][2 das_me], box 2 das_me x 128
    alignas(64) CUtensorMap tm_E;     // E16 as [Kb * F_pad][2 das_me], box 2 das_me x 128
    int num_sms = 148;
    bool pair_srp = true;          // SRP GEMM on CTA pairs (cta_group::2); Q_pad is then a multiple of 256
    // host-buffer path: two staging slots + a copy stream so chunk i+1's H2D overlaps chunk i's compute
    float* d_stage = nullptr;
    int64_t stage_elems = 0;           // elements per slot
    cudaStream_t copy_stream = nullptr;
    cudaEvent_t ev_copied[2] = {nullptr, nullptr};
    cudaEvent_t ev_done[2] = {nullptr, nullptr};
    // method BOTH: the SVD chain runs on svd_stream, forked after the STFT and joined before the finalize, so its
    // kernels fill the SMs released by the SRP GEMM's last (partial) wave
    cudaStream_t svd_stream = nullptr;   // lowest priority
    cudaStream_t srp_stream = nullptr;   // highest priority: its CTAs are dispatched before the SVD chain's
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr, ev_z = nullptr;
    int32_t* d_doa_stage = nullptr;
    float* d_score_stage = nullptr;
    int64_t last_frames = 0;
    int last_method = 0;
    // streaming host path (svdphat_submit_host): two staging slots
    struct HostSlot {
        float* d_audio = nullptr;
        int64_t elems = 0;
        int32_t* d_doa = nullptr;
        float* d_score = nullptr;
        cudaEvent_t h2d = nullptr, comp = nullptr, d2h = nullptr;
        int64_t ticket = -1;
    } slots[2];
    cudaStream_t up_stream = nullptr, down_stream = nullptr;
    int64_t next_ticket = 0;
    int options = 0;              // svdphat_plan_desc.options (SVDPHAT_OPT_*)
    // per-stage profiling
    bool prof_on = false;
    int prof_cap = 0, prof_n = 0;
    std::vector<cudaEvent_t> prof_ev;   // 2 * prof_cap
    std::vector<int> prof_stage;
};

// Per-call band limit (NEXT-3): bins [k_lo, k_hi) -> active bin chunks [c_lo, c_hi); optional per-frame TF mask.
// Passed explicitly to every launcher (the plan stays immutable after creation).
struct Band {
    int k_lo = 0, k_hi = 0, c_lo = 0, c_hi = 0;
    const uint8_t* mask = nullptr;
    int64_t mask_stride = 0;
};
Band make_band(const Plan& p, int k_lo, int k_hi, const uint8_t* mask, int64_t mask_stride);
inline Band full_band(const Plan& p) { return make_band(p, 0, p.Kb, nullptr, 0); }

// ---------------------------------------------------------------- error plumbing
void set_error(const std::string& msg);
#define SVD_CUDA_TRY(expr)                                                                                    \
    do {                                                                                                      \
        cudaError_t _e = (expr);                                                                              \
        if (_e != cudaSuccess) {                                                                              \
            ::svdphat::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" __FILE__ ":" +     \
                                 std::to_string(__LINE__));                                                   \
            return SVDPHAT_CUDA;                                                                              \
        }                                                                                                     \
    } while (0)

// ---------------------------------------------------------------- launchers (return cudaError_t)
cudaError_t launch_stft_phat(const Plan& p, const Band& b, const float* audio, int64_t cs, int64_t fstride, int F,
                             cudaStream_t s);
// mode: 0 = SRP argmax (A = W16, B = producer), 1 = SVD GEMM1 store Z (A = V16, B = producer),
//       2 = SVD search argmax + candidate lists (A = R16, B = Zs16 via TMA), 3 = SRP power map -> d_S,
//       4 = SVD search power map -> d_S, 5 = SVD search score map -> d_Smap (small batches, rescored per frame)
// both: a localize(BOTH) call, where the SRP tail rows travel through the projection (Plan::tail_n)
cudaError_t launch_gemm(const Plan& p, const Band& b, int mode, int F, cudaStream_t s, bool both = false);
cudaError_t launch_zsplit(const Plan& p, const Band& b, int F, cudaStream_t s, bool both = false);
int srp_split_ways(const Plan& p, const Band& b, int F);   // > 1: the SRP call takes the small-batch split-K path
cudaError_t launch_split_argmax(const Plan& p, int F, int S, cudaStream_t s);
constexpr int MAX_KSPLIT = 32;               // cap on K splits (chunk ranges) of the store-mode GEMMs
// FP16 search + exact rescore: a row enters a frame's candidate list when its FP16 score is within SEARCH_TAU of the
// frame's running FP16 maximum.  SEARCH_TAU = 2.5e-3 >= twice the FP16 error bound of a unit-vector dot product
// (2^-10 + FP32 accumulation), so the exact argmax is always a candidate; lists longer than SEARCH_CAP fall back to
// an exact scan of every class for that frame.
constexpr int SEARCH_CAP = 128;
constexpr float SEARCH_TAU = 2.5e-3f;
cudaError_t launch_rescore(const Plan& p, int F, cudaStream_t s);
struct ProjShape {
    bool pair;
    int m_tiles, n_tiles, ksplit;   // pair: m = 256-frame tiles, n = proj_nt-row V tiles; 1-CTA: m = 128-row V tiles
};
ProjShape proj_shape(const Plan& p, const Band& b, int F);   // tiles and K splits of the SVD projection GEMM
// method SRP|SVD|BOTH; doa[0]/score[0] receive SRP results, doa[1]/score[1] SVD results
cudaError_t launch_finalize(const Plan& p, int method, int F, int32_t* const doa[2], float* const score[2],
                            cudaStream_t s);
// multi-source: greedy top-k with angular suppression over d_S -> class lists, then Y_q of each peak
cudaError_t launch_topk(const Plan& p, int F, int k, float cos_sep, cudaStream_t s);
cudaError_t launch_finalize_topk(const Plan& p, int F, int k, int32_t* doa, float* score, cudaStream_t s);
cudaError_t gemm_set_attributes();   // per-device kernel attributes, set at plan creation
cudaError_t stft_set_attributes();
cudaError_t topk_set_attributes();

// delay-and-sum SRP (das.cu): E16 from the phasor records, then the per-bin GEMM + sum of squares + argmax -> SRP keys
int das_me(int M);
bool das_active(const Plan& p, int F);     // plan has the operands and F fills the CTA pairs
cudaError_t launch_das_bins(const Plan& p, const Band& b, int F, cudaStream_t s);
cudaError_t launch_das(const Plan& p, const Band& b, int F, cudaStream_t s);
cudaError_t das_set_attributes();

// setup (float64, device)
svdphat_status setup_das_operand(Plan& p, const double* h_delay_cls);
// folded form: h_delay_fold [fold_rows][M] = delays of each fold row's first class (d_fold_cls[0][r])
svdphat_status setup_das_fold_operand(Plan& p, const double* h_delay_fold);
svdphat_status setup_srp_operand(Plan& p, const double* d_tau_cls);
svdphat_status setup_svd_operands(Plan& p, const double* d_tau_cls, int rank_D);

}  // namespace svdphat
