/*
 * svdphat.h — C-ABI of libsvdphat.so, the B200 (sm_100a) per-frame localisation hot path of
 * SVD-PHAT and of the exact SRP-PHAT it approximates (Grondin & Glass, arXiv 1811.11785).
 *
 * Citations: PAPER.md = /root/reference/PAPER.md (line numbers, section / equation / algorithm).
 * Readings of silent or ambiguous passages are the R* items of DESIGN.md.
 *
 * Boundary: plain pointers and sizes only, no torch types.  A plan is created once
 * (Alg. 1 "Offline") and then localises batches of frames (Alg. 1 "Online",
 * PAPER.md:191-197; SRP-PHAT eqs. 5-6).
 *
 * Error behaviour: every call returns an svdphat_status and never throws across the ABI.  All arguments are
 * validated before any kernel is launched; on a non-OK status no output is written and
 * svdphat_last_error() returns a thread-local human-readable detail.  Asynchronous device faults surface at
 * the caller's next synchronisation of the stream.
 */
#ifndef SVDPHAT_H_
#define SVDPHAT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SVDPHAT_OK = 0,
    SVDPHAT_INVALID_ARG = 1,   /* argument violates a documented precondition                          */
    SVDPHAT_ALLOC = 2,         /* device or host allocation failed                                      */
    SVDPHAT_CUDA = 3,          /* a CUDA runtime / driver / cuBLAS / cuSOLVER call failed               */
    SVDPHAT_NUMERIC = 4,       /* setup produced non-finite values (e.g. eigensolver failure)           */
    SVDPHAT_UNSUPPORTED = 5,   /* valid but not supported by this build (e.g. no sm_100a device)        */
    SVDPHAT_TOO_LARGE = 6      /* the plan would not fit the device memory or index ranges              */
} svdphat_status;

enum { SVDPHAT_FIELD_FAR = 0, SVDPHAT_FIELD_NEAR = 1 };
enum { SVDPHAT_METHOD_SRP = 1, SVDPHAT_METHOD_SVD = 2, SVDPHAT_METHOD_BOTH = 3 };

typedef struct svdphat_plan_s* svdphat_plan_t;

/* Plan description.  All pointers are HOST pointers, read only during svdphat_plan_create (not retained). */
typedef struct {
    int32_t M;                 /* microphones, 2..32 ("array with M microphones")                */
    const double* mic_xyz;     /* M x 3 row-major, metres, finite (r_i)                          */
    double fs;                 /* sample rate f_S > 0, Hz                                        */
    double c;                  /* speed of sound c > 0, m/s                                      */
    int32_t N;                 /* frame size, power of two in [16, 2048]                         */
    int32_t hop;               /* hop Delta N, 0 < hop <= N; informational for streams            */
    int32_t field;             /* SVDPHAT_FIELD_FAR: eq. 2 on directions s_q (normalised here);
                                  SVDPHAT_FIELD_NEAR: eq. 1 on points s_q in metres             */
    int32_t Q;                 /* candidates, 1..2^24                                             */
    const double* points_xyz;  /* Q x 3 row-major; FAR: any non-zero finite vector; NEAR: finite position      */
    int32_t rank_D;            /* SVD rank: > 0 explicit, 0 = rule of eq. 11 with delta          */
    double delta;              /* eq. 11 tolerance, 0 < delta < 1 (BASELINE cfg1: 1e-5)                         */
    int32_t methods;           /* bitmask of SVDPHAT_METHOD_SRP | SVDPHAT_METHOD_SVD                           */
    int64_t max_frames;        /* largest n_frames of a single localize call (sizes the device workspace)       */
    int32_t device;            /* CUDA device ordinal                                                          */
    int32_t options;           /* 0 = the product configuration; bits of SVDPHAT_OPT_* select equivalent
                                  alternative kernels (same results up to FP32 summation order; for tests and
                                  A/B measurements).  Unknown bits -> INVALID_ARG.                             */
} svdphat_plan_desc;

/* Plan options (svdphat_plan_desc.options).  Each selects an alternative evaluation of the same equations:
 *   NO_SRP_FOLD   SRP GEMM on one row per steering class instead of antipodal fold rows (R22);
 *   NO_SVD_FOLD   complex V_D (2D real-split rows) instead of the real-basis V_D of a centrally symmetric grid;
 *   ONE_CTA_SRP   1-CTA 128-row SRP GEMM tiles instead of CTA pairs (implies NO_SRP_FOLD);
 *   ONE_CTA_PROJ  1-CTA V-on-M projection GEMM instead of the frames-on-M CTA-pair kernel (implies NO_SVD_FOLD);
 *   NO_DAS        SRP-PHAT always through eq. 9's GEMM Y = Re{W X}, never through the delay-and-sum form of eq. 5
 *                 (Y_q = 1/2 sum_k |sum_m e_m[k] e^{j 2 pi k delta_qm / N}|^2 - n_k, tau_qij = delta_qi - delta_qj), which
 *                 the library uses by default for M >= 17 on batches that fill the GPU (NEXT-4);
 *   DAS           the delay-and-sum form for every M and every batch size;
 *   DAS_FOLD      the antipodally folded delay-and-sum kernel also for 9..16 microphones (default only for 17..32):
 *                 one (cos, sin) row pair per antipodal class pair (delta_q'm = -delta_qm + const, reading R22)
 *                 against (Re e, Im e) frame columns, both classes' |a|^2 from the four real products. */
enum {
    SVDPHAT_OPT_NO_SRP_FOLD = 1,
    SVDPHAT_OPT_NO_SVD_FOLD = 2,
    SVDPHAT_OPT_ONE_CTA_SRP = 4,
    SVDPHAT_OPT_ONE_CTA_PROJ = 8,
    SVDPHAT_OPT_NO_DAS = 16,
    SVDPHAT_OPT_DAS = 32,
    SVDPHAT_OPT_DAS_FOLD = 64
};

typedef struct {
    int32_t M, P, N, K_bins;   /* P = M(M-1)/2 pairs, K_bins = N/2+1                             */
    int64_t PK;                /* length of the X vector, P*(N/2+1) (eq. 7)                        */
    int32_t Q;                 /* candidates                                                                    */
    int32_t Q_classes;         /* distinct steering rows of W (bitwise-identical rows merged; R11)    */
    int32_t D;                 /* retained SVD rank (paper's K, eq. 11), 0 if SVD not planned                   */
    double energy_kept;        /* sum_{d<=D} sigma_d^2 / Tr{W W^H}                                              */
    double trace_WWH;          /* Tr{W W^H} = Q*P*(N/2+1) exactly (|W| = 1)                                     */
    int32_t methods;
    int32_t gemm_k;            /* padded contraction length of the device real-split GEMMs                      */
    int64_t max_frames;
    int64_t bytes_W;           /* device bytes of the FP16 real-split steering matrix (SRP)                     */
    int64_t bytes_V;           /* device bytes of the FP16 real-split V_D (SVD)                                 */
    int64_t bytes_R;           /* device bytes of the split-FP16 normalised dictionary rows (SVD)               */
    int64_t bytes_workspace;   /* per-call workspace (phasors, keys, Z, ...)                                    */
    double setup_seconds;      /* wall time of svdphat_plan_create                                              */
    int32_t srp_rows;          /* rows of the SRP GEMM: Q_classes, or the antipodal fold rows when the grid is
                                  centrally symmetric in tau (class pairs tau_c' = -tau_c; R22)        */
    int32_t svd_rows;          /* rows of the SVD projection GEMM: 2*D (complex V, real-split) or D (real V when
                                  every class has its antipode; R22); 0 if SVD not planned             */
    int32_t das_rows;          /* rows of the delay-and-sum SRP GEMM (2 per class: Re a_q, Im a_q; padded to 256);
                                  0 if the plan has no delay-and-sum operand (M < 12 or SVDPHAT_OPT_NO_DAS)       */
    int32_t das_me;            /* microphones of its contraction, padded to 8/16/32 (K = 2*das_me per bin)       */
    int64_t srp_gemm_k;        /* contraction length the eq. 9 SRP GEMM executes (padded, fold layout if folded)  */
    int32_t srp_gemm_rows;     /* W rows it holds (256-row tiles)                                               */
    int32_t srp_tail_rows;     /* fold rows past the last full tile that BOTH calls score through the projection */
} svdphat_plan_info_t;

/* Alg. 1 offline steps 1-3: TDOAs (eq. 1/2), W (eqs. 4, 8), SVD (eq. 10) with the rank rule
 * (eq. 11), dictionary rows D = US (eq. 13) normalised.  Float64 setup, run once; the k-d tree of
 * step 4 is replaced by an exhaustive contraction.  *out receives an opaque plan owned by the caller
 * (free with svdphat_plan_destroy).  Returns INVALID_ARG for bad descriptors (M<2 or >32, N not a power of two,
 * hop<=0 or >N, fs<=0, c<=0, non-finite coordinates, zero FAR direction, delta outside (0,1), methods==0,
 * max_frames<0, unknown option bits), UNSUPPORTED if the device is not sm_100, TOO_LARGE if the operands or the
 * float64 setup workspace (SVD: a Q_classes^2 Gram matrix, Q_classes <= 65535) would not fit the device or the
 * launch ranges, ALLOC if an allocation fails.  Every entry point of this header restores the caller's current CUDA
 * device before returning (calls run on the plan's device). */
svdphat_status svdphat_plan_create(const svdphat_plan_desc* desc, svdphat_plan_t* out);

/* Fills *out (host struct).  INVALID_ARG on NULL. */
svdphat_status svdphat_plan_info(svdphat_plan_t plan, svdphat_plan_info_t* out);

/* Copies the first min(n, Q_classes) squared singular values sigma_d^2 of W, descending (host array), so that a
 * caller can re-apply eq. 11 for any delta (Fig. 2b/2c).  INVALID_ARG if SVD was not planned. */
svdphat_status svdphat_plan_sigma2(svdphat_plan_t plan, double* out, int32_t n);

/* Localise n_frames frames on `stream` (a cudaStream_t, NULL = legacy default stream); asynchronous, no host
 * synchronisation and no allocation (graph-capturable).
 *   method   SVDPHAT_METHOD_SRP: eqs. 5-6 = Y = Re{W X} (eq. 9) + argmax;
 *            SVDPHAT_METHOD_SVD: Alg. 1 online: Z = V^H X (eq. 12), nearest normalised
 *            dictionary row (eqs. 14-15), then Y_q from the row of W.
 *            SVDPHAT_METHOD_BOTH: both from one STFT pass; d_doa / d_score then hold 2*n_frames entries,
 *            SRP results first, SVD results second.
 *   d_audio  DEVICE float32 samples: sample n of channel m in frame l is d_audio[m*channel_stride +
 *            l*frame_stride + n] (stream [M][L]: channel_stride=L, frame_stride=hop; framed [B][M][N]:
 *            channel_stride=N, frame_stride=M*N).  Must be 4-byte aligned.
 *   d_doa    DEVICE int32[n_frames]: 0-based index into the plan's points; lowest index among exact ties
 *            (R10); -1 when the frame's X vector is identically 0 (R4).
 *   d_score  DEVICE float32[n_frames]: Y_q_bar (eq. 5 at q_bar), 0 when d_doa = -1.
 * Buffers are owned by the caller.  0 <= n_frames <= max_frames.  One localize in flight per plan (the plan's
 * workspace is shared).  INVALID_ARG on violated preconditions, CUDA on launch failure. */
svdphat_status svdphat_localize(svdphat_plan_t plan, int32_t method, const float* d_audio, int64_t n_frames,
                                int64_t channel_stride, int64_t frame_stride, int32_t* d_doa, float* d_score,
                                void* stream);

/* Same with HOST buffers: copies audio elements [0, audio_elems) host->device, localises, copies results back
 * (2*n_frames entries for SVDPHAT_METHOD_BOTH) and synchronises `stream`.  h_audio should be pinned for full bandwidth.  The device staging buffer is
 * allocated on first use and kept by the plan (ALLOC on failure). */
svdphat_status svdphat_localize_host(svdphat_plan_t plan, int32_t method, const float* h_audio,
                                     int64_t audio_elems, int64_t n_frames, int64_t channel_stride,
                                     int64_t frame_stride, int32_t* h_doa, float* h_score, void* stream);

/* Streaming host path: enqueue one batch (H2D copy of audio elements [0, audio_elems) on an internal upload
 * stream, localisation on `stream`, D2H of the results on an internal download stream) and return at once with a
 * ticket.  Two batches may be in flight per plan (double-buffered device staging, allocated on first use): the
 * upload of batch i+1 overlaps the kernels of batch i.  A third submit first waits for the oldest batch.  Host
 * buffers must stay valid and unmodified until svdphat_wait(ticket) returns (pinned memory for full bandwidth).
 * Outputs as svdphat_localize_host. */
svdphat_status svdphat_submit_host(svdphat_plan_t plan, int32_t method, const float* h_audio, int64_t audio_elems,
                                   int64_t n_frames, int64_t channel_stride, int64_t frame_stride, int32_t* h_doa,
                                   float* h_score, void* stream, int64_t* ticket);
/* Blocks until the batch of `ticket` has been copied back (INVALID_ARG for an unknown ticket). */
svdphat_status svdphat_wait(svdphat_plan_t plan, int64_t ticket);

/* Multi-source extension (future work: "investigate multiple source localization").  For each frame,
 * the k (1..4) strongest peaks of the method's power map — SRP: Y_q (eq. 5); SVD: Re{D_hat_q . Z_hat} (eq. 14) —
 * taken greedily, each peak excluding all candidates whose direction is within min_sep_deg of a stronger peak
 * (directions from the array centroid; steering classes of DESIGN.md R11 count as one candidate).
 *   d_doa[f*k + j], d_score[f*k + j] (DEVICE): peak j of frame f (point index, Y_q of eq. 5), strongest first;
 *   -1 / 0 when fewer than j+1 candidates remain or the frame is degenerate (R4).
 * method SRP or SVD.  On first use allocates a float32 power-map workspace of max_frames x Q_classes (ALLOC on
 * failure).  Q_classes must be <= 49152 (the map of one frame is staged in shared memory); INVALID_ARG otherwise. */
svdphat_status svdphat_localize_topk(svdphat_plan_t plan, int32_t method, const float* d_audio, int64_t n_frames,
                                     int64_t channel_stride, int64_t frame_stride, int32_t k, double min_sep_deg,
                                     int32_t* d_doa, float* d_score, void* stream);

/* Binary time-frequency masks (future work: "binary time-frequency mask, which could reduce even more
 * the amount of computations").  As svdphat_localize, but bin k of frame l enters the X vector (eq. 7) only if
 * k_lo <= k < k_hi and (d_mask == NULL or d_mask[l*mask_stride + k] != 0); excluded entries of eq. 3 are 0.  The band
 * [k_lo, k_hi) is skipped at bin-chunk granularity by the projection GEMMs (compute ~ (k_hi-k_lo)/(N/2+1)); the
 * DEVICE per-frame mask (uint8, mask_stride 0 = one row for all frames) changes the result, not the work.
 * 0 <= k_lo < k_hi <= N/2+1, else INVALID_ARG. */
svdphat_status svdphat_localize_masked(svdphat_plan_t plan, int32_t method, const float* d_audio, int64_t n_frames,
                                       int64_t channel_stride, int64_t frame_stride, int32_t k_lo, int32_t k_hi,
                                       const uint8_t* d_mask, int64_t mask_stride, int32_t* d_doa, float* d_score,
                                       void* stream);

/* Releases all device and host memory of the plan (NULL is a no-op).  The caller must have synchronised any
 * stream a localize was issued on. */
void svdphat_plan_destroy(svdphat_plan_t plan);

/* Number of frames of an L-sample stream without padding: 1 + floor((L - N)/hop), 0 if L < N (R3). */
int64_t svdphat_frame_count(int64_t L, int32_t N, int32_t hop);

const char* svdphat_status_str(svdphat_status s);
const char* svdphat_last_error(void);

/* ---- per-stage device timing (CUDA events recorded on the launching stream, for bench.py's roofline) ----
 * After svdphat_profile_begin(plan, capacity), every localize records a start/end event pair around each of its
 * kernels (up to `capacity` pairs).  svdphat_profile_end synchronises the events, writes up to `max` records
 * (stage id, milliseconds) in launch order, returns the number written (negative status on error) and stops
 * profiling.  Stage ids: */
enum {
    SVDPHAT_STAGE_STFT = 1,        /* sine-window STFT + PHAT phasors                                           */
    SVDPHAT_STAGE_SRP_GEMM = 2,    /* Y = Re{W X} with fused cross-spectrum producer and argmax (eqs. 3, 5-9)   */
    SVDPHAT_STAGE_SVD_PROJ = 3,    /* Z = V^H X with fused cross-spectrum producer (eq. 12)                     */
    SVDPHAT_STAGE_SVD_NORM = 4,    /* Zhat = Z / ||Z|| (FP16 search operand, FP32 rescore operand)              */
    SVDPHAT_STAGE_SVD_SEARCH = 5,  /* Re{Dhat_q Zhat} in FP16 + fused running argmax and candidate lists (eq. 14)  */
    SVDPHAT_STAGE_FINALIZE = 6,    /* Y_q of the chosen q (eq. 5; Alg. 1 online step 4)                         */
    SVDPHAT_STAGE_SVD_RESCORE = 7, /* exact FP32 Re{Dhat_q Zhat} of the search candidates -> q_bar (eqs. 14-15)  */
    SVDPHAT_STAGE_SRP_BINS = 8,    /* phasors re-laid per bin for the delay-and-sum SRP GEMM                     */
    SVDPHAT_STAGE_SRP_DAS = 9      /* delay-and-sum SRP: per-bin GEMM, sum of |a_q[k]|^2 over bins, argmax (eq. 5) */
};
svdphat_status svdphat_profile_begin(svdphat_plan_t plan, int32_t capacity);
int32_t svdphat_profile_end(svdphat_plan_t plan, int32_t* stage_ids, float* ms, int32_t max);

/* ---- test-only introspection (not part of the product path; used by tests/ for kernel-unit parity) ---- */
enum {
    SVDPHAT_DUMP_PHASORS = 1,  /* FP16 unit phasors of the last call, decoded to float32 [F][M][K_bins][2]     */
    SVDPHAT_DUMP_Z = 2,        /* float32 Z of the last SVD call [F][2*D] (Re then Im), scaled by sqrt(PK)       */
    SVDPHAT_DUMP_CLASS_REP = 3,/* int32 [Q_classes]: representative (lowest) point index of each steering class */
    SVDPHAT_DUMP_KEYS = 4,     /* uint64 [F]: packed (score, class) argmax keys of the last call                 */
    SVDPHAT_DUMP_POWER = 5     /* float32 [F][Q_classes]: the power map of the last svdphat_localize_topk call -
                                  SRP: Y_q of eq. 9 per steering class; SVD: Re{D^_q Z^} of eq. 14 - the raw GEMM
                                  outputs, for element-wise parity                                               */
};
svdphat_status svdphat_debug_dump(svdphat_plan_t plan, int32_t what, int64_t n_frames, void* host_out,
                                  int64_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* SVDPHAT_H_ */
