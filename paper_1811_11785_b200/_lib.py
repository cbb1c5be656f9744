"""Thin ctypes binding of libsvdphat.so (include/svdphat.h).  Argument marshalling only: every step of the
localisation path runs in the library's CUDA kernels.  There is no CPU fallback: if the shared library is missing
or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsvdphat.so")

OK, INVALID_ARG, ALLOC, CUDA, NUMERIC, UNSUPPORTED, TOO_LARGE = range(7)
FIELD_FAR, FIELD_NEAR = 0, 1
METHOD_SRP, METHOD_SVD, METHOD_BOTH = 1, 2, 3
STAGES = {1: "stft_phat", 2: "srp_gemm", 3: "svd_proj", 4: "svd_norm", 5: "svd_search", 6: "finalize",
          7: "svd_rescore", 8: "srp_bins", 9: "srp_das"}
_METHOD = {"srp": METHOD_SRP, "svd": METHOD_SVD, "both": METHOD_BOTH}
DUMP_PHASORS, DUMP_Z, DUMP_CLASS_REP, DUMP_KEYS, DUMP_POWER = 1, 2, 3, 4, 5
# svdphat_plan_desc.options: equivalent alternative kernels (tests / A-B measurements), 0 = product configuration
OPT_NO_SRP_FOLD, OPT_NO_SVD_FOLD, OPT_ONE_CTA_SRP, OPT_ONE_CTA_PROJ, OPT_NO_DAS, OPT_DAS, OPT_DAS_FOLD = 1, 2, 4, 8, 16, 32, 64


class PlanDesc(C.Structure):
    _fields_ = [("M", C.c_int32), ("mic_xyz", C.POINTER(C.c_double)), ("fs", C.c_double), ("c", C.c_double),
                ("N", C.c_int32), ("hop", C.c_int32), ("field", C.c_int32), ("Q", C.c_int32),
                ("points_xyz", C.POINTER(C.c_double)), ("rank_D", C.c_int32), ("delta", C.c_double),
                ("methods", C.c_int32), ("max_frames", C.c_int64), ("device", C.c_int32), ("options", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("M", C.c_int32), ("P", C.c_int32), ("N", C.c_int32), ("K_bins", C.c_int32), ("PK", C.c_int64),
                ("Q", C.c_int32), ("Q_classes", C.c_int32), ("D", C.c_int32), ("energy_kept", C.c_double),
                ("trace_WWH", C.c_double), ("methods", C.c_int32), ("gemm_k", C.c_int32),
                ("max_frames", C.c_int64), ("bytes_W", C.c_int64), ("bytes_V", C.c_int64), ("bytes_R", C.c_int64),
                ("bytes_workspace", C.c_int64), ("setup_seconds", C.c_double),
                ("srp_rows", C.c_int32), ("svd_rows", C.c_int32), ("das_rows", C.c_int32),
                ("das_me", C.c_int32), ("srp_gemm_k", C.c_int64), ("srp_gemm_rows", C.c_int32),
                ("srp_tail_rows", C.c_int32)]


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1811_11785_b200/build.py` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64, st = C.c_void_p, C.c_int32, C.c_int64, C.c_int
    sig = {
        "svdphat_plan_create": (st, [C.POINTER(PlanDesc), C.POINTER(vp)]),
        "svdphat_plan_info": (st, [vp, C.POINTER(PlanInfo)]),
        "svdphat_plan_sigma2": (st, [vp, C.POINTER(C.c_double), i32]),
        "svdphat_localize": (st, [vp, i32, vp, i64, i64, i64, vp, vp, vp]),
        "svdphat_localize_host": (st, [vp, i32, vp, i64, i64, i64, i64, vp, vp, vp]),
        "svdphat_plan_destroy": (None, [vp]),
        "svdphat_frame_count": (i64, [i64, i32, i32]),
        "svdphat_status_str": (C.c_char_p, [st]),
        "svdphat_last_error": (C.c_char_p, []),
        "svdphat_debug_dump": (st, [vp, i32, i64, vp, i64]),
        "svdphat_profile_begin": (st, [vp, i32]),
        "svdphat_localize_topk": (st, [vp, i32, vp, i64, i64, i64, i32, C.c_double, vp, vp, vp]),
        "svdphat_localize_masked": (st, [vp, i32, vp, i64, i64, i64, i32, i32, vp, i64, vp, vp, vp]),
        "svdphat_submit_host": (st, [vp, i32, vp, i64, i64, i64, i64, vp, vp, vp, C.POINTER(i64)]),
        "svdphat_wait": (st, [vp, i64]),
        "svdphat_profile_end": (i32, [vp, C.POINTER(i32), C.POINTER(C.c_float), i32]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    return lib


lib = _load()


class SvdPhatError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {lib.svdphat_status_str(status).decode()} "
                         f"({lib.svdphat_last_error().decode()})")


def _check(status: int, where: str) -> None:
    if status != OK:
        raise SvdPhatError(status, where)


def frame_count(L: int, N: int, hop: int) -> int:
    return int(lib.svdphat_frame_count(L, N, hop))


def _ptr(x) -> int:
    """Device/host address of a torch tensor, numpy array or raw int."""
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


class Plan:
    """svdphat_plan_create / _localize / _destroy.  `points` are unit-or-not directions (field='far', eq. 2) or
    positions in metres (field='near', eq. 1)."""

    def __init__(self, mics, points, fs: float, c: float, N: int, hop: int, field: str = "far", rank_D: int = 0,
                 delta: float = 1e-5, methods=("srp", "svd"), max_frames: int = 1024, device: int = 0,
                 options: int = 0):
        self._mics = np.ascontiguousarray(mics, dtype=np.float64)
        self._pts = np.ascontiguousarray(points, dtype=np.float64)
        m = (METHOD_SRP if "srp" in methods else 0) | (METHOD_SVD if "svd" in methods else 0)
        d = PlanDesc(self._mics.shape[0], self._mics.ctypes.data_as(C.POINTER(C.c_double)), fs, c, N, hop,
                     FIELD_FAR if field == "far" else FIELD_NEAR, self._pts.shape[0],
                     self._pts.ctypes.data_as(C.POINTER(C.c_double)), rank_D, delta, m, max_frames, device,
                     options)
        h = C.c_void_p()
        _check(lib.svdphat_plan_create(C.byref(d), C.byref(h)), "svdphat_plan_create")
        self._h = h
        self.N, self.hop, self.M = N, hop, self._mics.shape[0]

    def info(self) -> dict:
        inf = PlanInfo()
        _check(lib.svdphat_plan_info(self._h, C.byref(inf)), "svdphat_plan_info")
        return {k: getattr(inf, k) for k, _ in PlanInfo._fields_}

    def sigma2(self, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.float64)
        _check(lib.svdphat_plan_sigma2(self._h, out.ctypes.data_as(C.POINTER(C.c_double)), n), "sigma2")
        return out

    def localize(self, method: str, audio, n_frames: int, channel_stride: int, frame_stride: int, doa, score,
                 stream: int = 0) -> None:
        """Device path: audio/doa/score are CUDA tensors (float32 / int32 / float32); async on `stream`.
        method "srp" | "svd" | "both" (doa/score then hold 2*n_frames: SRP first, SVD second)."""
        _check(lib.svdphat_localize(self._h, _METHOD[method], _ptr(audio), n_frames,
                                    channel_stride, frame_stride, _ptr(doa), _ptr(score), stream),
               "svdphat_localize")

    def localize_host(self, method: str, audio, audio_elems: int, n_frames: int, channel_stride: int,
                      frame_stride: int, doa, score, stream: int = 0) -> None:
        """Host path: audio/doa/score are host buffers (pinned for full bandwidth); synchronous."""
        _check(lib.svdphat_localize_host(self._h, _METHOD[method], _ptr(audio),
                                         audio_elems, n_frames, channel_stride, frame_stride, _ptr(doa), _ptr(score),
                                         stream), "svdphat_localize_host")

    def localize_topk(self, method: str, audio, n_frames: int, channel_stride: int, frame_stride: int, k: int,
                      min_sep_deg: float, doa, score, stream: int = 0) -> None:
        """Multi-source: the k strongest peaks per frame (doa/score: CUDA tensors of n_frames*k), separated by at
        least min_sep_deg; method "srp" or "svd"."""
        _check(lib.svdphat_localize_topk(self._h, _METHOD[method], _ptr(audio), n_frames, channel_stride,
                                         frame_stride, k, min_sep_deg, _ptr(doa), _ptr(score), stream),
               "svdphat_localize_topk")

    def submit_host(self, method: str, audio, audio_elems: int, n_frames: int, channel_stride: int,
                    frame_stride: int, doa, score, stream: int = 0) -> int:
        """Streaming host path: enqueue H2D -> localise -> D2H and return a ticket (two batches in flight)."""
        t = C.c_int64()
        _check(lib.svdphat_submit_host(self._h, _METHOD[method], _ptr(audio), audio_elems, n_frames, channel_stride,
                                       frame_stride, _ptr(doa), _ptr(score), stream, C.byref(t)),
               "svdphat_submit_host")
        return t.value

    def wait(self, ticket: int) -> None:
        _check(lib.svdphat_wait(self._h, ticket), "svdphat_wait")

    def localize_masked(self, method: str, audio, n_frames: int, channel_stride: int, frame_stride: int, k_lo: int,
                        k_hi: int, mask, mask_stride: int, doa, score, stream: int = 0) -> None:
        """Band limit [k_lo, k_hi) (skipped by the GEMMs) + optional per-frame binary TF mask (uint8 CUDA tensor)."""
        _check(lib.svdphat_localize_masked(self._h, _METHOD[method], _ptr(audio), n_frames, channel_stride,
                                           frame_stride, k_lo, k_hi, _ptr(mask), mask_stride, _ptr(doa), _ptr(score),
                                           stream), "svdphat_localize_masked")

    def profile_begin(self, capacity: int) -> None:
        _check(lib.svdphat_profile_begin(self._h, capacity), "profile_begin")

    def profile_end(self, max_records: int = 1 << 16) -> list[tuple[str, float]]:
        ids = (C.c_int32 * max_records)()
        ms = (C.c_float * max_records)()
        n = lib.svdphat_profile_end(self._h, ids, ms, max_records)
        if n < 0:
            raise SvdPhatError(-n, "profile_end")
        return [(STAGES[ids[i]], float(ms[i])) for i in range(n)]

    def debug_dump(self, what: int, n_frames: int) -> np.ndarray:
        inf = self.info()
        if what == DUMP_PHASORS:
            out = np.zeros((n_frames, inf["M"], inf["K_bins"], 2), dtype=np.float32)
        elif what == DUMP_Z:
            out = np.zeros((n_frames, 2 * inf["D"]), dtype=np.float32)
        elif what == DUMP_CLASS_REP:
            out = np.zeros(inf["Q_classes"], dtype=np.int32)
        elif what == DUMP_POWER:
            out = np.zeros((n_frames, inf["Q_classes"]), dtype=np.float32)
        else:
            out = np.zeros(n_frames, dtype=np.uint64)
        _check(lib.svdphat_debug_dump(self._h, what, n_frames, out.ctypes.data, out.nbytes), "debug_dump")
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib.svdphat_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
