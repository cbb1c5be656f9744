"""bench.py — frames/s of the SVD-PHAT + SRP-PHAT per-frame localisation hot path on B200.

Workload (BASELINE.json metric "frames/sec (SVD-PHAT & SRP-PHAT) at M=16, Q=10242"): configs[2] (cfg3): the
16-mic two-ring array, N=1024, Q=10242 far-field grid, a batch of 10^4 seeded synthetic frames (float32, 655 MB,
larger than L2).  One step = one svdphat_localize(method=BOTH) over the batch: STFT+PHAT once, SRP-PHAT (eqs. 5-9)
and SVD-PHAT (Alg. 1 online) for every frame, outputs (DOA index, Y_q) for both methods.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--cfg 3]

N>1: launch with torchrun (one process per GPU); each rank localises its own 10^4-frame batch (weak scaling, no
data-path collective: frames are independent); time = max over ranks of device time.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
METRIC = "frames/sec (SVD-PHAT & SRP-PHAT) at M=16, Q=10242; % of HBM/tensor roofline"
UNIT = "frames/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cfg", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-frames", type=int, default=32)
    return ap.parse_args()


# ------------------------------------------------------------------------------------------------ clocks
def _nvml_index(cuda_index: int) -> int:
    """NVML numbers every GPU of the node; CUDA only the visible ones."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [v.strip() for v in vis.split(",") if v.strip()]
    if ids and all(v.isdigit() for v in ids) and cuda_index < len(ids):
        return int(ids[cuda_index])
    return cuda_index


class ClockSampler:
    """SM clock, power and clock-event (throttle) reasons sampled through NVML every 10 ms during the timed region
    (nvidia-smi every 200 ms if NVML is unavailable)."""
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device_index: int, period_s: float = 0.01):
        self.dev = _nvml_index(device_index)
        self.period = period_s
        self.sm: list[float] = []
        self.power: list[float] = []
        self.reasons: set[str] = set()
        self.sm_max = None
        self.src = "nvml"
        self._nv = None
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _nvml_open(self) -> bool:
        """NVML is initialised here, on the caller's thread, BEFORE the timed region (inside the sampling thread the
        import + nvmlInit took longer than a 0.1 s region when the process is pinned to few cores: 0 samples)."""
        try:
            import pynvml as nv
            nv.nvmlInit()
            self._nv = nv
            self._h = nv.nvmlDeviceGetHandleByIndex(self.dev)
            self.sm_max = float(nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM))
            self._bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                          nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
            return True
        except Exception:
            self._nv = None
            return False

    def _sample_nvml(self):
        nv, h = self._nv, self._h
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
        self.power.append(nv.nvmlDeviceGetPowerUsage(h) / 1e3)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        self.reasons.update(n for n, b in zip(self.NAMES, self._bits) if r & b)

    def _run_nvml(self):
        while not self._stop.is_set():
            self._sample_nvml()
            self._stop.wait(self.period)

    def _run_smi(self):
        self.src = "nvidia-smi"
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                r = [x.strip() for x in out.stdout.strip().split(",")]
                self.sm.append(float(r[0]))
                self.sm_max = float(r[1])
                self.power.append(float(r[2]))
                self.reasons.update(n for n, v in zip(self.NAMES, r[3:7]) if v == "Active")
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        if self._nv is not None:
            try:
                self._run_nvml()
                return
            except Exception:
                pass
        self._run_smi()

    def __enter__(self):
        self._nvml_open()
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if self._nv is not None:
            try:
                if not self.sm:
                    self._sample_nvml()       # never leave the line without a reading
                self._nv.nvmlShutdown()
            except Exception:
                pass

    def summary(self) -> dict:
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.sm_max, "sm_min_mhz": min(self.sm),
                "power_w_median": float(np.median(self.power)) if self.power else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "period_ms": 1e3 * self.period,
                "src": self.src}


# ------------------------------------------------------------------------------------------------ helpers
def _peaks() -> dict:
    p = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"tensor_burst": d.get("bf16_tflops"), "tensor_sustained": d.get("bf16_tflops_sustained"),
                "hbm": d.get("hbm_gbs"), "src": "measured (MEASURED_PEAKS.json)"}
    return {"tensor_burst": 1590.0, "tensor_sustained": 1400.0, "hbm": 6650.0,
            "src": "fallback (B200_PROFILING.md)"}


def _ncu_traffic() -> dict:
    p = os.path.join(HERE, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def _oracle_frames(w, idx):
    from oracle import srpphat as srp
    if w.layout == "framed":
        return np.stack([w.audio[i].astype(np.float64) for i in idx])
    return srp.extract_frames(w.audio, w.n_frames, w.M, w.N, w.channel_stride, w.frame_stride)[idx]


def oracle_factors(w):
    """Alg. 1 offline steps 1-3 by the oracle (untimed setup of the SVD leg): returns (tau, factors, seconds)."""
    from oracle import srpphat as srp
    from oracle import svdphat as svd
    t = time.perf_counter()
    tau = srp.tdoa(w.mics, w.points, w.fs, w.c, w.field)
    fac = svd.svd_factors(tau, w.N, w.delta, n_top=1024 if tau.shape[0] > 4096 else None)
    return tau, fac, time.perf_counter() - t


def cpu_baseline(w, n_frames: int, svd_leg: bool = True, factors=None) -> dict:
    """The float64 oracle, as it stands, on a bounded sample of the same workload (rank 0, N=1 only).

    SRP leg (timed): direct-DFT STFT, explicit PHAT cross-spectra (eq. 3), Y = Re{WX} with W regenerated in row
    chunks (eq. 9), tie-aware argmax (eq. 6).  SVD leg: the offline factors (Alg. 1 offline 1-3: one pass over W for
    the Gram matrix W W^H, top-subset eigh, eq. 11 rank rule, V_D = W^H U_D S_D^-1) are computed untimed
    (`svd_setup_seconds`); timed is Alg. 1 online: STFT + X, Z = V^H x (eq. 12), brute-force nearest normalised
    row (eq. 15), Y_q from the row of W (step 4).  `value` = frames / (SRP leg + SVD leg), the same both-methods
    metric as the GPU line.  The oracle's DOAs and its power maps for the same frames are returned for the
    bench line's parity statistics."""
    from oracle import srpphat as srp  # test infrastructure; only this leg of bench.py executes it
    from oracle import svdphat as svd
    cores = len(os.sched_getaffinity(0))
    idx = np.linspace(0, w.n_frames - 1, n_frames).astype(int)
    tau = srp.tdoa(w.mics, w.points, w.fs, w.c, w.field)
    t0 = time.perf_counter()
    x = srp.frames_to_x(_oracle_frames(w, idx))
    Y = srp.srp_energy(tau, x, w.N)
    q_srp, _ = srp.argmax_tie(Y)
    q_srp[srp.degenerate(x)] = -1
    dt_srp = time.perf_counter() - t0
    out = {"unit": UNIT, "cores": cores, "kind": "oracle", "frames": idx, "q_srp": q_srp, "Y_srp": Y,
           "srp_seconds": dt_srp}
    sample = (f"{n_frames} cfg{w.cfg} frames (evenly spaced) through the float64 oracle: SRP-PHAT online "
              "(direct-DFT STFT, explicit PHAT cross-spectra, Y=Re{WX} with W regenerated in 256-row chunks, "
              "tie-aware argmax)")
    dt = dt_srp
    if svd_leg:
        _, fac, out["svd_setup_seconds"] = factors if factors is not None else oracle_factors(w)
        t2 = time.perf_counter()
        x2 = srp.frames_to_x(_oracle_frames(w, idx))
        q_svd, _ = svd.svd_localize(fac, tau, x2, w.N)
        dt_svd = time.perf_counter() - t2
        dt += dt_svd
        Z = svd.project(fac["V"], x)
        nz = np.linalg.norm(Z, axis=1, keepdims=True)
        out.update(q_svd=q_svd, S_svd=svd.search_scores(fac["Rhat"], Z / np.where(nz > 0, nz, 1.0)),
                   svd_seconds=dt_svd, D=fac["D"])
        sample += (" + SVD-PHAT online (direct-DFT STFT, X, Z = V^H x, brute-force nearest normalised row, Y_q "
                   f"from the W row; offline factors untimed, D={fac['D']})")
    out.update(value=n_frames / dt, seconds=dt,
               sample=sample + "; numpy/OpenBLAS threads = host cores; value = frames / (SRP leg + SVD leg)")
    return out


def parity_stats(q_gpu: np.ndarray, q_or: np.ndarray, P_or: np.ndarray, tol: float = 2e-3) -> dict:
    """GPU DOAs of the timed run vs the oracle's on the cpu_baseline frames (north_star rule: a disagreement must be
    a near-tie of the oracle's own power, gap <= tol * |P_best|)."""
    agree = q_gpu == q_or
    ties = 0
    for f in np.nonzero(~agree)[0]:
        g, o = int(q_gpu[f]), int(q_or[f])
        if 0 <= g < P_or.shape[1] and o >= 0 and P_or[f, o] - P_or[f, g] <= tol * abs(P_or[f, o]):
            ties += 1
    return {"frames": int(len(q_or)), "agree": float(np.mean(agree)) if len(q_or) else 1.0,
            "disagree_near_tie": ties, "disagree_not_tie": int(np.sum(~agree)) - ties}


def aggregate(ms_local: float, frames_local: int, dist=None, device=None) -> tuple[float, float]:
    """Weak scaling, no data-path collective: step time = MAX over ranks of each rank's device time; value = all
    ranks' frames / that time.  Returns (ms_per_step, frames_per_second)."""
    ms, fr = ms_local, float(frames_local)
    if dist is not None and dist.is_initialized():
        import torch
        t = torch.tensor([ms, fr], dtype=torch.float64, device=device)
        m = t.clone()
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        ms, fr = float(m[0]), float(t[1])
    return ms, fr / (ms / 1e3)


def frame_shard(n_total: int, rank: int, ws: int) -> tuple[int, int]:
    """Contiguous, balanced shard of the global frame index space owned by `rank`: (first frame, count).  Frames are
    independent, so the shards need no data-path collective."""
    base, rem = divmod(n_total, ws)
    return rank * base + min(rank, rem), base + (1 if rank < rem else 0)


def gather_frames(local, n_total: int, dist=None):
    """Per-frame results of every rank's shard, concatenated in global frame order (all_gather of the shards, padded
    to the largest shard; 8 B per frame, outside any timed region).  `local` is a 1-D tensor on the rank's device."""
    if dist is None or not dist.is_initialized():
        return local
    import torch
    ws = dist.get_world_size()
    n_max = frame_shard(n_total, 0, ws)[1]
    buf = torch.zeros(n_max, dtype=local.dtype, device=local.device)
    buf[:local.numel()] = local
    parts = [torch.empty_like(buf) for _ in range(ws)]
    dist.all_gather(parts, buf)
    return torch.cat([parts[r][:frame_shard(n_total, r, ws)[1]] for r in range(ws)])


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws == 1:
        return None, 0, 1, 0
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    return dist, rank, ws, local


def workload_config(cfg: int, w, Q: int, D: int, ws: int) -> dict:
    """`config` of the JSON line: names the workload; identical for both arms (the reference arm times a bounded
    sample of it per step and says so in cpu_baseline.sample)."""
    return {"workload": f"cfg{cfg}", "name": w.name, "frames_per_step": w.n_frames, "M": w.M, "N": w.N,
            "Q": int(Q), "D": int(D), "delta": w.delta, "methods": "SRP-PHAT+SVD-PHAT",
            "l2": "inputs larger than L2 (audio 655 MB, W 2.57 GB per step)", "parallelism": f"frames x{ws}"}


def run_reference(a) -> None:
    """--impl reference: the oracle (the deliberately slow CPU program) on the box's host cores, same metric."""
    dist, rank, ws, local = _dist()
    if rank != 0:
        return
    from workloads import make
    w = make(a.cfg)
    per = 32  # frames per step: every oracle pass regenerates the whole W (~13 s at cfg3), so 32 frames cost ~2 frames
    factors = oracle_factors(w)   # Alg. 1 offline (setup, untimed, once)
    for _ in range(a.warmup):
        cpu_baseline(w, per, factors=factors)
    t = []
    for _ in range(a.steps):
        t.append(cpu_baseline(w, per, factors=factors)["seconds"])
    sec = float(np.sum(t))
    v = per * a.steps / sec
    cores = len(os.sched_getaffinity(0))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * sec / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(a.cfg, w, len(w.points), factors[1]["D"], ws), "reference_frames_per_step": per,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": (f"{per} cfg{a.cfg} frames per step through the oracle's SRP-PHAT online path "
                                        "(W regenerated per step) and SVD-PHAT online path (factors computed once, "
                                        f"untimed, {factors[2]:.0f} s)")},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _p16_bytes(info, w, F) -> float:
    """Algorithmic bytes of the per-frame phasor records: M mics x K bins x FP16 complex (DESIGN.md §6 P16)."""
    return float(w.M * info["K_bins"] * 4 * F)


def roofline(info, w, F, stage_ms, clocks) -> dict:
    """Roofline of the dominant kernel of the timed step (the SRP stage: 80-90% of the step's kernel time, ncu launch list).

    Delay-and-sum SRP (das_kernel, NEXT-4): per (class, bin, frame) a_q[k] = sum_m e_m e^{j phi_qm} is M
    complex MACs = 8 M flops, so 8 Q_classes M K F algorithmic flops per launch; the kernel executes
    2 das_rows (2 das_me) K F_tiles on the tensor cores (rows and frames padded to 256, mics to 8/16/32).  Every
    accumulator element is also read back from TMEM once per bin for |a|^2 (the epilogue), reported per SM-clock.
    Eq. 9 GEMM (srp_gemm): 4 srp_rows PK F (SURVEY §8d's 4 Q PK per frame on the rows the GEMM executes, R11/R22).
    Peak: the measured burst dense FP16/BF16 rate (a kernel of a few ms timed inside a sub-second region)."""
    pk = _peaks()
    # the SRP stage: in a BOTH step the SVD chain runs on a low-priority stream beside it, so an SVD stage's event
    # time includes waiting for the SMs the SRP kernel holds and is not a kernel duration
    dom = next((k for k in ("srp_das", "srp_gemm") if k in stage_ms), max(stage_ms, key=stage_ms.get))
    ms = stage_ms[dom]
    F_exec = -(-F // 256) * 256
    traffic = _ncu_traffic()
    if dom == "srp_das":
        Qc, M, ME, Kb, R = info["Q_classes"], w.M, info["das_me"], info["K_bins"], info["das_rows"]
        flops = 8.0 * Qc * M * Kb * F
        executed = 2.0 * R * 2 * ME * Kb * F_exec
        kern, basis = "srp_das (das_kernel<%d>, CTA pairs)" % ME, f"8*Q_classes*M*K*F (Q_classes={Qc}, M={M}, K={Kb})"
        tmem_elems = float(R) * F_exec * Kb
        sm_hz = (clocks.get("sm_mhz") or 1965.0) * 1e6
        extra = {"epilogue_tmem_elems_per_launch": tmem_elems,
                 "epilogue_elems_per_clk_per_sm": tmem_elems / (ms / 1e3) / sm_hz / 148,
                 "epilogue_note": "accumulator elements read from TMEM (tcgen05.ld) and squared per bin; "
                                  "tools/microbench_tmem.cu measures ~100 elements/clk/SM for ld + FFMA2"}
        tkey = "srp_das_dram_bytes_per_launch"
    elif dom == "srp_gemm":
        flops = 4.0 * info["srp_rows"] * info["PK"] * F
        # executed: the W rows of the tiles the GEMM runs (BOTH calls skip the tail tile, whose rows ride in the SVD
        # projection) x the contraction the MMAs cover x 256-frame tiles.  The fold layout stores 128 unit slots per
        # bin chunk for 120 pairs (srp_gemm_k, what TMA streams), but the issuer skips the two empty K steps of each
        # chunk's last slab pair (kHalfPair, gemm_tc.cu), so the MMAs cover gemm_k = chunks x units x 8 halves
        rows_exec = info["srp_gemm_rows"] - (256 if info["srp_tail_rows"] > 0 else 0)
        executed = 2.0 * rows_exec * info["gemm_k"] * F_exec
        kern, basis = "srp_gemm (gemm2_kernel, CTA pairs)", f"4*srp_rows*PK*F, srp_rows={info['srp_rows']}"
        extra, tkey = {}, "srp_gemm_dram_bytes_per_launch"
    else:
        return {"bound": "tensor", "kernel": dom, "note": "dominant stage without a roofline model"}
    achieved = flops / (ms / 1e3) / 1e12
    peak = pk["tensor_burst"]
    out = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
           "traffic": traffic.get(tkey), "kernel": kern, "stage_ms": ms, "flops_basis": basis,
           "flops_per_launch": flops, "executed_mma_flops_per_launch": executed,
           "executed_over_algorithmic": executed / flops,
           "peak_src": pk["src"] + " bf16_tflops (burst; fp16 = bf16 rate)",
           "peak_sustained": pk["tensor_sustained"], "frac_sustained": achieved / pk["tensor_sustained"],
           "frac_executed": executed / (ms / 1e3) / 1e12 / peak}
    out.update(extra)
    return out


def roofline_svd(info, w, F, svd_ms, st) -> dict:
    """SVD-PHAT path (method=svd run): each kernel's ideal time max(flops / tensor peak, bytes / HBM peak) on
    algorithmic work, summed, against the measured path time.  STFT: audio read + phasor records written; projection
    Z = V^T x: 4 svd_rows PK F flops (real V, R22; 8 D PK with a complex V), V + records read; search Re{D^_q Z^}:
    4 Q D F flops; finalize: records read once; zsplit / rescore: O(F D) (counted as 0)."""
    pk = _peaks()
    tp, bw = pk["tensor_burst"] * 1e12, pk["hbm"] * 1e9
    p16 = _p16_bytes(info, w, F)
    audio = float(F * w.M * w.N * 4)
    ideal = {
        "stft_phat": (audio + p16) / bw,
        "svd_proj": max(4.0 * info["svd_rows"] * info["PK"] * F / tp, (info["bytes_V"] + p16) / bw),
        "svd_search": 4.0 * info["Q"] * info["D"] * F / tp,
        "finalize": p16 / bw,
    }
    ideal_ms = 1e3 * sum(ideal.values())
    proj_ms = st.get("svd_proj", float("nan"))
    proj_flops = 4.0 * info["svd_rows"] * info["PK"] * F
    return {"bound": "tensor+hbm (per kernel)", "path_ms": svd_ms, "ideal_ms": ideal_ms, "frac": ideal_ms / svd_ms,
            "ideal_ms_per_kernel": {k: 1e3 * v for k, v in ideal.items()}, "stage_ms": st,
            "proj_achieved_tflops": proj_flops / (proj_ms / 1e3) / 1e12,
            "proj_frac_tensor": proj_flops / (proj_ms / 1e3) / 1e12 / pk["tensor_burst"],
            "proj_bytes_per_launch": float(info["bytes_V"]) + p16,
            "peaks": {"tensor_tflops": pk["tensor_burst"], "hbm_gbs": pk["hbm"], "src": pk["src"]}}


def _factors_child(cfg, conn, cores):
    """Child process (forked before CUDA is initialised): the oracle's offline SVD factors for the cpu_baseline SVD
    leg, computed while the GPU legs run, on all host cores but the one left to the GPU driver thread."""
    if cores:
        os.sched_setaffinity(0, cores)
    from workloads import make
    tau, fac, sec = oracle_factors(make(cfg))
    conn.send((tau, {k: fac[k] for k in ("V", "Rhat", "D")}, sec))
    conn.close()


def main() -> None:
    a = _args()
    if a.impl == "reference":
        run_reference(a)
        return
    all_cores = sorted(os.sched_getaffinity(0))
    fac_proc = fac_conn = None
    if not a.no_cpu_baseline and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        fac_conn, child = ctx.Pipe(duplex=False)
        fac_proc = ctx.Process(target=_factors_child, args=(a.cfg, child, all_cores[2:] or all_cores), daemon=True)
        fac_proc.start()
        os.sched_setaffinity(0, all_cores[:2])     # the launch thread and the clock sampler
    import torch

    import paper_1811_11785_b200 as S
    from workloads import make

    dist, rank, ws, local = _dist()
    if dist is not None:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)

    w = make(a.cfg)
    if w.layout != "framed":
        raise SystemExit("bench.py times the framed batch configs (3, 4)")
    F = w.n_frames
    plan = S.Plan(w.mics, w.points, w.fs, w.c, w.N, w.hop, w.field, delta=w.delta, methods=("srp", "svd"),
                  max_frames=F, device=local)
    info = plan.info()
    audio = torch.from_numpy(w.audio).to(dev)
    doa = torch.empty(2 * F, dtype=torch.int32, device=dev)
    score = torch.empty(2 * F, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def step(method="both"):
        plan.localize(method, audio, F, w.channel_stride, w.frame_stride, doa, score, sh)

    def barrier():
        if dist is not None:
            dist.barrier()

    def timed(method, n, warm=3):
        for _ in range(warm):
            step(method)
        torch.cuda.synchronize(dev)
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        for _ in range(n):
            step(method)
        x1.record(stream)
        torch.cuda.synchronize(dev)
        return x0.elapsed_time(x1) / n

    # ---------------------------------------------------------------- SVD-PHAT alone (method=svd), with stage events
    # Timed before the SRP legs: inside the "both" step the SVD chain shares the SMs with the SRP GEMM, and right after
    # a run of SRP GEMMs the board sits at its power cap with the SM clock ~30% down for a while (r02: every SVD kernel
    # measured 1.23-1.33x slower there), which an SVD-only caller never sees.
    n_svd = max(20, 2 * a.steps)
    plan.profile_begin(8 * n_svd + 16)
    svd_ms = timed("svd", n_svd)
    svd_stages: dict[str, list[float]] = {}
    for name, ms in plan.profile_end():
        svd_stages.setdefault(name, []).append(ms)
    svd_stage_ms = {k: float(np.mean(v)) for k, v in svd_stages.items()}

    for _ in range(max(3, a.warmup)):
        step()
    torch.cuda.synchronize(dev)

    # ---------------------------------------------------------------- timed region (device time, CUDA events)
    plan.profile_begin(8 * a.steps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(a.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
    prof = plan.profile_end()
    q_last = doa.clone()          # DOAs of the last timed step (parity statistics against the oracle)
    ms_step, value = aggregate(e0.elapsed_time(e1) / a.steps, F, dist, dev)

    # per-stage averages inside the timed region
    stages: dict[str, list[float]] = {}
    for name, ms in prof:
        stages.setdefault(name, []).append(ms)
    stage_ms = {k: float(np.mean(v)) for k, v in stages.items()}
    launches = len(prof)

    # ---------------------------------------------------------------- SRP-PHAT alone (same protocol)
    srp_ms = timed("srp", max(3, a.steps // 2), warm=2)

    # ---------------------------------------------------------------- end to end through the host-buffer C-ABI
    # svdphat_submit_host: every step uploads its 655 MB of pinned float32 audio, localises and downloads the
    # (doa, score) results; two steps in flight, so step i+1's upload overlaps step i's kernels (serving pattern).
    h_audio = torch.from_numpy(w.audio).pin_memory()
    h_doa = torch.empty(2 * F, dtype=torch.int32).pin_memory()
    h_score = torch.empty(2 * F, dtype=torch.float32).pin_memory()
    n_elems = w.audio.size

    def submit():
        return plan.submit_host("both", h_audio, n_elems, F, w.channel_stride, w.frame_stride, h_doa, h_score, sh)
    plan.wait(submit())
    # a streaming pipeline: the first upload and the last step's kernels are not overlapped with anything, so the
    # fill/drain (one H2D + one compute) is amortised over at least 20 steps (5 steps reported 13.8 ms per step for
    # an 11.8 ms upload period)
    e2e_steps = max(20, a.steps)
    barrier()
    t0 = time.perf_counter()
    last = None
    for _ in range(e2e_steps):
        last = submit()
    plan.wait(last)
    e2e_ms, e2e_value = aggregate(1e3 * (time.perf_counter() - t0) / e2e_steps, F, dist, dev)

    # ---------------------------------------------------------------- roofline of the dominant kernel
    roof = roofline(info, w, F, stage_ms, clk.summary())
    roof_svd = roofline_svd(info, w, F, svd_ms, svd_stage_ms)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps, "warmup": max(3, a.warmup),
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic",
        "config": workload_config(a.cfg, w, info["Q"], info["D"], ws),
        "srp_fps": F * ws / (srp_ms / 1e3), "svd_fps": F * ws / (svd_ms / 1e3),
        "stage_ms": stage_ms, "gpu_launches": launches,
        "roofline": roof, "roofline_svd": roof_svd,
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(w.audio.nbytes),
                "d2h_bytes_per_step": int(2 * F * 8), "api": "svdphat_submit_host/svdphat_wait (2 in flight)",
                "steps": e2e_steps},
        "setup_seconds": info["setup_seconds"],
    }
    if fac_proc is not None:
        factors = fac_conn.recv()
        fac_proc.join()
        os.sched_setaffinity(0, all_cores)
        cb = cpu_baseline(w, a.cpu_frames, factors=factors)
        q_run = q_last.cpu().numpy()
        fr = cb["frames"]
        line["parity"] = {"srp": parity_stats(q_run[:F][fr], cb["q_srp"], cb["Y_srp"])}
        if "q_svd" in cb:
            line["parity"]["svd"] = parity_stats(q_run[F:][fr], cb["q_svd"], cb["S_svd"])
        line["parity"]["note"] = ("DOAs of the last timed localize(BOTH) vs the float64 oracle on the cpu_baseline "
                                  "frames; a disagreement counts as a near-tie if the oracle's power gap <= 2e-3")
        line["cpu_baseline"] = {k: (float(v) if isinstance(v, (np.floating,)) else v) for k, v in cb.items()
                                if k in ("value", "unit", "cores", "kind", "sample", "srp_seconds", "svd_seconds",
                                         "svd_setup_seconds", "D")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
