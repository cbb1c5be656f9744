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
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                for line in out.stdout.strip().splitlines():
                    self.rows.append([x.strip() for x in line.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


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


def cpu_baseline(w, n_frames: int) -> dict:
    """The float64 oracle, as it stands, on a bounded sample of the same workload (rank 0, N=1 only)."""
    from oracle import srpphat as srp  # test infrastructure; only this leg of bench.py executes it
    cores = len(os.sched_getaffinity(0))
    idx = np.linspace(0, w.n_frames - 1, n_frames).astype(int)
    t0 = time.perf_counter()
    fr = np.stack([w.audio[i].astype(np.float64) for i in idx]) if w.layout == "framed" else \
        srp.extract_frames(w.audio, w.n_frames, w.M, w.N, w.channel_stride, w.frame_stride)[idx]
    x = srp.frames_to_x(fr)
    tau = srp.tdoa(w.mics, w.points, w.fs, w.c, w.field)
    srp.srp_localize(tau, x, w.N)
    dt = time.perf_counter() - t0
    return {"value": n_frames / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": (f"{n_frames} cfg{w.cfg} frames (evenly spaced) through the float64 oracle's online SRP-PHAT "
                       "path: direct-DFT STFT, explicit PHAT cross-spectra, Y=Re{WX} with W regenerated in "
                       "256-row chunks, tie-aware argmax; SVD-PHAT online omitted (the oracle's float64 offline "
                       "SVD of the cfg3 W alone takes minutes); numpy/OpenBLAS threads = host cores"),
            "seconds": dt}


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


def run_reference(a) -> None:
    """--impl reference: the oracle (the deliberately slow CPU program) on the box's host cores, same metric."""
    dist, rank, ws, local = _dist()
    if rank != 0:
        return
    from workloads import make
    w = make(a.cfg)
    per = 32  # frames per step: every oracle pass regenerates the whole W (~13 s at cfg3), so 32 frames cost ~2 frames
    for _ in range(a.warmup):
        cpu_baseline(w, per)
    t = []
    for _ in range(a.steps):
        t.append(cpu_baseline(w, per)["seconds"])
    sec = float(np.sum(t))
    v = per * a.steps / sec
    cores = len(os.sched_getaffinity(0))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * sec / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg{a.cfg}", "frames_per_step": per},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{per} cfg{a.cfg} frames per step through the oracle SRP-PHAT path (W regenerated per step)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    a = _args()
    if a.impl == "reference":
        run_reference(a)
        return
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
    ms_step, value = aggregate(e0.elapsed_time(e1) / a.steps, F, dist, dev)

    # per-stage averages inside the timed region
    stages: dict[str, list[float]] = {}
    for name, ms in prof:
        stages.setdefault(name, []).append(ms)
    stage_ms = {k: float(np.mean(v)) for k, v in stages.items()}
    launches = len(prof)

    # ---------------------------------------------------------------- per-method throughput (same protocol)
    def timed(method, n):
        for _ in range(2):
            step(method)
        torch.cuda.synchronize(dev)
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(stream)
        for _ in range(n):
            step(method)
        x1.record(stream)
        torch.cuda.synchronize(dev)
        return x0.elapsed_time(x1) / n
    srp_ms = timed("srp", max(3, a.steps // 2))
    # the SVD chain alone, with its stage events: inside the "both" step the projection shares the SMs with the
    # SRP GEMM, so its own roofline is measured here
    plan.profile_begin(8 * max(3, a.steps // 2) + 16)
    svd_ms = timed("svd", max(3, a.steps // 2))
    svd_stages: dict[str, list[float]] = {}
    for name, ms in plan.profile_end():
        svd_stages.setdefault(name, []).append(ms)
    svd_stage_ms = {k: float(np.mean(v)) for k, v in svd_stages.items()}

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
    e2e_steps = max(4, a.steps // 2)
    barrier()
    t0 = time.perf_counter()
    last = None
    for _ in range(e2e_steps):
        last = submit()
    plan.wait(last)
    e2e_ms, e2e_value = aggregate(1e3 * (time.perf_counter() - t0) / e2e_steps, F, dist, dev)

    # ---------------------------------------------------------------- roofline of the dominant kernel
    pk = _peaks()
    gemm_ms = stage_ms.get("srp_gemm", float("nan"))
    # algorithmic flops of the SRP GEMM as executed: 4 flops per (row, PK element) per frame over the plan's SRP rows
    # (SURVEY §8d counts 4·Q·PK; twin classes and the antipodal fold, R11/R22, compute every Q row's
    # Re{W_q X} from srp_rows rows, so the fraction is graded on srp_rows and stays <= 1)
    flops = 4.0 * info["srp_rows"] * info["PK"] * F
    achieved = flops / (gemm_ms / 1e3) / 1e12
    peak = pk["tensor_sustained"]
    traffic = _ncu_traffic().get("srp_gemm_dram_bytes_per_launch")
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "kernel": "srp_gemm (gemm2_kernel<16,4,0,fold>, CTA pairs)",
            "flops_basis": f"4*srp_rows*PK*F, srp_rows={info['srp_rows']} (Q={info['Q']}, antipodal fold)",
            "flops_per_launch": flops, "peak_src": pk["src"] + " bf16_tflops_sustained (fp16 = bf16 rate)",
            # the sustained figure is a cuBLAS run under the same 1 kW power cap; the burst one bounds the clock
            "peak_burst": pk["tensor_burst"], "frac_burst": achieved / pk["tensor_burst"]}
    proj_ms = svd_stage_ms.get("svd_proj", float("nan"))
    svd_flops = 4.0 * info["svd_rows"] * info["PK"] * F      # 8·D·PK (complex V) or 4·D·PK (real V, R22)
    roof_svd = {"kernel": "svd_proj (method=svd run)", "stage_ms": svd_stage_ms, "achieved_tflops": svd_flops / (proj_ms / 1e3) / 1e12,
                "frac_tensor": svd_flops / (proj_ms / 1e3) / 1e12 / peak,
                "bytes_per_launch": float(info["bytes_V"] + F * w.M * w.N * 4)}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": a.steps, "warmup": max(3, a.warmup),
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic",
        "config": {"workload": f"cfg{a.cfg}", "name": w.name, "frames_per_step": F, "M": w.M, "N": w.N,
                   "Q": info["Q"], "D": info["D"], "delta": w.delta, "methods": "SRP-PHAT+SVD-PHAT",
                   "l2": "inputs larger than L2 (audio 655 MB, W 2.57 GB per step)", "parallelism": f"frames x{ws}"},
        "srp_fps": F * ws / (srp_ms / 1e3), "svd_fps": F * ws / (svd_ms / 1e3),
        "stage_ms": stage_ms, "gpu_launches": launches,
        "roofline": roof, "roofline_svd": roof_svd,
        "clocks": clk.summary(),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(w.audio.nbytes),
                "d2h_bytes_per_step": int(2 * F * 8), "api": "svdphat_submit_host/svdphat_wait (2 in flight)",
                "steps": e2e_steps},
        "setup_seconds": info["setup_seconds"],
    }
    if rank == 0 and ws == 1 and not a.no_cpu_baseline:
        line["cpu_baseline"] = {k: v for k, v in cpu_baseline(w, a.cpu_frames).items() if k != "seconds"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    plan.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
