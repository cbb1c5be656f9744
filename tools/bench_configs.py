"""Frames/s of SRP-PHAT, SVD-PHAT and both on all five BASELINE.json configs (device-resident inputs, CUDA-event
timing on the launching stream), plus per-call latency for cfg5's 256-frame streaming calls.  One JSON line per
config.  bench.py remains the driver contract (cfg3); this is the per-config table of DESIGN.md.

  python tools/bench_configs.py [cfg ...]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1811_11785_b200 as S  # noqa: E402
from workloads import make  # noqa: E402


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(cfg):
    t = time.time()
    w = make(cfg)
    gen = time.time() - t
    per = w.frames_per_call
    plan = S.Plan(w.mics, w.points, w.fs, w.c, w.N, w.hop, w.field, delta=w.delta, methods=("srp", "svd"),
                  max_frames=per)
    info = plan.info()
    audio = torch.from_numpy(w.audio).cuda()
    d = torch.empty(2 * per, dtype=torch.int32, device="cuda")
    sc = torch.empty(2 * per, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    calls = [(c0, min(per, w.n_frames - c0)) for c0 in range(0, w.n_frames, per)]

    def all_calls(method):
        def f():
            for c0, n in calls:
                plan.localize(method, audio.data_ptr() + 4 * c0 * w.frame_stride, n, w.channel_stride,
                              w.frame_stride, d, sc, st)
        return f
    reps = 3 if w.n_frames >= 10_000 else 10
    out = {"cfg": cfg, "name": w.name, "M": w.M, "N": w.N, "Q": w.Q, "Q_classes": info["Q_classes"], "D": info["D"],
           "frames": w.n_frames, "frames_per_call": per, "calls": len(calls), "setup_s": round(info["setup_seconds"], 2),
           "gen_s": round(gen, 1)}
    # SVD first (as bench.py): right after the SRP GEMMs of the large configs the board sits at its power cap and every
    # kernel runs slower for a while, a state an SVD-only caller never sees
    for m in ("svd", "srp", "both"):
        ms = timed(all_calls(m), reps if m != "svd" else max(reps, 10))
        out[f"{m}_fps"] = w.n_frames / (ms / 1e3)
        out[f"{m}_ms_total"] = ms
    if len(calls) > 1:                                   # per-call latency (cfg5): each call timed alone
        lat = []
        for c0, n in calls[:200]:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.localize("both", audio.data_ptr() + 4 * c0 * w.frame_stride, n, w.channel_stride, w.frame_stride,
                          d, sc, st)
            e1.record()
            torch.cuda.synchronize()
            lat.append(e0.elapsed_time(e1))
        out["call_latency_ms_p50"] = float(np.percentile(lat, 50))
        out["call_latency_ms_p99"] = float(np.percentile(lat, 99))
        # the same call captured once as a CUDA graph and replayed (streaming deployment: new audio is written
        # into a fixed device window before each replay)
        n = calls[0][1]
        s2 = torch.cuda.Stream()
        src = audio.clone()
        with torch.cuda.stream(s2):
            plan.localize("both", src, n, w.channel_stride, w.frame_stride, d, sc, s2.cuda_stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s2):
            plan.localize("both", src, n, w.channel_stride, w.frame_stride, d, sc, s2.cuda_stream)
        glat = []
        for _ in range(200):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            glat.append(e0.elapsed_time(e1))
        out["call_latency_graph_ms_p50"] = float(np.percentile(glat, 50))
        out["call_latency_graph_ms_p99"] = float(np.percentile(glat, 99))
    plan.close()
    return out


if __name__ == "__main__":
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
    for c in cfgs:
        print(json.dumps(run(c)), flush=True)
