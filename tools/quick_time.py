"""Quick timing of the hot path on one config (dev tool; bench.py is the contract)."""
import sys
import time

import numpy as np
import torch

import paper_1811_11785_b200 as S
from workloads import make

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
frames = int(sys.argv[2]) if len(sys.argv) > 2 else None
methods = sys.argv[3].split(",") if len(sys.argv) > 3 else ["srp", "svd"]
t = time.time()
w = make(cfg, frames)
print(f"workload cfg{cfg}: {w.audio.shape} frames={w.n_frames} gen {time.time() - t:.1f}s", flush=True)
t = time.time()
plan = S.Plan(w.mics, w.points, w.fs, w.c, w.N, w.hop, w.field, delta=w.delta, methods=methods,
              max_frames=w.frames_per_call)
print(f"plan {time.time() - t:.1f}s", plan.info(), flush=True)
audio = torch.from_numpy(w.audio).cuda()
F = w.frames_per_call
doa = torch.zeros(F, dtype=torch.int32, device="cuda")
sc = torch.zeros(F, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for m in methods:
    for _ in range(2):
        plan.localize(m, audio, F, w.channel_stride, w.frame_stride, doa, sc, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    e0.record()
    for _ in range(n):
        plan.localize(m, audio, F, w.channel_stride, w.frame_stride, doa, sc, st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{m}: {ms:.3f} ms / {F} frames = {F / ms * 1e3:.4g} frames/s", flush=True)
    q = doa.cpu().numpy()
    if w.field == "far" and "u" in w.truth and cfg in (3, 4):
        ang = np.degrees(np.arccos(np.clip(np.sum(w.points[q] * w.truth["u"][:F], axis=1), -1, 1)))
        print(f"  median angular error vs truth {np.median(ang):.2f} deg")
