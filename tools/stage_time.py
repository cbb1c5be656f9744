"""Per-stage device times (the library's profile events) of localize calls: python tools/stage_time.py CFG METHOD [N]
(dev tool; bench.py is the contract)."""
import sys

import numpy as np
import torch

import paper_1811_11785_b200 as S
from workloads import make

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
method = sys.argv[2] if len(sys.argv) > 2 else "svd"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 10
w = make(cfg)
plan = S.Plan(w.mics, w.points, w.fs, w.c, w.N, w.hop, w.field, delta=w.delta, methods=("srp", "svd"),
              max_frames=w.frames_per_call)
audio = torch.from_numpy(w.audio).cuda()
F = w.frames_per_call
k = 2 if method == "both" else 1
doa = torch.zeros(k * F, dtype=torch.int32, device="cuda")
sc = torch.zeros(k * F, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    plan.localize(method, audio, F, w.channel_stride, w.frame_stride, doa, sc, st)
torch.cuda.synchronize()
plan.profile_begin(16 * n)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    plan.localize(method, audio, F, w.channel_stride, w.frame_stride, doa, sc, st)
e1.record()
torch.cuda.synchronize()
prof = plan.profile_end()
ms = e0.elapsed_time(e1) / n
stages = {}
for name, t in prof:
    stages.setdefault(name, []).append(t)
print(f"cfg{cfg} {method}: {ms:.3f} ms/call = {F / ms * 1e3:.4g} frames/s  D={plan.info()['D']}  " +
      "  ".join(f"{k}={np.mean(v):.3f}" for k, v in stages.items()), flush=True)
