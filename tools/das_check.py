"""Delay-and-sum SRP (das.cu) vs eq. 9's GEMM on the same plan geometry: DOA agreement, score agreement, stage times,
and oracle parity on a frame sample.  python tools/das_check.py CFG [n_oracle_frames]  (dev tool)."""
import sys

import numpy as np
import torch

import paper_1811_11785_b200 as S
from oracle import srpphat as srp
from tests import _parity as PP
from workloads import make

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n_or = int(sys.argv[2]) if len(sys.argv) > 2 else 64
w = make(cfg)
F = w.frames_per_call
audio = torch.from_numpy(w.audio).cuda()
st = torch.cuda.current_stream().cuda_stream
res = {}
for name, opt in (("das", 0), ("w", S.OPT_NO_DAS)):
    plan = S.Plan(w.mics, w.points, w.fs, w.c, w.N, w.hop, w.field, delta=w.delta, methods=("srp",),
                  max_frames=F, options=opt)
    doa = torch.zeros(F, dtype=torch.int32, device="cuda")
    sc = torch.zeros(F, dtype=torch.float32, device="cuda")
    for _ in range(3):
        plan.localize("srp", audio, F, w.channel_stride, w.frame_stride, doa, sc, st)
    torch.cuda.synchronize()
    plan.profile_begin(256)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    n = 10
    for _ in range(n):
        plan.localize("srp", audio, F, w.channel_stride, w.frame_stride, doa, sc, st)
    e1.record()
    torch.cuda.synchronize()
    stages = {}
    for nm, t in plan.profile_end():
        stages.setdefault(nm, []).append(t)
    ms = e0.elapsed_time(e1) / n
    print(f"cfg{cfg} {name}: {ms:.3f} ms/call = {F / ms * 1e3:.4g} frames/s  " +
          "  ".join(f"{k}={np.mean(v):.3f}" for k, v in stages.items()), flush=True)
    res[name] = (doa.cpu().numpy(), sc.cpu().numpy())
    plan.close()
a, b = res["das"], res["w"]
agree = np.mean(a[0] == b[0])
rel = np.max(np.abs(a[1] - b[1]) / np.maximum(np.abs(b[1]), 1e-30))
print(f"das vs W GEMM: DOA agreement {agree:.5f} ({np.sum(a[0] != b[0])} of {F}), max score rel diff {rel:.2e}")
if n_or > 0:
    idx = np.linspace(0, F - 1, n_or).astype(int)
    tau = srp.tdoa(w.mics, w.points, w.fs, w.c, w.field)
    _, x = PP.oracle_inputs(w, idx)
    Y, Y_at = PP.srp_reference(tau, x, w.N)
    stt = PP.compare(a[0][idx], a[1][idx], Y, Y_at, f"cfg{cfg} das vs oracle")
    print("das vs oracle:", stt)
