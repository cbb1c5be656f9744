"""Dev A/B of SRP kernel variants (plan options) on one config: stage times and DOA agreement with the first
variant.  python tools/das_ab.py CFG  (bench.py is the contract)."""
import sys

import numpy as np
import torch

import paper_1811_11785_b200 as S
from workloads import make

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
method = sys.argv[2] if len(sys.argv) > 2 else "srp"
w = make(cfg)
F = w.frames_per_call
audio = torch.from_numpy(w.audio).cuda()
st = torch.cuda.current_stream().cuda_stream
ref = None
variants = [("das", 0), ("fold", S.OPT_DAS_FOLD), ("eq9", S.OPT_NO_DAS)]
for name, opt in variants:
    plan = S.Plan(w.mics, w.points, w.fs, w.c, w.N, w.hop, w.field, delta=w.delta, methods=("srp", "svd") if method == "both" else ("srp",), max_frames=F,
                  options=opt)
    doa = torch.zeros(2 * F, dtype=torch.int32, device="cuda")
    sc = torch.zeros(2 * F, dtype=torch.float32, device="cuda")
    for _ in range(3):
        plan.localize(method, audio, F, w.channel_stride, w.frame_stride, doa, sc, st)
    torch.cuda.synchronize()
    plan.profile_begin(256)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        plan.localize(method, audio, F, w.channel_stride, w.frame_stride, doa, sc, st)
    e1.record()
    torch.cuda.synchronize()
    stages = {}
    for n, t in plan.profile_end():
        stages.setdefault(n, []).append(t)
    q = doa.cpu().numpy()
    if ref is None:
        ref = q
    print(f"cfg{cfg} {method} {name:10s} {e0.elapsed_time(e1) / 10:7.3f} ms/call  agree {np.mean(q == ref):.4f}  " +
          "  ".join(f"{k}={np.mean(v):.3f}" for k, v in stages.items()), flush=True)
    plan.close()
