"""Small driver for ncu: cfg3 (or argv[1]) plan, one warm-up and one profiled localize (argv[2]: both|srp|svd)."""
import sys

import torch

import paper_1811_11785_b200 as S
from workloads import make

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
METHOD = sys.argv[2] if len(sys.argv) > 2 else "both"
w = make(cfg)
plan = S.Plan(w.mics, w.points, w.fs, w.c, w.N, w.hop, w.field, delta=w.delta, methods=("srp", "svd"),
              max_frames=w.frames_per_call)
a = torch.from_numpy(w.audio).cuda()
F = w.frames_per_call
doa = torch.empty(2 * F, dtype=torch.int32, device="cuda")
sc = torch.empty(2 * F, dtype=torch.float32, device="cuda")
for _ in range(2):
    plan.localize(METHOD, a, F, w.channel_stride, w.frame_stride, doa, sc, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", plan.info()["D"])
