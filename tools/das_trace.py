"""Dev tool: latency trace of the folded delay-and-sum kernel (library built with -DDAS_TRACE by
tools/gpu_das_trace.sh).  Leader CTA of pair 0, per TMEM region step s: MMA issue (after its empty-barrier wait),
epilogue warp 2 wake (full barrier) and release (after its loads); clock64 cycles on that SM."""
import ctypes as C
import sys

import numpy as np
import torch

import paper_1811_11785_b200 as S
from paper_1811_11785_b200 import _lib
from workloads import make

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = make(cfg)
F = w.frames_per_call
plan = S.Plan(w.mics, w.points, w.fs, w.c, w.N, w.hop, w.field, delta=w.delta, methods=("srp",), max_frames=F,
              options=S.OPT_DAS | S.OPT_DAS_FOLD)
audio = torch.from_numpy(w.audio).cuda()
doa = torch.zeros(F, dtype=torch.int32, device="cuda")
sc = torch.zeros(F, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    plan.localize("srp", audio, F, w.channel_stride, w.frame_stride, doa, sc, st)
torch.cuda.synchronize()
buf = np.zeros((3, 8192), dtype=np.int64)
fn = _lib.lib.svdphat_dev_das_trace
fn.argtypes = [C.c_void_p, C.c_int]
assert fn(buf.ctypes.data, buf.size) == 0
t_iss, t_wake, t_rel = buf[0].astype(np.float64), buf[1].astype(np.float64), buf[2].astype(np.float64)
s = np.arange(200, 8000)
print("cfg", cfg, "per-region-step cycles (median, p10, p90):")
for name, v in (("issue -> epilogue wake (MMA + commit + wake)", t_wake[s] - t_iss[s]),
                ("wake -> release (loads)", t_rel[s] - t_wake[s]),
                ("release -> MMA reissue of that region (arrivals + wake)", t_iss[s + 4] - t_rel[s]),
                ("issue period (per region step)", t_iss[s + 1] - t_iss[s]),
                ("epilogue wake period", t_wake[s + 1] - t_wake[s])):
    print(f"  {name:58s} {np.median(v):8.0f} {np.percentile(v, 10):8.0f} {np.percentile(v, 90):8.0f}")
