"""Dev check of the narrow last frame tile of the pair SRP GEMM: cfg3 SRP DOAs of the default plan (CTA pairs, fold,
last tile N = 32) against the 1-CTA unfolded kernel (an independent code path) on all 10^4 frames, and the last 16
frames against a 16-frame call (split-K path)."""
import numpy as np
import torch

import paper_1811_11785_b200 as S
from workloads import make

w = make(3)
F = w.n_frames
a = torch.from_numpy(w.audio).cuda()
st = torch.cuda.current_stream().cuda_stream
out = {}
for name, opt in (("pair", 0), ("one_cta", S.OPT_ONE_CTA_SRP | S.OPT_NO_SRP_FOLD)):
    plan = S.Plan(w.mics, w.points, w.fs, w.c, w.N, w.hop, w.field, delta=w.delta, methods=("srp",), max_frames=F,
                  options=opt)
    doa = torch.empty(F, dtype=torch.int32, device="cuda")
    sc = torch.empty(F, dtype=torch.float32, device="cuda")
    plan.localize("srp", a, F, w.channel_stride, w.frame_stride, doa, sc, st)
    torch.cuda.synchronize()
    out[name] = (doa.cpu().numpy(), sc.cpu().numpy())
    if name == "pair":
        d2 = torch.empty(16, dtype=torch.int32, device="cuda")
        s2 = torch.empty(16, dtype=torch.float32, device="cuda")
        plan.localize("srp", a.data_ptr() + 4 * (F - 16) * w.frame_stride, 16, w.channel_stride, w.frame_stride, d2, s2, st)
        torch.cuda.synchronize()
        out["tail16"] = (d2.cpu().numpy(), s2.cpu().numpy())
    plan.close()
same = out["pair"][0] == out["one_cta"][0]
print("pair vs one_cta: agree %.5f (%d differ), last 32 frames agree %d/32, max |score diff| %.3g"
      % (same.mean(), (~same).sum(), same[-32:].sum(), np.abs(out["pair"][1] - out["one_cta"][1]).max()))
print("last 16 frames vs 16-frame call: %d/16 equal" % (out["pair"][0][-16:] == out["tail16"][0]).sum())
