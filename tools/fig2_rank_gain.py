"""NEXT-2: Fig. 2b/2c of the paper (rank K and gain Q/K vs delta) from the device float64 setup.

Table 1 parameters + Table 2 arrays (tests/golden/), icosphere level 4 (Q = 2562); one plan per array, sigma^2 via
svdphat_plan_sigma2, eq. 11 applied for each delta.  Writes CSV rows geometry,delta,K,gain (needs a GPU).
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1811_11785_b200 as S  # noqa: E402
from workloads import geometry as G  # noqa: E402

gold = os.path.join(ROOT, "tests", "golden")
t1 = json.load(open(os.path.join(gold, "paper_table1.json")))
arrays = json.load(open(os.path.join(gold, "paper_table2_cm.json")))
grid = G.icosphere(4)
out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01", "fig2bc_rank_gain.csv")
rows = ["geometry,delta,K,gain"]
for name in ("1d", "2d", "3d"):
    mics = np.asarray(arrays[name], dtype=np.float64) / 100.0
    plan = S.Plan(mics, grid, t1["fs"], t1["c"], t1["N"], t1["hop"], "far", delta=1e-5, methods=("svd",),
                  max_frames=16)
    info = plan.info()
    s2 = plan.sigma2(info["Q_classes"])
    csum = np.cumsum(s2)
    for delta in (1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6):
        K = int(np.nonzero(csum >= (1 - delta) * info["trace_WWH"])[0][0]) + 1
        rows.append(f"{name},{delta:g},{K},{t1['Q'] / K:.1f}")
    plan.close()
open(out, "w").write("\n".join(rows) + "\n")
print("\n".join(rows))
