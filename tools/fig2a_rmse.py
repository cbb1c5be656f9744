"""NEXT-2: Fig. 2a of the paper (Delta RMSE = RMSE(SVD-PHAT) - RMSE(SRP-PHAT) vs delta) through
the GPU path, on synthetic scenes that stand in for the paper's TIMIT speech in image-method rooms (not
available): per configuration one white-Gaussian plane wave from a seeded uniform direction s_0, SNR ~ U[0, 30] dB
(P:360), frames of Table 1 (N = 256, fs = 16 kHz), Table 2 arrays, icosphere grid Q = 2562.  Per configuration the
energy-weighted RMSE of eq. results_rmse (oracle/rmse.py: f_1 / f_2 / f_3, test infrastructure) of each method's
(q_bar, Y_q_bar) over the frames; the CSV gives the mean over configurations.

  python tools/fig2a_rmse.py [n_conf=300] [frames=32] [out.csv]   (needs a GPU)
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1811_11785_b200 as S  # noqa: E402
from oracle import rmse as R  # noqa: E402
from workloads import geometry as G  # noqa: E402
from workloads import scenes as SC  # noqa: E402

DELTAS = (1e-1, 1e-2, 1e-3, 1e-4, 1e-5, 1e-6)
ALPHA = {"1d": 1, "2d": 2, "3d": 3}


def scenes(mics, n_conf, frames, seed, fs, c, N):
    """(audio (n_conf*frames, M, N) float32, s0 (n_conf, 3)): one direction and SNR per configuration."""
    rng = np.random.default_rng(seed)
    s0 = rng.standard_normal((n_conf, 3))
    s0 /= np.linalg.norm(s0, axis=1, keepdims=True)
    snr = rng.uniform(0.0, 30.0, n_conf)
    audio = SC.plane_wave_frames(rng, mics, fs, c, N, np.repeat(s0, frames, axis=0), np.repeat(snr, frames))
    return audio, s0


def localize(plan, audio, method):
    B, M, N = audio.shape
    d = torch.from_numpy(np.ascontiguousarray(audio)).cuda()
    doa = torch.empty(2 * B if method == "both" else B, dtype=torch.int32, device="cuda")
    sc = torch.empty_like(doa, dtype=torch.float32)
    plan.localize(method, d, B, N, M * N, doa, sc, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return doa.cpu().numpy(), sc.cpu().numpy()


def rmse_per_conf(alpha, grid, q, Y, s0, frames):
    return np.array([R.rmse_from_indices(alpha, grid, q[i * frames:(i + 1) * frames], Y[i * frames:(i + 1) * frames],
                                         s0[i]) for i in range(s0.shape[0])])


def main():
    n_conf = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 32
    out = sys.argv[3] if len(sys.argv) > 3 else os.path.join(ROOT, "profiles", "r02", "fig2a_delta_rmse.csv")
    t1 = json.load(open(os.path.join(ROOT, "tests", "golden", "paper_table1.json")))
    grid = G.icosphere(4)
    rows = ["geometry,delta,K,rmse_srp,rmse_svd,delta_rmse,delta_rmse_p90,n_conf,frames"]
    for gi, name in enumerate(("1d", "2d", "3d")):
        mics = G.paper_array(name)
        audio, s0 = scenes(mics, n_conf, frames, 4100 + gi, t1["fs"], t1["c"], t1["N"])
        for delta in DELTAS:
            plan = S.Plan(mics, grid, t1["fs"], t1["c"], t1["N"], t1["hop"], "far", delta=delta,
                          methods=("srp", "svd"), max_frames=audio.shape[0])
            q, Y = localize(plan, audio, "both")
            B = audio.shape[0]
            r_srp = rmse_per_conf(ALPHA[name], grid, q[:B], Y[:B], s0, frames)
            r_svd = rmse_per_conf(ALPHA[name], grid, q[B:], Y[B:], s0, frames)
            d = r_svd - r_srp
            ok = np.isfinite(d)
            rows.append(f"{name},{delta:g},{plan.info()['D']},{np.nanmean(r_srp):.5f},{np.nanmean(r_svd):.5f},"
                        f"{np.mean(d[ok]):.5f},{np.percentile(d[ok], 90):.5f},{n_conf},{frames}")
            print(rows[-1], flush=True)
            plan.close()
    os.makedirs(os.path.dirname(out), exist_ok=True)
    open(out, "w").write("\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
