"""CPU-side checks of the C-ABI boundary and the host logic (no GPU needed, no compute calls).

* libsvdphat.so builds for sm_100a, loads, and exports every function include/svdphat.h declares;
* argument validation happens before any device access (INVALID_ARG on CPU, UNSUPPORTED only for valid descs);
* frame counting (R3) and status strings;
* bench.py's multi-rank aggregation (max over ranks, sum of frames) under a world_size-2 gloo group.
"""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "svdphat.h")
LIB = os.path.join(ROOT, "paper_1811_11785_b200", "libsvdphat.so")


@pytest.fixture(scope="module")
def lib():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "paper_1811_11785_b200", "build.py")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    import paper_1811_11785_b200 as S
    return S


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(svdphat_\w+)\s*\(", src)))


def test_header_symbols_exported(lib):
    names = _declared()
    assert "svdphat_plan_create" in names and "svdphat_localize" in names and len(names) >= 12
    so = ctypes.CDLL(LIB)
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing
    nm = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", nm, flags=re.M), n          # extern "C": unmangled


def test_sass_is_tcgen05(lib):
    """The GEMMs compile to tcgen05 (UTCHMMA, incl. the CTA-pair form) fed by TMA (UTMALDG), not mma.sync."""
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and "UTCHMMA.2CTA" in out and "UTMALDG" in out and "LDTM" in out
    assert not re.search(r"\bHMMA\.", out)


def test_frame_count_and_status(lib):
    S = lib
    assert S.frame_count(32000, 512, 256) == 124
    assert S.frame_count(960000, 512, 256) == 3749
    assert S.frame_count(511, 512, 256) == 0
    assert S.frame_count(512, 512, 256) == 1
    assert S.frame_count(25_600_256, 512, 256) == 100_000
    assert S.lib.svdphat_status_str(0) == b"OK"
    assert S.lib.svdphat_status_str(1) == b"INVALID_ARG"


BAD = [
    dict(mics=np.zeros((1, 3))),                       # M < 2
    dict(mics=np.zeros((33, 3))),                      # M > 32
    dict(N=500),                                       # not a power of two
    dict(N=8),
    dict(hop=0), dict(hop=1025),
    dict(fs=0.0), dict(c=-1.0),
    dict(points=np.zeros((3, 3))),                     # zero far-field direction
    dict(points=np.array([[np.nan, 0, 1.0]])),
    dict(mics=np.array([[0, 0, 0], [np.inf, 0, 0]])),
    dict(delta=0.0), dict(delta=1.0),
    dict(methods=()),
    dict(max_frames=-1),
    dict(rank_D=-2),
    dict(options=128),                                 # unknown option bit
]


@pytest.mark.parametrize("bad", BAD)
def test_validation_before_device(lib, bad):
    S = lib
    kw = dict(mics=np.array([[0.05, 0, 0], [-0.05, 0, 0], [0, 0.05, 0]]), points=np.eye(3), fs=16000.0, c=343.0,
              N=1024, hop=512, delta=1e-5, methods=("srp", "svd"), max_frames=16, rank_D=0, options=0)
    kw.update(bad)
    with pytest.raises(S.SvdPhatError) as ei:
        S.Plan(kw["mics"], kw["points"], kw["fs"], kw["c"], kw["N"], kw["hop"], "far", rank_D=kw["rank_D"],
               delta=kw["delta"], methods=kw["methods"], max_frames=kw["max_frames"], options=kw["options"])
    assert ei.value.status == 1, str(ei.value)                  # INVALID_ARG
    assert S.lib.svdphat_last_error()


def test_valid_desc_without_gpu_is_unsupported(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    S = lib
    with pytest.raises(S.SvdPhatError) as ei:
        S.Plan(np.array([[0.05, 0, 0], [-0.05, 0, 0]]), np.eye(3), 16000.0, 343.0, 64, 32)
    assert ei.value.status == 5                                   # UNSUPPORTED: no device, no CPU fallback


def _split_worker(rank, ws, port, n_total, q):
    """One rank of the frame-sharded run: its contiguous shard of the global frame index space, its (stand-in)
    per-frame results, and the gather of all ranks' results to every rank (bench.frame_shard / bench.gather_frames)."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    sys.path.insert(0, ROOT)
    import bench
    f0, n = bench.frame_shard(n_total, rank, ws)
    local = torch.arange(f0, f0 + n, dtype=torch.int32) * 3          # frame g's "result" = 3 g
    allr = bench.gather_frames(local, n_total, dist)
    q.put((rank, f0, n, allr.numpy().tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_total", [10_001, 5])
def test_frame_split_two_ranks(n_total):
    """frames are sharded across ranks with no data-path collective; every frame is processed
    by exactly one rank (contiguous, balanced shards) and the gathered results are in global frame order."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30500 + (os.getpid() % 1000) + n_total % 7
    ps = [ctx.Process(target=_split_worker, args=(r, 2, port, n_total, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = sorted(q.get(timeout=10) for _ in range(2))
    owned = np.zeros(n_total, dtype=int)
    for _, f0, n, allr in res:
        owned[f0:f0 + n] += 1
        assert allr == [3 * g for g in range(n_total)]
    assert np.all(owned == 1)
    assert abs(res[0][2] - res[1][2]) <= 1


def _agg_worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    sys.path.insert(0, ROOT)
    import bench
    ms, v = bench.aggregate(10.0 * (rank + 1), 1000, dist, "cpu")
    q.put((rank, ms, v))
    dist.destroy_process_group()


def test_bench_aggregation_two_ranks():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    ps = [ctx.Process(target=_agg_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = sorted(q.get(timeout=10) for _ in range(2))
    for _, ms, v in res:
        assert ms == 20.0                       # max over ranks
        assert v == pytest.approx(2000 / 0.020)  # all ranks' frames / max time


def test_bench_arms_share_the_workload_config():
    """Both bench arms print the same `config` (the reference arm times a bounded sample of that workload)."""
    import bench
    from workloads import make
    w = make(1)
    a = bench.workload_config(1, w, len(w.points), 39, 1)
    b = bench.workload_config(1, w, len(w.points), 39, 1)
    assert a == b and a["workload"] == "cfg1" and a["frames_per_step"] == w.n_frames
    assert "model" not in a


def test_committed_launch_list_parses_and_names_the_dominant_kernel():
    """profiles/r02/final: the ncu launch list of the bench command summarises to per-step shares in which the SRP
    GEMM is the dominant kernel (the kernel bench.py's `roofline` object describes)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    csv_path = os.path.join(root, "profiles", "r02", "final", "ncu_launches_bench.csv")
    if not os.path.exists(csv_path):
        pytest.skip("no committed launch list")
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "launch_summary.py"), csv_path],
                         capture_output=True, text=True, check=True).stdout
    step = out[out.index("per localize(BOTH) step"):]
    first = [ln for ln in step.splitlines()[1:] if ln.startswith("svdphat::")][0]
    assert "gemm2_kernel" in first and float(first.split()[-1].rstrip("%")) > 70.0
