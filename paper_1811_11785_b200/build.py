"""Build libsvdphat.so in-tree: nvcc for sm_100a (-gencode arch=compute_100a,code=sm_100a), -lineinfo, O3.

Usage: python paper_1811_11785_b200/build.py [--force] [--verbose]   (does not import the package)
Writes paper_1811_11785_b200/libsvdphat.so and build/ptxas.log (registers / spills per kernel).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsvdphat.so")
BUILD = os.path.join(ROOT, "build")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include")]
SOURCES = ["api.cu", "setup.cu", "stft_phat.cu", "gemm_tc.cu", "finalize.cu", "das.cu"]
HEADERS = ["internal.h", "ptx.cuh"]


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "svdphat.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _obj_fresh(src: str, obj: str) -> bool:
    """The object is newer than its source, the shared headers and the build flags (this file)."""
    if not os.path.exists(obj):
        return False
    deps = [os.path.join(CSRC, src)] + [os.path.join(CSRC, h) for h in HEADERS] + \
        [os.path.join(ROOT, "include", "svdphat.h"), os.path.abspath(__file__)]
    t = os.path.getmtime(obj)
    return all(os.path.getmtime(d) <= t for d in deps)


def _compile(src: str, force: bool = False) -> tuple[str, str]:
    obj = os.path.join(BUILD, os.path.splitext(src)[0] + ".o")
    log = obj + ".ptxas.log"
    if not force and _obj_fresh(src, obj) and os.path.exists(log):
        return obj, open(log).read()
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    with open(log, "w") as f:
        f.write(r.stderr)
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        res = list(ex.map(lambda f: _compile(f, force), SOURCES))
    objs = [o for o, _ in res]
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        for _, log in res:
            f.write(log)
    lib = os.path.join(CUDA, "lib64")
    cmd = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-L" + lib, "-lcublas", "-lcusolver", "-lcudart",
           "-Xlinker", "-rpath," + lib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    if verbose:
        print(open(os.path.join(BUILD, "ptxas.log")).read())
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
