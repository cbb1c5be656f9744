"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): per svdphat kernel, launches, total and
mean time, and share of the svdphat kernel time (plan-creation cuSOLVER/cuBLAS kernels are listed apart).
Usage: python tools/launch_summary.py gpurun_out/s_launches.csv > profiles/r02/.../launch_summary.txt"""
import collections
import csv
import io
import sys

txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
agg = collections.defaultdict(lambda: [0, 0.0])
calls = []                                   # localize calls: each begins with an STFT launch
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = r["Kernel Name"].split("(")[0].replace("void ", "")
    us = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else 1.0)   # -> us
    agg[name][0] += 1
    agg[name][1] += us
    if "stft_phat_kernel" in name:
        calls.append([])
    if calls and name.startswith("svdphat::"):
        calls[-1].append((name, us))
own = {k: v for k, v in agg.items() if k.startswith("svdphat::") and "pack_" not in k and "gram" not in k
       and "bmat" not in k and "setup" not in k and "ucplx" not in k and "rwchunk" not in k}
tot = sum(v[1] for v in own.values())
print(f"{'kernel (svdphat hot path)':60s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s} {'share':>7s}")
for k, (c, t) in sorted(own.items(), key=lambda x: -x[1][1]):
    print(f"{k[:60]:60s} {c:8d} {t / 1e3:10.3f} {t / c:10.1f} {100 * t / tot:6.1f}%")
print(f"{'total':60s} {'':8s} {tot / 1e3:10.3f}")
rest = {k: v for k, v in agg.items() if k not in own}
print(f"\nplan creation / library kernels (not in the step): {len(rest)} kinds, "
      f"{sum(v[1] for v in rest.values()) / 1e3:.1f} ms")

# the bench step = one localize(BOTH): the calls that run an SRP kernel and the SVD projection
both = [c for c in calls if any("gemm2_kernel" in n or "das" in n for n, _ in c) and any("gemm2p" in n or "gemm2f" in n for n, _ in c)]
if both:
    st = collections.defaultdict(lambda: [0, 0.0])
    for c in both:
        for n, us in c:
            st[n][0] += 1
            st[n][1] += us
    tt = sum(v[1] for v in st.values())
    print(f"\nper localize(BOTH) step ({len(both)} steps in the list; the bench's SVD-only and SRP-only legs excluded):")
    for k, (c, t) in sorted(st.items(), key=lambda x: -x[1][1]):
        print(f"{k[:60]:60s} {c / len(both):8.1f} {t / len(both) / 1e3:10.3f} {t / c:10.1f} {100 * t / tt:6.1f}%")
    print(f"{'kernel time per step (serialised, cold cache)':60s} {'':8s} {tt / len(both) / 1e3:10.3f}")
