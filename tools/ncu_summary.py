"""Key metrics of every kernel in an ncu --set full report: duration, SM clock, tensor / issue / warp activity, DRAM and
L2 traffic and throughput, top warp stall reasons.
Usage: python tools/ncu_summary.py report.ncu-rep [kernel-substring] > profiles/r02/.../ncu_summary.txt"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
filt = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def get(r, *names):
    for n in names:
        if n in col and r[col[n]] not in ("", "n/a"):
            try:
                return float(r[col[n]].replace(",", ""))
            except ValueError:
                return r[col[n]]
    return None


KEYS = [
    ("duration_us", ("gpu__time_duration.sum",), "time"),
    ("sm_clock_ghz", ("sm__cycles_elapsed.avg.per_second",), "freq"),
    ("tensor_active_pct", ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                           "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active"), ""),
    ("tensor_mem_active_pct", ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",), ""),
    ("issue_active_pct", ("sm__issue_active.avg.pct_of_peak_sustained_active",
                          "smsp__issue_active.avg.pct_of_peak_sustained_active"), ""),
    ("warps_active_pct", ("sm__warps_active.avg.pct_of_peak_sustained_active",), ""),
    ("dram_read_MB", ("dram__bytes_read.sum",), "bytes"),
    ("dram_write_MB", ("dram__bytes_write.sum",), "bytes"),
    ("dram_pct_peak", ("dram__throughput.avg.pct_of_peak_sustained_elapsed",
                       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), ""),
    ("l2_pct_peak", ("lts__throughput.avg.pct_of_peak_sustained_elapsed",), ""),
    ("l2_to_sm_MB", ("l1tex__m_xbar2l1tex_read_bytes.sum",), "bytes"),
    ("l2_to_sm_TBps", ("l1tex__m_xbar2l1tex_read_bytes.sum.per_second",), "rate"),
    ("sm_throughput_pct", ("sm__throughput.avg.pct_of_peak_sustained_elapsed",), ""),
    ("registers", ("launch__registers_per_thread",), ""),
    ("inst_executed_M", ("smsp__inst_executed.sum", "sm__inst_executed.sum"), "count"),
]
CONV = {
    "time": {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6},
    "freq": {"Ghz": 1.0, "GHz": 1.0, "Mhz": 1e-3, "MHz": 1e-3, "hz": 1e-9, "cycle/second": 1e-9},
    "bytes": {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6, "sector": 32e-6},
    "rate": {"Tbyte/s": 1.0, "Gbyte/s": 1e-3, "Mbyte/s": 1e-6, "byte/s": 1e-12},
    "count": {"": 1e-6, "inst": 1e-6, "Kinst": 1e-3, "Minst": 1.0, "Ginst": 1e3},
}
# ncu prefixes some columns with their section ("TPC.TriageCompute.sm__..."): match on the metric suffix
bare = {}
for i, h in enumerate(hdr):
    bare.setdefault(h.split(".", 2)[-1] if h[:1].isupper() and h.count(".") >= 2 else h, i)
    bare.setdefault(h, i)

for r in data:
    name = r[col["Kernel Name"]]
    if filt and filt not in name:
        continue
    print(f"== {name.split('(')[0]}  grid {r[col['Grid Size']]} block {r[col['Block Size']]}")
    for key, names, kind in KEYS:
        for n in names:
            i = bare.get(n)
            if i is None or r[i] in ("", "n/a"):
                continue
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            if kind:
                v *= CONV[kind].get(units[i], 1.0)
            print(f"  {key:22s} {v:14.3f}")
            break
    stalls = []
    for h, i in col.items():
        if "average_warp_latency_issue_stalled_" in h or \
                ("pcsamp_warps_issue_stalled_" in h and not h.endswith("_not_issued")):
            try:
                stalls.append((float(r[i].replace(",", "")), h.split("stalled_")[-1]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    if stalls:
        print("  top stalls:", ", ".join(f"{n}={v:.3g}" for v, n in stalls[:6]))
