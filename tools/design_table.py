"""Print the DESIGN.md per-config table from profiles/r01/bench_configs.jsonl (tools/bench_configs.py output)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "r01", "bench_configs.jsonl")
print("| cfg | array | M | N | Q (classes) | D | frames/call | SRP frames/s | SVD frames/s | both frames/s | notes |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for line in open(path):
    d = json.loads(line)
    note = ""
    if "call_latency_graph_ms_p50" in d:
        note = (f"per 256-frame call (both): {d['call_latency_ms_p50']:.3f} ms eager, "
                f"{d['call_latency_graph_ms_p50']:.3f} ms as a CUDA graph (p50)")
    print(f"| {d['cfg']} | {d['name']} | {d['M']} | {d['N']} | {d['Q']} ({d['Q_classes']}) | {d['D']} | "
          f"{d['frames_per_call']} | {d['srp_fps']:.3g} | {d['svd_fps']:.3g} | {d['both_fps']:.3g} | {note} |")
