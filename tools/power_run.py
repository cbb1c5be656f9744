"""Long SRP run with nvidia-smi power/clock sampling (dev tool): is the GEMM at the power cap?"""
import subprocess, sys, time, threading
import torch
import paper_1811_11785_b200 as S
from workloads import make
w = make(3)
plan = S.Plan(w.mics, w.points, w.fs, w.c, w.N, w.hop, w.field, delta=w.delta, methods=("srp",), max_frames=w.n_frames)
a = torch.from_numpy(w.audio).cuda(); F = w.n_frames
doa = torch.empty(F, dtype=torch.int32, device="cuda"); sc = torch.empty(F, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(3): plan.localize("srp", a, F, w.channel_stride, w.frame_stride, doa, sc, st)
torch.cuda.synchronize()
rows = []; stop = threading.Event()
def samp():
    while not stop.is_set():
        o = subprocess.run(["nvidia-smi","--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap","--format=csv,noheader,nounits"],capture_output=True,text=True).stdout.strip()
        rows.append(o); time.sleep(0.1)
th = threading.Thread(target=samp); th.start()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
plan.profile_begin(4 * n)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n): plan.localize("srp", a, F, w.channel_stride, w.frame_stride, doa, sc, st)
e1.record(); torch.cuda.synchronize(); stop.set(); th.join()
prof = plan.profile_end()
g = [ms for nm, ms in prof if nm == "srp_gemm"]
print("steps", n, "ms/step %.3f" % (e0.elapsed_time(e1) / n), "gemm ms avg %.3f min %.3f max %.3f" % (sum(g)/len(g), min(g), max(g)),
      "TF/s %.0f" % (4.0 * 10242 * 61560 * F / (sum(g)/len(g)/1e3) / 1e12))
print("\n".join(rows[::5]))
