"""HBM copy bandwidth, burst (best of 10 single copies) and sustained (back to back for
~3 s, the regime of a long solve phase under the board power cap), the way
MEASURED_PEAKS.json measures the burst figure: b.copy_(a), read + write bytes."""
import json
import statistics
import subprocess
import threading
import time

import torch

n = 1 << 30                                   # doubles: 8 GiB per buffer
a = torch.randn(n, dtype=torch.float64, device="cuda")
b = torch.empty_like(a)
by = 2 * 8 * n
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
best = 1e30
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
samples = []
p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                      "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [samples.append(l.strip()) for l in p.stdout], daemon=True).start()
time.sleep(0.5)
reps = 600
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    b.copy_(a)
e1.record()
torch.cuda.synchronize()
p.terminate()
sus = e0.elapsed_time(e1) / reps
sm = [float(s.split(",")[0]) for s in samples[5:] if s]
pw = [float(s.split(",")[1]) for s in samples[5:] if s]
print(json.dumps({"burst_gbs": by / best / 1e6, "sustained_gbs": by / sus / 1e6, "sustained_s": sus * reps / 1e3,
                  "sm_mhz_median": statistics.median(sm) if sm else None, "power_w_median": statistics.median(pw) if pw else None}))
