"""c5-shaped long pass through lsrn_debug_rowpass: average over a short burst (5 passes)
and over a sustained run (100 passes, ~1.2 s of back-to-back streaming, like the solve's
iteration phase), with nvidia-smi's SM clock and power sampled during the sustained run."""
import json
import os
import subprocess
import sys
import threading

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402

R, C = 1000000, 10000
Y = torch.randn(R, C, dtype=torch.float64, device="cuda")
t = torch.randn(C, dtype=torch.float64, device="cuda") * 1e-3
z = torch.randn(R, dtype=torch.float64, device="cuda")
ctx = lsrn.Context()
ctx.debug_rowpass(Y, t, z, (0.5, 0.1, 0.0), reps=2)
out = {}
for reps in (5, 100, 5, 100):
    samples = []
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    th = threading.Thread(target=lambda: [samples.append(l.strip()) for l in p.stdout], daemon=True)
    th.start()
    import time
    time.sleep(0.5)
    ms = ctx.debug_rowpass(Y, t, z, (0.5, 0.1, 0.0), reps=reps, per_rep=True)[1] if False else None
    # time all reps with CUDA events around the whole loop
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ctx.debug_rowpass(Y, t, z, (0.5, 0.1, 0.0), reps=1)
    e1.record()
    torch.cuda.synchronize()
    p.terminate()
    avg = e0.elapsed_time(e1) / reps
    print(json.dumps({"passes": reps, "avg_ms_per_pass_incl_colreduce": avg, "gbs": 8.0016e10 / avg / 1e6,
                      "smi": samples[-8:]}), flush=True)
