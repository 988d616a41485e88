import os
import sys
"""Time the dense sketch on the c2 shape under tuning env settings (one process per setting)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1109_5981_b200 import lsrn
m, n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000, int(sys.argv[2]) if len(sys.argv) > 2 else 2000
torch.manual_seed(0)
X = torch.randn(m, n, dtype=torch.float64, device="cuda")
ctx = lsrn.Context()
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _opts import apply_env_options  # noqa: E402
apply_env_options(ctx)
with torch.cuda.stream(ctx.stream):
    for _ in range(2):
        ctx.sketch(X, m, n)
    torch.cuda.synchronize()
    ms = []
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream); ctx.sketch(X, m, n); e1.record(ctx.stream); torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
s = int(2 * n)
print(json.dumps({"m": m, "n": n, "env": {k: v for k, v in os.environ.items() if k.startswith("LSRN_OPT_")},
                  "ms_min": min(ms), "tflops": 2 * s * n * m / min(ms) / 1e9}))
