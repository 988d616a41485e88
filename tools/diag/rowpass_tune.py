import os
import sys
"""Long-pass (K6) timing on a c2/c5-shaped solve under tuning env settings."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1109_5981_b200 import lsrn
from synth.generate import make_problem
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
kw = {}
if cfg == "c5s":      # c5 recipe at 1/8 of the rows (one rank's shard at 8 GPUs)
    p = make_problem("c5", device="cuda", shard=(0, 125000)); m, n = 125000, 10000
    X, b = p.X, p.b
else:
    p = make_problem(cfg, device="cuda"); m, n = p.m, p.n
    X, b = p.X, p.b
ctx = lsrn.Context()
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _opts import apply_env_options  # noqa: E402
apply_env_options(ctx)
ctx.set_profiling(True)
out = []
with torch.cuda.stream(ctx.stream):
    for it in range(3):
        x, rep = ctx.solve(X, b, m, n, solver="lsqr", **kw)
        st = ctx.stats()
        out.append((st["long_pass_ms"], rep["t_iter"], st["long_pass_bytes"]))
lp, ti, by = min(out)
print(json.dumps({"cfg": cfg, "env": {k: v for k, v in os.environ.items() if k.startswith("LSRN_OPT_")},
                  "long_pass_ms": lp, "gbs": by / lp / 1e6, "t_iter_s": ti, "iters": rep["iters"]}))
