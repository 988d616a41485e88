import os
import sys
"""CSR long-pass (K6-CSR) timing on a c4-shaped problem: 20 random + 50 heavy columns per row.
argv: m n [solver]; prints the library's per-launch long-pass time and algorithmic GB/s."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1109_5981_b200 import lsrn
from synth.generate import make_problem
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
solver = sys.argv[3] if len(sys.argv) > 3 else "cs"
p = make_problem("c4", device="cuda", m=m, n=n)
X = lsrn.Csr(p.rowptr, p.colind, p.val)
ctx = lsrn.Context()
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _opts import apply_env_options  # noqa: E402
apply_env_options(ctx)
ctx.set_profiling(True)
out = []
with torch.cuda.stream(ctx.stream):
    for it in range(2):
        x, rep = ctx.solve(X, p.b, m, n, solver=solver)
        st = ctx.stats()
        out.append((st["long_pass_ms"], rep["t_iter"], st["long_pass_bytes"], rep["t_sketch"], rep["t_svd"]))
lp, ti, by, tsk, tsvd = min(out)
print(json.dumps({"m": m, "n": n, "nnz": int(p.val.numel()), "solver": solver,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("LSRN_OPT_")},
                  "long_pass_ms": lp, "gbs": by / lp / 1e6, "bytes": by, "t_iter_s": ti, "iters": rep["iters"],
                  "t_sketch": tsk, "t_svd": tsvd}))
