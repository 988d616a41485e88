"""Long-pass time per option set on a full config: each argument after the config is a
comma-separated list of name=value library options (lsrn.OPTIONS; '-' = defaults).
Prints the average long-pass time (library CUDA events, best of 3 solves), its
algorithmic bytes and GB/s, the iteration-stage time, and x against the first set.
argv: config [solver=cs] optsets...   e.g.  c4 - csr_colgather=4 csr_colgather=8"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

cfg = sys.argv[1]
args = sys.argv[2:]
solver = "cs"
if args and args[0].startswith("solver="):
    solver = args.pop(0).split("=", 1)[1]
sets = args or ["-"]
p = make_problem(cfg, device="cuda")
X = lsrn.Csr(p.rowptr, p.colind, p.val) if p.kind == "csr" else p.X
ctx = lsrn.Context()
ctx.set_profiling(True)
xs = []
for st_ in sets:
    kv = {} if st_ == "-" else dict(a.split("=", 1) for a in st_.split(","))
    kv = {k: int(v) for k, v in kv.items()}
    with ctx.options(**kv):
        best = None
        for _ in range(3):
            x, rep = ctx.solve(X, p.b, p.m, p.n, solver=solver)
            torch.cuda.synchronize()
            s = ctx.stats()
            if best is None or s["long_pass_ms"] < best[0]:
                best = (s["long_pass_ms"], s["long_pass_bytes"], rep["t_iter"], rep["iters"])
    xs.append(x.clone())
    lp, by, ti, it = best
    rel = float(torch.linalg.norm(x - xs[0]) / torch.linalg.norm(xs[0]))
    print(json.dumps({"cfg": cfg, "opts": kv, "long_pass_ms": lp, "bytes": by, "gbs": by / lp / 1e6, "t_iter": ti,
                      "iters": it, "x_rel_vs_first": rel}), flush=True)
