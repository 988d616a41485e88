"""SVD stage (t_svd, outside the hot path) of a full solve per LSRN_OPT_SVD method on a
config; prints the stage times, the method actually used and the relative difference
of x between methods.  argv: config [methods...] (default: jw polar)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
methods = sys.argv[2:] or ["jw", "polar"]
p = make_problem(cfg, device="cuda")
X = lsrn.Csr(p.rowptr, p.colind, p.val) if p.kind == "csr" else p.X
ctx = lsrn.Context()
xs = {}
for meth in methods:
    ctx.set_option("svd", meth)
    for rep_ in range(2):
        x, rep = ctx.solve(X, p.b, p.m, p.n, solver="cs" if cfg == "c4" else "lsqr", lam=p.lam)
    torch.cuda.synchronize()
    xs[meth] = x.clone()
    print(json.dumps({"cfg": cfg, "svd": meth, "svd_used": rep["svd_used"], "t_svd": rep["t_svd"],
                      "t_sketch": rep["t_sketch"], "t_iter": rep["t_iter"], "t_total": rep["t_total"],
                      "r": rep["r"], "iters": rep["iters"]}), flush=True)
ms = list(xs)
for a in ms[1:]:
    d = float(torch.linalg.norm(xs[a] - xs[ms[0]]) / torch.linalg.norm(xs[ms[0]]))
    print(json.dumps({"cfg": cfg, "x_reldiff": [ms[0], a], "value": d}), flush=True)
