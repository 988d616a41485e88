"""precision = 1 vs 0: x error against the oracle's long-double mode and solve time,
on c1 (2000 x 100, kappa 1e6) and on a c5-recipe 200000 x 2000 instance (cost at size)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.lsrn import solve as orc_solve  # noqa: E402
from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

ctx = lsrn.Context()
ctx.set_option("profiling", 1)
for solver in ("lsqr", "cs"):
    p = make_problem("c1")
    orc = orc_solve(p.X.numpy(), p.b.numpy(), solver=solver, extended=True)
    for prec in (0, 1):
        x, rep = ctx.solve(p.X.cuda(), p.b.cuda(), p.m, p.n, solver=solver, precision=prec)
        x, rep = ctx.solve(p.X.cuda(), p.b.cuda(), p.m, p.n, solver=solver, precision=prec)
        rel = float(np.linalg.norm(x.cpu().numpy() - orc["x"]) / np.linalg.norm(orc["x"]))
        print(json.dumps({"cfg": "c1", "solver": solver, "precision": prec, "x_rel_vs_oracle_ext": rel,
                          "t_iter_ms": rep["t_iter"] * 1e3, "iters": rep["iters"]}), flush=True)
p = make_problem("c5", m=200000, n=2000, device="cuda")
for prec in (0, 1):
    x, rep = ctx.solve(p.X, p.b, p.m, p.n, solver="lsqr", precision=prec)
    x, rep = ctx.solve(p.X, p.b, p.m, p.n, solver="lsqr", precision=prec)
    torch.cuda.synchronize()
    if prec == 0:
        x0 = x.clone()
    print(json.dumps({"cfg": "c5-200000x2000", "solver": "lsqr", "precision": prec, "iters": rep["iters"],
                      "t_iter_ms": rep["t_iter"] * 1e3, "ms_per_iter": rep["t_iter"] * 1e3 / rep["iters"],
                      "x_rel_vs_prec0": float(torch.linalg.norm(x - x0) / torch.linalg.norm(x0))}), flush=True)
