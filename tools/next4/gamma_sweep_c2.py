"""NEXT-4 on the bench workload: per-stage times vs gamma for c2 (1e5 x 2000, rank
1800, LSQR, tol 1e-14), and lsrn_choose_gamma's pick from a probe at gamma = 2.
The bench itself keeps BASELINE.json's gamma = 2.  One JSON line per gamma."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

p = make_problem("c2", device="cuda")
ctx = lsrn.Context()
best = None
for gamma in (1.2, 1.4, 1.6, 1.8, 2.0, 2.2, 2.5, 3.0):
    rows = [ctx.solve(p.X, p.b, p.m, p.n, gamma=gamma)[1] for _ in range(3)]
    rep = min(rows[1:], key=lambda d: d["t_total"])
    line = {"gamma": gamma, "s": rep["s"], "r": rep["r"], "iters": rep["iters"], "t_sketch": rep["t_sketch"],
            "t_svd": rep["t_svd"], "t_iter": rep["t_iter"], "t_total": rep["t_total"]}
    print(json.dumps(line), flush=True)
    if best is None or line["t_total"] < best["t_total"]:
        best = line
probe = ctx.solve(p.X, p.b, p.m, p.n, gamma=2.0)[1]
print(json.dumps({"best_gamma": best["gamma"], "best_t_total": best["t_total"],
                  "choose_gamma_from_probe_at_2": lsrn.choose_gamma(probe, p.m, p.n)}), flush=True)
