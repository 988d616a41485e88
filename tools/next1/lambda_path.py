"""NEXT-1 (§5): a Tikhonov path solved with one sketch of A.

c3 (2000 x 2e5, the wide Tikhonov config) for lambda in {1e-1, 1e-2, 1e-3, 1e-4}:
fresh solves vs Context.solve_path (LSRN_REUSE_SKETCH after the first), stage
times from the library's CUDA events.  One JSON line per (mode, lambda)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.getcwd())
from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

p = make_problem("c3", device="cuda")
ctx = lsrn.Context()
lams = [1e-1, 1e-2, 1e-3, 1e-4]
ctx.solve(p.X, p.b, p.m, p.n, lam=lams[0])          # warm-up
for mode in ("fresh", "path"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if mode == "fresh":
        reps = [ctx.solve(p.X, p.b, p.m, p.n, lam=lam)[1] for lam in lams]
    else:
        reps = [r for _, r in ctx.solve_path(p.X, p.b, p.m, p.n, lams)]
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    for lam, r in zip(lams, reps):
        print(json.dumps({"mode": mode, "lambda": lam, "iters": r["iters"], "t_sketch": r["t_sketch"],
                          "t_svd": r["t_svd"], "t_iter": r["t_iter"], "t_total": r["t_total"]}))
    print(json.dumps({"mode": mode, "wall_s_all_lambdas": wall}), flush=True)
