"""c5 LSQR with the library's per-pass profiling events on and off: t_iter and t_total."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

p = make_problem("c5", device="cuda")
ctx = lsrn.Context()
for prof in (1, 0, 1, 0):
    ctx.set_option("profiling", prof)
    x, rep = ctx.solve(p.X, p.b, p.m, p.n, solver="lsqr")
    x, rep = ctx.solve(p.X, p.b, p.m, p.n, solver="lsqr")
    torch.cuda.synchronize()
    print(json.dumps({"profiling": prof, "t_iter": rep["t_iter"], "t_total": rep["t_total"]}), flush=True)
