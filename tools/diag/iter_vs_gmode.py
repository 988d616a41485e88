"""c5 LSQR iterations and long-pass time with the dense sketch's G stored (default) or
generated in registers (sketch_g = 0): does the stored-G workspace change the passes?
Order -1, 0, -1 in one process."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

p = make_problem("c5", device="cuda")
ctx = lsrn.Context()
ctx.set_option("profiling", 1)
for g in (-1, 0, -1, 0):
    ctx.set_option("sketch_g", g)
    ctx._ws = None
    torch.cuda.empty_cache()
    x, rep = ctx.solve(p.X, p.b, p.m, p.n, solver="lsqr")
    torch.cuda.synchronize()
    st = ctx.stats()
    print(json.dumps({"sketch_g": g, "t_iter": rep["t_iter"], "t_sketch": rep["t_sketch"], "t_svd": rep["t_svd"],
                      "long_pass_ms": st.get("long_pass_ms"), "ws_gb": ctx._ws.numel() / 1e9}), flush=True)
