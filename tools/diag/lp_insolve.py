"""c5: the long pass inside the solve (library per-pass events) vs the same pass on the
same 80 GB A through lsrn_debug_rowpass, for L2 prefetch distances 0-2."""
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
t = torch.randn(p.n, dtype=torch.float64, device="cuda") * 1e-3
z = torch.randn(p.m, dtype=torch.float64, device="cuda")
for pf in (1, 0, 2):
    ctx.set_option("rowpass_pf", pf)
    x, rep = ctx.solve(p.X, p.b, p.m, p.n, solver="lsqr")
    x, rep = ctx.solve(p.X, p.b, p.m, p.n, solver="lsqr")
    torch.cuda.synchronize()
    st = ctx.stats()
    ms_dbg = min(ctx.debug_rowpass(p.X, t, z, (0.5, 0.1, 0.0), reps=5)[1] for _ in range(3))
    print(json.dumps({"pf": pf, "t_iter": rep["t_iter"], "long_pass_ms_insolve": st["long_pass_ms"],
                      "long_pass_ms_debug": ms_dbg, "gbs_debug": 8.0008e10 / ms_dbg / 1e6}), flush=True)
