"""CSR long pass (K6-CSR) per variant on a full config: average kernel time of the long
pass (library CUDA events), its algorithmic bytes and GB/s; LSRN_OPT_CSR_ROWDOT values
given on the command line (-1 = planner).  argv: config [variants...]"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "t4"
variants = [int(a) for a in sys.argv[2:]] or [-1, 3]
p = make_problem(cfg, device="cuda")
X = lsrn.Csr(p.rowptr, p.colind, p.val)
ctx = lsrn.Context()
ctx.set_profiling(True)
xs = {}
for v in variants:
    ctx.set_option("csr_rowdot", v)
    for _ in range(2):
        x, rep = ctx.solve(X, p.b, p.m, p.n, solver="cs")
    torch.cuda.synchronize()
    st = ctx.stats()
    xs[v] = x.clone()
    print(json.dumps({"cfg": cfg, "csr_rowdot": v, "long_pass_ms": st["long_pass_ms"], "bytes": st["long_pass_bytes"],
                      "gbs": st["long_pass_bytes"] / st["long_pass_ms"] / 1e6 if st["long_pass_ms"] else None,
                      "t_iter": rep["t_iter"], "iters": rep["iters"]}), flush=True)
ks = list(xs)
for v in ks[1:]:
    print(json.dumps({"x_reldiff": [ks[0], v], "value": float(torch.linalg.norm(xs[v] - xs[ks[0]]) / torch.linalg.norm(xs[ks[0]]))}))
