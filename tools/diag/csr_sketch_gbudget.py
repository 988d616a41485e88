"""CSR stored-G sketch (csr_sketch = 2) per G budget (LSRN_OPT_SKETCH_G, MB; -1 = the 8 GB
default) on a full config: sketch stage time (library CUDA events) and the relative
Frobenius difference from the first budget's sketch.  A budget that fits in L2 keeps each
chunk's G block L2-resident between its generation and the light kernel's gathers.
argv: config budgets..."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

cfg = sys.argv[1]
budgets = [int(a) for a in sys.argv[2:]] or [-1, 64]
p = make_problem(cfg, device="cuda")
X = lsrn.Csr(p.rowptr, p.colind, p.val)
ctx = lsrn.Context()
ctx.set_profiling(True)
ref = None
for mb in budgets:
    ctx.set_option("sketch_g", mb)
    ms = []
    for _ in range(2):
        At = ctx.sketch(X, p.m, p.n)
        torch.cuda.synchronize()
        ms.append(ctx.stats()["sketch_ms"])
    if ref is None:
        ref = At.clone()
    d = float(torch.linalg.norm(At - ref) / torch.linalg.norm(ref))
    print(json.dumps({"cfg": cfg, "sketch_g_mb": mb, "sketch_ms": min(ms), "relfro_vs_first": d}), flush=True)
    del At
    torch.cuda.empty_cache()
