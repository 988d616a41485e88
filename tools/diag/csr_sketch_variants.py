"""CSR sketch stage time (library CUDA events, lsrn_last_stats sketch_ms) of the two
light-sketch kernels on a full config: per-nonzero (csr_sketch = 0) vs generate-once
slab (csr_sketch = 1); prints both and their relative Frobenius difference.
argv: config (t4 | c4) [reps]"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "t4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
p = make_problem(cfg, device="cuda")
X = lsrn.Csr(p.rowptr, p.colind, p.val)
ctx = lsrn.Context()
out = {"cfg": cfg, "nnz": int(p.val.numel())}
res = {}
for light in (1, 0):
    ctx.set_option("csr_sketch", light)
    ms = []
    for _ in range(reps):
        At = ctx.sketch(X, p.m, p.n)
        torch.cuda.synchronize()
        ms.append(ctx.stats()["sketch_ms"])
    res[light] = At
    out[f"sketch_ms_light{light}"] = min(ms)
d = torch.linalg.norm(res[0] - res[1]) / torch.linalg.norm(res[0])
out["relfro_between"] = float(d)
print(json.dumps(out), flush=True)
