"""Time the CSR sketch (K4) on the full c4 recipe."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1109_5981_b200 import lsrn
from synth.generate import make_problem
p = make_problem("c4", device="cuda")
X = lsrn.Csr(p.rowptr, p.colind, p.val)
ctx = lsrn.Context()
ctx.sketch(X, p.m, p.n)
torch.cuda.synchronize()
with torch.cuda.stream(ctx.stream):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ctx.stream); ctx.sketch(X, p.m, p.n); e1.record(ctx.stream); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
nnz = p.val.numel(); s = 2 * p.n
print(json.dumps({"cfg": "c4", "sketch_ms": ms, "flops": 2.0 * s * nnz, "tflops": 2.0 * s * nnz / ms / 1e9,
                  "normals_once": s * p.m}))
