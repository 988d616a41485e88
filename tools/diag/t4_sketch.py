"""Time the CSR sketch on the t4 (NEXT-2) shape."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1109_5981_b200 import lsrn
from synth.generate import make_problem
p = make_problem("t4", device="cuda")
X = lsrn.Csr(p.rowptr, p.colind, p.val)
ctx = lsrn.Context()
ctx.sketch(X, p.m, p.n)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(ctx.stream):
    e0.record(ctx.stream); ctx.sketch(X, p.m, p.n); e1.record(ctx.stream)
torch.cuda.synchronize()
print(json.dumps({"cfg": "t4", "sketch_ms": e0.elapsed_time(e1)}))
