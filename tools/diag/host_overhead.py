"""Host-side overhead of one c2 solve: time of lsrn_workspace_size and of the whole
solve call vs its device time (t_total), to find GPU-idle gaps between solves."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1109_5981_b200 import lsrn
from synth.generate import make_problem
p = make_problem("c2", device="cuda")
ctx = lsrn.Context()
for _ in range(3):
    ctx.solve(p.X, p.b, p.m, p.n)
torch.cuda.synchronize()
mat, _k = lsrn.describe(p.X, p.m, p.n, 0, None)
opts = lsrn.Opts(gamma=2.0, lambda_=0.0, tol=1e-14, alpha=-1.0, seed=5981, mode=0, max_iter=0, flags=0)
t0 = time.perf_counter()
for _ in range(10):
    ctx.workspace_size(mat, opts)
t1 = time.perf_counter()
print("workspace_size ms", (t1 - t0) / 10 * 1e3)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(ctx.stream)
t0 = time.perf_counter()
for _ in range(5):
    x, rep = ctx.solve(p.X, p.b, p.m, p.n)
t1 = time.perf_counter()
e1.record(ctx.stream)
torch.cuda.synchronize()
print("wall per solve ms", (t1 - t0) / 5 * 1e3, "device per solve ms", e0.elapsed_time(e1) / 5, "t_total ms", rep["t_total"] * 1e3)
