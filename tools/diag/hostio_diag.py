"""Stage times of a c2 solve: device-resident vs LSRN_HOST_IO (streamed chunks)."""
import time

import torch

from paper_1109_5981_b200 import lsrn
from synth.generate import make_problem

p = make_problem("c2", device="cuda")
c = lsrn.Context()
Xh = p.X.cpu().pin_memory()
bh = p.b.cpu().pin_memory()
for name, X, b, hio in (("device", p.X, p.b, False), ("host", Xh, bh, True)):
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = c.solve(X, b, p.m, p.n, host_io=hio)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
    print(name, f"wall {1e3 * (t1 - t0):.1f} ms", {k: round(v * 1e3, 2) for k, v in rep.items() if k.startswith("t_")})
t = torch.empty_like(p.X)
torch.cuda.synchronize()
t0 = time.perf_counter()
t.copy_(Xh, non_blocking=True)
torch.cuda.synchronize()
print("plain H2D of A", 1e3 * (time.perf_counter() - t0), "ms")
