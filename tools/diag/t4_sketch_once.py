"""One t4 CSR sketch with the slab light kernel (ncu target)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "t4"
p = make_problem(cfg, device="cuda")
X = lsrn.Csr(p.rowptr, p.colind, p.val)
ctx = lsrn.Context()
ctx.set_option("csr_sketch", int(os.environ.get("LIGHT", "1")))
ctx.sketch(X, p.m, p.n)
torch.cuda.synchronize()
print("sketch_ms", ctx.stats()["sketch_ms"])
