"""CSR sketch stage time (library CUDA events) per LSRN_OPT_CSR_SKETCH mode on a full
config, with the relative Frobenius difference of each mode's sketch from the first.
argv: config modes..."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

cfg = sys.argv[1]
modes = [int(a) for a in sys.argv[2:]] or [0, 2]
p = make_problem(cfg, device="cuda")
X = lsrn.Csr(p.rowptr, p.colind, p.val)
ctx = lsrn.Context()
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _opts import apply_env_options  # noqa: E402
apply_env_options(ctx)               # LSRN_OPT_* of the environment (e.g. LSRN_OPT_CSR_HEAVY_FMA)
ref = None
for mode in modes:
    ctx.set_option("csr_sketch", mode)
    ms = []
    for _ in range(2):
        At = ctx.sketch(X, p.m, p.n)
        torch.cuda.synchronize()
        ms.append(ctx.stats()["sketch_ms"])
    if ref is None:
        ref = At.clone()
    d = float(torch.linalg.norm(At - ref) / torch.linalg.norm(ref))
    print(json.dumps({"cfg": cfg, "csr_sketch": mode, "sketch_ms": min(ms), "relfro_vs_first": d}), flush=True)
    del At
    torch.cuda.empty_cache()
