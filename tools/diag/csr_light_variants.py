"""Stored-G CSR light-sketch kernel per LSRN_OPT_CSR_LIGHT value (10 * columns per CTA +
gathers in flight per thread; -1 = default), optionally "@MB" with a G budget
(LSRN_OPT_SKETCH_G), on a full config: sketch stage time (library CUDA events, best of 3)
and bitwise equality with the first value's sketch (the per-column accumulation order does
not depend on either parameter).  argv: config values...  (e.g. 14 18@256)"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

cfg = sys.argv[1]
vals = sys.argv[2:] or ["-1", "48"]
p = make_problem(cfg, device="cuda")
X = lsrn.Csr(p.rowptr, p.colind, p.val)
ctx = lsrn.Context()
ctx.set_profiling(True)
ref = None
for a in vals:
    v, _, mb = a.partition("@")
    v, mb = int(v), int(mb) if mb else -1
    ctx.set_option("csr_light", v)
    ctx.set_option("sketch_g", mb)
    ms = []
    for _ in range(3):
        At = ctx.sketch(X, p.m, p.n)
        torch.cuda.synchronize()
        ms.append(ctx.stats()["sketch_ms"])
    if ref is None:
        ref = At.clone()
    print(json.dumps({"cfg": cfg, "csr_light": v, "sketch_g_mb": mb, "sketch_ms": min(ms), "bitwise_equal_to_first": bool(torch.equal(At, ref))}),
          flush=True)
    del At
