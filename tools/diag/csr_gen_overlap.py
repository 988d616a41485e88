"""Stored-G CSR sketch with and without the overlapped generation (LSRN_OPT_CSR_GEN_OVERLAP
0 = serial, one G block; -1 = default, two blocks): sketch stage time (library CUDA events,
best of 3) and whether the two sketches are bitwise equal.  argv: configs..."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402
from synth.generate import make_problem  # noqa: E402

args = sys.argv[1:] or ["t4", "c4"]
modes = [int(a) for a in args if a.lstrip("-").isdigit()] or [0, -1]
for cfg in [a for a in args if not a.lstrip("-").isdigit()]:
    p = make_problem(cfg, device="cuda")
    X = lsrn.Csr(p.rowptr, p.colind, p.val)
    ctx = lsrn.Context()
    ctx.set_profiling(True)
    out = {}
    for ov in modes:
        ctx.set_option("csr_gen_overlap", ov)
        ms = []
        for _ in range(3):
            At = ctx.sketch(X, p.m, p.n)
            torch.cuda.synchronize()
            ms.append(ctx.stats()["sketch_ms"])
        out[ov] = At
        print(json.dumps({"cfg": cfg, "csr_gen_overlap": ov, "sketch_ms": min(ms), "all_ms": ms}), flush=True)
    print(json.dumps({"cfg": cfg, "bitwise_equal_to_first": [bool(torch.equal(out[modes[0]], v)) for v in out.values()]}),
          flush=True)
    del out, At, X, p
    ctx.close()
    torch.cuda.empty_cache()
