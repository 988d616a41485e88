import os
import sys
"""Time the fused row pass (lsrn_debug_rowpass) on an R x C device matrix under the
current LSRN_OPT_ROWPASS_* environment (applied through lsrn_ctx_set_option).  argv: R C [reps]; prints ms and GB/s (8 C + 16
bytes per row)."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1109_5981_b200 import lsrn
R, C = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
g = torch.Generator(device="cuda").manual_seed(1)
Y = torch.randn(R, C, generator=g, dtype=torch.float64, device="cuda")
t = torch.randn(C, generator=g, dtype=torch.float64, device="cuda") * 1e-3
z = torch.randn(R, generator=g, dtype=torch.float64, device="cuda")
ctx = lsrn.Context()
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _opts import apply_env_options  # noqa: E402
apply_env_options(ctx)
ctx.debug_rowpass(Y, t, z, (0.5, 0.1, 0.0), reps=2)
best = min(ctx.debug_rowpass(Y, t, z, (0.5, 0.1, 0.0), reps=reps)[1] for _ in range(3))
by = R * (8.0 * C + 16)
print(json.dumps({"R": R, "C": C, "env": {k: v for k, v in os.environ.items() if k.startswith("LSRN_OPT_")},
                  "ms": best, "gbs": by / best / 1e6}))
