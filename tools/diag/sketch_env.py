"""Dense sketch stage time on an m x n Gaussian X under LSRN_OPT_* settings of this
process (applied through lsrn_ctx_set_option).  argv: m n [reps]"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _opts import apply_env_options  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
torch.manual_seed(0)
X = torch.randn(m, n, dtype=torch.float64, device="cuda")
ctx = lsrn.Context()
used = apply_env_options(ctx)
ms = []
for _ in range(reps):
    ctx.sketch(X, m, n)
    torch.cuda.synchronize()
    ms.append(ctx.stats()["sketch_ms"])
print(json.dumps({"m": m, "n": n, "opts": used, "ms": min(ms), "tflops": 4.0 * n * n * m / min(ms) / 1e9}), flush=True)
