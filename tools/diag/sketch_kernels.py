"""Dense sketch stage time per kernel variant (LSRN_OPT_SKETCH_KERNEL: 0 warp-specialized
with RNG producer warps, 2 DMMA warps generating G) on an m x n Gaussian X; prints
ms, TFLOP/s (2 s k L) and the relative difference between the variants' sketches.
argv: m n [kernels...]"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1109_5981_b200 import lsrn  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
kernels = [int(a) for a in sys.argv[3:]] or [0, 2]
torch.manual_seed(0)
X = torch.randn(m, n, dtype=torch.float64, device="cuda")
ctx = lsrn.Context()
res = {}
for kern in kernels:
    ctx.set_option("sketch_kernel", kern)
    ms = []
    for _ in range(3):
        At = ctx.sketch(X, m, n)
        torch.cuda.synchronize()
        ms.append(ctx.stats()["sketch_ms"])
    res[kern] = At
    s = 2 * n
    print(json.dumps({"m": m, "n": n, "kernel": kern, "ms": min(ms), "tflops": 2 * s * n * m / min(ms) / 1e9}),
          flush=True)
ks = list(res)
for kk in ks[1:]:
    print(json.dumps({"relfro": float(torch.linalg.norm(res[kk] - res[ks[0]]) / torch.linalg.norm(res[ks[0]])),
                      "kernels": [ks[0], kk]}))
