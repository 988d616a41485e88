"""NEXT-4: the paper's gamma study (§6.3, Figure 2) on the GPU.

Problem 1e5 x 1e3, kappa = 1e6 (sigma log-spaced 1 -> 1e-6, U, V Haar), b ~ N(0,1),
tol 1e-14, LSQR, gamma in [1.2, 3].  Stage times from the library's own CUDA-event
report (lsrn_report: t_sketch = randn + mult, fused here; t_svd; t_iter), minimum
over `reps` solves.  One JSON line per gamma on stdout; the last line names the
best gamma and what lsrn_choose_gamma predicts from a probe solve at gamma = 2.
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_1109_5981_b200 import lsrn  # noqa: E402

M, N = 100_000, 1_000


def main():
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(1035)
    U, _ = torch.linalg.qr(torch.randn(M, N, generator=g, dtype=torch.float64, device=dev))
    V, _ = torch.linalg.qr(torch.randn(N, N, generator=g, dtype=torch.float64, device=dev))
    sig = torch.logspace(0, -6, N, dtype=torch.float64, device=dev)
    A = ((U * sig) @ V.T).contiguous()
    b = torch.randn(M, generator=g, dtype=torch.float64, device=dev)
    ctx = lsrn.Context()
    reps = int(os.environ.get("SWEEP_REPS", "3"))
    best = None
    for gamma in (1.2, 1.4, 1.6, 1.8, 2.0, 2.2, 2.5, 2.8, 3.0):
        rows = []
        for _ in range(reps + 1):
            _, rep = ctx.solve(A, b, M, N, gamma=gamma, tol=1e-14)
            rows.append(rep)
        rep = min(rows[1:], key=lambda d: d["t_total"])
        line = {"gamma": gamma, "s": rep["s"], "iters": rep["iters"], "t_sketch": rep["t_sketch"],
                "t_svd": rep["t_svd"], "t_iter": rep["t_iter"], "t_total": rep["t_total"]}
        print(json.dumps(line), flush=True)
        if best is None or line["t_total"] < best["t_total"]:
            best = line
    _, probe = ctx.solve(A, b, M, N, gamma=2.0, tol=1e-14)
    pred = lsrn.choose_gamma(probe, M, N, tol=1e-14, solver="lsqr")
    print(json.dumps({"best_gamma": best["gamma"], "best_t_total": best["t_total"],
                      "choose_gamma_from_probe_at_2": pred}), flush=True)


if __name__ == "__main__":
    main()
