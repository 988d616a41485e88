"""NEXT-4: reproduce the paper's Figure 1 (§6.2) on the GPU.

Left: kappa(AN) vs kappa_+(A) for several (r, s), with the estimate
(1 + sqrt(r/s)) / (1 - sqrt(r/s)) (Thm 4.4 with alpha ignored).
Right: LSQR iterations (adaptive mode, tol 1e-14) vs r/s, with the bound
(log eps - log 2) / log sqrt(r/s) (Thm 4.5).

A in R^{1e4 x 1e3} of rank r, A = U diag(sigma) V^T with U, V Haar (QR of
Gaussian) and sigma log-spaced 1 -> 1/kappa_+ (the paper's "randomly generated
with condition numbers ranged from 1e2 to 1e8").  As in the paper, each point
is the largest value over `runs` independent runs (different seeds for A and G).

The sketch and the solve go through the library (ctx.sketch, ctx.solve); the
SVD of the sketch and of A N here are measurement code (torch on the GPU), not
the product path.  Output: one JSON line per (r, s, kappa_+) point on stdout.
"""
import json
import math
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_1109_5981_b200 import lsrn  # noqa: E402

M, N = 10_000, 1_000
EPS = 1e-14


def make(r, kappa, seed, dev):
    g = torch.Generator(device=dev).manual_seed(seed)
    U, _ = torch.linalg.qr(torch.randn(M, r, generator=g, dtype=torch.float64, device=dev))
    V, _ = torch.linalg.qr(torch.randn(N, r, generator=g, dtype=torch.float64, device=dev))
    sig = torch.logspace(0, -math.log10(kappa), r, dtype=torch.float64, device=dev)
    A = (U * sig) @ V.T
    b = torch.randn(M, generator=g, dtype=torch.float64, device=dev)
    return A.contiguous(), b


def kappa_AN(ctx, A, gamma, seed):
    At = ctx.sketch(A, M, N, gamma, 0.0, seed=seed)               # s x n, the library's G A
    _, S, Vh = torch.linalg.svd(At, full_matrices=False)
    s = At.shape[0]
    r = int((S > max(s, N) * 2.0 ** -52 * S[0]).sum())          # rank rule C4
    Nm = Vh[:r].T / S[:r]
    sv = torch.linalg.svdvals(A @ Nm)
    return float(sv[0] / sv[-1]), r, s


def main():
    runs = int(os.environ.get("FIG1_RUNS", "5"))
    dev = "cuda"
    ctx = lsrn.Context()
    kappas = [1e2, 1e3, 1e4, 1e5, 1e6, 1e7, 1e8]
    for r in (1000, 800, 500):
        for gamma in (1.2, 1.5, 2.0, 3.0):
            for kp in kappas:
                worst_k, worst_it = 0.0, 0
                for run in range(runs):
                    A, b = make(r, kp, 1000 * run + r, dev)
                    kap, rr, s = kappa_AN(ctx, A, gamma, seed=77 + run)
                    _, rep = ctx.solve(A, b, M, N, gamma=gamma, tol=EPS, mode="adaptive", seed=77 + run)
                    worst_k = max(worst_k, kap)
                    worst_it = max(worst_it, int(rep["iters"]))
                rs = rr / s
                est = (1 + math.sqrt(rs)) / (1 - math.sqrt(rs))
                it_bound = (math.log(EPS) - math.log(2)) / math.log(math.sqrt(rs))
                print(json.dumps({"r": r, "s": s, "rank_found": rr, "gamma": gamma, "kappa_plus": kp,
                                  "runs": runs, "kappa_AN_max": worst_k, "kappa_estimate": est,
                                  "lsqr_iters_max": worst_it, "iter_bound": it_bound}), flush=True)


if __name__ == "__main__":
    main()
