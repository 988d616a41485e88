"""Reading C18 measured: how the fp64 error of an LSRN solve against the exact x* grows
with n at fixed kappa (the c1 recipe, kappa = 1e6, m = n + 1900, gamma = 1.5 -- the
shapes of tests/test_gpu_parity.py::test_wide_rows_vs_pseudoinverse).  For each n: the
GPU solve (LSQR, CS) and the oracle's solve in fp64 (and, up to n = 2000, with long-
double products) against x* = V diag(1/sigma) U^T b from the generator's factors:
relative 2-norm error and the A-norm form ||A dx|| / ||A x*||."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle.lsrn import solve as orc_solve  # noqa: E402
from synth.generate import make_problem  # noqa: E402

ns = [int(a) for a in sys.argv[1:]] or [250, 1000, 2000, 4100, 9000]
gpu = torch.cuda.is_available()
if gpu:
    from paper_1109_5981_b200 import lsrn
    ctx = lsrn.Context()
for n in ns:
    p = make_problem("c1", m=n + 1900, n=n, keep_factors=True)
    U, V, sig = p.meta["U"].numpy(), p.meta["V"].numpy(), p.meta["sigma"].numpy()
    b = p.b.numpy()
    xs = V @ ((U.T @ b) / sig)

    def errs(x):
        dx = x - xs
        return (float(np.linalg.norm(dx) / np.linalg.norm(xs)),
                float(np.linalg.norm(sig * (V.T @ dx)) / np.linalg.norm(sig * (V.T @ xs))))
    for solver in ("lsqr", "cs"):
        row = {"n": n, "m": n + 1900, "kappa": float(sig[0] / sig[-1]), "solver": solver}
        if gpu:
            x, rep = ctx.solve(p.X.cuda(), p.b.cuda(), p.m, p.n, solver=solver, gamma=1.5)
            row["gpu_rel"], row["gpu_anorm"] = errs(x.cpu().numpy())
        if n <= 4100:
            A = p.X.numpy()
            o = orc_solve(A, b, solver=solver, gamma=1.5)
            row["oracle_rel"], row["oracle_anorm"] = errs(o["x"])
            if n <= 2000:
                oe = orc_solve(A, b, solver=solver, gamma=1.5, extended=True, At=o["At"])
                row["oracle_ext_rel"], row["oracle_ext_anorm"] = errs(oe["x"])
        print(json.dumps(row), flush=True)
