"""Diagnose the CSR solve path against the dense path on the same matrix."""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, scipy.sparse as sp
from paper_1109_5981_b200 import lsrn
from synth.generate import small
from oracle.lsrn import solve as orc_solve

ctx = lsrn.Context()
def run(A, b, label):
    A = sp.csr_matrix(A); A.sort_indices()
    m, n = A.shape
    X = lsrn.Csr(torch.from_numpy(A.indptr.astype(np.int64)).cuda(), torch.from_numpy(A.indices.astype(np.int32)).cuda(),
                 torch.from_numpy(A.data).cuda())
    for solver in ("lsqr", "cs"):
        xc, rc = ctx.solve(X, torch.from_numpy(b).cuda(), m, n, solver=solver)
        xd, rd = ctx.solve(torch.from_numpy(A.toarray()).cuda(), torch.from_numpy(b).cuda(), m, n, solver=solver)
        orc = orc_solve(A, b, solver=solver)
        e = lambda x: np.linalg.norm(x.cpu().numpy() - orc["x"]) / np.linalg.norm(orc["x"])
        print(label, solver, "iters", rc["iters"], rd["iters"], orc["iters"], "r", rc["r"], rd["r"], "err csr %.3e dense %.3e" % (e(xc), e(xd)), flush=True)

p = small("c4")
A = p.to_scipy(); b = p.b.numpy()
cnt = np.bincount(A.indices, minlength=A.shape[1])
print("small c4", A.shape, "col counts min/max", cnt.min(), cnt.max(), "heavy thr", (A.shape[0] + 31) // 32, "n heavy cand", (cnt >= (A.shape[0]+31)//32).sum())
run(A, b, "small_c4")
rng = np.random.default_rng(0)
# light only: 3 random per row, 3000 x 200 -> each column ~45 < thr 94
B = sp.random(3000, 200, density=0.015, random_state=1, format="csr"); B.data = rng.standard_normal(B.nnz)
B = B + sp.csr_matrix(np.eye(3000, 200))
run(B, rng.standard_normal(3000), "light_only")
# heavy only: dense matrix as CSR
C = rng.standard_normal((2000, 40))
run(C, rng.standard_normal(2000), "heavy_only")
