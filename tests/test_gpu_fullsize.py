"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py uses.

The oracle cannot redo a full-size solve in seconds, so these tests check
  * sampled sketch entries, each recomputed one by one by the oracle
    (oracle.sketch.sketch_entries: G[i, :] regenerated, dot with column c);
  * closed forms: for c2 the generator's own factors give the exact
    min-length solution x* = V diag(1/sigma) U^T b, so x is checked
    against A^+ b directly; iteration counts against Thm 4.5 / Alg. 3 (P:643,
    P:694) and the rank against the generator's rank;
  * invariants at any size: x in range(A^T) and the normal equations.
  * at c2, the WHOLE sketch against the oracle's (relative Frobenius <= 1e-12,
    the north star's bar), since the oracle finishes it in under a minute.
Every BASELINE config runs: c2, c3 (3.2 GB), c4 (CSR, 1.4e8 nonzeros: sampled
sketch and a full CS solve), c5 (80 GB) and t4 (NEXT-2), in the launch
configuration bench.py times (default plans, one context).
"""
import numpy as np
import pytest
import torch

from oracle import bounds
from oracle.sketch import plan as orc_plan
from oracle.sketch import sketch_entries
from synth.generate import SKETCH_SEED, make_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1109_5981_b200 import lsrn
    c = lsrn.Context()
    yield c
    c.close()


def _sampled_sketch_check(At, Xcol, s, L, sx=1.0, si=0.0, nsamp=12, seed=0):
    """Compare nsamp entries of At (s x k, device) with the oracle, one by one."""
    rng = np.random.default_rng(seed)
    k = At.shape[1]
    rows = list(rng.integers(0, s, nsamp - 2)) + [0, s - 1]
    cols = list(rng.integers(0, k, nsamp - 2)) + [k - 1, 0]
    cols_data = {c: Xcol(c) for c in set(cols)}
    ref = sketch_entries(cols_data, rows, cols, SKETCH_SEED, sx, si, L=L)
    got = At[torch.tensor(rows), torch.tensor(cols)].cpu().numpy()
    # each entry is sx * (length-L dot product of N(0,1) draws with a column) + si * G: compare
    # against its natural scale sx * sqrt(sum_j X[j,c]^2) + si (the entry's standard deviation)
    scale = np.array([sx * np.linalg.norm(cols_data[c]) + si for c in cols])
    err = np.abs(got - ref) / scale
    assert err.max() <= 1e-12, (err.max(), rows, cols)


def test_c2_full_sketch_vs_oracle(ctx):
    """The whole c2 sketch (4000 x 2000 from 1e5 x 2000) against the oracle's blocked
    explicit-G product (oracle.sketch.sketch): relative Frobenius <= 1e-12."""
    from oracle.sketch import sketch as orc_sketch
    p = make_problem("c2", device="cuda")
    At = ctx.sketch(p.X, p.m, p.n, 2.0, 0.0, seed=SKETCH_SEED).cpu().numpy()
    X = p.X.cpu().numpy()
    del p
    ref = orc_sketch(X, 4000, SKETCH_SEED, block=8192, precise=True)
    rel = np.linalg.norm(At - ref) / np.linalg.norm(ref)
    assert rel <= 1e-12, rel


def test_c2_full(ctx):
    p = make_problem("c2", device="cuda", keep_factors=True)
    m, n = p.m, p.n
    At = ctx.sketch(p.X, m, n, 2.0, 0.0, seed=SKETCH_SEED)
    s = At.shape[0]
    assert s == 4000
    Xc = p.X
    _sampled_sketch_check(At, lambda c: Xc[:, c].cpu().numpy(), s, m)
    del At
    U = p.meta["U"].cpu().numpy()
    V = p.meta["V"].cpu().numpy()
    sig = p.meta["sigma"].cpu().numpy()
    b = p.b.cpu().numpy()
    xstar = V @ ((U.T @ b) / sig)                     # A^+ b from the generator's SVD
    del U
    for solver in ("lsqr", "cs"):
        x, rep = ctx.solve(p.X, p.b, m, n, solver=solver, seed=SKETCH_SEED)
        assert rep["r"] == 1800 and rep["s"] == 4000
        alpha = bounds.default_alpha(s)
        sl, su = bounds.sigma_bounds(s, 1800, alpha)
        want = bounds.lsqr_count(1e-14, 1800, s) if solver == "lsqr" else bounds.cs_passes(sl, su, 1e-14)
        assert rep["iters"] == want == (83 if solver == "lsqr" else 89)
        xg = x.cpu().numpy()
        rel = np.linalg.norm(xg - xstar) / np.linalg.norm(xstar)
        assert rel <= 1e-9, (solver, rel)
        leak = np.linalg.norm(xg - V @ (V.T @ xg)) / np.linalg.norm(xg)    # x in range(A^T)
        assert leak <= 1e-10, leak


def test_c3_full_tikhonov(ctx):
    p = make_problem("c3", device="cuda")
    m, n, lam = p.m, p.n, p.lam
    pl = orc_plan(m, n, 2.0, lam)
    At = ctx.sketch(p.X, m, n, 2.0, lam, seed=SKETCH_SEED)
    Xc = p.X                                          # X = A^T (n x m)
    _sampled_sketch_check(At, lambda c: Xc[:, c].cpu().numpy(), pl["s"], n, pl["sigma_x"], pl["sigma_i"])
    del At
    for solver in ("lsqr", "cs"):
        x, rep = ctx.solve(p.X, p.b, m, n, solver=solver, lam=lam)
        assert rep["r"] == 2000
        # ridge normal equations A^T (b - A x) = lam^2 x  (W = lam I)
        A_T = p.X
        res = A_T @ (p.b - A_T.T @ x) - lam ** 2 * x
        fro = torch.linalg.norm(A_T)                   # ||A||_F >= ||A||_2: a looser, cheap scale
        scale = fro ** 2 * torch.linalg.norm(x) + torch.linalg.norm(A_T @ p.b)
        assert float(torch.linalg.norm(res) / scale) <= 1e-12


def test_c4_full_sketch(ctx):
    from paper_1109_5981_b200.lsrn import Csr
    p = make_problem("c4", device="cuda")
    X = Csr(p.rowptr, p.colind, p.val)
    At = ctx.sketch(X, p.m, p.n, 2.0, 0.0, seed=SKETCH_SEED)
    A = p.to_scipy().tocsc()

    def col(c):
        return np.asarray(A[:, c].toarray()).ravel()
    _sampled_sketch_check(At, col, At.shape[0], p.m, nsamp=8)


def test_c4_full_solve(ctx):
    """c4 end to end with CS (the config's solver): Alg. 3's pass count from the Thm 4.4
    bounds at r = k = 2e4, s = 4e4, and the normal equations
    A^T (b - A x) = 0 to the iteration tolerance (Thm 4.5's A-norm bound, as for c5)."""
    from paper_1109_5981_b200.lsrn import Csr
    p = make_problem("c4", device="cuda")
    X = Csr(p.rowptr, p.colind, p.val)
    x, rep = ctx.solve(X, p.b, p.m, p.n, solver="cs")
    s = 40000
    sl, su = bounds.sigma_bounds(s, 20000, bounds.default_alpha(s))
    assert rep["r"] == 20000 and rep["iters"] == bounds.cs_passes(sl, su, 1e-14)
    A = p.to_scipy()
    xh, b = x.cpu().numpy(), p.b.cpu().numpy()
    g = A.T @ (b - A @ xh)
    an = np.sqrt((A.data ** 2).sum())                     # ||A||_F >= ||A||_2
    assert np.linalg.norm(g) <= 10 * 2e-14 * an * np.linalg.norm(b)


def test_c5_full(ctx):
    p = make_problem("c5", device="cuda")
    m, n = p.m, p.n
    At = ctx.sketch(p.X, m, n, 2.0, 0.0, seed=SKETCH_SEED)
    Xc = p.X
    _sampled_sketch_check(At, lambda c: Xc[:, c].cpu().numpy(), At.shape[0], m, nsamp=6)
    del At
    x, rep = ctx.solve(p.X, p.b, m, n, solver="cs")
    s = 20000
    sl, su = bounds.sigma_bounds(s, 10000, bounds.default_alpha(s))
    assert rep["r"] == 10000 and rep["iters"] == bounds.cs_passes(sl, su, 1e-14) == 99
    # normal equations A^T (b - A x) = 0 up to the iteration tolerance: Thm 4.5 bounds
    # ||A(x - x*)|| by ~2 eps ||A x*||, so ||A^T r|| <~ ||A||_2 2 eps ||b||; checked with the
    # cheaper ||A||_F >= ||A||_2 and a 10x margin
    r = p.b - p.X @ x
    g = p.X.T @ r
    an = float(torch.linalg.norm(p.X))
    assert float(torch.linalg.norm(g)) <= 10 * 2e-14 * an * float(torch.linalg.norm(p.b))


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
def test_t4_full(ctx, solver):
    """NEXT-2 at its full size (1024 x 4e6, the CSR of A^T, 21 nonzeros per column of A):
    sampled sketch entries one by one against the oracle, the Table 3 CS pass count
    (106), and the min-length characterisation of an under-determined solve:
    A x = b (consistent, full row rank) and x in range(A^T)."""
    from paper_1109_5981_b200.lsrn import Csr
    p = make_problem("t4", device="cuda")
    m, n = p.m, p.n
    X = Csr(p.rowptr, p.colind, p.val)                    # rows of X = columns of A
    At = ctx.sketch(X, m, n, 2.0, 0.0, seed=SKETCH_SEED)
    assert At.shape == (2048, 1024)
    Xs = p.to_scipy().T.tocsc()                           # X = A^T as CSC: column c = row c of A

    def col(c):
        return np.asarray(Xs[:, c].toarray()).ravel()
    _sampled_sketch_check(At, col, 2048, n, nsamp=8)
    del At
    x, rep = ctx.solve(X, p.b, m, n, solver=solver)
    if solver == "cs":
        assert rep["iters"] == 106
    A = p.to_scipy()                                      # m x n
    xh = x.cpu().numpy()
    b = p.b.cpu().numpy()
    res = np.linalg.norm(A @ xh - b) / np.linalg.norm(b)
    assert res <= 1e-10, res
    # x = A^T y for the y solving (A A^T) y = A x: the component outside range(A^T) vanishes
    AAt = (A @ A.T).toarray()
    y = np.linalg.solve(AAt, A @ xh)
    leak = np.linalg.norm(xh - A.T @ y) / np.linalg.norm(xh)
    assert leak <= 1e-10, leak
