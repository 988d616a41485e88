"""precision = 1 (LSRN_COMPENSATED, reading C18(ii)) against the oracle's
long-double product mode (oracle/lsrn.py, extended=True).

With fp64 products the x parity floor is ~15 kappa(A) u: up to
1.7e-9 on c1's kappa = 1e6 shape, so the fp64 tests gate x at max(1e-9, 20 kappa u).
Here the products carry N v and A^T u as double-double pairs with compensated
accumulation, and x is held to the north star's literal bar, relative 2-norm
<= 1e-9 with no kappa term, plus the Thm 4.5 A-norm form at 1e-12.
"""
import numpy as np
import pytest
import torch

from oracle.lsrn import solve as orc_solve
from synth.generate import make_problem, small

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1109_5981_b200 import lsrn
    c = lsrn.Context()
    yield c
    c.close()


def _rel(x, ref):
    return float(np.linalg.norm(x - ref) / np.linalg.norm(ref))


def _anorm(A, x, ref):
    return float(np.linalg.norm(A @ (x - ref)) / np.linalg.norm(A @ ref))


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
@pytest.mark.parametrize("seed", [None, 11, 12])
def test_c1_compensated_meets_literal_bar(ctx, solver, seed):
    p = make_problem("c1", seed=seed) if seed is not None else make_problem("c1")
    A, b = p.X.numpy(), p.b.numpy()
    orc = orc_solve(A, b, solver=solver, extended=True)
    x1, rep1 = ctx.solve(p.X.cuda(), p.b.cuda(), p.m, p.n, solver=solver, precision=1)
    x0, rep0 = ctx.solve(p.X.cuda(), p.b.cuda(), p.m, p.n, solver=solver, precision=0)
    assert rep1["r"] == orc["r"] == 100 and rep1["iters"] == orc["iters"] == rep0["iters"]
    x1, x0 = x1.cpu().numpy(), x0.cpu().numpy()
    rel1, rel0 = _rel(x1, orc["x"]), _rel(x0, orc["x"])
    assert rel1 <= 1e-9, (rel1, rel0)
    assert _anorm(A, x1, orc["x"]) <= 1e-12
    # the compensated products remove the kappa u floor of the fp64 ones
    assert rel1 < 0.1 * rel0 or rel0 < 1e-11, (rel1, rel0)


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_small_configs_compensated(ctx, solver, name):
    """Rank-deficient tall (c2), wide with the Tikhonov block (c3), tall graded columns (c5)."""
    p = small(name)
    A = p.dense_A().numpy()
    b = p.b.numpy()
    orc = orc_solve(A, b, solver=solver, lam=p.lam, extended=True)
    x, rep = ctx.solve(p.X.cuda(), p.b.cuda(), p.m, p.n, solver=solver, lam=p.lam, precision=1)
    assert rep["r"] == orc["r"] and rep["s"] == orc["s"] and rep["iters"] == orc["iters"]
    x = x.cpu().numpy()
    Aop = np.vstack([A, p.lam * np.eye(p.n)]) if (p.lam > 0 and p.tall) else A
    assert _rel(x, orc["x"]) <= 1e-9
    assert _anorm(Aop, x, orc["x"]) <= 1e-12


def test_adaptive_lsqr_compensated(ctx):
    p = make_problem("c1")
    A, b = p.X.numpy(), p.b.numpy()
    orc = orc_solve(A, b, solver="lsqr", mode="adaptive", extended=True)
    x, rep = ctx.solve(p.X.cuda(), p.b.cuda(), p.m, p.n, solver="lsqr", mode="adaptive", precision=1)
    assert rep["converged"] == 1 and abs(rep["iters"] - orc["iters"]) <= 2
    assert _rel(x.cpu().numpy(), orc["x"]) <= 1e-9


def test_compensated_ragged_multi_block(ctx):
    """Rows spread over many blocks with a ragged last block, k not a multiple of 32."""
    p = make_problem("c1", m=9001, n=77)
    A, b = p.X.numpy(), p.b.numpy()
    orc = orc_solve(A, b, solver="cs", extended=True)
    x, rep = ctx.solve(p.X.cuda(), p.b.cuda(), p.m, p.n, solver="cs", precision=1)
    assert rep["iters"] == orc["iters"]
    assert _rel(x.cpu().numpy(), orc["x"]) <= 1e-9


def test_compensated_deterministic_and_graph_reuse(ctx):
    p = make_problem("c1")
    X, b = p.X.cuda(), p.b.cuda()
    xa, _ = ctx.solve(X, b, p.m, p.n, solver="lsqr", precision=1)
    xa = xa.clone()
    xb, _ = ctx.solve(X, b, p.m, p.n, solver="lsqr", precision=1)     # reused graph
    assert torch.equal(xa, xb)
    xc, _ = ctx.solve(X, b, p.m, p.n, solver="lsqr", precision=0)     # different graph: fp64 products
    assert not torch.equal(xa, xc)


def test_compensated_csr_unsupported(ctx):
    from paper_1109_5981_b200 import lsrn
    q = small("c4")
    X = lsrn.Csr(q.rowptr.cuda(), q.colind.cuda(), q.val.cuda())
    with pytest.raises(RuntimeError, match="EUNSUPPORTED"):
        ctx.solve(X, q.b.cuda(), q.m, q.n, solver="cs", precision=1)
