"""Pins for oracle/lsrn.py and oracle/brute.py (no GPU).

brute (tiny inputs): long-double Jacobi min-length solution vs numpy.linalg.lstsq
/ pinv (LAPACK, library pin); long-double ridge vs numpy.linalg.solve of the
normal equations (library pin).
lsrn (Alg. 1/2 + §5): x̂ = A^+ b (Thm 4.1) for tall/wide, full-rank and
rank-deficient, LSQR and CS; Tikhonov tall/wide vs ridge; b = 0
(S:307); x in range(A^T) and ||A^T(b - Ax)|| ~ 0 (north star invariants);
rank-deficiency reduces the LSQR count; Thm 4.5 A-norm form.
"""
import numpy as np
import pytest

from oracle import brute
from oracle.lsrn import solve
from synth.generate import small


def _rand_lowrank(m, n, r, seed, kappa=1e3):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, r)))
    V, _ = np.linalg.qr(rng.standard_normal((n, r)))
    sig = np.logspace(0, -np.log10(kappa), r)
    return (U * sig) @ V.T, V if m >= n else U


@pytest.mark.parametrize("shape,r", [((60, 12), 12), ((60, 12), 7), ((12, 60), 12), ((12, 60), 5)])
def test_brute_min_length_vs_lapack(shape, r):
    A, _ = _rand_lowrank(*shape, r, seed=r)
    b = np.random.default_rng(1).standard_normal(shape[0])
    x, rr = brute.min_length(A, b)
    assert rr == r
    ref = np.linalg.lstsq(A, b, rcond=1e-10)[0]
    assert np.linalg.norm(x - ref) <= 1e-10 * np.linalg.norm(ref)
    assert np.linalg.norm(x - np.linalg.pinv(A, rcond=1e-10) @ b) <= 1e-10 * np.linalg.norm(ref)


@pytest.mark.parametrize("shape", [(80, 10), (10, 80)])
def test_brute_ridge_vs_normal_equations(shape):
    rng = np.random.default_rng(2)
    A = rng.standard_normal(shape)
    b = rng.standard_normal(shape[0])
    lam = 0.7
    x = brute.ridge(A, b, lam)
    ref = np.linalg.solve(A.T @ A + lam ** 2 * np.eye(shape[1]), A.T @ b)
    assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
@pytest.mark.parametrize("shape,r", [((400, 20), 20), ((400, 20), 13), ((20, 400), 20), ((20, 400), 9)])
def test_lsrn_min_length(solver, shape, r):
    A, Vr = _rand_lowrank(*shape, r, seed=10 + r)
    b = np.random.default_rng(3).standard_normal(shape[0])
    rep = solve(A, b, gamma=2.0, tol=1e-14, seed=77, solver=solver)
    x_ref, rr = brute.min_length(A, b)
    assert rep["r"] == r == rr
    assert np.linalg.norm(rep["x"] - x_ref) <= 1e-9 * np.linalg.norm(x_ref)
    # invariants: x in range(A^T); A^T (b - A x) ~ 0
    x = rep["x"]
    rowspace = Vr if shape[0] >= shape[1] else np.linalg.svd(A, full_matrices=False)[2][:r].T
    assert np.linalg.norm(x - rowspace @ (rowspace.T @ x)) <= 1e-10 * np.linalg.norm(x)
    res = b - A @ x
    nA = np.linalg.norm(A, 2)
    assert np.linalg.norm(A.T @ res) <= nA * (1e-9 * np.linalg.norm(res) +
                                              1e-12 * (nA * np.linalg.norm(x) + np.linalg.norm(b)))


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
@pytest.mark.parametrize("shape", [(300, 15), (15, 300)])
def test_lsrn_tikhonov(solver, shape):
    rng = np.random.default_rng(4)
    A = rng.standard_normal(shape) * np.logspace(0, -3, shape[1])
    b = rng.standard_normal(shape[0])
    lam = 1e-2
    rep = solve(A, b, gamma=2.0, lam=lam, tol=1e-14, seed=5, solver=solver)
    ref = brute.ridge(A, b, lam)
    assert np.linalg.norm(rep["x"] - ref) <= 1e-9 * np.linalg.norm(ref)
    # huge lambda drives x -> 0
    big = solve(A, b, lam=1e8 * np.linalg.norm(A, 2), seed=5, solver=solver)["x"]
    assert np.linalg.norm(big) <= 1e-6 * np.linalg.norm(np.linalg.lstsq(A, b, rcond=None)[0])


def test_lsrn_b_zero_and_rank_deficiency_counts():
    A, _ = _rand_lowrank(500, 40, 40, seed=1)
    rep = solve(A, np.zeros(500), solver="lsqr")
    assert rep["iters"] == 0 and not np.any(rep["x"])
    assert not np.any(solve(A, np.zeros(500), solver="cs")["x"])
    Ad, _ = _rand_lowrank(500, 40, 24, seed=2)
    b = np.random.default_rng(0).standard_normal(500)
    full = solve(A, b, solver="lsqr")
    defic = solve(Ad, b, solver="lsqr")
    assert defic["r"] == 24 and defic["iters"] < full["iters"]
    ad = solve(Ad, b, solver="lsqr", mode="adaptive")
    assert ad["converged"] and ad["iters"] <= 2 * defic["lsqr_count"]


def test_lsrn_c1_small_all_modes():
    """c1 recipe at full c1 size (2000 x 100, κ = 1e6): LSQR/CS/extended agree (C18)."""
    p = small("c1")
    A = p.X.numpy()
    b = p.b.numpy()
    ref = np.linalg.lstsq(A, b, rcond=None)[0]          # LAPACK gelsd (library pin)
    reps = {}
    for solver in ("lsqr", "cs"):
        for ext in (False, True):
            rep = solve(A, b, solver=solver, extended=ext)
            reps[(solver, ext)] = rep
            assert rep["r"] == 100 and rep["s"] == 200
            # Thm 4.5 A-norm form: ||A(x - x*)|| <= eps-ish ||A x*||
            assert np.linalg.norm(A @ (rep["x"] - ref)) <= 1e-11 * np.linalg.norm(A @ ref)
    assert reps[("lsqr", False)]["iters"] == 96 and reps[("cs", False)]["iters"] == 133
    xl, xe = reps[("lsqr", False)]["x"], reps[("lsqr", True)]["x"]
    kappa = 1e6
    assert np.linalg.norm(xl - xe) <= max(1e-9, 20 * kappa * 2 ** -53) * np.linalg.norm(xe)
