"""Pins for oracle/bounds.py and oracle/krylov.py (no GPU).

bounds: paper values (tests/golden/paper_values.json: Table 3's 106 CS passes,
P:1283-1284; 84 LSQR iterations <= the Thm 4.5 bound; κ < 3 at s = 4r, P:294-296;
κ < 6 at s = 2r; N_iter ~ 100 at γ = 2), SPEC's sigma_bounds
example, the identity (σU-σL)/(σU+σL) = α + sqrt(r/s).
CS (Alg. 3, reading C1): the closed-form Chebyshev error polynomial on a diagonal
operator at EVERY pass (numpy.polynomial.chebyshev as the library routine), which
fails for the literal k = 1 step of P:706; the c = 0 collapse.
LSQR: identity and diag(1,2,4), fixed count vs numpy lstsq.
"""
import json
import math
import os

import numpy as np
import pytest
from numpy.polynomial import chebyshev as npcheb

from oracle import bounds
from oracle.krylov import chebyshev, cs_schedule, lsqr


def _paper(golden_dir):
    with open(os.path.join(golden_dir, "paper_values.json")) as f:
        return json.load(f)


def test_table3_counts(golden_dir):
    pv = _paper(golden_dir)
    t = pv["table3_cs_iterations"]
    r, s, eps = t["r"], t["s"], t["eps"]
    lo, hi = bounds.sigma_bounds(s, r, bounds.default_alpha(s))
    assert bounds.cs_passes(lo, hi, eps) == t["value"]                 # 106
    assert pv["table3_lsqr_iterations"]["value"] <= bounds.lsqr_count(eps, r, s)  # 84 <= 96


def test_bound_values(golden_dir):
    pv = _paper(golden_dir)
    # r=100, s=400, α=0.1 -> σ_U = 0.125, σ_L = 0.03125
    lo, hi = bounds.sigma_bounds(400, 100, 0.1)
    assert abs(hi - 0.125) < 1e-15 and abs(lo - 0.03125) < 1e-16
    assert bounds.kappa_bound(400, 100, 1e-12) < pv["kappa_s_eq_4r"]["value"] + 1e-9
    assert bounds.kappa_bound(400, 200, 1e-12) < pv["kappa_s_gt_2r"]["value"]
    # γ = 2, ε = 1e-14, full rank: N_iter ≈ 100
    n_it = bounds.lsqr_count(pv["eps_default"]["value"], 1000, 2000)
    assert abs(n_it - pv["niter_gamma2"]["value"]) <= 5
    # erratum of S:249/S:316: ⌈95.014⌉ = 96
    assert bounds.lsqr_count(1e-14, 1, 2) == 96
    assert bounds.lsqr_count(1e-14, 1, 16) == 24
    assert bounds.lsqr_count(2.0, 1, 4) == 0
    for s, r in [(200, 100), (4000, 1800), (2048, 1024), (40000, 20000)]:
        a = bounds.default_alpha(s)
        lo, hi = bounds.sigma_bounds(s, r, a)
        assert abs((hi - lo) / (hi + lo) - (a + math.sqrt(r / s))) < 1e-15
    assert bounds.cs_passes(2.0, 2.0, 1e-14) == 1                      # c = 0


def _T(k, x):
    return npcheb.chebval(x, [0] * k + [1])


def test_cs_closed_form_every_pass():
    sl, su = 0.3, 1.7
    d, c = (su * su + sl * sl) / 2, (su * su - sl * sl) / 2
    sig = np.linspace(sl, su, 25)
    xs = np.random.default_rng(0).standard_normal(25)
    A = np.diag(sig)
    b = A @ xs
    for k in range(12):
        x = chebyshev(lambda v: A @ v, lambda u: A.T @ u, b, sl, su, k + 1)
        ratio = (xs - x) / xs
        pred = _T(k + 1, (d - sig ** 2) / c) / _T(k + 1, d / c)
        assert np.max(np.abs(ratio - pred)) < 1e-12, k
    # the literal k = 1 step of P:706 (alpha = d - c^2/(2d)) breaks the closed form
    sched = cs_schedule(d, c, 2)
    lit_alpha1 = d - c * c / (2 * d)
    assert abs(sched[1][1] - lit_alpha1) > 0.1


def test_cs_c0_collapse():
    A = 2.0 * np.eye(5)
    b = np.arange(1.0, 6.0)
    x = chebyshev(lambda v: A @ v, lambda u: A.T @ u, b, 2.0, 2.0, 1)
    assert np.allclose(x, b / 2, rtol=0, atol=1e-15)


def test_lsqr_small_cases():
    b = np.random.default_rng(1).standard_normal(10)
    I = np.eye(10)
    y, it, _ = lsqr(lambda v: I @ v, lambda u: I @ u, b, iters=2)
    assert np.allclose(y, b, atol=1e-14)
    D = np.diag([1.0, 2.0, 4.0])
    y, it, _ = lsqr(lambda v: D @ v, lambda u: D @ u, np.array([1.0, 2.0, 4.0]), iters=3)
    assert np.allclose(y, 1.0, atol=1e-12)
    y, it, info = lsqr(lambda v: D @ v, lambda u: D @ u, np.zeros(3), iters=3)
    assert it == 0 and not np.any(y)


def test_lsqr_fixed_and_adaptive_vs_lstsq():
    rng = np.random.default_rng(2)
    U, _ = np.linalg.qr(rng.standard_normal((300, 20)))
    V, _ = np.linalg.qr(rng.standard_normal((20, 20)))
    A = (U * np.linspace(1.0, 0.2, 20)) @ V.T
    b = rng.standard_normal(300)
    ref = np.linalg.lstsq(A, b, rcond=None)[0]
    y, it, _ = lsqr(lambda v: A @ v, lambda u: A.T @ u, b, iters=60)
    assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)
    y2, it2, info = lsqr(lambda v: A @ v, lambda u: A.T @ u, b, tol=1e-14, max_iter=200,
                         mode="adaptive")
    assert info["converged"] and it2 < 200
    assert np.linalg.norm(y2 - ref) <= 1e-11 * np.linalg.norm(ref)
    # CS with exact bounds converges to the same solution
    lo, hi = 0.2 - 1e-12, 1.0 + 1e-12
    x = chebyshev(lambda v: A @ v, lambda u: A.T @ u, b, lo, hi, bounds.cs_passes(lo, hi, 1e-14))
    assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("kind,tol,seed", [("precond", 1e-14, 1), ("precond", 1e-10, 2), ("precond", 1e-14, 3),
                                           ("plain", 1e-8, 4), ("plain", 1e-6, 5), ("rankdef", 1e-10, 6),
                                           ("wide", 1e-12, 7)])
def test_lsqr_adaptive_stop_matches_scipy(kind, tol, seed):
    """Reading C5's adaptive mode is the Paige-Saunders stopping rule with atol = btol = tol:
    ||r|| <= tol ||b|| + tol ||A|| ||x||  or  ||A^T r|| <= tol ||A|| ||r||, ||A|| the running
    Frobenius estimate.  scipy.sparse.linalg.lsqr implements the same published rule (its
    ||x|| is a recurrence estimate, conlim disabled here), so the two stop within one
    iteration of each other on fixed operators -- a wrong ||A^T r|| estimate (e.g. a stale
    alpha) or a wrong ||A|| would shift the count by several.  (On ill-conditioned plain
    operators at tight tolerances the count itself is not reproducible across fp64
    implementations -- reading C5 -- so those stay at tol >= 1e-8.)"""
    scipy_lsqr = pytest.importorskip("scipy.sparse.linalg").lsqr
    rng = np.random.default_rng(seed)
    if kind == "precond":            # what LSRN iterates on: an orthonormal-ish A N (kappa ~ 6)
        Q, _ = np.linalg.qr(rng.standard_normal((400, 60)))
        A = Q * np.linspace(1.0, 1.0 / 6.0, 60)
    elif kind == "plain":
        A = rng.standard_normal((300, 40)) * np.logspace(0, -1, 40)
    elif kind == "rankdef":
        A = rng.standard_normal((200, 30)) @ rng.standard_normal((30, 50))[:, :50] @ np.diag(np.logspace(0, -2, 50))
    else:
        A = rng.standard_normal((40, 300))
    b = rng.standard_normal(A.shape[0])
    y, it, info = lsqr(lambda v: A @ v, lambda u: A.T @ u, b, tol=tol, max_iter=2000, mode="adaptive")
    res = scipy_lsqr(A, b, atol=tol, btol=tol, conlim=1e300, iter_lim=2000)
    itn = res[2]
    assert info["converged"]
    assert abs(it - itn) <= 1, (it, itn)
    assert np.linalg.norm(y - res[0]) <= max(1e-6, 1e3 * tol) * np.linalg.norm(res[0])
