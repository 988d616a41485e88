"""The two iterative solvers of Alg. 1 step 6, on an abstract operator (oracle).

LSQR: Paige & Saunders, "LSQR: an algorithm for sparse linear equations and
sparse least squares", ACM TOMS 8 (1982) -- cited by the paper at P:107-109
(§1) and P:185-187 (§2.1) but not spelled out there.  The recurrences below are
the published bidiagonalisation + Givens QR of that paper (§4.1 of P&S), started
from y0 = 0 so the iterates stay in range(Abar^T).

Stopping (reading C5; the paper is silent):
  mode 'predictable' : exactly `iters` iterations, iters = Thm 4.5 count at
                       alpha = 0 (bounds.lsqr_count, Fig. 1 right),
                       fewer only if the bidiagonalisation terminates exactly
                       (alpha or beta == 0: y is then exact, P&S §3);
  mode 'adaptive'    : P&S tests with atol = btol = tol:
                       ||r|| <= tol ||b|| + tol ||Abar|| ||y||   or
                       ||Abar^T r|| <= tol ||Abar|| ||r||,
                       capped at max_iter (2x the Thm 4.5 count).

CS: Alg. 3 verbatim except the k = 1 step size, which the paper
prints as "alpha <- d - c^2/(2d)"; reading C1 uses its reciprocal
alpha_1 = 1 / (d - c^2/(2d)) (the classical Chebyshev recurrence; pinned by the
closed form in tests/test_oracle_krylov.py).  beta is evaluated before alpha in
each pass, so beta_k uses alpha_{k-1}.

Both take `matvec(y) = Abar y` and `rmatvec(u) = Abar^T u`.  Vectors are fp64
unless the operator returns long double (the extended-precision product mode of
reading C18), in which case the recurrences run in long double too.
"""
import math

import numpy as np


def _norm(x):
    return np.sqrt(np.sum(x * x))


def lsqr(matvec, rmatvec, b, iters=None, tol=1e-14, max_iter=None, mode="predictable"):
    """Return (y, n_iter, info). `iters` is the fixed count for 'predictable'."""
    if mode not in ("predictable", "adaptive"):
        raise ValueError("mode must be 'predictable' or 'adaptive'")
    cap = iters if mode == "predictable" else max_iter
    if cap is None:
        raise ValueError("iteration count / cap required")
    beta = _norm(b)
    if beta == 0:                                   # b = 0 -> y = 0
        return np.zeros_like(rmatvec(b)), 0, dict(converged=True, rnorm=0.0, arnorm=0.0)
    u = b / beta
    v = rmatvec(u)
    alpha = _norm(v)
    y = np.zeros_like(v)
    if alpha == 0:
        return y, 0, dict(converged=True, rnorm=float(beta), arnorm=0.0)
    v = v / alpha
    w = v.copy()
    phibar, rhobar = beta, alpha
    bnorm = beta
    anorm2 = 0.0
    converged = mode == "predictable"
    it = 0
    rnorm, arnorm = beta, alpha * beta
    while it < cap:
        it += 1
        # bidiagonalisation (P&S eq. 3.2)
        u = matvec(v) - alpha * u
        beta_new = _norm(u)
        if beta_new > 0:
            u = u / beta_new
        anorm2 = anorm2 + alpha * alpha + beta_new * beta_new
        v = rmatvec(u) - beta_new * v
        alpha_new = _norm(v)
        if alpha_new > 0:
            v = v / alpha_new
        # Givens rotation (P&S eq. 4.6-4.12)
        rho = np.hypot(rhobar, beta_new)
        c = rhobar / rho
        sn = beta_new / rho
        theta = sn * alpha_new
        rhobar = -c * alpha_new
        phi = c * phibar
        phibar = sn * phibar
        y = y + (phi / rho) * w
        w = v - (theta / rho) * w
        alpha = alpha_new
        rnorm = phibar
        arnorm = phibar * alpha_new * abs(c)
        if alpha_new == 0 or beta_new == 0:
            # the bidiagonalisation terminated: y is the exact LS solution (P&S §3)
            converged = True
            break
        if mode == "adaptive":
            anorm = math.sqrt(float(anorm2))
            ynorm = float(_norm(y))
            if float(rnorm) <= tol * float(bnorm) + tol * anorm * ynorm or \
               float(arnorm) <= tol * anorm * float(rnorm):
                converged = True
                break
    return y, it, dict(converged=converged, rnorm=float(rnorm), arnorm=float(arnorm))


def cs_schedule(d, c, passes):
    """[(beta_k, alpha_k)] for k = 0..passes-1 (Alg. 3 line 4, reading C1)."""
    out = []
    alpha = None
    for k in range(passes):
        if k == 0:
            beta, alpha = 0.0, 1.0 / d
        elif k == 1:
            beta = 0.5 * (c / d) ** 2
            alpha = 1.0 / (d - c * c / (2.0 * d))
        else:
            beta = (alpha * c / 2.0) ** 2
            alpha = 1.0 / (d - alpha * c * c / 4.0)
        out.append((beta, alpha))
    return out


def chebyshev(matvec, rmatvec, b, sig_l, sig_u, passes):
    """Alg. 3: returns x after `passes` loop passes (k = 0..passes-1)."""
    d = (sig_u ** 2 + sig_l ** 2) / 2.0
    c = (sig_u ** 2 - sig_l ** 2) / 2.0
    r = b.copy()
    x = None
    v = None
    for beta, alpha in cs_schedule(d, c, passes):
        atr = rmatvec(r)
        if v is None:
            v = np.zeros_like(atr)
            x = np.zeros_like(atr)
        v = beta * v + atr                    # line 5
        x = x + alpha * v                     # line 6
        r = r - alpha * matvec(v)             # line 7
    return x
