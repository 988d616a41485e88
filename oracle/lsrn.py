"""LSRN drivers: Alg. 1 (m >= n), Alg. 2 (m < n) and the §5 Tikhonov forms (oracle).

Alg. 1                       Alg. 2
 1 s = ceil(gamma n)                      1 s = ceil(gamma m)
 2 G = randn(s, m)                        2 G = randn(n, s)
 3 Ã = G A                                3 Ã = A G
 4 SVD Ã = Ũ Σ̃ Ṽ^T, r = rank(Ã)           4 SVD, only Ũ, Σ̃ needed
 5 N = Ṽ Σ̃^-1                            5 M = Ũ Σ̃^-1
 6 y = argmin ||A N y - b|| (min-length)  6 x = min-length argmin ||M^T A x - M^T b||
 7 x = N y                                7 return x

§5, W = lambda I, penalty (1/2)||Wx||^2 = (lambda^2/2)||x||^2
(reading C11): tall -> Alg. 1 on [A; lambda I], rhs [b; 0]; wide -> Alg. 2 on
[A/lambda, I_m], x = z / lambda.

All of it is written through the tall-form long operator (sketch.py)
    P t   = [sigma_X X t ; sigma_I t]        (R^k -> R^{L(+k)})
    P^T u = sigma_X X^T u_X + sigma_I u_I    (R^{L(+k)} -> R^k)
tall:  Abar = P N          (y in R^r),      rhs = b (or [b; 0]),  x = N y
wide:  Abar = N^T P^T      (z in R^{L(+k)}), rhs = N^T b,          x = sigma_X z_X
(for the wide case the paper's Ũ is the V of the tall-form sketch, so M = N.)
"""
import time

import numpy as np

from . import bounds as _bounds
from .krylov import chebyshev, lsqr
from .precond import factor
from .sketch import plan as _plan
from .sketch import sketch as _sketch


def _is_sparse(A):
    return hasattr(A, "tocsr") and not isinstance(A, np.ndarray)


class LongOperator:
    """P and P^T of the tall form; `extended` carries products in long double."""

    def __init__(self, X, sigma_x, sigma_i, extended=False):
        self.X = X
        self.L, self.k = X.shape
        self.sx = sigma_x
        self.si = sigma_i
        self.ext = extended and not _is_sparse(X)
        self.Xe = X.astype(np.longdouble) if self.ext else None
        self.dim = self.L + (self.k if sigma_i != 0.0 else 0)

    def P(self, t):
        if self.ext:
            xt = self.Xe @ np.asarray(t, dtype=np.longdouble)
        else:
            xt = self.X @ t
        top = self.sx * xt if self.sx != 1.0 else xt
        if self.si == 0.0:
            return top
        return np.concatenate([top, self.si * t])

    def PT(self, u):
        uX = u[: self.L]
        if self.ext:
            out = self.Xe.T @ np.asarray(uX, dtype=np.longdouble)
        else:
            out = self.X.T @ uX
        if self.sx != 1.0:
            out = self.sx * out
        if self.si != 0.0:
            out = out + self.si * u[self.L:]
        return out


def solve(A, b, gamma=2.0, lam=0.0, tol=1e-14, seed=5981, solver="lsqr",
          alpha=None, mode="predictable", extended=False, precise_g=True,
          sketch_block=4096, At=None):
    """Return a report dict: x, iters, r, s, sigma_l, sigma_u, stage times."""
    A_is_sparse = _is_sparse(A)
    m, n = A.shape
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (m,):
        raise ValueError("b must have length m")
    p = _plan(m, n, gamma, lam)
    X = A if p["tall"] else (A.T.tocsr() if A_is_sparse else np.ascontiguousarray(A.T))
    t0 = time.perf_counter()
    if At is None:
        At = _sketch(X, p["s"], seed, p["sigma_x"], p["sigma_i"], block=sketch_block,
                     precise=precise_g)
    t1 = time.perf_counter()
    N, sig, r = factor(At)
    t2 = time.perf_counter()
    s = p["s"]
    if alpha is None:
        alpha = _bounds.default_alpha(s)
    sig_l, sig_u = _bounds.sigma_bounds(s, r, alpha)
    op = LongOperator(X, p["sigma_x"], p["sigma_i"], extended=extended)
    Ne = N.astype(np.longdouble) if op.ext else N
    if p["tall"]:
        rhs = b if p["sigma_i"] == 0.0 else np.concatenate([b, np.zeros(n)])
        mv = lambda y: op.P(Ne @ y)                      # Abar y = A (N y)
        rmv = lambda u: Ne.T @ op.PT(u)                  # Abar^T u = N^T (A^T u)
    else:
        rhs = Ne.T @ (b.astype(np.longdouble) if op.ext else b)   # M^T b
        mv = lambda z: Ne.T @ op.PT(z)                   # Abar z = M^T (B z)
        rmv = lambda q: op.P(Ne @ q)                     # Abar^T q = B^T (M q)
    kl = _bounds.lsqr_count(tol, r, s, 0.0)
    if solver == "lsqr":
        if mode == "predictable":
            sol, iters, info = lsqr(mv, rmv, rhs, iters=kl, tol=tol, mode="predictable")
        else:
            sol, iters, info = lsqr(mv, rmv, rhs, tol=tol, max_iter=2 * kl, mode="adaptive")
        converged = info["converged"]
    elif solver == "cs":
        iters = _bounds.cs_passes(sig_l, sig_u, tol)
        sol = chebyshev(mv, rmv, rhs, sig_l, sig_u, iters)
        converged = True
    else:
        raise ValueError("solver must be 'lsqr' or 'cs'")
    if p["tall"]:
        x = Ne @ sol
    else:
        x = p["sigma_x"] * sol[: p["L"]]
    t3 = time.perf_counter()
    return dict(x=np.asarray(x, dtype=np.float64), iters=int(iters), converged=bool(converged),
                r=int(r), s=int(s), sigma_l=sig_l, sigma_u=sig_u, alpha=alpha, sig=sig,
                At=At, N=N, plan=p, lsqr_count=kl,
                t_sketch=t1 - t0, t_svd=t2 - t1, t_iter=t3 - t2)
