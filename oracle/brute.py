"""Closed-form solutions for tiny inputs (oracle pins; test infrastructure only).

Min-length least squares (§1): x* = A^+ b = V_r Σ_r^-1 U_r^T b.
Ridge with W = lambda I (eq. l2_reg, reading C11):
    x_lambda = (A^T A + lambda^2 I)^-1 A^T b = A^T (A A^T + lambda^2 I)^-1 b.

`min_length` uses a long-double one-sided Jacobi SVD (Hestenes) written out
here, independent of LAPACK, so that tests can cross-check it against
numpy.linalg.lstsq / pinv (library pins).  `ridge` solves the smaller normal
system with long-double Gaussian elimination with partial pivoting.
"""
import numpy as np


def jacobi_svd(A, sweeps=60):
    """One-sided Jacobi SVD in long double: returns (U, s, V) with A = U diag(s) V^T."""
    W = np.array(A, dtype=np.longdouble)
    m, n = W.shape
    V = np.eye(n, dtype=np.longdouble)
    eps = np.finfo(np.longdouble).eps
    for _ in range(sweeps):
        off = 0
        for p in range(n - 1):
            for q in range(p + 1, n):
                a = W[:, p] @ W[:, p]
                bb = W[:, q] @ W[:, q]
                g = W[:, p] @ W[:, q]
                if abs(g) <= eps * np.sqrt(a * bb) or g == 0:
                    continue
                off += 1
                zeta = (bb - a) / (2 * g)
                t = np.sign(zeta) / (abs(zeta) + np.sqrt(1 + zeta * zeta)) if zeta != 0 else np.longdouble(1)
                c = 1 / np.sqrt(1 + t * t)
                sn = c * t
                Wp, Wq = W[:, p].copy(), W[:, q].copy()
                W[:, p] = c * Wp - sn * Wq
                W[:, q] = sn * Wp + c * Wq
                Vp, Vq = V[:, p].copy(), V[:, q].copy()
                V[:, p] = c * Vp - sn * Vq
                V[:, q] = sn * Vp + c * Vq
        if off == 0:
            break
    s = np.sqrt(np.sum(W * W, axis=0))
    order = np.argsort(-s.astype(np.float64), kind="stable")
    s = s[order]
    V = V[:, order]
    W = W[:, order]
    U = np.zeros_like(W)
    nz = s > 0
    U[:, nz] = W[:, nz] / s[nz]
    return U, s, V


def min_length(A, b, rtol=None):
    """x* = A^+ b via the long-double Jacobi SVD (works on A or A^T, whichever is tall)."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    tall = m >= n
    U, s, V = jacobi_svd(A if tall else A.T)
    if rtol is None:
        rtol = max(m, n) * 2.0 ** -52
    r = int(np.count_nonzero(s > rtol * s[0])) if s[0] > 0 else 0
    bl = np.asarray(b, dtype=np.longdouble)
    if tall:     # A = U S V^T
        x = V[:, :r] @ ((U[:, :r].T @ bl) / s[:r])
    else:        # A^T = U S V^T  ->  A = V S U^T,  A^+ = U S^-1 V^T
        x = U[:, :r] @ ((V[:, :r].T @ bl) / s[:r])
    return x.astype(np.float64), r


def _solve_ld(M, rhs):
    M = np.array(M, dtype=np.longdouble)
    y = np.array(rhs, dtype=np.longdouble)
    n = M.shape[0]
    for c in range(n):
        p = c + int(np.argmax(np.abs(M[c:, c].astype(np.float64))))
        if p != c:
            M[[c, p]] = M[[p, c]]
            y[[c, p]] = y[[p, c]]
        piv = M[c, c]
        f = M[c + 1:, c] / piv
        M[c + 1:, c:] -= np.outer(f, M[c, c:])
        y[c + 1:] -= f * y[c]
    x = np.zeros(n, dtype=np.longdouble)
    for c in range(n - 1, -1, -1):
        x[c] = (y[c] - M[c, c + 1:] @ x[c + 1:]) / M[c, c]
    return x


def ridge(A, b, lam):
    """x = argmin 1/2||Ax-b||^2 + 1/2 lam^2 ||x||^2 via the smaller normal system."""
    Al = np.asarray(A, dtype=np.longdouble)
    bl = np.asarray(b, dtype=np.longdouble)
    m, n = Al.shape
    l2 = np.longdouble(lam) ** 2
    if m >= n:
        x = _solve_ld(Al.T @ Al + l2 * np.eye(n, dtype=np.longdouble), Al.T @ bl)
    else:
        x = Al.T @ _solve_ld(Al @ Al.T + l2 * np.eye(m, dtype=np.longdouble), bl)
    return x.astype(np.float64)
