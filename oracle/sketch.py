"""Plan and sketch: Alg. 1/2 steps 1 and 3 plus the §5 Tikhonov blocks (oracle).

Alg. 1 (m >> n): s = ceil(gamma n) (step 1), Ã = G A (step 3,
P:487).  Alg. 2 (m << n): s = ceil(gamma m), Ã = A G.
§5, W = lambda I:
  tall  : min ||[A; lambda I] x - [b; 0]||   (eq. l2_reg_eq)
          -> Ã = G[:, :m] A + lambda G[:, m:m+n]
  wide  : min-length solution of [A/lambda, I_m] (z; r) = b, x = z/lambda
          (eq. l2_reg_eq_under)
          -> Ã = (1/lambda) A G[:n, :] + G[n:n+m, :]

Everything is expressed in the "tall form": X is the L x k
long-index-major matrix (X = A when m >= n, X = A^T when m < n) and
    Ãt = sigma_X * (G[:, :L] X) + sigma_I * G[:, L:L+k]        (s x k)
with (sigma_X, sigma_I) = (1, lambda) tall, (1/lambda, 1) wide, (1, 0) when
lambda = 0.  For the wide case the paper's Ã (m x s) is Ãt^T.  m == n goes to the
tall path.
"""
import math

import numpy as np

from .gaussian import gaussian, gaussian_block


def plan(m, n, gamma, lam=0.0):
    """a0 of SURVEY §8(a): orientation, s, the long/short dimensions and scales."""
    if not gamma > 1.0:
        raise ValueError("oversampling factor must exceed 1 (Alg. 1 step 1, P:480)")
    if lam < 0:
        raise ValueError("lambda must be >= 0")
    tall = m >= n
    L, k = (m, n) if tall else (n, m)
    s = int(math.ceil(gamma * k))                      # P:480 / P:508, reading C10
    if lam > 0:
        sigma_x, sigma_i = (1.0, float(lam)) if tall else (1.0 / lam, 1.0)
    else:
        sigma_x, sigma_i = 1.0, 0.0
    return dict(tall=tall, m=m, n=n, L=L, k=k, s=s, lam=float(lam),
                sigma_x=sigma_x, sigma_i=sigma_i)


def sketch(X, s, seed, sigma_x=1.0, sigma_i=0.0, block=None, precise=True):
    """Ãt = sigma_X (G[:, :L] X) + sigma_I G[:, L:L+k]  (s x k), X dense or scipy CSR.

    The oracle's sketch is the naive-loop C code (oracle/c/lsrn_oracle.c,
    orc_sketch_dense / orc_sketch_csr): for every sketch row i and column c the sum
    over the long index in increasing order, in fixed blocks of 256 (C17), with
    G[i, j] evaluated in long double (C9).  `block` and `precise` are accepted for
    the explicit-G variant below (precise=False selects it with fp64 libm normals).
    """
    from . import _c
    if not precise:
        return sketch_blas(X, s, seed, sigma_x, sigma_i, block=block or 4096, precise=False)
    if hasattr(X, "toarray") and not isinstance(X, np.ndarray):
        return _c.sketch_csr(X, s, seed, sigma_x, sigma_i)
    return _c.sketch_dense(X, s, seed, sigma_x, sigma_i)


def sketch_blas(X, s, seed, sigma_x=1.0, sigma_i=0.0, block=4096, precise=True):
    """The same product through explicit G blocks and a library matmul (a pin of the
    naive loops: same definition, different summation order)."""
    L, k = X.shape
    acc = np.zeros((s, k), dtype=np.float64)
    for j0 in range(0, L, block):
        j1 = min(L, j0 + block)
        G = gaussian_block(seed, 0, s, j0, j1, precise=precise)
        Xb = X[j0:j1]
        if hasattr(Xb, "toarray") and not isinstance(Xb, np.ndarray):
            acc += np.asarray((Xb.T @ G.T).T)          # sparse block: (X^T G^T)^T
        else:
            acc += G @ Xb
    At = sigma_x * acc
    if sigma_i != 0.0:
        At = At + sigma_i * gaussian_block(seed, 0, s, L, L + k, precise=precise)
    return At


def sketch_entries(Xcols, rows, cols, seed, sigma_x=1.0, sigma_i=0.0, L=None,
                   block=1 << 16, precise=False):
    """Sampled entries Ãt[rows[t], cols[t]] one by one (full-size parity).

    Xcols: dict col -> the dense length-L column X[:, col].
    """
    out = np.empty(len(rows), dtype=np.float64)
    for t, (i, c) in enumerate(zip(rows, cols)):
        x = Xcols[c]
        Lx = x.shape[0] if L is None else L
        acc = 0.0
        for j0 in range(0, Lx, block):
            j1 = min(Lx, j0 + block)
            g = gaussian(seed, [i], np.arange(j0, j1), precise=precise)[0]
            acc += float(g @ x[j0:j1])
        val = sigma_x * acc
        if sigma_i != 0.0:
            val += sigma_i * gaussian(seed, [i], [Lx + c], precise=precise)[0, 0]
        out[t] = val
    return out
