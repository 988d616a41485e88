"""Alg. 1/2 steps 4-5: SVD of the sketch and the preconditioner (oracle).

Alg. 1 step 4: economy SVD Ã = Ũ Σ̃ Ṽ^T, r = rank(Ã); only Σ̃, Ṽ
are needed.  Step 5: N = Ṽ Σ̃^-1.  Alg. 2 steps 4-5:
M = Ũ Σ̃^-1.  In the tall form (sketch.py) both are V_r Σ_r^-1 of Ãt, because
the wide Ã = Ãt^T.

The SVD is the one-sided (Hestenes) Jacobi SVD of oracle/c/lsrn_oracle.c
(orc_jacobi_svd) for k <= 2048 -- every configuration the oracle solves in
full (c1, c2 and all the small test instances).  Above that (c3's augmented
k = 2000 is below; c4 k = 2e4 and c5 k = 1e4 only appear in bench.py's staged
CPU timing) LAPACK's gesdd (numpy.linalg.svd) stands in for it: O(s k^2) per
Jacobi sweep at k = 1e4 is hours on the host.  Both are true SVDs (never an
eigendecomposition of Ã^T Ã); reading C20.  Rank rule
(reading C4, the paper says only "r = rank(Ã)"):
r = #{σ̃_i > max(s, k) * 2^-52 * σ̃_1}.
"""
import numpy as np

JACOBI_MAX_K = 2048


class RankZeroError(ValueError):
    pass


def rank_threshold(sig, s, k):
    return max(s, k) * 2.0 ** -52 * (sig[0] if sig.size else 0.0)


def svd(At):
    """(sigma descending, V with the right singular vectors as columns)."""
    s, k = At.shape
    if k <= JACOBI_MAX_K:
        from . import _c
        sig, V, _sweeps = _c.jacobi_svd(At)
        return sig, V
    _, sig, Vt = np.linalg.svd(At, full_matrices=False)
    return sig, Vt.T


def factor(At):
    """Return (N, sig, r): N = V_r diag(1/σ_r) (k x r), σ̃ all, r numerical rank."""
    s, k = At.shape
    sig, V = svd(At)
    tau = rank_threshold(sig, s, k)
    r = int(np.count_nonzero(sig > tau)) if sig.size and sig[0] > 0 else 0
    if r == 0:
        raise RankZeroError("sketch has numerical rank 0")
    N = V[:, :r] / sig[:r]
    return N, sig, r
