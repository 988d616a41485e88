"""Alg. 1/2 steps 4-5: SVD of the sketch and the preconditioner (oracle).

Alg. 1 step 4: economy SVD Ã = Ũ Σ̃ Ṽ^T, r = rank(Ã); only Σ̃, Ṽ
are needed.  Step 5: N = Ṽ Σ̃^-1.  Alg. 2 steps 4-5:
M = Ũ Σ̃^-1.  In the tall form (sketch.py) both are V_r Σ_r^-1 of Ãt, because
the wide Ã = Ãt^T.

The SVD is LAPACK's (numpy.linalg.svd, a true SVD -- never an eigen-
decomposition of Ã^T Ã).  Rank rule (reading C4, the paper says only
"r = rank(Ã)"): r = #{σ̃_i > max(s, k) * 2^-52 * σ̃_1}.
"""
import numpy as np


class RankZeroError(ValueError):
    pass


def rank_threshold(sig, s, k):
    return max(s, k) * 2.0 ** -52 * (sig[0] if sig.size else 0.0)


def factor(At):
    """Return (N, sig, r): N = V_r diag(1/σ_r) (k x r), σ̃ all, r numerical rank."""
    s, k = At.shape
    _, sig, Vt = np.linalg.svd(At, full_matrices=False)
    tau = rank_threshold(sig, s, k)
    r = int(np.count_nonzero(sig > tau)) if sig.size and sig[0] > 0 else 0
    if r == 0:
        raise RankZeroError("sketch has numerical rank 0")
    N = Vt[:r].T / sig[:r]
    return N, sig, r
