"""Closed-form bounds and iteration counts (oracle).

Thm 4.4 (eq. sgm_concentration): for alpha in (0, 1 - sqrt(r/s)),
    sigma_U = 1 / ((1 - alpha) sqrt(s) - sqrt(r)),
    sigma_L = 1 / ((1 + alpha) sqrt(s) + sqrt(r)),
hold with probability >= 1 - 2 exp(-alpha^2 s / 2).
Default alpha = 1/sqrt(s) (reading C3: t = 1 in Lemma 4.3; reproduces
Table 3's 106 CS iterations).

Alg. 3 loop: for k = 0, 1, ..., K with
    K = ceil((log eps - log 2) / log((sigma_U - sigma_L) / (sigma_U + sigma_L)))
i.e. K + 1 passes (reading C2; K <= 0 -> 1 pass).

Thm 4.5: a CG-like method converges within
    (log eps - log 2) / log(alpha + sqrt(r/s))
iterations.  LSQR's predictable count (reading C5) is that bound at alpha = 0:
    K_L = ceil((log eps - log 2) / log(sqrt(r/s))).
"""
import math


def default_alpha(s):
    return 1.0 / math.sqrt(s)


def sigma_bounds(s, r, alpha):
    if not (r >= 1 and s > r):
        raise ValueError("need s > r >= 1")
    if not (0.0 < alpha < 1.0 - math.sqrt(r / s)):
        raise ValueError("alpha must lie in (0, 1 - sqrt(r/s)) (Thm 4.4, P:620)")
    sig_u = 1.0 / ((1.0 - alpha) * math.sqrt(s) - math.sqrt(r))
    sig_l = 1.0 / ((1.0 + alpha) * math.sqrt(s) + math.sqrt(r))
    return sig_l, sig_u


def kappa_bound(s, r, alpha):
    """eq. cond_concentration: (1 + alpha + sqrt(r/s)) / (1 - alpha - sqrt(r/s))."""
    q = math.sqrt(r / s)
    return (1.0 + alpha + q) / (1.0 - alpha - q)


def cs_passes(sig_l, sig_u, eps):
    """Number of loop passes of Alg. 3 = K + 1 (reading C2)."""
    if not (0.0 < sig_l <= sig_u):
        raise ValueError("need 0 < sigma_L <= sigma_U")
    rho = (sig_u - sig_l) / (sig_u + sig_l)
    if rho == 0.0:
        return 1
    K = math.ceil((math.log(eps) - math.log(2.0)) / math.log(rho))
    return max(K, 0) + 1


def lsqr_count(eps, r, s, alpha=0.0):
    """Thm 4.5 bound ceil((log eps - log 2) / log(alpha + sqrt(r/s)))."""
    rate = alpha + math.sqrt(r / s)
    if not (0.0 < rate < 1.0):
        raise ValueError("oversampling too small for requested alpha")
    return max(0, math.ceil((math.log(eps) - math.log(2.0)) / math.log(rate)))
