"""NEXT-4: lsrn_choose_gamma (§6.3), host-only, runs without a GPU.

Pins: the choice minimises the stage-time model whose iteration counts come from
the oracle's own Thm 4.5 / Alg. 3 bounds (oracle.bounds, written from the paper);
the limiting regimes of §6.3's Figure 2 discussion (randn / mult / svd grow
linearly in gamma, iter falls): iteration-dominated -> the top of the range,
sketch-dominated -> the bottom; bad probes are rejected."""
import math

import pytest

from oracle import bounds

M, N = 100_000, 1_000


def probe(**kw):
    d = dict(s=2000, r=1000, iters=94, converged=1, sigma_L=0.0, sigma_U=0.0, alpha=0.0,
             t_sketch=0.010, t_allreduce=0.0, t_svd=0.020, t_iter=0.050, t_total=0.080, rnorm_est=0.0)
    d.update(kw)
    return d


def model(p, gamma, solver, tol=1e-14):
    """T(gamma) of include/lsrn.h with the oracle's counts (None if Thm 4.4 excludes gamma)."""
    k = min(M, N)
    s = math.ceil(gamma * k)
    a = bounds.default_alpha(s)
    if not a < 1 - math.sqrt(p["r"] / s):
        return None
    if solver == "lsqr":
        it = bounds.lsqr_count(1e-14, p["r"], s)
    else:
        it = bounds.cs_passes(*bounds.sigma_bounds(s, p["r"], a), tol)
    svd = lambda ss: 2 * ss * k * k + 11 * k ** 3  # noqa: E731
    return p["t_sketch"] * s / p["s"] + p["t_svd"] * svd(s) / svd(p["s"]) + p["t_iter"] / p["iters"] * it


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
@pytest.mark.parametrize("kw", [{}, {"t_iter": 0.2}, {"t_sketch": 0.1}, {"t_svd": 0.001, "r": 600}])
def test_choice_minimises_model(solver, kw):
    from paper_1109_5981_b200 import lsrn
    p = probe(**kw)
    got = lsrn.choose_gamma(p, M, N, solver=solver)
    grid = [1.2 + 0.01 * i for i in range(181)]
    ts = [(model(p, g, solver), g) for g in grid]
    ts = [(t, g) for t, g in ts if t is not None]
    tbest = min(ts)[0]
    assert abs(got["t_model"] - model(p, got["gamma"], solver)) <= 1e-12 * tbest
    assert got["t_model"] <= tbest * (1 + 1e-12)


def test_limiting_regimes():
    from paper_1109_5981_b200 import lsrn
    assert lsrn.choose_gamma(probe(t_iter=50.0), M, N)["gamma"] == 3.0     # iterations dominate
    assert lsrn.choose_gamma(probe(t_iter=1e-6), M, N)["gamma"] == 1.2     # sketch + SVD dominate


def test_bad_probe_rejected():
    from paper_1109_5981_b200 import lsrn
    for kw in ({"iters": 0}, {"r": 2000}, {"t_iter": 0.0}):
        with pytest.raises(lsrn.LsrnError):
            lsrn.choose_gamma(probe(**kw), M, N)
    with pytest.raises(lsrn.LsrnError):
        lsrn.choose_gamma(probe(), M, N, lo=3.0, hi=2.0)
