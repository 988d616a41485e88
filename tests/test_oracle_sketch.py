"""Pins for oracle/sketch.py and oracle/precond.py (no GPU).

Sketch (Alg. 1/2 step 3; §5 blocks): explicit-G product via one
library matmul over the whole G, zero/linearity, CSR == dense,
wide == transposed tall, the Tikhonov block equals G[:, L:L+k], sampled entries.
Precond (steps 4-5): LAPACK-independent SVD checks (reconstruction,
orthogonality), the rank rule on a constructed spectrum, Lemma 4.2
spectrum transfer with the generator's U, Thm 4.1 / Thm 3.2
range(N) = range(A^T), Thm 4.4 window.
"""
import math

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import bounds
from oracle.gaussian import gaussian_block
from oracle.precond import RankZeroError, factor
from oracle.sketch import plan, sketch, sketch_entries
from synth.generate import CONFIGS, make_problem, small


def test_plan_configs():
    exp_s = {"c1": 200, "c2": 4000, "c3": 4000, "c4": 40000, "c5": 20000, "t4": 2048}   # Table 3: s = 2048
    for c, cfg in CONFIGS.items():
        p = plan(cfg["m"], cfg["n"], cfg["gamma"], cfg["lam"])
        assert p["s"] == exp_s[c]
        assert p["tall"] == (cfg["m"] >= cfg["n"])
    p = plan(2000, 200000, 2.0, 1e-3)
    assert (p["sigma_x"], p["sigma_i"]) == (1e3, 1.0) and p["L"] == 200000 and p["k"] == 2000
    p = plan(100, 10, 2.0, 0.5)
    assert (p["sigma_x"], p["sigma_i"]) == (1.0, 0.5)
    assert plan(50, 50, 1.5)["tall"]                                  # m == n -> tall
    assert plan(100, 10, 1.1)["s"] == math.ceil(1.1 * 10)             # reading C10
    with pytest.raises(ValueError):
        plan(100, 10, 1.0)


def test_sketch_explicit_g_and_linearity():
    rng = np.random.default_rng(1)
    X = rng.standard_normal((10000, 100))
    Y = rng.standard_normal((10000, 100))
    s = 200
    G = gaussian_block(7, 0, s, 0, 10000)
    ref = G @ X                                                      # one library matmul
    got = sketch(X, s, 7, block=777)                                 # blocked, ragged tail
    assert np.linalg.norm(got - ref) <= 1e-13 * np.linalg.norm(ref)
    assert not np.any(sketch(np.zeros((300, 10)), 20, 7))
    lin = sketch(2.0 * X - 3.0 * Y, s, 7, block=4096)
    comb = 2.0 * got - 3.0 * sketch(Y, s, 7, block=2048)
    assert np.linalg.norm(lin - comb) <= 1e-13 * np.linalg.norm(lin)


def test_sketch_csr_equals_dense_and_wide_is_transposed_tall():
    p = small("c4")
    Xs = p.to_scipy()
    Xd = Xs.toarray()
    a = sketch(Xs, 60, 11, block=1000)
    b = sketch(Xd, 60, 11, block=1000)
    assert np.linalg.norm(a - b) <= 1e-13 * np.linalg.norm(b)
    # Alg. 2's Ã = A G with G_wide(j, i) = G(i, j): A G = (G^T... ) = sketch_tall(A^T)^T
    A = np.random.default_rng(3).standard_normal((30, 500))
    s = 60
    Gw = gaussian_block(11, 0, s, 0, 500).T                         # n x s
    assert np.linalg.norm(A @ Gw - sketch(A.T, s, 11).T) <= 1e-13 * np.linalg.norm(A @ Gw)


def test_sketch_tikhonov_blocks():
    rng = np.random.default_rng(4)
    X = rng.standard_normal((400, 20))
    s = 40
    G = gaussian_block(9, 0, s, 0, 420)
    lam = 0.37
    # tall: G [A; lam I] (§5 eq. l2_reg_eq)
    stacked = np.vstack([X, lam * np.eye(20)])
    assert np.allclose(sketch(X, s, 9, 1.0, lam), G @ stacked, rtol=0, atol=1e-12)
    # wide: [A/lam, I] G_wide  (eq. l2_reg_eq_under), in tall form
    Aw = X.T                                                         # 20 x 400 wide
    aug = np.hstack([Aw / lam, np.eye(20)])                          # 20 x 420
    ref = aug @ G.T                                                  # m x s
    assert np.allclose(sketch(X, s, 9, 1.0 / lam, 1.0).T, ref, rtol=0, atol=1e-11)
    # pure identity block
    assert np.array_equal(sketch(np.zeros((400, 20)), s, 9, 1.0, 1.0), G[:, 400:420])


def test_sketch_sampled_entries():
    rng = np.random.default_rng(5)
    X = rng.standard_normal((3000, 30))
    full = sketch(X, 64, 21, 1.0, 0.25, precise=False)
    rows = [0, 5, 63, 17]
    cols = [0, 29, 3, 17]
    got = sketch_entries({c: X[:, c] for c in cols}, rows, cols, 21, 1.0, 0.25, block=700)
    assert np.allclose(got, full[rows, cols], rtol=1e-13, atol=1e-12)


def test_svd_and_rank_rule():
    rng = np.random.default_rng(6)
    U, _ = np.linalg.qr(rng.standard_normal((40, 10)))
    V, _ = np.linalg.qr(rng.standard_normal((10, 10)))
    sig = np.ones(10)
    sig[-1] = 1e-20
    At = (U * sig) @ V.T                                              # r = 9
    N, s_all, r = factor(At)
    assert r == 9
    B = rng.standard_normal((80, 12))
    N, s_all, r = factor(B)
    assert r == 12
    # N = V Σ^-1  =>  B N = U (orthonormal columns), N^T B^T B N = I
    Q = B @ N
    assert np.linalg.norm(Q.T @ Q - np.eye(12)) < 1e-13
    assert np.allclose(np.sort(s_all)[::-1], np.linalg.svd(B, compute_uv=False), rtol=1e-14)
    with pytest.raises(RankZeroError):
        factor(np.zeros((8, 4)))


def _c1_like(m=2000, n=100, rank=None, seed=0):
    rng = np.random.default_rng(seed)
    rank = n if rank is None else rank
    U, _ = np.linalg.qr(rng.standard_normal((m, rank)))
    V, _ = np.linalg.qr(rng.standard_normal((n, rank)))
    sig = 10.0 ** (-6 * np.arange(rank) / max(rank - 1, 1))
    return (U * sig) @ V.T, U, V, sig


def test_lemma_4_2_spectrum_transfer_and_range():
    A, U, V, sig = _c1_like(m=1000, n=60, rank=40)
    s = 120
    At = sketch(A, s, 5981)
    N, _, r = factor(At)
    assert r == 40
    sv_AN = np.linalg.svd(A @ N, compute_uv=False)
    G1 = gaussian_block(5981, 0, s, 0, 1000) @ U                    # G U_r
    sv_G1 = np.linalg.svd(G1, compute_uv=False)
    # Lemma 4.2: σ(AN) = σ((GU)^+) = 1 / σ(GU), independent of A's spectrum
    assert np.allclose(np.sort(sv_AN), np.sort(1.0 / sv_G1), rtol=1e-9)
    # Thm 4.1 via Thm 3.2: range(N) = range(A^T) = range(V)
    P = N - V @ (V.T @ N)
    assert np.linalg.norm(P) <= 1e-10 * np.linalg.norm(N)


def test_thm_4_4_window_on_c1_small():
    p = small("c1")
    A = p.X.numpy()
    s = 200
    N, _, r = factor(sketch(A, s, 5981))
    sv = np.linalg.svd(A @ N, compute_uv=False)
    alpha = bounds.default_alpha(s)
    lo, hi = bounds.sigma_bounds(s, r, alpha)
    assert sv.min() >= lo and sv.max() <= hi
    assert sv.max() / sv.min() <= bounds.kappa_bound(s, r, alpha)
    assert sv.max() / sv.min() < 6                                   # P:971-973 (s = 2r)
