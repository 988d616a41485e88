"""The N > 1 decomposition on CPU: world_size-2 gloo process groups.

The GPU path shards the long dimension (§4.3): rank p sketches its
rows with GLOBAL Philox indices, the partial sketches are allreduced, and each
iteration does local long passes plus one allreduce of the short vector.  These
tests run that decomposition with gloo collectives on the oracle's arithmetic
and check it against the single-process oracle, and they exercise the host-side
plumbing of paper_1109_5981_b200.dist (shard bounds, NCCL-id exchange).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1109_5981_b200.dist import exchange_unique_id, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world=2):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_entry, args=(fn, r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = [q.get() for _ in range(world)]
    for r in res:
        assert r[1] == "ok", r
    return sorted(res)


def _entry(fn, rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        fn(rank, world)
        q.put((rank, "ok"))
    except Exception as ex:  # report to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("L,world", [(10, 3), (7, 7), (0, 2), (100_000, 8), (5, 8)])
def test_shard_bounds_partition(L, world):
    b = [shard_bounds(L, world, r) for r in range(world)]
    assert b[0][0] == 0 and b[-1][1] == L
    for (lo, hi), (lo2, _) in zip(b, b[1:]):
        assert hi == lo2 and hi >= lo
    sizes = [hi - lo for lo, hi in b]
    assert max(sizes) - min(sizes) <= 1


def _id_exchange(rank, world):
    got = exchange_unique_id(lambda: bytes(range(rank, rank + 128)))
    assert got == bytes(range(0, 128)), got[:4]


def test_unique_id_exchange_gloo():
    _run(_id_exchange)


def _sketch_shards(rank, world):
    from oracle.gaussian import gaussian_block
    from oracle.sketch import sketch
    rng = np.random.default_rng(3)
    L, k, s, seed = 1001, 13, 26, 5981
    X = rng.standard_normal((L, k))
    lo, hi = shard_bounds(L, world, rank)
    part = gaussian_block(seed, 0, s, lo, hi) @ X[lo:hi]           # global indices j = lo..hi-1
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    full = sketch(X, s, seed)
    err = np.linalg.norm(t.numpy() - full) / np.linalg.norm(full)
    assert err <= 1e-13, err


def test_sharded_sketch_allreduce_equals_full():
    _run(_sketch_shards)


def _cs_shards(rank, world):
    """Alg. 3 with row-sharded A N: local products + one allreduce per pass."""
    from oracle import bounds
    from oracle.krylov import chebyshev, cs_schedule
    from oracle.precond import factor
    from oracle.sketch import sketch
    rng = np.random.default_rng(5)
    m, n = 900, 20
    A = rng.standard_normal((m, n)) * np.logspace(0, -3, n)
    b = rng.standard_normal(m)
    s = 40
    N, _, r = factor(sketch(A, s, 5981))
    sl, su = bounds.sigma_bounds(s, r, bounds.default_alpha(s))
    passes = bounds.cs_passes(sl, su, 1e-14)
    ref = N @ chebyshev(lambda y: A @ (N @ y), lambda u: N.T @ (A.T @ u), b, sl, su, passes)
    lo, hi = shard_bounds(m, world, rank)
    Ap, rp = A[lo:hi], b[lo:hi].copy()
    d = (su ** 2 + sl ** 2) / 2.0
    c = (su ** 2 - sl ** 2) / 2.0
    v = np.zeros(r)
    y = np.zeros(r)
    for beta, alpha in cs_schedule(d, c, passes):
        w = torch.from_numpy(Ap.T @ rp)          # local long pass
        dist.all_reduce(w)                       # the one collective per pass
        v = beta * v + N.T @ w.numpy()
        y = y + alpha * v
        rp = rp - alpha * (Ap @ (N @ v))
    x = N @ y
    err = np.linalg.norm(x - ref) / np.linalg.norm(ref)
    assert err <= 1e-10, err


def test_sharded_chebyshev_allreduce_equals_single_process():
    _run(_cs_shards)


@pytest.mark.parametrize("name", ["c4", "t4"])
def test_csr_recipes_are_canonical(name):
    """The CSR generators honour lsrn.h's contract: sorted, distinct columns per row of X."""
    from synth.generate import small
    p = small(name)
    rp, ci = p.rowptr.numpy(), p.colind.numpy()
    assert all(np.all(np.diff(ci[rp[i]:rp[i + 1]]) > 0) for i in range(p.m))
    assert ci.min() >= 0 and ci.max() < min(p.m, p.n)


def _lsqr_shards(rank, world, two_sync):
    """LSQR (Paige & Saunders) on row-sharded A N: per iteration the local long pass
    gives A_p^T u_p and ||u_p||^2; they are reduced together (one collective, the
    library's packed form) or one after the other (two collectives, the textbook
    count the paper compares CS against).  Both equal the one-process
    oracle LSQR with the same fixed iteration count."""
    from oracle import bounds
    from oracle.krylov import lsqr
    from oracle.precond import factor
    from oracle.sketch import sketch
    rng = np.random.default_rng(6)
    m, n = 800, 18
    A = rng.standard_normal((m, n)) * np.logspace(0, -2, n)
    b = rng.standard_normal(m)
    s = 40
    N, _, r = factor(sketch(A, s, 5981))
    iters = bounds.lsqr_count(1e-14, r, s)
    ref = N @ lsqr(lambda y: A @ (N @ y), lambda u: N.T @ (A.T @ u), b, iters=iters)[0]
    lo, hi = shard_bounds(m, world, rank)
    Ap = A[lo:hi]
    ncoll = [0]

    def reduce_pair(vec, nrm2):
        if two_sync:
            t = torch.tensor([nrm2])
            dist.all_reduce(t)
            w = torch.from_numpy(vec.copy())
            dist.all_reduce(w)
            ncoll[0] += 2
            return w.numpy(), float(t[0])
        packed = torch.from_numpy(np.concatenate([vec, [nrm2]]))
        dist.all_reduce(packed)
        ncoll[0] += 1
        return packed.numpy()[:-1], float(packed[-1])
    # bidiagonalisation with the long vector u sharded (u_p = rows lo..hi) and v replicated
    up = b[lo:hi].copy()
    atu, beta2 = reduce_pair(Ap.T @ up, float(up @ up))
    beta = np.sqrt(beta2)
    up /= beta
    v = N.T @ (atu / beta)
    alpha = np.linalg.norm(v)
    v /= alpha
    w = v.copy()
    y = np.zeros(r)
    phibar, rhobar = beta, alpha
    for _ in range(iters):
        up = Ap @ (N @ v) - alpha * up
        atu, beta2 = reduce_pair(Ap.T @ up, float(up @ up))
        beta = np.sqrt(beta2)
        up /= beta
        v = N.T @ (atu / beta) - beta * v
        alpha = np.linalg.norm(v)
        v /= alpha
        rho = np.hypot(rhobar, beta)
        c_, s_ = rhobar / rho, beta / rho
        theta = s_ * alpha
        rhobar = -c_ * alpha
        phi = c_ * phibar
        phibar = s_ * phibar
        y = y + (phi / rho) * w
        w = v - (theta / rho) * w
    x = N @ y
    err = np.linalg.norm(x - ref) / np.linalg.norm(ref)
    assert err <= 1e-10, err
    assert ncoll[0] == (iters + 1) * (2 if two_sync else 1)


@pytest.mark.parametrize("two_sync", [False, True])
def test_sharded_lsqr_equals_single_process(two_sync):
    import functools
    _run(functools.partial(_lsqr_shards, two_sync=two_sync))


def _wide_cs_shards(rank, world):
    """Alg. 2 with Tikhonov (§5): the wide operator [A/lambda, I] is column-sharded --
    each rank holds a block of columns of A (rank 0 also the I block) -- so the
    sketch partials A_p G_p and, per pass, the short products A_p v_p are summed by one
    allreduce of m doubles; x comes back per column shard."""
    from oracle import bounds
    from oracle.gaussian import gaussian_block
    from oracle.krylov import cs_schedule
    from oracle.lsrn import solve as orc_solve
    from oracle.precond import factor
    rng = np.random.default_rng(9)
    m, n, lam = 12, 700, 0.05
    A = rng.standard_normal((m, n)) * np.logspace(0, -2, m)[:, None]
    b = rng.standard_normal(m)
    ref = orc_solve(A, b, solver="cs", lam=lam)
    s, seed = 24, 5981
    sx, si = 1.0 / lam, 1.0
    X = np.ascontiguousarray(A.T)                       # tall form: n x m
    lo, hi = shard_bounds(n, world, rank)
    part = sx * (gaussian_block(seed, 0, s, lo, hi) @ X[lo:hi])
    if rank == 0:
        part = part + si * gaussian_block(seed, 0, s, n, n + m)
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    N, _, r = factor(t.numpy())
    sl, su = bounds.sigma_bounds(s, r, bounds.default_alpha(s))
    passes = bounds.cs_passes(sl, su, 1e-14)
    assert passes == ref["iters"]
    d = (su ** 2 + sl ** 2) / 2.0
    c = (su ** 2 - sl ** 2) / 2.0
    # CS on Abar = N^T [sx X_p^T | si I], long vector z sharded by columns (+ I block on rank 0)
    Xp = X[lo:hi]
    rvec = N.T @ b
    zp = np.zeros(hi - lo)
    zi = np.zeros(m) if rank == 0 else None
    vp = np.zeros(hi - lo)
    vi = np.zeros(m) if rank == 0 else None
    for beta, alpha in cs_schedule(d, c, passes):
        q = N @ rvec                                     # replicated short vector
        vp = beta * vp + sx * (Xp @ q)
        zp = zp + alpha * vp
        if rank == 0:
            vi = beta * vi + si * q
            zi = zi + alpha * vi
        loc = sx * (Xp.T @ vp) + (si * vi if rank == 0 else 0.0)
        tt = torch.from_numpy(np.asarray(loc, dtype=np.float64).copy())
        dist.all_reduce(tt)                              # one collective per pass: m doubles
        rvec = rvec - alpha * (N.T @ tt.numpy())
    xp = sx * zp
    err = np.linalg.norm(xp - ref["x"][lo:hi]) / np.linalg.norm(ref["x"])
    assert err <= 1e-9, err


def test_column_sharded_wide_tikhonov_cs():
    _run(_wide_cs_shards)
