"""liblsrn.so's own nranks = 2 path, on the one GPU the pool gives.

Two processes, one gloo process group.  Each process creates an lsrn context
with nranks = 2 and host-staged collectives (lsrn_ctx_set_host_collectives via
paper_1109_5981_b200.dist.host_context: the library copies the operand to the
host and calls back into torch.distributed for the sum / broadcast -- the
paper's MPI_Reduce, MPI_Bcast(N) and per-iteration MPI_Allreduce).
Both processes share the GPU, but no kernel waits on another rank's kernel: the
ranks meet only on the host, inside the collectives.

What runs here that a one-rank run never exercises: the GLOBAL Philox long index
of each shard (lo > 0), the Tikhonov block held by rank 0 only (has_I), the
per-rank long vectors, the sketch allreduce of partial sketches, the broadcast
of sigma and N from rank 0 (LSRN_OPT_BCAST_N), the per-pass
reductions (packed, or the two-collective LSQR of LSRN_OPT_LSQR_SYNC = 1) and
the column-sharded wide form (Alg. 2) with x returned per shard.

Each sharded solve is compared with the oracle on the full problem (same rank,
identical iteration counts, x within the DESIGN.md C18 bar) and with the
library's own one-rank solve.
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
U_ = 2.0 ** -53


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1109_5981_b200 import dist as ldist
        from paper_1109_5981_b200 import lsrn
        from synth.generate import small
        torch.cuda.set_device(0)
        p = small(case["name"])
        L = max(p.m, p.n)
        lo, hi = ldist.shard_bounds(L, world, rank)
        ctx = ldist.host_context()
        for k_, v_ in case.get("opts", {}).items():
            ctx.set_option(k_, v_)
        if p.kind == "csr":
            rp = p.rowptr[lo:hi + 1]
            X = lsrn.Csr((rp - rp[0]).contiguous().cuda(), p.colind[rp[0]:rp[-1]].contiguous().cuda(),
                         p.val[rp[0]:rp[-1]].contiguous().cuda())
        else:
            X = p.X[lo:hi].contiguous().cuda()
        b = (p.b[lo:hi] if p.tall else p.b).contiguous().cuda()
        x, rep = ctx.solve(X, b, p.m, p.n, solver=case["solver"], lam=p.lam, lo=lo, cnt=hi - lo)
        q.put((rank, "ok", (lo, hi), x.cpu().numpy(), rep))
        ctx.close()
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc(), None, None, None))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _run_two(case):
    import torch.multiprocessing as mp
    port = _free_port()
    mpc = mp.get_context("spawn")
    q = mpc.SimpleQueue()
    procs = [mpc.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get() for _ in range(2)]
    for p in procs:
        p.join(300)
    for r in res:
        assert r[1] == "ok", r[1]
    return sorted(res, key=lambda r: r[0])


CASES = [
    dict(name="c2", solver="lsqr"),                                   # tall dense, rank-deficient
    dict(name="c2", solver="cs"),
    dict(name="c2", solver="lsqr", opts=dict(lsqr_sync=1)),           # textbook LSQR: 2 collectives / half-step
    dict(name="c2", solver="cs", opts=dict(bcast_n=0)),               # every rank computes the SVD itself
    dict(name="c5", solver="lsqr"),
    dict(name="c3", solver="lsqr"),                                   # wide + Tikhonov: column shards, I block on rank 0
    dict(name="c3", solver="cs"),
    dict(name="c4", solver="cs"),                                     # CSR, heavy + light columns
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c['name']}-{c['solver']}-{'-'.join(map(str, c.get('opts', {}).items()))}")
def test_two_ranks_match_oracle(case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle.lsrn import solve as orc_solve
    from synth.generate import small
    p = small(case["name"])
    res = _run_two(case)
    reps = [r[4] for r in res]
    if p.tall:
        x = res[0][3]
        assert np.array_equal(res[0][3], res[1][3])            # x replicated: identical on both ranks
    else:
        x = np.concatenate([res[0][3], res[1][3]])             # wide: each rank returns its columns
    A = p.to_scipy() if p.kind == "csr" else p.dense_A().numpy()
    orc = orc_solve(A, p.b.numpy(), solver=case["solver"], lam=p.lam)
    for rep in reps:
        assert rep["r"] == orc["r"] and rep["s"] == orc["s"]
        assert rep["iters"] == orc["iters"]
    # collectives per rank: sketch allreduce + non-finite flag + (sigma, N broadcasts) + passes
    passes = orc["iters"] + 1 if case["solver"] == "lsqr" else orc["iters"]
    bc = 0 if case.get("opts", {}).get("bcast_n") == 0 else 2
    per_pass = 2 if case.get("opts", {}).get("lsqr_sync") == 1 else 1
    if p.tall:
        assert reps[0]["collectives"] == 2 + bc + per_pass * passes, reps[0]["collectives"]
    Ad = A.toarray() if hasattr(A, "toarray") else A
    if p.lam > 0:
        Aop = np.vstack([Ad, p.lam * np.eye(p.n)]) if p.tall else Ad
    else:
        Aop = Ad
    sv = np.linalg.svd(Ad, compute_uv=False)
    kappa = sv[0] / sv[sv > sv[0] * 1e-12][-1]
    rel = np.linalg.norm(x - orc["x"]) / np.linalg.norm(orc["x"])
    assert rel <= max(1e-9, 20 * kappa * U_), rel
    an = np.linalg.norm(Aop @ (x - orc["x"])) / np.linalg.norm(Aop @ orc["x"])
    assert an <= 1e-11, an


def _worker_full(rank, world, port, name, solver, q):
    """Full-size: rank p generates only its shard of the config (synth's block-seeded
    recipe, bytes identical to the same rows of the whole matrix) and solves through
    the library's sharded path with host-staged collectives."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_1109_5981_b200 import dist as ldist
        from synth.generate import CONFIGS, SKETCH_SEED, make_problem
        torch.cuda.set_device(0)
        cfg = CONFIGS[name]
        L = max(cfg["m"], cfg["n"])
        lo, hi = ldist.shard_bounds(L, world, rank)
        p = make_problem(name, device="cuda", shard=(lo, hi))
        ctx = ldist.host_context()
        x, rep = ctx.solve(p.X, p.b, p.m, p.n, solver=solver, lo=lo, cnt=hi - lo, seed=SKETCH_SEED)
        # normal equations on this shard: A_p^T (b_p - A_p x), summed over the ranks
        g = p.X.T @ (p.b - p.X @ x)
        nb = torch.tensor([float(torch.linalg.norm(p.b)) ** 2, float(torch.linalg.norm(p.X)) ** 2])
        gt = g.cpu()
        dist.all_reduce(gt)
        dist.all_reduce(nb)
        q.put((rank, "ok", float(torch.linalg.norm(gt)), nb.tolist(), rep, x[:8].cpu().numpy()))
        ctx.close()
    except Exception:
        import traceback
        q.put((rank, traceback.format_exc(), None, None, None, None))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("solver", ["cs"])
def test_two_ranks_full_c5(solver):
    """c5 at full size (1e6 x 1e4, 80 GB) split over two ranks of 500000 rows (40 GB each)
    on the one GPU: the library's sharded sketch (global Philox index), the 1.6 GB sketch
    allreduce, rank 0's SVD broadcast and the per-pass reductions.  Checks the pass count of
    Alg. 3 at r = k, identical x on both ranks, and the normal equations
    A^T (b - A x) = 0 to the iteration tolerance (Thm 4.5's bound, as tests/test_gpu_fullsize.py
    checks for the one-rank solve)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.synchronize()
    torch.cuda.empty_cache()                 # earlier tests' cached blocks back to the device
    free, total = torch.cuda.mem_get_info()
    if free < 120e9:
        pytest.skip("needs ~110 GB of device memory for two 40 GB shards and their workspaces")
    import torch.multiprocessing as mp
    from oracle import bounds
    port = _free_port()
    mpc = mp.get_context("spawn")
    q = mpc.SimpleQueue()
    procs = [mpc.Process(target=_worker_full, args=(r, 2, port, "c5", solver, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = sorted([q.get() for _ in range(2)], key=lambda r: r[0])
    for pr in procs:
        pr.join(600)
    for r in res:
        assert r[1] == "ok", r[1]
    s = 20000
    sl, su = bounds.sigma_bounds(s, 10000, bounds.default_alpha(s))
    for r in res:
        assert r[4]["r"] == 10000 and r[4]["iters"] == bounds.cs_passes(sl, su, 1e-14) == 99
    assert np.array_equal(res[0][5], res[1][5])               # x replicated bit for bit (same N on both)
    gnorm, (b2, a2) = res[0][2], res[0][3]
    assert gnorm <= 10 * 2e-14 * np.sqrt(a2) * np.sqrt(b2), (gnorm, a2, b2)
