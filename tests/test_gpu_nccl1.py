"""The NCCL collective path on one GPU: a context built with nranks = 1 and an NCCL
unique id owns a one-rank communicator, so the sketch allreduce and the per-pass
allreduce of k + 1 doubles are issued through NCCL (the per-pass ones inside the
captured iteration graph).  This exercises communicator set-up and NCCL calls under
stream capture on the one GPU the pool gives; NCCL completes a one-rank in-place
allreduce without moving data, so the results must equal the communicator-free
context bit for bit -- dense and CSR, LSQR and CS, tall and wide.  The cross-rank
data path itself is covered on the host side by tests/test_multirank_gloo.py."""
import numpy as np
import pytest
import torch

from synth.generate import small

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pair():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1109_5981_b200 import lsrn
    try:
        nid = lsrn.nccl_unique_id()
    except lsrn.LsrnError:
        pytest.skip("built without NCCL")
    a = lsrn.Context()
    b = lsrn.Context(nranks=1, rank=0, nccl_id=nid)
    yield a, b
    a.close()
    b.close()


@pytest.mark.parametrize("name", ["c1", "c3", "c4"])
@pytest.mark.parametrize("solver", ["lsqr", "cs"])
def test_one_rank_nccl_equals_plain(pair, name, solver):
    from paper_1109_5981_b200 import lsrn
    plain, nccl = pair
    p = small(name)
    if p.kind == "csr":
        X = lsrn.Csr(p.rowptr.cuda(), p.colind.cuda(), p.val.cuda())
    else:
        X = p.X.cuda()
    b = p.b.cuda()
    x1, r1 = plain.solve(X, b, p.m, p.n, solver=solver, lam=p.lam)
    x2, r2 = nccl.solve(X, b, p.m, p.n, solver=solver, lam=p.lam)
    assert r1["iters"] == r2["iters"] and r1["r"] == r2["r"]
    assert torch.equal(x1, x2)
    assert np.isfinite(x2.cpu().numpy()).all()


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_one_rank_nccl_lsqr_two_collectives(pair, name):
    """LSRN_OPT_LSQR_SYNC = 1 (textbook LSQR: ||u||^2 reduced first, then the vector,
    P:301-304) issues two NCCL allreduces per half-step instead of one packed one;
    the arithmetic is unchanged, so x equals the packed run bit for bit."""
    plain, nccl = pair
    p = small(name)
    X, b = p.X.cuda(), p.b.cuda()
    x1, r1 = nccl.solve(X, b, p.m, p.n, solver="lsqr", lam=p.lam)
    with nccl.options(lsqr_sync=1):
        x2, r2 = nccl.solve(X, b, p.m, p.n, solver="lsqr", lam=p.lam)
    assert torch.equal(x1, x2) and r1["iters"] == r2["iters"]
    # sketch allreduce + non-finite flag + one (packed) or two per long pass
    passes = r1["iters"] + 1
    assert r1["collectives"] == 2 + passes, r1["collectives"]
    assert r2["collectives"] == 2 + 2 * passes, r2["collectives"]
