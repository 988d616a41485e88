"""The C-ABI contract of include/lsrn.h on the GPU: error codes, "outputs only on
LSRN_OK", the NULL (legacy) stream, workspace alignment, CSR nnz validation,
options, and the lambda path starting at lambda = 0."""
import ctypes

import numpy as np
import pytest
import torch

from oracle import brute
from synth.generate import small

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1109_5981_b200 import lsrn
    c = lsrn.Context()
    yield c
    c.close()


def test_null_stream_context_solves():
    """lsrn_ctx_create(stream = NULL): the context runs on its own stream joined to the
    legacy stream (the iteration graph cannot be captured on the legacy stream)."""
    from paper_1109_5981_b200 import lsrn
    p = small("c5")
    X, b = p.X.cuda(), p.b.cuda()
    ref, rr = lsrn.Context().solve(X, b, p.m, p.n, solver="lsqr")
    c = lsrn.Context(null_stream=True)
    x, rep = c.solve(X, b, p.m, p.n, solver="lsqr")
    # ordered on the legacy stream: visible to a legacy-stream consumer without a sync
    y = x * 2.0
    torch.cuda.synchronize()
    assert torch.equal(x, ref) and torch.equal(y, 2.0 * ref) and rep["iters"] == rr["iters"]
    At = c.sketch(X, p.m, p.n, 2.0)
    assert At.shape[0] == rep["s"]
    c.close()


@pytest.mark.parametrize("where", ["b_nan", "b_inf", "A_nan", "A_inf"])
@pytest.mark.parametrize("solver", ["lsqr", "cs"])
def test_nonfinite_inputs_return_enonfinite(ctx, where, solver):
    """NaN / Inf in b or A -> LSRN_ENONFINITE, and x_out is not written."""
    from paper_1109_5981_b200.lsrn import LsrnError
    p = small("c2")
    X, b = p.X.clone().cuda(), p.b.clone().cuda()
    bad = float("nan") if where.endswith("nan") else float("inf")
    if where.startswith("b"):
        b[17] = bad
    else:
        X[123, 45] = bad
    x_out = torch.full((p.n,), 7.0, dtype=torch.float64, device="cuda")
    with pytest.raises(LsrnError, match="ENONFINITE"):
        ctx.solve(X, b, p.m, p.n, solver=solver, x_out=x_out)
    torch.cuda.synchronize()
    assert torch.all(x_out == 7.0)


def test_csr_nnz_mismatch_is_edim(ctx):
    from paper_1109_5981_b200 import lsrn
    p = small("c4")
    A = lsrn.Csr(p.rowptr.cuda(), p.colind.cuda(), p.val.cuda())
    b = p.b.cuda()
    mat, _ = lsrn.csr(A, p.m, p.n)
    mat.nnz = mat.nnz - 5                          # inconsistent with rowptr[cnt] - rowptr[0]
    opts = lsrn.Opts(gamma=2.0, lambda_=0.0, tol=1e-14, alpha=-1.0, seed=5981)
    ws = ctx.workspace(ctx.workspace_size(mat, opts))
    x = torch.full((p.n,), 3.0, dtype=torch.float64, device="cuda")
    rep = lsrn.Report()
    rc = lsrn.lib().lsrn_solve_cs(ctx.h, ctypes.byref(mat), lsrn._ptr(b), ctypes.byref(opts), lsrn._ptr(ws),
                                  ws.numel(), lsrn._ptr(x), ctypes.byref(rep))
    assert rc == -2 and b"nnz" in lsrn.lib().lsrn_last_error()
    assert torch.all(x == 3.0)


@pytest.mark.parametrize("offset", [8, 24, 136])
def test_misaligned_workspace(ctx, offset):
    """Any workspace alignment works (the carve-up is aligned to 256 bytes of the absolute
    address inside the slack lsrn_workspace_size adds); results are bit for bit those of an
    aligned workspace."""
    from paper_1109_5981_b200 import lsrn
    p = small("c5")
    X, b = p.X.cuda(), p.b.cuda()
    ref, _ = ctx.solve(X, b, p.m, p.n, solver="lsqr")
    mat, _ = lsrn.dense(X, p.m, p.n)
    opts = lsrn.Opts(gamma=2.0, lambda_=0.0, tol=1e-14, alpha=-1.0, seed=5981)
    need = ctx.workspace_size(mat, opts)
    raw = torch.empty(need + offset, dtype=torch.uint8, device="cuda")
    x = torch.empty(p.n, dtype=torch.float64, device="cuda")
    rep = lsrn.Report()
    with torch.cuda.stream(ctx.stream):
        rc = lsrn.lib().lsrn_solve_lsqr(ctx.h, ctypes.byref(mat), lsrn._ptr(b), ctypes.byref(opts),
                                        ctypes.c_void_p(raw.data_ptr() + offset), need, lsrn._ptr(x),
                                        ctypes.byref(rep))
    torch.cuda.synchronize()
    assert rc == 0, lsrn.lib().lsrn_last_error()
    assert torch.equal(x, ref)


def test_workspace_too_small_is_enomem(ctx):
    from paper_1109_5981_b200 import lsrn
    p = small("c5")
    X, b = p.X.cuda(), p.b.cuda()
    mat, _ = lsrn.dense(X, p.m, p.n)
    opts = lsrn.Opts(gamma=2.0, lambda_=0.0, tol=1e-14, alpha=-1.0, seed=5981)
    need = ctx.workspace_size(mat, opts)
    raw = torch.empty(need, dtype=torch.uint8, device="cuda")
    x = torch.full((p.n,), 5.0, dtype=torch.float64, device="cuda")
    rep = lsrn.Report()
    rc = lsrn.lib().lsrn_solve_lsqr(ctx.h, ctypes.byref(mat), lsrn._ptr(b), ctypes.byref(opts),
                                    lsrn._ptr(raw), need // 2, lsrn._ptr(x), ctypes.byref(rep))
    assert rc == -6
    torch.cuda.synchronize()
    assert torch.all(x == 5.0)


def test_options_are_validated(ctx):
    from paper_1109_5981_b200.lsrn import LsrnError
    with pytest.raises(LsrnError, match="EINVAL"):
        ctx.set_option("svd", 9)
    with pytest.raises(LsrnError, match="EINVAL"):
        ctx.set_option("rowpass_nt", 300)
    from paper_1109_5981_b200 import lsrn
    assert lsrn.lib().lsrn_ctx_set_option(ctx.h, 9999, 1) == -1
    with pytest.raises(LsrnError, match="EUNSUPPORTED"):          # JW needs k <= 16384
        with ctx.options(svd="jw"):
            m, n = 16500, 16400                    # refused at planning, before any device work
            X = torch.empty(m, n, dtype=torch.float64, device="cuda")
            ctx.solve(X, torch.zeros(m, dtype=torch.float64, device="cuda"), m, n)


@pytest.mark.parametrize("shape", [(3000, 40), (40, 3000)])
def test_lambda_path_from_zero(ctx, shape):
    """A path that starts at lambda = 0 and moves to lambda > 0 (the Tikhonov block grows the
    long vectors; solve_path sizes one workspace for the whole path, so the cached sketch of
    G A stays valid)."""
    rng = np.random.default_rng(3)
    m, n = shape
    A = rng.standard_normal((m, n))
    b = rng.standard_normal(m)
    X = torch.from_numpy(A if m >= n else np.ascontiguousarray(A.T)).cuda()
    bd = torch.from_numpy(b).cuda()
    path = ctx.solve_path(X, bd, m, n, [0.0, 0.1, 0.0], solver="cs")
    for lam, (x, rep) in zip([0.0, 0.1, 0.0], path):
        ref = brute.ridge(A, b, lam) if lam > 0 else brute.min_length(A, b)[0]
        assert np.linalg.norm(x.cpu().numpy() - ref) <= 1e-9 * np.linalg.norm(ref)


def test_binding_rejects_bad_vectors(ctx):
    p = small("c5")
    X = p.X.cuda()
    with pytest.raises(TypeError):
        ctx.solve(X, p.b.float().cuda(), p.m, p.n)
    with pytest.raises(ValueError):
        ctx.solve(X, p.b, p.m, p.n)                          # b on the CPU
    with pytest.raises(ValueError):
        ctx.solve(X, p.b.cuda()[:-1], p.m, p.n)              # wrong length
    with pytest.raises(ValueError):
        ctx.solve(X, torch.stack([p.b, p.b], 1).cuda()[:, 0], p.m, p.n)   # non-contiguous
    with pytest.raises(ValueError):
        ctx.solve(p.X, p.b.cuda(), p.m, p.n)                 # A on the CPU without host_io
    with pytest.raises(ValueError):
        ctx.solve(X, p.b.cuda(), p.m, p.n, x_out=torch.empty(p.n + 1, dtype=torch.float64, device="cuda"))
