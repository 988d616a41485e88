"""GPU parity of the CSR path (K4 sketch, CSR long pass) against the CPU oracle.

Sketch Ã = G A for sparse A (Alg. 1 step 3; "automatically speeds up
when A is sparse"): relative Frobenius <= 1e-12 (north star).  Solves:
identical iteration counts and rank, x within max(1e-9, 20 kappa u) and the
A-norm form (C18).  Cases cover the heavy/light column split (none,
some, more than the 64-column cap), empty rows and columns, shards with a
non-zero global offset, the Tikhonov block and host buffers.
"""
import numpy as np
import pytest
import scipy.sparse as sp
import torch

from oracle.lsrn import solve as orc_solve
from oracle.sketch import plan as orc_plan
from oracle.sketch import sketch as orc_sketch
from synth.generate import make_problem, small

pytestmark = pytest.mark.gpu
U = 2.0 ** -53


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1109_5981_b200 import lsrn
    c = lsrn.Context()
    yield c
    c.close()


def _gpu_csr(A):
    from paper_1109_5981_b200.lsrn import Csr
    A = sp.csr_matrix(A)
    A.sort_indices()
    return Csr(torch.from_numpy(A.indptr.astype(np.int64)).cuda(),
               torch.from_numpy(A.indices.astype(np.int32)).cuda(),
               torch.from_numpy(A.data.astype(np.float64)).cuda())


def _random_csr(m, n, nnz_row, dense_cols=0, dense_scale=1.0, empty_rows=0, seed=0):
    rng = np.random.default_rng(seed)
    rows, cols, vals = [], [], []
    light = n - dense_cols
    for i in range(m):
        if i < empty_rows:
            continue
        cs = rng.choice(light, size=min(nnz_row, light), replace=False) if light > 0 else np.array([], int)
        cs = np.concatenate([cs, np.arange(light, n)])
        v = rng.standard_normal(cs.size)
        v[cs >= light] *= dense_scale
        rows += [i] * cs.size
        cols += list(cs)
        vals += list(v)
    return sp.csr_matrix((vals, (rows, cols)), shape=(m, n))


def _relfro(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("m,n,nnz_row,dense_cols,lam,empty", [
    (3000, 120, 6, 0, 0.0, 0),       # light columns only (no heavy block)
    (4000, 150, 5, 7, 0.0, 17),      # heavy block ND=16 + empty rows
    (2500, 100, 3, 80, 0.0, 0),      # 80 dense columns: capped at 64 heavy, 16 dense ones stay light
    (3000, 90, 4, 20, 0.5, 0),       # heavy ND=32 + tall Tikhonov block
    (777, 61, 2, 3, 0.0, 5),         # odd s = 122? (gamma 2 -> 122), ragged everything
    (2597, 1300, 9, 0, 0.0, 3),      # 3 column tiles of the slab kernel, ragged last chunk and tile
    (1100, 530, 4, 40, 0.25, 0),     # 2 tiles, heavy + light, Tikhonov block
])
@pytest.mark.parametrize("light,gmb,hfma", [(0, -1, -1), (1, -1, -1), (2, -1, -1), (2, 1, -1), (2, -1, 1)])
def test_csr_sketch_vs_oracle(ctx, m, n, nnz_row, dense_cols, lam, empty, light, gmb, hfma):
    """light = 0: per-nonzero light sketch (G[:, j] regenerated per nonzero); light = 1:
    the generate-once slab kernel (each G[i, j] once per 512-column tile); light = 2: G
    generated once per chunk of rows and read by the heavy and light kernels (gmb = 1: a
    1 MB G budget, so several chunks; hfma = 1: the FP64-FMA heavy kernel instead of DMMA)."""
    A = _random_csr(m, n, nnz_row, dense_cols, 1e3, empty, seed=m + n)
    with ctx.options(csr_sketch=light, sketch_g=gmb, csr_heavy_fma=hfma):
        At = ctx.sketch(_gpu_csr(A), m, n, 2.0, lam, seed=5981).cpu().numpy()
    p = orc_plan(m, n, 2.0, lam)
    ref = orc_sketch(A, p["s"], 5981, p["sigma_x"], p["sigma_i"])
    assert _relfro(At, ref) <= 1e-12


def test_csr_sketch_equals_dense_sketch(ctx):
    A = _random_csr(2000, 80, 5, 4, 10.0, 3, seed=11)
    Ad = torch.from_numpy(A.toarray()).cuda()
    a1 = ctx.sketch(_gpu_csr(A), 2000, 80).cpu().numpy()
    a2 = ctx.sketch(Ad, 2000, 80).cpu().numpy()
    assert _relfro(a1, a2) <= 1e-13


@pytest.mark.parametrize("light,gmb", [(0, -1), (1, -1), (2, -1), (2, 1)])
def test_csr_sketch_shards_sum_to_full(ctx, light, gmb):
    m, n = 3100, 70
    A = _random_csr(m, n, 4, 5, 100.0, 0, seed=2)
    with ctx.options(csr_sketch=light, sketch_g=gmb):
        full = ctx.sketch(_gpu_csr(A), m, n).cpu().numpy()
        acc = np.zeros_like(full)
        for lo, hi in [(0, 999), (999, 1000), (1000, 3100)]:
            acc += ctx.sketch(_gpu_csr(A[lo:hi]), m, n, lo=lo, cnt=hi - lo).cpu().numpy()
    assert _relfro(acc, full) <= 1e-13


def test_csr_sketch_repeatable_bitwise(ctx):
    A = _random_csr(3000, 100, 6, 5, 1e3, 0, seed=9)
    G = _gpu_csr(A)
    a1 = ctx.sketch(G, 3000, 100)
    a2 = ctx.sketch(G, 3000, 100)
    assert torch.equal(a1, a2)


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
def test_csr_solve_small_c4(ctx, solver):
    p = small("c4")
    A = p.to_scipy()
    b = p.b.numpy()
    from paper_1109_5981_b200.lsrn import Csr
    X = Csr(p.rowptr.cuda(), p.colind.cuda(), p.val.cuda())
    x, rep = ctx.solve(X, p.b.cuda(), p.m, p.n, solver=solver)
    orc = orc_solve(A, b, solver=solver)
    assert rep["r"] == orc["r"] and rep["s"] == orc["s"]
    assert rep["iters"] == orc["iters"]
    sv = np.linalg.svd(A.toarray(), compute_uv=False)
    kappa = sv[0] / sv[-1]
    xg = x.cpu().numpy()
    rel = np.linalg.norm(xg - orc["x"]) / np.linalg.norm(orc["x"])
    assert rel <= max(1e-9, 20 * kappa * U), rel
    an = np.linalg.norm(A @ (xg - orc["x"])) / np.linalg.norm(A @ orc["x"])
    assert an <= 1e-11, an


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
def test_csr_solve_tikhonov_and_dense_agree(ctx, solver):
    A = _random_csr(1500, 60, 4, 6, 30.0, 2, seed=4)
    b = np.random.default_rng(1).standard_normal(1500)
    lam = 0.3
    x1, r1 = ctx.solve(_gpu_csr(A), torch.from_numpy(b).cuda(), 1500, 60, solver=solver, lam=lam)
    x2, r2 = ctx.solve(torch.from_numpy(A.toarray()).cuda(), torch.from_numpy(b).cuda(), 1500, 60, solver=solver,
                       lam=lam)
    orc = orc_solve(A, b, solver=solver, lam=lam)
    assert r1["iters"] == r2["iters"] == orc["iters"]
    for x in (x1, x2):
        rel = np.linalg.norm(x.cpu().numpy() - orc["x"]) / np.linalg.norm(orc["x"])
        assert rel <= 1e-9, rel


def test_csr_host_io_matches_device(ctx):
    from paper_1109_5981_b200.lsrn import Csr
    p = small("c4")
    xd, rd = ctx.solve(Csr(p.rowptr.cuda(), p.colind.cuda(), p.val.cuda()), p.b.cuda(), p.m, p.n, solver="cs")
    Xh = Csr(p.rowptr.pin_memory(), p.colind.pin_memory(), p.val.pin_memory())
    xh, rh = ctx.solve(Xh, p.b.pin_memory(), p.m, p.n, solver="cs", host_io=True)
    assert torch.equal(xd.cpu(), xh) and rd["iters"] == rh["iters"]


@pytest.mark.parametrize("lam", [0.0, 0.05])
def test_csr_wide_sketch_vs_oracle(ctx, lam):
    """Wide sparse A (m < n) given as the CSR of A^T (Alg. 2; §5 wide form)."""
    AT = _random_csr(3000, 60, 4, 3, 10.0, 2, seed=21)          # X = A^T: 3000 x 60, A: 60 x 3000
    m, n = 60, 3000
    At = ctx.sketch(_gpu_csr(AT), m, n, 2.0, lam, seed=5981).cpu().numpy()
    p = orc_plan(m, n, 2.0, lam)
    ref = orc_sketch(AT, p["s"], 5981, p["sigma_x"], p["sigma_i"])
    assert _relfro(At, ref) <= 1e-12


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
@pytest.mark.parametrize("lam", [0.0, 0.05])
def test_csr_wide_solve_vs_oracle_and_dense(ctx, solver, lam):
    """Wide CSR solves (NEXT-2 shape: few rows, many sparse columns) against the oracle and the
    dense wide path on the same matrix."""
    AT = _random_csr(2500, 50, 5, 2, 5.0, 0, seed=33)
    A = AT.T.tocsr()
    m, n = 50, 2500
    b = np.random.default_rng(2).standard_normal(m)
    x1, r1 = ctx.solve(_gpu_csr(AT), torch.from_numpy(b).cuda(), m, n, solver=solver, lam=lam)
    x2, r2 = ctx.solve(torch.from_numpy(AT.toarray()).cuda(), torch.from_numpy(b).cuda(), m, n, solver=solver,
                       lam=lam)
    orc = orc_solve(A, b, solver=solver, lam=lam)
    assert r1["iters"] == r2["iters"] == orc["iters"] and r1["r"] == orc["r"]
    for x in (x1, x2):
        rel = np.linalg.norm(x.cpu().numpy() - orc["x"]) / np.linalg.norm(orc["x"])
        assert rel <= 1e-9, rel


@pytest.mark.parametrize("bad", ["dup", "unsorted", "range"])
def test_csr_rejects_non_canonical(ctx, bad):
    from paper_1109_5981_b200.lsrn import Csr, LsrnError
    rowptr = torch.tensor([0, 3, 5, 7, 8, 9, 10], dtype=torch.int64)          # 6 x 5, tall
    good = [0, 2, 3, 1, 3, 0, 4, 1, 2, 4]
    cols = {"dup": [0, 2, 2, 1, 3, 0, 4, 1, 2, 4], "unsorted": [0, 3, 2, 1, 3, 0, 4, 1, 2, 4],
            "range": [0, 2, 5, 1, 3, 0, 4, 1, 2, 4]}[bad]
    ones = torch.ones(10, dtype=torch.float64).cuda()
    ctx.sketch(Csr(rowptr.cuda(), torch.tensor(good, dtype=torch.int32).cuda(), ones), 6, 5, 1.5)
    X = Csr(rowptr.cuda(), torch.tensor(cols, dtype=torch.int32).cuda(), ones)
    with pytest.raises(LsrnError, match="EINVAL"):
        ctx.sketch(X, 6, 5, 1.5)


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
def test_csr_small_t4_vs_oracle(ctx, solver):
    """NEXT-2 recipe (tnimg-shaped: few rows, ~21 nonzeros per column) at test size."""
    from paper_1109_5981_b200.lsrn import Csr
    p = small("t4")
    A = p.to_scipy()
    b = p.b.numpy()
    x, rep = ctx.solve(Csr(p.rowptr.cuda(), p.colind.cuda(), p.val.cuda()), p.b.cuda(), p.m, p.n, solver=solver)
    orc = orc_solve(A, b, solver=solver)
    assert rep["iters"] == orc["iters"] and rep["r"] == orc["r"]
    rel = np.linalg.norm(x.cpu().numpy() - orc["x"]) / np.linalg.norm(orc["x"])
    assert rel <= 1e-9, rel


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
@pytest.mark.parametrize("m,nnz_row,dense,empty,lam", [
    (4400, 4, 3, 0, 0.0),       # heavy ND = 16 (one heavy column per lane)
    (4600, 40, 40, 25, 0.0),    # ND = 64 (two per lane, 40 used), 40 light entries per row, empty rows
    (4400, 6, 0, 0, 0.3),       # no heavy block, tall Tikhonov block
])
def test_csr_solve_wide_k_uses_csc_gather(ctx, solver, m, nnz_row, dense, empty, lam):
    """k > 2048: the CSR long pass runs in the heavy-dense + light-CSR form (csr_rowdot_hl) and
    gathers the light part of w = A^T u from the CSC copy (for k <= 2048 it accumulates w in
    shared memory in one pass)."""
    n = 2100
    A = _random_csr(m, n, nnz_row, dense, 20.0, empty, seed=41 + m)
    b = np.random.default_rng(3).standard_normal(m)
    x, rep = ctx.solve(_gpu_csr(A), torch.from_numpy(b).cuda(), m, n, solver=solver, gamma=1.5, lam=lam)
    orc = orc_solve(A, b, solver=solver, gamma=1.5, lam=lam, precise_g=False)
    assert rep["iters"] == orc["iters"] and rep["r"] == orc["r"]
    rel = np.linalg.norm(x.cpu().numpy() - orc["x"]) / np.linalg.norm(orc["x"])
    assert rel <= 1e-9, rel


def _ragged_csr(m, n, seed):
    """Row lengths mixed: empty rows, rows of 3..45 entries, a 32-row chunk of 40-entry
    rows and one 120-entry row (longer than a warp)."""
    rng = np.random.default_rng(seed)
    lens = rng.choice([0, 3, 7, 21, 45], size=m, p=[0.05, 0.4, 0.3, 0.2, 0.05])
    lens[200:232] = 40
    lens[300] = 120
    rows, cols, vals = [], [], []
    for i, L in enumerate(lens):
        cs = rng.choice(n, size=min(int(L), n), replace=False)
        rows += [i] * cs.size
        cols += list(cs)
        vals += list(rng.standard_normal(cs.size))
    return sp.csr_matrix((vals, (rows, cols)), shape=(m, n))


@pytest.mark.parametrize("solver", ["lsqr", "cs"])
@pytest.mark.parametrize("rowdot,variant", [(-1, -1), (3, -1), (-1, 0), (-1, 6), (-1, 10)])
def test_csr_single_pass_staged_and_direct_chunks(ctx, solver, rowdot, variant):
    """k <= 2048 long pass on ragged rows (empty rows, rows longer than a warp, a chunk of
    long rows): the single-pass kernels (LSRN_OPT_CSR_ALL: 0 one pair of rows in flight,
    6 / 10 the pipelined groups, 10 with t in shared memory) and the two-kernel CSC-gather form (LSRN_OPT_CSR_ROWDOT = 3)
    against the oracle."""
    A = _ragged_csr(5000, 300, seed=8)
    b = np.random.default_rng(9).standard_normal(A.shape[0])
    with ctx.options(csr_rowdot=rowdot, csr_all=variant):
        x, rep = ctx.solve(_gpu_csr(A), torch.from_numpy(b).cuda(), A.shape[0], A.shape[1], solver=solver)
    orc = orc_solve(A, b, solver=solver)
    assert rep["iters"] == orc["iters"] and rep["r"] == orc["r"]
    xg = x.cpu().numpy()
    sv = np.linalg.svd(A.toarray(), compute_uv=False)
    kappa = sv[0] / sv[sv > sv[0] * 1e-12][-1]
    rel = np.linalg.norm(xg - orc["x"]) / np.linalg.norm(orc["x"])
    assert rel <= max(1e-9, 20 * kappa * U), rel
    an = np.linalg.norm(A @ (xg - orc["x"])) / np.linalg.norm(A @ orc["x"])
    assert an <= 1e-11, an


@pytest.mark.parametrize("variant", [0, 6, 10])
@pytest.mark.parametrize("lam", [0.0, 0.05])
def test_csr_single_pass_variants_wide_ragged(ctx, variant, lam):
    """Wide ragged CSR (X = A^T with empty, short and > 32-entry rows; CS keeps the
    acc_j += ca u_j update of the wide form in the same pass) for every single-pass
    variant: iteration count, rank and x against the oracle."""
    AT = _ragged_csr(4100, 260, seed=17)
    A = AT.T.tocsr()
    m, n = AT.shape[1], AT.shape[0]
    b = np.random.default_rng(3).standard_normal(m)
    with ctx.options(csr_all=variant):
        x, rep = ctx.solve(_gpu_csr(AT), torch.from_numpy(b).cuda(), m, n, solver="cs", lam=lam)
    orc = orc_solve(A, b, solver="cs", lam=lam)
    assert rep["iters"] == orc["iters"] and rep["r"] == orc["r"]
    rel = np.linalg.norm(x.cpu().numpy() - orc["x"]) / np.linalg.norm(orc["x"])
    assert rel <= 1e-9, rel


@pytest.mark.parametrize("light", [-1, 14, 48, 162, 22])
@pytest.mark.parametrize("m,n,dense_cols,gamma", [(3000, 150, 7, 2.0), (2500, 61, 0, 2.01), (1800, 300, 3, 1.5)])
def test_csr_light_kernel_variants_vs_oracle(ctx, light, m, n, dense_cols, gamma):
    """Stored-G light kernel (LSRN_OPT_CSR_LIGHT = 10 columns per CTA + gathers in flight),
    with several G chunks (1 MB budget), an odd s and a partial last sketch-row block:
    relative Frobenius <= 1e-12 against the oracle's sketch."""
    A = _random_csr(m, n, 5, dense_cols, 4.0, 3, seed=51)
    with ctx.options(csr_light=light, sketch_g=1):
        At = ctx.sketch(_gpu_csr(A), m, n, gamma).cpu().numpy()
    p = orc_plan(m, n, gamma, 0.0)
    assert At.shape[0] == p["s"]
    ref = orc_sketch(A, p["s"], 5981, p["sigma_x"], p["sigma_i"])
    assert _relfro(At, ref) <= 1e-12
