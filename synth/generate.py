"""Synthetic problem generators for configs c1..c5 (BASELINE.json) and scaled variants.

Recipe:
  c1  dense 2000 x 100, A = U diag(sigma) V^T, U, V Haar (QR of a Gaussian,
      sign-fixed so diag(R) > 0), sigma_i = 10^(-6 i / 99) (1 -> 1e-6),
      b = A x0 + 1e-3 N(0,1), x0 ~ N(0, I).             Stand-in for §6.2.
  c2  dense 1e5 x 2000, rank 1800, sigma_i = 10^(-4 i / 1799) for i < 1800, 0 after,
      b ~ N(0,1).                                          Stand-in for P:1079-1087.
  c3  dense 2000 x 2e5 (wide), A_ij ~ N(0,1) * 10^(-3 i / 1999) (row scales),
      b ~ N(0,1), lambda = 1e-3.                           Stand-in for P:1064-1077 + §5.
  c4  CSR 2e6 x 2e4: per row 20 distinct columns drawn uniformly without
      replacement from the first 19 950 (C15: rejection of rows with a repeated
      column, so every 20-subset is equally likely), sorted, plus the 50 dense
      columns 19 950..19 999; values N(0,1), dense-column values x 1e3,
      b ~ N(0,1).                                          Stand-in for P:1115-1153.
  t4  the same recipe with 21 random columns and no dense ones, as the CSR of A^T.
  c5  dense 1e6 x 1e4, A_ij ~ N(0,1) * 10^(-5 j / 9999) (column scales),
      b = A x0 + 1e-3 N(0,1).                              Stand-in for Table 3.
Seeds: data seed = 1109 * 1000 + config number (C16); the sketch seed is 5981.

Layout: the long index is the major one ("long-index-major"): tall dense A is
row-major m x n; wide dense A is stored as X = A^T row-major (n x m), i.e. A
column-major.  CSR is row-major CSR of the tall A (rowptr int64, colind int32,
val fp64).
"""
import math
from dataclasses import dataclass, field

import torch

SKETCH_SEED = 5981

CONFIGS = {
    "c1": dict(num=1, kind="dense", m=2000, n=100, gamma=2.0, lam=0.0,
               spectrum="haar", rank=100, log_range=6.0, rhs="model"),
    "c2": dict(num=2, kind="dense", m=100_000, n=2000, gamma=2.0, lam=0.0,
               spectrum="haar", rank=1800, log_range=4.0, rhs="randn"),
    "c3": dict(num=3, kind="dense", m=2000, n=200_000, gamma=2.0, lam=1e-3,
               spectrum="rowscale", log_range=3.0, rhs="randn"),
    "c4": dict(num=4, kind="csr", m=2_000_000, n=20_000, gamma=2.0, lam=0.0,
               nnz_random=20, dense_cols=50, dense_scale=1e3, rhs="randn"),
    "c5": dict(num=5, kind="dense", m=1_000_000, n=10_000, gamma=2.0, lam=0.0,
               spectrum="colscale", log_range=5.0, rhs="model"),
    # NEXT-2: the shape of the paper's cluster workload tnimg_4 (Table 3,
    # P:1207-1219): 1024 x 4e6, ~21 nonzeros per column; the real
    # TinyImages data is not available, so columns get 21 distinct uniform rows, N(0,1).
    "t4": dict(num=6, kind="csr", m=1024, n=4_000_000, gamma=2.0, lam=0.0,
               nnz_random=21, dense_cols=0, dense_scale=1.0, rhs="randn"),
}


@dataclass
class Problem:
    name: str
    m: int
    n: int
    kind: str                 # "dense" or "csr"
    gamma: float
    lam: float
    b: torch.Tensor
    X: torch.Tensor = None    # dense, long-index-major (A if m >= n else A^T), row-major
    rowptr: torch.Tensor = None
    colind: torch.Tensor = None
    val: torch.Tensor = None
    x0: torch.Tensor = None
    meta: dict = field(default_factory=dict)

    @property
    def tall(self):
        return self.m >= self.n

    def dense_A(self):
        """A itself (a view for dense; materialised for CSR)."""
        if self.kind == "dense":
            return self.X if self.tall else self.X.T
        L, k = max(self.m, self.n), min(self.m, self.n)
        X = torch.zeros(L, k, dtype=torch.float64, device=self.val.device)
        rows = torch.repeat_interleave(torch.arange(L, device=self.val.device),
                                       self.rowptr[1:] - self.rowptr[:-1])
        X[rows, self.colind.long()] = self.val
        return X if self.tall else X.T

    def to_scipy(self):
        """A itself as scipy CSR (for a wide A the stored CSR is that of A^T)."""
        import scipy.sparse as sp
        L, k = max(self.m, self.n), min(self.m, self.n)
        X = sp.csr_matrix((self.val.cpu().numpy(), self.colind.cpu().numpy(),
                           self.rowptr.cpu().numpy()), shape=(L, k))
        return X if self.tall else X.T.tocsr()


def _haar(L, r, gen, device):
    """L x r matrix with orthonormal columns, Haar distributed (sign-fixed QR)."""
    Z = torch.randn(L, r, generator=gen, dtype=torch.float64, device=device)
    Q, R = torch.linalg.qr(Z)
    d = torch.sign(torch.diagonal(R))
    d[d == 0] = 1
    return Q * d


BLOCK = 8192   # long-index rows per independently seeded block (shard-invariant data)


def _block_gen(seed, g, device):
    gen = torch.Generator(device=device)
    gen.manual_seed(seed * 1_000_003 + 7919 * g + 1)
    return gen


def make_problem(name, device="cpu", m=None, n=None, seed=None, shard=None, keep_factors=False, **over):
    """Build config `name` (c1..c5), optionally rescaled (m, n overrides).

    keep_factors=True keeps the generator's U, V (Haar recipes) in meta, so tests can
    form the exact pseudoinverse solution at full size.
    shard=(lo, hi) generates only long-index rows [lo, hi) of X (and the matching
    rows of b for a tall A) -- the bytes are identical to the same rows of the
    full problem for the i.i.d. recipes (c3, c4, c5), which are generated in
    independently seeded blocks of BLOCK long-index rows.  The Haar recipes
    (c1, c2) need the full matrix and are sliced after generation.
    """
    cfg = dict(CONFIGS[name])
    cfg.update(over)
    m = cfg["m"] if m is None else m
    n = cfg["n"] if n is None else n
    seed = 1109 * 1000 + cfg["num"] if seed is None else seed
    f64 = dict(dtype=torch.float64, device=device)
    kind = cfg["kind"]
    L, k = max(m, n), min(m, n)
    lo, hi = (0, L) if shard is None else (int(shard[0]), int(shard[1]))
    meta = dict(seed=seed, cfg=cfg, shard=(lo, hi))
    x0 = None
    if kind == "dense" and cfg["spectrum"] == "haar":
        gen = torch.Generator(device=device)
        gen.manual_seed(seed)
        base = CONFIGS[name]
        frac = base["rank"] / min(base["m"], base["n"])     # c1: 1.0, c2: 0.9
        rank = cfg["rank"] if "rank" in over else max(1, int(round(frac * k)))
        rank = min(rank, k)
        i = torch.arange(rank, **f64)
        sig = 10.0 ** (-cfg["log_range"] * i / max(rank - 1, 1))
        U = _haar(L, rank, gen, device)
        V = _haar(k, rank, gen, device)
        X = (U * sig) @ V.T                           # long-index-major L x k
        meta.update(rank=rank, sigma=sig, kappa=float(sig[0] / sig[-1]))
        if keep_factors:                              # X = U diag(sig) V^T (test pins: exact pseudoinverse)
            meta.update(U=U, V=V)
        del U
        if cfg["rhs"] == "model":
            x0 = torch.randn(n, generator=gen, **f64)
            b = (X @ x0 if m >= n else X.T @ x0) + 1e-3 * torch.randn(m, generator=gen, **f64)
        else:
            b = torch.randn(m, generator=gen, **f64)
        if shard is not None:
            X = X[lo:hi].contiguous()
            if m >= n:
                b = b[lo:hi].contiguous()
        return Problem(name, m, n, "dense", cfg["gamma"], cfg["lam"], b, X=X.contiguous(), x0=x0, meta=meta)

    gx = torch.Generator(device=device)
    gx.manual_seed(seed * 7 + 3)
    if cfg.get("rhs") == "model":
        x0 = torch.randn(n, generator=gx, **f64)
    blocks = range(lo // BLOCK, (hi + BLOCK - 1) // BLOCK) if hi > lo else range(0)
    if kind == "dense":
        sc = 10.0 ** (-cfg["log_range"] * torch.arange(k, **f64) / max(k - 1, 1))
        X = torch.empty(hi - lo, k, **f64)
        bt = torch.empty(hi - lo, **f64) if (m >= n) else None
        for g in blocks:
            g0, g1 = g * BLOCK, min(L, (g + 1) * BLOCK)
            gen = _block_gen(seed, g, device)
            blk = torch.randn(g1 - g0, k, generator=gen, **f64).mul_(sc)
            a0, a1 = max(g0, lo), min(g1, hi)
            X[a0 - lo:a1 - lo] = blk[a0 - g0:a1 - g0]
            if bt is not None:
                if cfg["rhs"] == "model":
                    bb = blk @ x0 + 1e-3 * torch.randn(g1 - g0, generator=gen, **f64)
                else:
                    bb = torch.randn(g1 - g0, generator=gen, **f64)
                bt[a0 - lo:a1 - lo] = bb[a0 - g0:a1 - g0]
        if m >= n:
            b = bt
            meta.update(col_scales=sc)
        else:       # wide: b is short (length m), replicated
            b = torch.randn(m, generator=gx, **f64)
            meta.update(row_scales=sc)
        return Problem(name, m, n, "dense", cfg["gamma"], cfg["lam"], b, X=X, x0=x0, meta=meta)

    if kind == "csr":
        nr = cfg["nnz_random"]
        nd = min(cfg["dense_cols"], k - nr) if k > nr else 0   # columns of X (k = min(m, n))
        pool = k - nd
        nnz_row = nr + nd
        cols_d = torch.arange(pool, k, device=device, dtype=torch.int64)
        rows = hi - lo
        colind = torch.empty(rows, nnz_row, dtype=torch.int32, device=device)
        val = torch.empty(rows, nnz_row, **f64)
        b = torch.empty(rows, **f64)
        for g in blocks:
            g0, g1 = g * BLOCK, min(L, (g + 1) * BLOCK)
            gen = _block_gen(seed, g, device)
            cr = _distinct_sorted(gen, g1 - g0, nr, pool, f64)
            ci = torch.cat([cr, cols_d.expand(g1 - g0, nd)], dim=1).to(torch.int32)
            vv = torch.randn(g1 - g0, nnz_row, generator=gen, **f64)
            vv[:, nr:] *= cfg["dense_scale"]
            bb = torch.randn(g1 - g0, generator=gen, **f64)
            a0, a1 = max(g0, lo), min(g1, hi)
            colind[a0 - lo:a1 - lo] = ci[a0 - g0:a1 - g0]
            val[a0 - lo:a1 - lo] = vv[a0 - g0:a1 - g0]
            b[a0 - lo:a1 - lo] = bb[a0 - g0:a1 - g0]
        rowptr = torch.arange(rows + 1, device=device, dtype=torch.int64) * nnz_row
        meta.update(nnz=rows * nnz_row, dense_cols=nd)
        if m < n:             # wide: X = A^T in CSR (A in CSC); b is short (length m), replicated
            b = torch.randn(m, generator=gx, **f64)
        return Problem(name, m, n, "csr", cfg["gamma"], cfg["lam"], b, rowptr=rowptr,
                       colind=colind.reshape(-1), val=val.reshape(-1), meta=meta)
    raise ValueError(f"unknown spectrum/kind for {name}")


def _draw_sorted(gen, rows, nr, pool, f64):
    u = torch.rand(rows, nr, generator=gen, **f64)
    c = torch.minimum((u * pool).floor().to(torch.int64), torch.tensor(pool - 1, device=u.device))
    return c.sort(dim=1).values


def _distinct_sorted(gen, rows, nr, pool, f64):
    """nr distinct columns per row, uniform over the nr-subsets of range(pool), sorted
    (C15): nr uniform draws per row, and any row with a repeat is drawn again whole
    (rejection keeps the subset distribution uniform)."""
    if nr > pool:
        raise ValueError(f"{nr} distinct columns out of {pool}")
    if 4 * nr > pool:         # dense rows: the first nr of a random permutation instead
        keys = torch.rand(rows, pool, generator=gen, **f64)
        return keys.argsort(dim=1)[:, :nr].sort(dim=1).values
    c = _draw_sorted(gen, rows, nr, pool, f64)
    if nr < 2:
        return c
    bad = (c[:, 1:] == c[:, :-1]).any(dim=1).nonzero().squeeze(1)
    while bad.numel():
        d = _draw_sorted(gen, bad.numel(), nr, pool, f64)
        c[bad] = d
        bad = bad[(d[:, 1:] == d[:, :-1]).any(dim=1)]
    return c


def small(name, device="cpu"):
    """Scaled-down instances used by CPU tests (same recipe, oracle-fast sizes)."""
    shapes = {"c1": (2000, 100), "c2": (3000, 120), "c3": (60, 3000),
              "c4": (6000, 200), "c5": (4000, 150), "t4": (64, 6000)}
    m, n = shapes[name]
    over = {}
    if name == "c4":
        over = dict(nnz_random=8, dense_cols=6)
    if name == "t4":
        over = dict(nnz_random=5)
    return make_problem(name, device=device, m=m, n=n, **over)


def kappa_of(sig):
    return float(sig.max() / sig.min()) if sig.numel() else math.inf
