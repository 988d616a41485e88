"""Synthetic problem generators for configs c1..c5 (BASELINE.json) and scaled variants.

Recipe:
  c1  dense 2000 x 100, A = U diag(sigma) V^T, U, V Haar (QR of a Gaussian,
      sign-fixed so diag(R) > 0), sigma_i = 10^(-6 i / 99) (1 -> 1e-6),
      b = A x0 + 1e-3 N(0,1), x0 ~ N(0, I).             Stand-in for §6.2.
  c2  dense 1e5 x 2000, rank 1800, sigma_i = 10^(-4 i / 1799) for i < 1800, 0 after,
      b ~ N(0,1).                                          Stand-in for P:1079-1087.
  c3  dense 2000 x 2e5 (wide), A_ij ~ N(0,1) * 10^(-3 i / 1999) (row scales),
      b ~ N(0,1), lambda = 1e-3.                           Stand-in for P:1064-1077 + §5.
  c4  CSR 2e6 x 2e4: per row 20 random columns among the first 19 950 (one
      uniform draw in each of 20 equal strata, so distinct and sorted) plus the 50
      dense columns 19 950..19 999; values N(0,1), dense-column values x 1e3,
      b ~ N(0,1).                                          Stand-in for P:1115-1153.
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
        A = torch.zeros(self.m, self.n, dtype=torch.float64, device=self.val.device)
        rows = torch.repeat_interleave(torch.arange(self.m, device=self.val.device),
                                       self.rowptr[1:] - self.rowptr[:-1])
        A[rows, self.colind.long()] = self.val
        return A

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val.cpu().numpy(), self.colind.cpu().numpy(),
                              self.rowptr.cpu().numpy()), shape=(self.m, self.n))


def _haar(L, r, gen, device):
    """L x r matrix with orthonormal columns, Haar distributed (sign-fixed QR)."""
    Z = torch.randn(L, r, generator=gen, dtype=torch.float64, device=device)
    Q, R = torch.linalg.qr(Z)
    d = torch.sign(torch.diagonal(R))
    d[d == 0] = 1
    return Q * d


def make_problem(name, device="cpu", m=None, n=None, seed=None, **over):
    """Build config `name` (c1..c5), optionally rescaled (m, n overrides)."""
    cfg = dict(CONFIGS[name])
    cfg.update(over)
    m = cfg["m"] if m is None else m
    n = cfg["n"] if n is None else n
    seed = 1109 * 1000 + cfg["num"] if seed is None else seed
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    f64 = dict(dtype=torch.float64, device=device)
    kind = cfg["kind"]
    x0 = None
    meta = dict(seed=seed, cfg=cfg)
    if kind == "dense" and cfg["spectrum"] == "haar":
        k = min(m, n)
        base = CONFIGS[name]
        frac = base["rank"] / min(base["m"], base["n"])     # c1: 1.0, c2: 0.9
        rank = cfg["rank"] if "rank" in over else max(1, int(round(frac * k)))
        rank = min(rank, k)
        i = torch.arange(rank, **f64)
        sig = 10.0 ** (-cfg["log_range"] * i / max(rank - 1, 1))
        U = _haar(max(m, n), rank, gen, device)
        V = _haar(min(m, n), rank, gen, device)
        Ut = U * sig                                  # L x rank
        X = Ut @ V.T                                  # long-index-major L x k
        meta.update(rank=rank, sigma=sig, kappa=float(sig[0] / sig[-1]))
    elif kind == "dense" and cfg["spectrum"] == "rowscale":
        # wide A (m < n): rows scaled; stored as X = A^T (n x m) row-major
        L, k = max(m, n), min(m, n)
        X = torch.randn(L, k, generator=gen, **f64)
        sc = 10.0 ** (-cfg["log_range"] * torch.arange(k, **f64) / max(k - 1, 1))
        X.mul_(sc)                                    # column c of X = row c of A
        meta.update(row_scales=sc)
    elif kind == "dense" and cfg["spectrum"] == "colscale":
        L, k = max(m, n), min(m, n)
        X = torch.empty(L, k, **f64)
        sc = 10.0 ** (-cfg["log_range"] * torch.arange(k, **f64) / max(k - 1, 1))
        step = max(1, (1 << 27) // k)
        for r0 in range(0, L, step):
            r1 = min(L, r0 + step)
            X[r0:r1] = torch.randn(r1 - r0, k, generator=gen, **f64)
            X[r0:r1].mul_(sc)
        meta.update(col_scales=sc)
    elif kind == "csr":
        nr = cfg["nnz_random"]
        nd = min(cfg["dense_cols"], n - nr) if n > nr else 0
        pool = n - nd
        nnz_row = nr + nd
        width = pool / nr
        lo = (torch.arange(nr, **f64) * width)
        u = torch.rand(m, nr, generator=gen, **f64)
        cols_r = torch.clamp((lo + u * width).floor().to(torch.int64),
                             max=pool - 1)
        # strata are disjoint and increasing: distinct and sorted
        cols_d = torch.arange(pool, n, device=device, dtype=torch.int64).expand(m, nd)
        colind = torch.cat([cols_r, cols_d], dim=1).to(torch.int32).reshape(-1)
        val = torch.randn(m, nnz_row, generator=gen, **f64)
        val[:, nr:] *= cfg["dense_scale"]
        rowptr = torch.arange(m + 1, device=device, dtype=torch.int64) * nnz_row
        b = torch.randn(m, generator=gen, **f64)
        meta.update(nnz=m * nnz_row, dense_cols=nd)
        return Problem(name, m, n, "csr", cfg["gamma"], cfg["lam"], b,
                       rowptr=rowptr, colind=colind, val=val.reshape(-1), meta=meta)
    else:
        raise ValueError(f"unknown spectrum/kind for {name}")
    if cfg["rhs"] == "model":
        x0 = torch.randn(n, generator=gen, **f64)
        if m >= n:
            b = X @ x0
        else:
            b = X.T @ x0
        b = b + 1e-3 * torch.randn(m, generator=gen, **f64)
    else:
        b = torch.randn(m, generator=gen, **f64)
    return Problem(name, m, n, "dense", cfg["gamma"], cfg["lam"], b, X=X.contiguous(),
                   x0=x0, meta=meta)


def small(name, device="cpu"):
    """Scaled-down instances used by CPU tests (same recipe, oracle-fast sizes)."""
    shapes = {"c1": (2000, 100), "c2": (3000, 120), "c3": (60, 3000),
              "c4": (6000, 200), "c5": (4000, 150)}
    m, n = shapes[name]
    over = {}
    if name == "c4":
        over = dict(nnz_random=8, dense_cols=6)
    return make_problem(name, device=device, m=m, n=n, **over)


def kappa_of(sig):
    return float(sig.max() / sig.min()) if sig.numel() else math.inf
