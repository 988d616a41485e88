"""The input recipes: CSR structure of c4 / t4 per SURVEY C15 (20
distinct columns per row drawn uniformly WITHOUT replacement, sorted, plus the
dense columns) and the shard property (any row shard is bit-identical to the same
rows of the whole matrix)."""
import itertools
import math

import numpy as np
import torch

from synth.generate import _distinct_sorted, make_problem


def test_distinct_sorted_is_uniform_over_subsets():
    # pool 9, 3 per row: 84 subsets; the rejection path (4 * 3 <= 9); chi-square at 60000 rows
    gen = torch.Generator().manual_seed(7)
    f64 = dict(dtype=torch.float64, device="cpu")
    c = _distinct_sorted(gen, 60000, 3, 9, f64)
    assert (c[:, 1:] > c[:, :-1]).all()
    idx = {s: i for i, s in enumerate(itertools.combinations(range(9), 3))}
    cnt = np.bincount([idx[tuple(r)] for r in c.tolist()], minlength=len(idx))
    e = 60000 / len(idx)
    chi2 = float(((cnt - e) ** 2 / e).sum())
    # 83 degrees of freedom: mean 83, sd 12.9; a stratified or biased draw is far outside
    assert chi2 < 83 + 5 * math.sqrt(2 * 83), chi2
    # the stratified recipe (one draw per third of the pool) could never give {0, 1, 2}
    assert cnt[idx[(0, 1, 2)]] > 0


def test_distinct_sorted_dense_rows_permutation_path():
    gen = torch.Generator().manual_seed(3)
    c = _distinct_sorted(gen, 20000, 4, 6, dict(dtype=torch.float64, device="cpu"))
    assert (c[:, 1:] > c[:, :-1]).all() and int(c.min()) == 0 and int(c.max()) == 5
    cnt = np.bincount(c.reshape(-1).numpy(), minlength=6)      # each column in 4/6 of the rows
    assert np.all(np.abs(cnt / 20000 - 4 / 6) < 0.02), cnt


def test_c4_recipe_structure_and_shards():
    p = make_problem("c4", m=20000, n=300, nnz_random=20, dense_cols=50)
    nz = p.colind.view(-1, 70).long()
    assert (nz[:, 1:] > nz[:, :-1]).all()                      # sorted, distinct
    assert (nz[:, 20:] == torch.arange(250, 300)).all()        # the dense columns
    assert int(nz[:, :20].max()) < 250
    # column frequency of the random part: uniform (each column in 20/250 of the rows)
    f = np.bincount(nz[:, :20].reshape(-1).numpy(), minlength=250) / 20000
    assert np.all(np.abs(f - 20 / 250) < 0.015)
    # adjacent columns co-occur as often as any pair (the stratified draw made pairs
    # inside one stratum impossible)
    adj = ((nz[:, :20].unsqueeze(2) == torch.arange(0, 249)).any(1)
           & (nz[:, :20].unsqueeze(2) == torch.arange(1, 250)).any(1)).sum().item()
    assert adj > 0
    q = make_problem("c4", m=20000, n=300, nnz_random=20, dense_cols=50, shard=(8000, 17000))
    assert torch.equal(q.colind, p.colind[8000 * 70:17000 * 70])
    assert torch.equal(q.val, p.val[8000 * 70:17000 * 70])
