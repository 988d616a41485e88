"""Pins for oracle/philox.py and oracle/gaussian.py (no GPU).

Philox: Random123 known-answer vectors (tests/golden/philox_kat.txt) and cuRAND's
curand_Philox4x32_10 compiled for the host (library routine, bitwise).
Box-Muller: exact uniform mapping, closed-form special values,
agreement with numpy's libm evaluation, moments and a KS test against scipy's
normal CDF, shard/tile invariance of the (i, j) -> G[i, j] definition.
"""
import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle.gaussian import box_muller, gaussian, gaussian_block, uniforms
from oracle.philox import philox4x32_10


def _kat(golden_dir):
    rows = []
    with open(os.path.join(golden_dir, "philox_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append([int(t, 16) for t in line.split()])
    return rows


def test_philox_known_answer_vectors(golden_dir):
    for r in _kat(golden_dir):
        out = philox4x32_10(r[0], r[1], r[2], r[3], r[4], r[5])
        assert [int(o) for o in out] == r[6:10]


CURAND_SRC = r"""
#include <cstdio>
#define QUALIFIERS static inline
#include <vector_types.h>
#include <vector_functions.h>
#include <curand_philox4x32_x.h>
int main() {
  unsigned a, b, c, d, e, f;
  while (scanf("%u %u %u %u %u %u", &a, &b, &c, &d, &e, &f) == 6) {
    uint4 o = curand_Philox4x32_10(make_uint4(a, b, c, d), make_uint2(e, f));
    printf("%u %u %u %u\n", o.x, o.y, o.z, o.w);
  }
  return 0;
}
"""


def test_philox_matches_curand_host(tmp_path):
    cxx = shutil.which("g++")
    inc = "/usr/local/cuda/include"
    if cxx is None or not os.path.exists(os.path.join(inc, "curand_philox4x32_x.h")):
        pytest.skip("g++ or cuRAND headers not available")
    src = tmp_path / "p.cpp"
    src.write_text(CURAND_SRC)
    exe = tmp_path / "p"
    subprocess.run([cxx, "-O1", "-I", inc, str(src), "-o", str(exe)], check=True)
    rng = np.random.default_rng(7)
    ctr = rng.integers(0, 2 ** 32, size=(2000, 6), dtype=np.uint64)
    ctr[:10, 1:4] = 0                                  # small counters too
    inp = "\n".join(" ".join(str(int(v)) for v in row) for row in ctr) + "\n"
    res = subprocess.run([str(exe)], input=inp, capture_output=True, text=True, check=True)
    ref = np.array([[int(t) for t in ln.split()] for ln in res.stdout.strip().splitlines()],
                   dtype=np.uint64)
    out = philox4x32_10(ctr[:, 0], ctr[:, 1], ctr[:, 2], ctr[:, 3], 0, 0)
    # keys differ per row: evaluate row by row for the key, vectorised otherwise
    got = np.empty_like(ref)
    for key in {(int(a), int(b)) for a, b in ctr[:, 4:6]}:
        sel = (ctr[:, 4] == key[0]) & (ctr[:, 5] == key[1])
        o = philox4x32_10(ctr[sel, 0], ctr[sel, 1], ctr[sel, 2], ctr[sel, 3], key[0], key[1])
        got[sel] = np.stack(o, axis=1)
    assert np.array_equal(got, ref)
    del out


def test_uniform_mapping_exact():
    seed = 0x123456789ABCDEF
    q = np.arange(50, dtype=np.uint64)
    j = np.arange(50, dtype=np.uint64) * np.uint64(977) + np.uint64(2 ** 33)
    u1, u2 = uniforms(seed, q, j)
    o = philox4x32_10(q, j & np.uint64(0xFFFFFFFF), j >> np.uint64(32), 0,
                      seed & 0xFFFFFFFF, seed >> 32)
    for t in range(50):
        w0 = int(o[0][t]) | (int(o[1][t]) << 32)
        w1 = int(o[2][t]) | (int(o[3][t]) << 32)
        assert u1[t] == ((w0 >> 11) + 1) / 2.0 ** 53
        assert u2[t] == (w1 >> 11) / 2.0 ** 53
    assert np.all(u1 > 0) and np.all(u1 <= 1) and np.all(u2 >= 0) and np.all(u2 < 1)


def test_box_muller_special_values():
    z0, z1 = box_muller(np.array([1.0, np.exp(-0.5), np.exp(-0.5), np.exp(-2.0)]),
                        np.array([0.3, 0.0, 0.25, 0.5]))
    assert z0[0] == 0.0 and z1[0] == 0.0                       # u1 = 1 -> rho = 0
    assert abs(z0[1] - 1.0) < 1e-16 and z1[1] == 0.0            # rho = 1, angle 0
    assert abs(z0[2]) < 1e-16 and abs(z1[2] - 1.0) < 1e-16      # angle pi/2
    assert abs(z0[3] + 2.0) < 4e-16 and abs(z1[3]) < 1e-15      # rho = 2, angle pi


def test_box_muller_precise_vs_libm():
    u1, u2 = uniforms(99, np.arange(20000) % 97, np.arange(20000))
    a0, a1 = box_muller(u1, u2, precise=True)
    b0, b1 = box_muller(u1, u2, precise=False)
    scale = np.maximum(1.0, np.sqrt(a0 ** 2 + a1 ** 2))
    assert np.max(np.abs(a0 - b0) / scale) < 2e-15
    assert np.max(np.abs(a1 - b1) / scale) < 2e-15


def test_gaussian_moments_and_ks():
    from scipy import stats
    G = gaussian_block(42, 0, 100, 0, 10000, precise=False).ravel()   # 1e6 draws
    assert abs(G.mean()) < 5e-3
    assert abs(G.var() - 1.0) < 5e-3
    assert abs(stats.skew(G)) < 0.01
    assert abs(stats.kurtosis(G)) < 0.02
    assert stats.kstest(G[:200000], "norm").pvalue > 1e-3
    Gp = gaussian_block(42, 0, 2, 0, 200000, precise=False)
    assert abs(np.corrcoef(Gp[0], Gp[1])[0, 1]) < 0.01                 # pair independence


def test_gaussian_determinism_seed_and_tiling():
    A = gaussian_block(42, 0, 37, 0, 101)
    B = gaussian_block(42, 0, 37, 0, 101)
    C = gaussian_block(43, 0, 37, 0, 101)
    assert np.array_equal(A, B)
    assert np.mean(A != C) > 0.99
    # any tile / shard of G is the same function of (i, j)
    T = gaussian_block(42, 5, 20, 33, 90)
    assert np.array_equal(T, A[5:20, 33:90])
    R = gaussian(42, [36, 3, 3, 0], [100, 1])
    assert np.array_equal(R, A[[36, 3, 3, 0]][:, [100, 1]])
    # large long index (hi32(j) != 0) is a different stream
    D = gaussian(42, [0, 1], [5, 5 + 2 ** 32])
    assert D[0, 0] != D[0, 1]
