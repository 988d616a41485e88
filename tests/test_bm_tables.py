"""CPU check of the table-driven Box-Muller transform (K1 v2, philox_bm.cuh) that the
GPU kernels use: the generated constants (csrc/bm_tables.h) and a host model of the
device arithmetic (same operation order, fma emulated exactly) against 40-digit
references of ln u1, sin / cos (2 pi u2) and the normals (reading C9).  The GPU
path itself is checked against the oracle in tests/test_gpu_parity.py."""
import decimal
import math
import os
import re
from decimal import Decimal as D

import numpy as np
import pytest

decimal.getcontext().prec = 40
HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1109_5981_b200", "csrc",
                   "bm_tables.h")
PI = D("3.14159265358979323846264338327950288419716939937510")


@pytest.fixture(scope="module")
def tab():
    src = open(HDR).read()
    sc = {m.group(1): float.fromhex(m.group(2)) for m in re.finditer(r"constexpr double (\w+) = ([^;]+);", src)}
    body = re.search(r"kTable\[TAB_SIZE\] = \{([^}]*)\}", src).group(1)
    t = [float.fromhex(x.strip()) for x in body.replace("\n", " ").split(",") if x.strip()]
    assert len(t) == 512
    return sc, t


def fma(a, b, c):
    return float(D(a) * D(b) + D(c))


def ln_u1(w0, sc, t):
    n1 = (w0 >> 11) + 1
    e = n1.bit_length() - 1
    mant = ((n1 << (52 - e)) & ((1 << 52) - 1)) if e <= 52 else 0
    m = 1.0 + mant * 2.0 ** -52
    i = mant >> 45
    r = fma(m, t[i], -1.0)
    p = sc["LOG1P_C8"]
    for k in (7, 6, 5, 4, 3, 2):
        p = fma(p, r, sc[f"LOG1P_C{k}"])
    poly = fma(r * r, p, r)
    E = float(e - 53)
    return fma(E, sc["LN2_HI"], t[128 + i]) + (fma(E, sc["LN2_LO"], t[256 + i]) + poly)


def sincos(w1, sc, t):
    n2 = w1 >> 11
    k, j, dm = n2 >> 51, (n2 >> 45) & 63, n2 & ((1 << 45) - 1)
    d = dm * 2.0 ** -45
    d2 = d * d
    sp = sc["SIN_C9"]
    for c in (7, 5, 3, 1):
        sp = fma(sp, d2, sc[f"SIN_C{c}"])
    sb = sp * d
    cp = sc["COS_C10"]
    for c in (8, 6, 4, 2):
        cp = fma(cp, d2, sc[f"COS_C{c}"])
    cb = fma(cp, d2, 1.0)
    sa, ca = t[384 + j], t[448 + j]
    s, c = fma(sa, cb, ca * sb), fma(ca, cb, -(sa * sb))
    return [(s, c), (c, -s), (-s, -c), (-c, s)][k]


def dsin(x):
    s, term, k = D(0), x, 1
    while abs(term) > D(10) ** -45:
        s += term
        term = -term * x * x / ((k + 1) * (k + 2))
        k += 2
    return s


def test_table_invariants(tab):
    sc, t = tab
    invc = t[:128]
    for i, ic in enumerate(invc):
        frac = (D(ic) * 512)
        assert frac == frac.to_integral_value() or i == 127        # 9 significant bits
        for m in (D(1) + D(i) / 128, D(1) + D(i + 1) / 128):
            assert abs(m * D(ic) - 1) < D(2) ** -7
    assert invc[127] == 0.5
    for i in range(128):                                            # heads have <= 42 bits
        h = t[128 + i]
        if h:
            assert float(h * 2.0 ** (41 - math.floor(math.log2(abs(h))))).is_integer()


def test_box_muller_model_accuracy(tab):
    sc, t = tab
    rng = np.random.default_rng(3)
    words = [(int(a), int(b)) for a, b in rng.integers(0, 2 ** 63, size=(3000, 2))]
    words += [((2 ** 64 - 1) - int(rng.integers(0, 2 ** min(k + 1, 62))), 0) for k in range(40)]
    words += [(int(rng.integers(0, 2 ** (k + 1))), (k % 4) << 62) for k in range(40)]
    words += [(0, ((q << 51) + (j << 45)) << 11) for q in range(4) for j in (0, 1, 63)]
    worst_ln = worst_sc = worst_z = 0.0
    for w0, w1 in words:
        u1 = D((w0 >> 11) + 1) * D(2) ** -53
        ref_ln = u1.ln()
        got = ln_u1(w0, sc, t)
        if ref_ln != 0:
            worst_ln = max(worst_ln, float(abs(D(got) - ref_ln) / abs(ref_ln)))
        else:
            assert got == 0.0
        a = 2 * PI * D(w1 >> 11) * D(2) ** -53
        rs, rc = dsin(a), dsin(a + PI / 2)
        s, c = sincos(w1, sc, t)
        worst_sc = max(worst_sc, float(abs(D(s) - rs)), float(abs(D(c) - rc)))
        rho = math.sqrt(-2.0 * got)
        rref = (-2 * ref_ln).sqrt()
        for z, zr in ((rho * c, rref * rc), (rho * s, rref * rs)):
            worst_z = max(worst_z, float(abs(D(z) - zr) / max(D(1), abs(zr))))
    assert worst_ln <= 4e-16, worst_ln
    assert worst_sc <= 4e-16, worst_sc
    assert worst_z <= 1e-15, worst_z
