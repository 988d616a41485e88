"""The Gaussian projection matrix G, defined entry-by-entry (oracle; test infra only).

Paper: Alg. 1 step 2 "Generate G = randn(s, m)" and Alg. 2 step 2
"G = randn(n, s)": i.i.d. standard normal entries.  The paper used a
threaded Ziggurat; this build fixes the counter-based definition of
SURVEY §8(c) C9 so that any tile of G can be regenerated anywhere:

  key      = (seed & 0xffffffff, seed >> 32)
  counter  = (q = i >> 1,  lo32(j),  hi32(j),  tag = 0)        i < s sketch row,
                                                               j long index
  o        = Philox4x32-10(counter, key)
  w0 = o.x | o.y << 32,  w1 = o.z | o.w << 32                  (uint64)
  u1 = ((w0 >> 11) + 1) * 2^-53  in (0, 1],   u2 = (w1 >> 11) * 2^-53  in [0, 1)
  rho = sqrt(-2 ln u1)
  G[2q, j] = rho cos(2 pi u2),   G[2q+1, j] = rho sin(2 pi u2)   (Box-Muller)

"Tall form": G is s x (L + k) where L is the long dimension and k the short one;
columns j >= L are the Tikhonov block (§5).  The wide sketch uses
G_wide(j, i) = G(i, j), so sketch_wide(A) = sketch_tall(A^T)^T.

Evaluation is in numpy long double (x87 80-bit) by default and rounded once to
fp64, so the oracle's normals are within ~1 ulp of the mathematical value.
"""
import numpy as np

from .philox import philox4x32_10

TWO_PI_LD = np.longdouble(8) * np.arctan(np.longdouble(1))
TWO_M53 = 2.0 ** -53


def _key(seed):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32


def uniforms(seed, q, j, tag=0):
    """(u1, u2) as exact fp64 values for counters (q, j) (broadcast arrays)."""
    k0, k1 = _key(seed)
    q = np.asarray(q, dtype=np.uint64)
    j = np.asarray(j, dtype=np.uint64)
    q, j = np.broadcast_arrays(q, j)
    lo = (j & np.uint64(0xFFFFFFFF)).astype(np.uint64)
    hi = (j >> np.uint64(32)).astype(np.uint64)
    o = philox4x32_10(q, lo, hi, np.full(q.shape, tag, dtype=np.uint64), k0, k1)
    return uniforms_from_words(o)


def uniforms_from_words(o):
    """(u1, u2) from the four uint32 Philox output words o = (x, y, z, w) (reading C9)."""
    w0 = np.asarray(o[0]).astype(np.uint64) | (np.asarray(o[1]).astype(np.uint64) << np.uint64(32))
    w1 = np.asarray(o[2]).astype(np.uint64) | (np.asarray(o[3]).astype(np.uint64) << np.uint64(32))
    # (w >> 11) < 2^53: exact in fp64; the scaling by 2^-53 is exact.
    u1 = ((w0 >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * TWO_M53
    u2 = (w1 >> np.uint64(11)).astype(np.float64) * TWO_M53
    return u1, u2


def box_muller(u1, u2, precise=True):
    """Box-Muller pair (z0, z1) = rho (cos 2 pi u2, sin 2 pi u2), rho = sqrt(-2 ln u1).

    precise=True evaluates in long double and rounds once to fp64.
    """
    if precise:
        u1 = np.asarray(u1, dtype=np.longdouble)
        u2 = np.asarray(u2, dtype=np.longdouble)
        rho = np.sqrt(np.longdouble(-2) * np.log(u1))
        ang = TWO_PI_LD * u2
        return (rho * np.cos(ang)).astype(np.float64), (rho * np.sin(ang)).astype(np.float64)
    rho = np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * np.pi * u2
    return rho * np.cos(ang), rho * np.sin(ang)


def gaussian(seed, rows, cols, precise=True):
    """G[rows][:, cols] as a dense fp64 array, rows/cols = integer index arrays."""
    rows = np.asarray(rows, dtype=np.int64).ravel()
    cols = np.asarray(cols, dtype=np.int64).ravel()
    out = np.empty((rows.size, cols.size), dtype=np.float64)
    if rows.size == 0 or cols.size == 0:
        return out
    qs, inv = np.unique(rows >> 1, return_inverse=True)
    u1, u2 = uniforms(seed, qs[:, None], cols[None, :])
    z0, z1 = box_muller(u1, u2, precise=precise)
    odd = (rows & 1).astype(bool)
    out[~odd] = z0[inv[~odd]]
    out[odd] = z1[inv[odd]]
    return out


def gaussian_block(seed, r0, r1, c0, c1, precise=True):
    """Contiguous block G[r0:r1, c0:c1]."""
    return gaussian(seed, np.arange(r0, r1), np.arange(c0, c1), precise=precise)
