"""ctypes loader of the oracle's C part (oracle/c/lsrn_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Built with gcc -O2 -fopenmp into oracle/_build/liboracle.so on first use (or by
__graft_entry__.build()).  No fast-math, no FMA contraction flags: the C code's
arithmetic is exactly what it spells out.  Only tests/, smoke() and bench.py's
CPU legs may load it; the product never does.
"""
import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "lsrn_oracle.c")
OUT = os.path.join(HERE, "_build", "liboracle.so")

_lib = None


def build(force=False):
    """Compile the C oracle (gcc) if the .so is missing or older than its source."""
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= os.path.getmtime(SRC):
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    tmp = OUT + ".tmp%d" % os.getpid()
    subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off", "-o", tmp, SRC, "-lm"],
                   check=True, capture_output=True)
    os.replace(tmp, OUT)
    return OUT


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64, u64, dbl, vp = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p
        L.orc_philox4x32_10.argtypes = [vp, ctypes.c_uint32, ctypes.c_uint32, vp]
        L.orc_philox4x32_10.restype = None
        L.orc_gaussian.argtypes = [u64, vp, vp, i64, vp]
        L.orc_gaussian.restype = None
        L.orc_sketch_dense.argtypes = [vp, i64, i64, i64, i64, u64, dbl, dbl, vp]
        L.orc_sketch_dense.restype = ctypes.c_int
        L.orc_sketch_csr.argtypes = [vp, vp, vp, i64, i64, i64, u64, dbl, dbl, vp]
        L.orc_sketch_csr.restype = ctypes.c_int
        L.orc_jacobi_svd.argtypes = [vp, i64, i64, ctypes.c_int, vp, vp]
        L.orc_jacobi_svd.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def philox(ctr, k0, k1):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    o = np.empty(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c), k0 & 0xFFFFFFFF, k1 & 0xFFFFFFFF, _p(o))
    return o


def gaussian(seed, rows, cols):
    """G[rows[t], cols[t]] for paired index arrays (long double Box-Muller, C9)."""
    r = np.ascontiguousarray(rows, dtype=np.int64).ravel()
    c = np.ascontiguousarray(cols, dtype=np.int64).ravel()
    out = np.empty(r.size, dtype=np.float64)
    lib().orc_gaussian(int(seed) & 0xFFFFFFFFFFFFFFFF, _p(r), _p(c), r.size, _p(out))
    return out


def sketch_dense(X, s, seed, sx=1.0, si=0.0):
    """Naive-loop Ãt = sx G[:, :L] X + si G[:, L:L+k] of a dense row-major X (L x k)."""
    X = np.ascontiguousarray(X, dtype=np.float64)
    L, k = X.shape
    At = np.empty((s, k), dtype=np.float64)
    rc = lib().orc_sketch_dense(_p(X), L, k, k, s, int(seed) & 0xFFFFFFFFFFFFFFFF, sx, si, _p(At))
    if rc != 0:
        raise RuntimeError(f"orc_sketch_dense failed ({rc})")
    return At


def sketch_csr(X, s, seed, sx=1.0, si=0.0):
    """The same for a scipy CSR X (canonical)."""
    X = X.tocsr()
    X.sort_indices()
    L, k = X.shape
    rp = np.ascontiguousarray(X.indptr, dtype=np.int64)
    ci = np.ascontiguousarray(X.indices, dtype=np.int32)
    v = np.ascontiguousarray(X.data, dtype=np.float64)
    At = np.empty((s, k), dtype=np.float64)
    rc = lib().orc_sketch_csr(_p(rp), _p(ci), _p(v), L, k, s, int(seed) & 0xFFFFFFFFFFFFFFFF, sx, si, _p(At))
    if rc != 0:
        raise RuntimeError(f"orc_sketch_csr failed ({rc})")
    return At


def jacobi_svd(A, max_sweeps=60):
    """One-sided Jacobi SVD of A (s x k): returns (sigma descending, V k x k, sweeps)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    s, k = A.shape
    sig = np.empty(k, dtype=np.float64)
    V = np.empty((k, k), dtype=np.float64)
    sw = lib().orc_jacobi_svd(_p(A), s, k, max_sweeps, _p(sig), _p(V))
    if sw < 0:
        raise RuntimeError(f"orc_jacobi_svd failed ({sw})")
    return sig, V, sw
