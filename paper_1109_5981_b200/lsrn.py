"""Thin ctypes binding of liblsrn.so (include/lsrn.h): argument marshalling only.

Every step of the LSRN path runs in the library's sm_100a kernels; torch is used
for device memory (tensors, the workspace), the CUDA stream and, for multi-GPU,
to exchange the NCCL unique id through torch.distributed.  There is no CPU
fallback: importing this module without the built library raises.
"""
import contextlib
import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblsrn.so")

LSRN_OK = 0
LSRN_DENSE, LSRN_CSR = 0, 1
MODE_PREDICTABLE, MODE_ADAPTIVE = 0, 1
HOST_IO = 1
SKETCH_ONLY = 2
REUSE_SKETCH = 4
COMPENSATED = 8            # precision = 1 (lsrn.h LSRN_COMPENSATED, C18(ii))
STATUS = {0: "LSRN_OK", -1: "LSRN_EINVAL", -2: "LSRN_EDIM", -3: "LSRN_ENONFINITE", -4: "LSRN_ERANK0",
          -5: "LSRN_ESVD", -6: "LSRN_ENOMEM", -7: "LSRN_ECUDA", -8: "LSRN_ENCCL", -9: "LSRN_EUNSUPPORTED"}

# every symbol include/lsrn.h declares
EXPORTS = ["lsrn_last_error", "lsrn_version", "lsrn_nccl_unique_id", "lsrn_ctx_create", "lsrn_ctx_destroy",
           "lsrn_ctx_set_profiling", "lsrn_workspace_size", "lsrn_sketch",
           "lsrn_solve_lsqr", "lsrn_solve_cs", "lsrn_debug_gaussian", "lsrn_debug_box_muller", "lsrn_debug_rowpass", "lsrn_last_stats",
           "lsrn_choose_gamma", "lsrn_ctx_set_option", "lsrn_ctx_set_host_collectives"]

# lsrn_ctx_set_option keys (include/lsrn.h)
OPTIONS = {"profiling": 1, "svd": 2, "graph_reuse": 3, "hostio_chunk_mb": 4, "lsqr_sync": 5, "bcast_n": 6,
           "sketch_kernel": 100, "sketch_tile": 101, "sketch_maxcl": 102, "sketch_nsplit": 103, "sketch_x_l2": 104,
           "sketch_chunks": 105, "sketch_g": 106,
           "rowpass_keep": 110, "rowpass_occ": 111, "rowpass_wide1": 112, "rowpass_wide2": 113,
           "rowpass_asyncx": 114, "rowpass_nt": 115, "rowpass_tr": 116, "rowpass_budget_kb": 117,
           "rowpass_wide_slice": 118, "rowpass_pf": 119, "csr_rowdot": 120, "csr_sketch": 121, "csr_heavy_fma": 123,
           "csr_all": 124, "csr_light": 126}
SVD_METHODS = {"auto": 0, "jw": 1, "gesvd": 2, "polar": 3, "qr": 4}
OPTION_DEFAULTS = {k: -1 for k in OPTIONS}
OPTION_DEFAULTS.update(profiling=0, svd=0, graph_reuse=1, hostio_chunk_mb=32, lsqr_sync=0, bcast_n=1)

HOST_ALLREDUCE = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64)
HOST_BCAST = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64,
                              ctypes.c_int)


class LsrnError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Matrix(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad_", ctypes.c_int32), ("m", ctypes.c_int64), ("n", ctypes.c_int64),
                ("lo", ctypes.c_int64), ("cnt", ctypes.c_int64), ("val", ctypes.c_void_p), ("ld", ctypes.c_int64),
                ("rowptr", ctypes.c_void_p), ("colind", ctypes.c_void_p), ("nnz", ctypes.c_int64)]


class Opts(ctypes.Structure):
    _fields_ = [("gamma", ctypes.c_double), ("lambda_", ctypes.c_double), ("tol", ctypes.c_double),
                ("alpha", ctypes.c_double), ("seed", ctypes.c_uint64), ("mode", ctypes.c_int32),
                ("max_iter", ctypes.c_int32), ("flags", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class Report(ctypes.Structure):
    _fields_ = [("s", ctypes.c_int64), ("r", ctypes.c_int64), ("iters", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("sigma_L", ctypes.c_double), ("sigma_U", ctypes.c_double),
                ("alpha", ctypes.c_double), ("t_sketch", ctypes.c_double), ("t_allreduce", ctypes.c_double),
                ("t_svd", ctypes.c_double), ("t_iter", ctypes.c_double), ("t_total", ctypes.c_double),
                ("rnorm_est", ctypes.c_double), ("svd_used", ctypes.c_int32), ("collectives", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib():
    """Load liblsrn.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} not built: run `python -m paper_1109_5981_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(_LIB_PATH)
        vp, i32, i64, u64, dbl, sz = (ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_uint64,
                                      ctypes.c_double, ctypes.c_size_t)
        L.lsrn_last_error.restype = ctypes.c_char_p
        L.lsrn_version.restype = ctypes.c_char_p
        sigs = {
            "lsrn_nccl_unique_id": [vp],
            "lsrn_ctx_create": [ctypes.POINTER(vp), vp, i32, i32, vp],
            "lsrn_ctx_destroy": [vp],
            "lsrn_ctx_set_profiling": [vp, i32],
            "lsrn_workspace_size": [vp, ctypes.POINTER(Matrix), ctypes.POINTER(Opts), ctypes.POINTER(sz)],
            "lsrn_sketch": [vp, ctypes.POINTER(Matrix), dbl, dbl, u64, vp, sz, vp, ctypes.POINTER(i64)],
            "lsrn_solve_lsqr": [vp, ctypes.POINTER(Matrix), vp, ctypes.POINTER(Opts), vp, sz, vp,
                                ctypes.POINTER(Report)],
            "lsrn_solve_cs": [vp, ctypes.POINTER(Matrix), vp, ctypes.POINTER(Opts), vp, sz, vp,
                              ctypes.POINTER(Report)],
            "lsrn_debug_gaussian": [vp, u64, vp, vp, i64, vp],
            "lsrn_debug_box_muller": [vp, vp, i64, i32, vp],
            "lsrn_last_stats": [vp, ctypes.POINTER(ctypes.c_double), i32],
            "lsrn_debug_rowpass": [vp, vp, i64, i64, i64, vp, vp, dbl, vp, vp, vp, i32, ctypes.POINTER(dbl)],
            "lsrn_choose_gamma": [ctypes.POINTER(Report), i64, i64, dbl, i32, dbl, dbl,
                                  ctypes.POINTER(dbl), ctypes.POINTER(dbl)],
            "lsrn_ctx_set_option": [vp, i32, i64],
            "lsrn_ctx_set_host_collectives": [vp, HOST_ALLREDUCE, HOST_BCAST, vp],
        }
        for name, args in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = ctypes.c_int
        _lib = L
    return _lib


def choose_gamma(probe, m, n, tol=1e-14, solver="lsqr", lo=1.2, hi=3.0):
    """lsrn_choose_gamma (NEXT-4, §6.3): the gamma minimising the stage-time
    model calibrated by a probe solve's report (a dict from Context.solve).  Host-only."""
    rep = Report(**{f: probe[f] for f, _ in Report._fields_ if f in probe})
    g, t = ctypes.c_double(), ctypes.c_double()
    _check(lib().lsrn_choose_gamma(ctypes.byref(rep), m, n, tol, 0 if solver == "lsqr" else 1, lo, hi,
                                   ctypes.byref(g), ctypes.byref(t)))
    return {"gamma": round(g.value, 2), "t_model": t.value}


def _check(code):
    if code != LSRN_OK:
        raise LsrnError(code, lib().lsrn_last_error().decode())


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _check_vec(name, v, length, device, host):
    """b / x_out: float64, contiguous, 1-D of the given length, on the device (or on the
    CPU for host IO) -- the C ABI takes raw pointers and cannot check any of this."""
    if not isinstance(v, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if v.dtype != torch.float64:
        raise TypeError(f"{name} must be float64, got {v.dtype}")
    if v.dim() != 1 or v.numel() != length:
        raise ValueError(f"{name} must be 1-D of length {length}, got shape {tuple(v.shape)}")
    if not v.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if host:
        if v.device.type != "cpu":
            raise ValueError(f"{name} must be a CPU tensor with host_io=True")
    elif v.device != device:
        raise ValueError(f"{name} must live on {device}, got {v.device}")


def _check_matrix_device(X, device, host):
    t = X.val if isinstance(X, Csr) else X
    if host:
        if t.device.type != "cpu":
            raise ValueError("A must be on the CPU with host_io=True")
    elif t.device != device:
        raise ValueError(f"A must live on {device}, got {t.device}")


def dense(X, m, n, lo=0, cnt=None):
    """Matrix descriptor for a long-index-major dense shard X (cnt x k, row-major)."""
    if X.dtype != torch.float64:
        raise TypeError("A must be float64")
    if X.dim() != 2 or (X.stride(1) != 1 and X.shape[1] > 1):   # a 1-column stride is immaterial
        raise ValueError("X must be a 2-D tensor with unit column stride (long-index-major)")
    cnt = X.shape[0] if cnt is None else cnt
    return Matrix(kind=LSRN_DENSE, m=m, n=n, lo=lo, cnt=cnt, val=X.data_ptr(), ld=X.stride(0) if cnt > 1 else
                  max(X.shape[1], 1), rowptr=None, colind=None, nnz=0), X


class Csr:
    """A row shard of a tall CSR A: rowptr int64[cnt+1], colind int32[nnz], val float64[nnz] (torch tensors)."""

    def __init__(self, rowptr, colind, val):
        if rowptr.dtype != torch.int64 or colind.dtype != torch.int32 or val.dtype != torch.float64:
            raise TypeError("CSR needs rowptr int64, colind int32, val float64")
        if not (rowptr.is_contiguous() and colind.is_contiguous() and val.is_contiguous()):
            raise ValueError("CSR arrays must be contiguous")
        self.rowptr, self.colind, self.val = rowptr, colind, val

    @property
    def rows(self):
        return self.rowptr.numel() - 1

    @property
    def device(self):
        return self.val.device


def csr(A, m, n, lo=0, cnt=None):
    """Matrix descriptor for a CSR row shard (see Csr)."""
    cnt = A.rows if cnt is None else cnt
    nnz = A.val.numel()
    return Matrix(kind=LSRN_CSR, m=m, n=n, lo=lo, cnt=cnt, val=A.val.data_ptr() if nnz else None, ld=0,
                  rowptr=A.rowptr.data_ptr(), colind=A.colind.data_ptr() if nnz else None, nnz=nnz), A


def describe(X, m, n, lo=0, cnt=None):
    """Descriptor for a dense long-index-major tensor or a Csr shard."""
    if isinstance(X, Csr):
        return csr(X, m, n, lo, cnt)
    return dense(X, m, n, lo, cnt)


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(lib().lsrn_nccl_unique_id(buf))
    return buf.raw


class Context:
    """An lsrn_ctx bound to the current CUDA device and a torch stream."""

    def __init__(self, stream=None, nranks=1, rank=0, nccl_id=None, null_stream=False):
        self.device = torch.device("cuda", torch.cuda.current_device())
        # a dedicated (capturable) stream: the iteration loop is captured as a CUDA graph.
        # null_stream=True passes NULL (the legacy stream) to the library, which then
        # runs on a stream of its own joined to the legacy stream at every call.
        if null_stream:
            self.stream = torch.cuda.default_stream(self.device)
            handle = None
        else:
            self.stream = stream if stream is not None else torch.cuda.Stream(self.device)
            handle = ctypes.c_void_p(self.stream.cuda_stream)
        h = ctypes.c_void_p()
        idbuf = ctypes.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        _check(lib().lsrn_ctx_create(ctypes.byref(h), handle, nranks, rank, idbuf))
        self.h = h
        self.nranks, self.rank = nranks, rank
        self._ws = None
        self._host_coll = None

    def close(self):
        if self.h:
            lib().lsrn_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_profiling(self, on=True):
        _check(lib().lsrn_ctx_set_profiling(self.h, 1 if on else 0))

    def set_option(self, name, value):
        """lsrn_ctx_set_option by name (OPTIONS); svd also takes 'auto' / 'jw' / 'gesvd' / 'polar'."""
        if name == "svd" and isinstance(value, str):
            value = SVD_METHODS[value]
        _check(lib().lsrn_ctx_set_option(self.h, OPTIONS[name], int(value)))

    @contextlib.contextmanager
    def options(self, **kv):
        """Set options for the duration of a with-block, then restore their defaults."""
        for k_, v_ in kv.items():
            self.set_option(k_, v_)
        try:
            yield self
        finally:
            for k_ in kv:
                self.set_option(k_, OPTION_DEFAULTS[k_])

    def set_host_collectives(self, allreduce, bcast):
        """Host-staged collectives (lsrn_ctx_set_host_collectives).  allreduce(arr) sums the
        float64 numpy array arr in place over the ranks; bcast(arr, root) broadcasts it.
        Python exceptions in the callbacks become LSRN_ENCCL."""
        import numpy as np

        def _ar(user, buf, count):
            try:
                allreduce(np.ctypeslib.as_array(buf, shape=(count,)))
                return 0
            except Exception:
                return 1

        def _bc(user, buf, count, root):
            try:
                bcast(np.ctypeslib.as_array(buf, shape=(count,)), root)
                return 0
            except Exception:
                return 1
        self._host_coll = (HOST_ALLREDUCE(_ar), HOST_BCAST(_bc))     # keep the thunks alive
        _check(lib().lsrn_ctx_set_host_collectives(self.h, self._host_coll[0], self._host_coll[1], None))

    def workspace(self, nbytes):
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = None
            self._ws = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        return self._ws

    def workspace_size(self, mat, opts):
        sz = ctypes.c_size_t()
        _check(lib().lsrn_workspace_size(self.h, ctypes.byref(mat), ctypes.byref(opts), ctypes.byref(sz)))
        return sz.value

    def stats(self):
        out = (ctypes.c_double * 8)()
        _check(lib().lsrn_last_stats(self.h, out, 8))
        keys = ["sketch_ms", "long_pass_ms", "reserved", "launches", "long_pass_timed", "long_pass_bytes",
                "sketch_flops", "graph_launches"]
        return dict(zip(keys, list(out)))

    # ---------------------------------------------------------------- calls
    def _enter(self):
        cur = torch.cuda.current_stream(self.device)
        if cur.cuda_stream != self.stream.cuda_stream:
            self.stream.wait_stream(cur)
        return cur

    def _leave(self, cur):
        if cur.cuda_stream != self.stream.cuda_stream:
            cur.wait_stream(self.stream)

    def sketch(self, X, m, n, gamma=2.0, lam=0.0, seed=5981, lo=0, cnt=None):
        """Tall-form sketch At (s x k) of the shard X (dense or Csr); returns a new device tensor."""
        _check_matrix_device(X, self.device, False)
        mat, _keep = describe(X, m, n, lo, cnt)
        k = min(m, n)
        s = int(torch.tensor(gamma * k, dtype=torch.float64).ceil().item())
        At = torch.empty(s, k, dtype=torch.float64, device=self.device)
        opts = Opts(gamma=gamma, lambda_=lam, tol=0.5, alpha=-1.0, seed=seed, flags=SKETCH_ONLY)
        ws = self.workspace(self.workspace_size(mat, opts))
        s_out = ctypes.c_int64()
        cur = self._enter()
        _check(lib().lsrn_sketch(self.h, ctypes.byref(mat), gamma, lam, seed, _ptr(ws), ws.numel(), _ptr(At),
                                 ctypes.byref(s_out)))
        self._leave(cur)
        assert s_out.value == s
        return At

    def solve(self, X, b, m, n, solver="lsqr", gamma=2.0, lam=0.0, tol=1e-14, seed=5981, alpha=-1.0,
              mode="predictable", max_iter=0, lo=0, cnt=None, x_out=None, host_io=False, reuse_sketch=False,
              precision=0):
        """LSRN solve; X a long-index-major dense shard or a Csr row shard (device, or pinned host with host_io).
        precision: 0 fp64 products, 1 compensated products (LSRN_COMPENSATED; dense, one rank)."""
        if solver not in ("lsqr", "cs"):
            raise ValueError("solver must be 'lsqr' or 'cs'")
        if precision not in (0, 1):
            raise ValueError("precision must be 0 (fp64) or 1 (compensated)")
        _check_matrix_device(X, self.device, host_io)
        if host_io and not isinstance(X, Csr):
            if X.dtype != torch.float64:
                raise TypeError("A must be float64")
            if X.dim() != 2 or (X.stride(1) != 1 and X.shape[1] > 1):   # a 1-column stride is immaterial
                raise ValueError("X must be row-major 2-D")
            cnt_ = X.shape[0] if cnt is None else cnt
            mat = Matrix(kind=LSRN_DENSE, m=m, n=n, lo=lo, cnt=cnt_, val=X.data_ptr(), ld=X.stride(0))
        else:
            mat, _keep = describe(X, m, n, lo, cnt)
        tall = m >= n
        xlen = n if tall else mat.cnt
        _check_vec("b", b, mat.cnt if tall else m, self.device, host_io)
        if x_out is None:
            x_out = torch.empty(xlen, dtype=torch.float64,
                                device="cpu" if host_io else self.device,
                                pin_memory=bool(host_io))
        else:
            _check_vec("x_out", x_out, xlen, self.device, host_io)
        opts = Opts(gamma=gamma, lambda_=lam, tol=tol, alpha=alpha, seed=seed,
                    mode=MODE_ADAPTIVE if mode == "adaptive" else MODE_PREDICTABLE, max_iter=max_iter,
                    flags=(HOST_IO if host_io else 0) | (REUSE_SKETCH if reuse_sketch else 0)
                    | (COMPENSATED if precision == 1 else 0))
        ws = self.workspace(self.workspace_size(mat, opts))
        rep = Report()
        fn = lib().lsrn_solve_lsqr if solver == "lsqr" else lib().lsrn_solve_cs
        cur = self._enter()
        _check(fn(self.h, ctypes.byref(mat), _ptr(b), ctypes.byref(opts), _ptr(ws), ws.numel(), _ptr(x_out),
                  ctypes.byref(rep)))
        self._leave(cur)
        return x_out, rep.as_dict()

    def solve_path(self, X, b, m, n, lambdas, **kw):
        """Solve for a sequence of Tikhonov lambdas, sketching A once (§5):
        the first solve computes G A, the others reuse it (LSRN_REUSE_SKETCH)."""
        # one workspace for the whole path: lambda > 0 adds the Tikhonov block to the long
        # vectors, and a workspace reallocated mid-path would lose the cached sketch
        mat, _keep = describe(X, m, n, kw.get("lo", 0), kw.get("cnt"))
        need = 0
        for lam in lambdas:
            o = Opts(gamma=kw.get("gamma", 2.0), lambda_=lam, tol=kw.get("tol", 1e-14), alpha=kw.get("alpha", -1.0),
                     seed=kw.get("seed", 5981), mode=MODE_PREDICTABLE, max_iter=0,
                     flags=COMPENSATED if kw.get("precision", 0) == 1 else 0)
            need = max(need, self.workspace_size(mat, o))
        self.workspace(need)
        out = []
        for i, lam in enumerate(lambdas):
            x, rep = self.solve(X, b, m, n, lam=lam, reuse_sketch=(i > 0), **kw)
            out.append((x.clone(), rep))
        return out

    def debug_rowpass(self, Y, t, z, coef, sx=1.0, acc=None, reps=1):
        """One fused row pass (lsrn_debug_rowpass) on device tensors; returns (out, ms)
        with out = [sx Y^T z_new ; ||z_new||^2] (z, acc updated in place)."""
        R, C = Y.shape
        out = torch.empty(C + 1, dtype=torch.float64, device=self.device)
        cf = torch.as_tensor(coef, dtype=torch.float64).to(self.device)
        ms = ctypes.c_double(0.0)
        cur = self._enter()
        _check(lib().lsrn_debug_rowpass(self.h, _ptr(Y), R, C, Y.stride(0), _ptr(t), _ptr(cf), sx, _ptr(z),
                                        _ptr(acc) if acc is not None else None, _ptr(out), reps, ctypes.byref(ms)))
        self._leave(cur)
        torch.cuda.synchronize(self.device)
        return out, ms.value

    def debug_box_muller(self, words, mode=0):
        """(count, 2) normals of the Box-Muller transform of (count, 4) uint32 Philox words."""
        w = torch.as_tensor(words).to(torch.int64).to(torch.int32).contiguous().to(self.device)
        n = w.shape[0]
        out = torch.empty(n, 2, dtype=torch.float64, device=self.device)
        cur = self._enter()
        _check(lib().lsrn_debug_box_muller(self.h, _ptr(w), n, mode, _ptr(out)))
        self._leave(cur)
        return out

    def debug_gaussian(self, seed, rows, cols):
        rows = rows.to(self.device, torch.int64).contiguous()
        cols = cols.to(self.device, torch.int64).contiguous()
        out = torch.empty(rows.numel(), dtype=torch.float64, device=self.device)
        cur = self._enter()
        _check(lib().lsrn_debug_gaussian(self.h, seed, _ptr(rows), _ptr(cols), rows.numel(), _ptr(out)))
        self._leave(cur)
        return out
