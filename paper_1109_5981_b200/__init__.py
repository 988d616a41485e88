"""B200-native (sm_100a) LSRN hot path: Gaussian sketch + fused LSQR / Chebyshev.

The compute lives in liblsrn.so (csrc/, C ABI in include/lsrn.h); this package is
the build script and a ctypes binding.  See DESIGN.md.
"""
from . import lsrn  # noqa: F401
from .lsrn import Context, LsrnError, lib  # noqa: F401
