"""The C-ABI library builds for sm_100a, loads, and exports every symbol that
include/lsrn.h declares (no compute calls: no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lsrn.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lsrn_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1109_5981_b200.build import build
    return build()


def test_header_symbols_exported(libpath):
    names = _declared()
    assert "lsrn_solve_lsqr" in names and "lsrn_solve_cs" in names and "lsrn_sketch" in names
    L = ctypes.CDLL(libpath)
    for n in names:
        assert hasattr(L, n), n
    from paper_1109_5981_b200 import lsrn
    assert sorted(lsrn.EXPORTS) == names
    assert b"sm_100a" in lsrn.lib().lsrn_version()


def test_sass_is_sm100a_and_uses_dmma(libpath):
    out = subprocess.run(["cuobjdump", "-lelf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    # the dense sketch (K2) runs on the fp64 tensor cores
    body = sass.split("sketch_dense_kernel", 1)[1]
    assert "DMMA.8x8x4" in body


def test_no_device_calls_without_gpu():
    import torch
    from paper_1109_5981_b200 import lsrn
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    # the binding loads; creating a context must fail loudly (no CPU fallback)
    h = ctypes.c_void_p()
    rc = lsrn.lib().lsrn_ctx_create(ctypes.byref(h), None, 1, 0, None)
    assert rc != 0
    assert lsrn.lib().lsrn_last_error()
