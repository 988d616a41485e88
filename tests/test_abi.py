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


def _sass_functions(libpath):
    """{mangled kernel name: SASS text} from cuobjdump -sass (one entry per function)."""
    sass = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    funcs = {}
    for chunk in sass.split("Function : ")[1:]:
        name, _, body = chunk.partition("\n")
        funcs[name.strip()] = funcs.get(name.strip(), "") + body
    return funcs


def test_sass_is_sm100a_and_uses_dmma(libpath):
    out = subprocess.run(["cuobjdump", "-lelf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    funcs = _sass_functions(libpath)
    # the dense sketch's default kernel (K2, warp-specialized) runs on the fp64 tensor
    # cores, its X tiles arrive by TMA bulk copies completing on mbarriers
    ws = {n: b for n, b in funcs.items() if "sketch_ws_kernel" in n}
    assert ws, "no sketch_ws_kernel instance in the library"
    for n, body in ws.items():
        assert "DMMA.8x8x4" in body, n
        assert "UBLKCP" in body, n
        assert "SYNCS" in body, n
    # the fallback kernel too
    fb = {n: b for n, b in funcs.items() if "sketch_dense_kernel" in n}
    assert fb and all("DMMA.8x8x4" in b for b in fb.values())


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


def test_binding_vector_checks_without_gpu():
    """The binding's argument checks (the C ABI takes raw pointers and cannot check dtype,
    length, contiguity or device)."""
    import torch
    from paper_1109_5981_b200 import lsrn
    dev = torch.device("cuda", 0)
    v = torch.zeros(10, dtype=torch.float64)
    lsrn._check_vec("b", v, 10, dev, host=True)
    with pytest.raises(TypeError):
        lsrn._check_vec("b", v.float(), 10, dev, host=True)
    with pytest.raises(ValueError):
        lsrn._check_vec("b", v, 11, dev, host=True)
    with pytest.raises(ValueError):
        lsrn._check_vec("b", torch.zeros(10, 2, dtype=torch.float64)[:, 0], 10, dev, host=True)
    with pytest.raises(ValueError):
        lsrn._check_vec("b", v, 10, dev, host=False)          # CPU tensor where the device is required
    with pytest.raises(ValueError):
        lsrn._check_matrix_device(torch.zeros(3, 2, dtype=torch.float64), dev, host=False)


def test_options_table_matches_header():
    """Every LSRN_OPT_* of include/lsrn.h has a name in the binding's OPTIONS, same value."""
    from paper_1109_5981_b200 import lsrn
    src = open(HEADER).read()
    hdr = {k.lower(): int(v) for k, v in re.findall(r"LSRN_OPT_([A-Z0-9_]+)\s*=\s*(\d+)", src)}
    assert hdr == lsrn.OPTIONS


def test_flag_constants_match_header():
    """The binding's lsrn_opts.flags bits and status codes equal include/lsrn.h's."""
    from paper_1109_5981_b200 import lsrn
    src = open(HEADER).read()
    for name in ("HOST_IO", "SKETCH_ONLY", "REUSE_SKETCH", "COMPENSATED"):
        v = re.search(rf"LSRN_{name}\s*=\s*(\d+)", src)
        assert v is not None and int(v.group(1)) == getattr(lsrn, name), name
    codes = {int(v): f"LSRN_{k}" for k, v in re.findall(r"LSRN_(E[A-Z0-9]+|OK)\s*=\s*(-?\d+)", src)}
    assert codes == lsrn.STATUS
