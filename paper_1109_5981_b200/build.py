"""Build the in-tree sm_100a shared library ``liblsrn.so`` with nvcc.

Every .cu under csrc/ is compiled with
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17
and linked into paper_1109_5981_b200/liblsrn.so against cuSOLVER and NCCL
(rpath to the CUDA toolkit).  Run: python -m paper_1109_5981_b200.build
"""
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "liblsrn.so")
OBJ = os.path.join(HERE, "_build")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nvcc():
    p = os.path.join(CUDA, "bin", "nvcc")
    return p if os.path.exists(p) else (shutil.which("nvcc") or "nvcc")


def _have_nccl():
    return os.path.exists("/usr/include/nccl.h")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "lsrn.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False, force=False):
    os.makedirs(OBJ, exist_ok=True)
    nvcc = _nvcc()
    defs = ["-DLSRN_WITH_NCCL"] if _have_nccl() else []
    flags = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
                    "-I", os.path.join(ROOT, "include"), "--expt-relaxed-constexpr"] + defs
    jobs = []
    for src in sources():
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        if force or _stale(obj, src):
            jobs.append([nvcc, "-c", src, "-o", obj] + flags)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose:
            sys.stderr.write(r.stdout + r.stderr)
        return r

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    objs = [os.path.join(OBJ, os.path.basename(s)[:-3] + ".o") for s in sources()]
    need_link = force or bool(jobs) or not os.path.exists(OUT) or \
        any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs)
    if need_link:
        libs = ["-lcusolver"] + (["-lnccl"] if defs else [])
        cmd = [nvcc, "-shared", "-o", OUT + ".tmp"] + ARCH + objs + [
            "-L", os.path.join(CUDA, "lib64"), "-Xlinker", "-rpath=" + os.path.join(CUDA, "lib64")] + libs
        run(cmd)
        os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
