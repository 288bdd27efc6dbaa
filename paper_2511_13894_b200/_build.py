"""Build libcpd.so in-tree with nvcc for sm_100a (no JIT cache, no CPU fallback)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# CPD_LIB: load/build another library file (tuning experiments only; default in-tree libcpd.so)
LIB = os.environ.get("CPD_LIB", os.path.join(PKG, "libcpd.so"))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xcompiler", "-fvisibility=hidden", "-Xptxas", "-v"]


def _nccl_dirs():
    try:
        import nvidia.nccl  # noqa: F401  (torch's bundled NCCL wheel)
        base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
    except Exception:
        return None, None
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    return (inc, lib) if os.path.exists(os.path.join(inc, "nccl.h")) else (None, None)


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "cpd.h")]


def source_hash() -> str:
    """sha256 (first 16 hex) of the library sources: tags profiles measured on a build."""
    import hashlib
    h = hashlib.sha256()
    for f in deps():
        with open(f, "rb") as fh:
            h.update(os.path.basename(f).encode() + b"\0" + fh.read())
    return h.hexdigest()[:16]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    objs = []
    inc, nlib = _nccl_dirs()
    extra_inc = ["-I" + os.path.join(ROOT, "include")] + (["-I" + inc] if inc else [])
    defs = ["-DCPD_HAVE_NCCL=1"] if inc else []
    build_dir = os.path.join(PKG, "build" + os.environ.get("CPD_BUILD_TAG", ""))
    os.makedirs(build_dir, exist_ok=True)
    for src in sources():
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        extra = os.environ.get("CPD_NVCC_DEFS", "").split()
        cmd = [NVCC, *ARCH, *FLAGS, *extra_inc, *defs, *extra, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stderr.write(r.stdout + r.stderr)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {src}")
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(r.stderr)
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    link = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    if nlib:
        link += [f"-L{nlib}", "-l:libnccl.so.2", f"-Xlinker", f"-rpath={nlib}"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
