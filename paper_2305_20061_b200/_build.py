"""Compile libpt_b200.so (CUDA sm_100a kernels + C++ host runtime) in-tree with nvcc."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libpt_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


STAMP = LIB + ".flags"


def _deps():
    """Every file the library's objects depend on: sources, private headers (.h and .cuh), the C-ABI
    header and this build script."""
    return (sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
            + glob.glob(os.path.join(INCLUDE, "*.h")) + [os.path.abspath(__file__)])


def _flags_key(defines=()) -> str:
    return " ".join([*ARCH, os.environ.get("PT_NVCC_EXTRA", ""), *[f"-D{d}" for d in defines]])


def _stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    try:
        if open(STAMP).read() != _flags_key():
            return True                   # built with other flags (PT_NVCC_EXTRA, defines)
    except OSError:
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile every source for sm_100a and link libpt_b200.so (or `out`, with extra -D defines; the
    environment variable PT_NVCC_EXTRA adds nvcc flags, for experiments)."""
    lib = os.path.abspath(out) if out else LIB
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    if not force and out is None and not _stale():
        return LIB
    objdir = os.path.join(ROOT, "build", "obj" if out is None else "obj_" + os.path.basename(lib))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    common = ["-O3", "-std=c++17", "-lineinfo", "-I", INCLUDE, "-I", CSRC,
              "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden"] + os.environ.get("PT_NVCC_EXTRA", "").split()
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *common, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        else:
            cmd += ["-x", "cu"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"])
    os.replace(tmp, lib)
    if out is None:
        with open(STAMP, "w") as f:
            f.write(_flags_key(defines))
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
