"""Build libspark.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2401_03378_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libspark.so")
# parity build: no FMA contraction, IEEE division / sqrt (R15/R16)
STRICT_LIB = os.path.join(LIBDIR, "libspark_strict.so")
STRICT_FLAGS = ("--fmad=false", "-DSPARK_STRICT_MATH")
# checked build: KB1's shared / global addresses and the halo-source mapping
# asserted in range (a trap on violation); compute-sanitizer is closed on the pool
CHECKED_LIB = os.path.join(LIBDIR, "libspark_checked.so")
CHECKED_FLAGS = ("-DSPARK_CHECKED",)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    """Headers and library of the NCCL that torch loads (one NCCL per process)."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia-nccl (torch's NCCL) not found")
    base = list(spec.submodule_search_locations)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(ROOT, "include", "*.h")))


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in sources() + headers() + [__file__])


def stale_lib(path: str) -> bool:
    if not os.path.exists(path):
        return True
    t = os.path.getmtime(path)
    return any(os.path.getmtime(f) > t for f in sources() + headers() + [__file__])


def build_strict(force: bool = False) -> str:
    """libspark_strict.so: the same sources with --fmad=false -DSPARK_STRICT_MATH."""
    if not force and not stale_lib(STRICT_LIB):
        return STRICT_LIB
    return build(force=True, out=STRICT_LIB, flags=STRICT_FLAGS)


def build_checked(force: bool = False) -> str:
    """libspark_checked.so: the same sources with -DSPARK_CHECKED."""
    if not force and not stale_lib(CHECKED_LIB):
        return CHECKED_LIB
    return build(force=True, out=CHECKED_LIB, flags=CHECKED_FLAGS)


def build_all(force: bool = False) -> list:
    """The production, strict and checked libraries, compiled concurrently."""
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(3) as ex:
        jobs = [ex.submit(build, force), ex.submit(build_strict, force), ex.submit(build_checked, force)]
        return [j.result() for j in jobs]


def build(force: bool = False, verbose: bool = False, out: str = LIB, defs=(), flags=()) -> str:
    """Build libspark.so (``out``/``defs``: design-experiment variants, tools/ablate.sh)."""
    if out == LIB and not force and not stale():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    inc, lib = nccl_paths()
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-Xptxas", "-v" if verbose else "-O3",
           *flags, *[f"-D{d}" for d in defs], "-I", os.path.join(ROOT, "include"), "-I", inc, *sources(),
           "-L", lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{lib}", "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    defs = [a[2:] for a in sys.argv[1:] if a.startswith("-D")]
    outs = [a[6:] for a in sys.argv[1:] if a.startswith("--out=")]
    if "--strict" in sys.argv:
        print(build_strict(force="--force" in sys.argv))
    elif "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv))
    elif "--all" in sys.argv:
        print("\n".join(build_all(force="--force" in sys.argv)))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, out=outs[0] if outs else LIB, defs=defs))
