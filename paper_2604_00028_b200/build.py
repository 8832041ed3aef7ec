"""Build libdecattn.so in-tree with nvcc for sm_100a.

    python paper_2604_00028_b200/build.py [--force] [--ptxas-verbose]

(run by path, or load it by path as __graft_entry__.build() does: importing it as a submodule
of the package would import the package first, which loads the library it is meant to build)

Sources: csrc/{plan.cpp, capi.cpp, fwd.cu, fwd_tc.cu, combine.cu}.  Output:
paper_2604_00028_b200/lib/libdecattn.so (git-ignored; travels to the GPU box
with the gpurun snapshot).  cudart is linked statically, so the library
loads on a machine without a GPU (the planner and the symbol checks run on
CPU) and does not depend on the toolkit's shared runtime at run time.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
BUILD = os.path.join(PKG, "build")
LIB = os.path.join(LIBDIR, "libdecattn.so")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")

SOURCES = ["plan.cpp", "capi.cpp", "fwd.cu", "fwd_tc.cu", "combine.cu"]
HEADERS = ["config.h", "internal.h", "ptx.cuh", "pub.cuh", "tile_common.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC,-fvisibility=hidden",
          "-I", CSRC, "-I", INCLUDE]


def nvcc() -> str:
    path = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(path):
        raise RuntimeError("nvcc not found: cannot build libdecattn.so")
    return path


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, ptxas_verbose: bool = False, quiet: bool = True,
          defines=(), lib: str | None = None, build_dir: str | None = None) -> str:
    """Compile + link.  ``defines``/``lib``/``build_dir`` build development variants
    (e.g. -DDECATTN_PREFETCH_TILES=0 into another .so); the default is the product library."""
    lib = lib or LIB
    bdir = build_dir or BUILD
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    os.makedirs(bdir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "decattn.h"),
                                                         os.path.abspath(__file__)]
    if not force and not _stale(lib, [os.path.join(CSRC, src) for src in SOURCES] + hdrs):
        return lib    # up to date with every source (the object directory need not exist)
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(bdir, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs):
            cmd = [nvcc()] + ARCH + COMMON + [f"-D{d}" for d in defines] + ["-c", s, "-o", o]
            if src.endswith(".cu") and ptxas_verbose:
                cmd += ["-Xptxas", "-v"]
            _run(cmd, quiet and not ptxas_verbose)
    if force or _stale(lib, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs
        _run(cmd, quiet)
    return lib


def _run(cmd, quiet):
    if not quiet:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {' '.join(cmd)}")
    if not quiet and (r.stdout or r.stderr):
        sys.stderr.write(r.stdout + r.stderr)


if __name__ == "__main__":
    build(force="--force" in sys.argv, ptxas_verbose="--ptxas-verbose" in sys.argv, quiet=False)
    print(LIB)
