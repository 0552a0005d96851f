"""Build libmpsp.so in-tree with nvcc for sm_100a (no torch extension needed:
the library exposes a plain C ABI, include/mpsp.h)."""
from __future__ import annotations

import fcntl
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libmpsp.so")
BUILD = os.path.join(PKG, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
         "-I" + os.path.join(ROOT, "include")]
SOURCES = ["spmv_kernels.cu", "spmv_wrow.cu", "spmv_wide.cu", "krylov.cu", "krylov_wide.cu", "xchg.cu", "mpsp_api.cpp"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _deps_mtime() -> float:
    m = 0.0
    for d in (CSRC, os.path.join(ROOT, "include")):
        for f in os.listdir(d):
            m = max(m, os.path.getmtime(os.path.join(d, f)))
    return max(m, os.path.getmtime(__file__))


def build(force: bool = False, verbose: bool = False, defines=(), name: str = "libmpsp.so") -> str:
    """Compile the library; `defines`/`name` build a tuning variant beside it.

    Safe to call from every rank of a torchrun job at once: an exclusive file
    lock serialises the builders, so the first one compiles and the others
    find the library current when they get the lock."""
    lib = os.path.join(PKG, name)
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= _deps_mtime():
        return lib
    os.makedirs(BUILD, exist_ok=True)
    with open(os.path.join(BUILD, name + ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if not force and os.path.exists(lib) and os.path.getmtime(lib) >= _deps_mtime():
                return lib
            return _compile(lib, verbose, defines, name)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)


def _compile(lib, verbose, defines, name):
    bdir = BUILD if name == "libmpsp.so" else os.path.join(BUILD, name)
    os.makedirs(bdir, exist_ok=True)
    nv = nvcc()

    def compile_one(src):
        obj = os.path.join(bdir, src + ".o")
        cmd = [nv, *ARCH, *FLAGS, *defines, "-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cu"):
            cmd += ["-Xptxas", "-v"] if verbose else []
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = f"{lib}.{os.getpid()}.tmp"
    cmd = [nv, *ARCH, "-shared", "--cudart", "shared", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    defs = [a for a in sys.argv[1:] if a.startswith("-D")]
    names = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--name=")]
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, defines=defs,
                name=names[0] if names else "libmpsp.so"))
