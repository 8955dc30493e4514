"""Build libboris.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_2104_04579_b200._build [--force] [--verbose]

Objects are compiled in parallel (one nvcc per translation unit) and linked
into ``paper_2104_04579_b200/libboris.so`` with the CUDA runtime linked
statically, so the library loads next to torch's own cudart without symbol
clashes.  The library travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "libboris.so")
BUILD_DIR = os.path.join(PKG, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                     "-I", INCLUDE, "-I", CSRC, "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found (CUDA 12.9 toolkit required to build libboris)")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  glob.glob(os.path.join(INCLUDE, "*.h")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), tag: str = "") -> str:
    """Build libboris.so, or with `tag` a variant tuning_libs/libboris_<tag>.so (outside
    the gpurun-ignored build/ directory, so it travels to the GPU box) compiled with
    extra -D `defines` (tuning experiments; the product is always libboris.so)."""
    srcs = sources()
    hdrs = headers()
    lib = LIB if not tag else os.path.join(PKG, "tuning_libs", f"libboris_{tag}.so")
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    if not force and not _stale(lib, srcs + hdrs + [__file__]):
        return lib
    os.makedirs(BUILD_DIR, exist_ok=True)
    cc = nvcc()
    extra = (["-Xptxas", "-v"] if verbose else []) + [f"-D{d}" for d in defines]

    def compile_one(src):
        obj = os.path.join(BUILD_DIR, os.path.basename(src) + (f".{tag}" if tag else "") + ".o")
        if force or _stale(obj, [src] + hdrs + [__file__]):
            cmd = [cc] + NVCC_FLAGS + extra + ["-c", src, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
            if verbose:
                sys.stderr.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, srcs))
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [cc] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--tag", default="")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, defines=a.defines, tag=a.tag))
