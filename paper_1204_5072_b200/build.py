"""Build the sm_100a library in-tree: paper_1204_5072_b200/_lib/liblfg.so.

    python -m paper_1204_5072_b200.build [--force] [--verbose]

nvcc cross-compiles for sm_100a without a GPU (-gencode
arch=compute_100a,code=sm_100a, -lineinfo for ncu source mapping).  The .so
is git-ignored but NOT gpurun-ignored, so it travels to the GPU box.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "liblfg.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "-Xptxas", "-v",
    "-shared",
]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _inputs() -> list[str]:
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "lfg.h"), os.path.join(ROOT, "include", "lfg_kmc.h"), os.path.abspath(__file__)]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _inputs())


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    target = out or LIB
    if not force and out is None and up_to_date():
        return LIB
    os.makedirs(os.path.dirname(target), exist_ok=True)
    tmp = target + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-o", tmp,
           *sources()]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = target + ".build.log"
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed (see {log})")
    if verbose:
        sys.stdout.write(res.stderr)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    args = sys.argv[1:]
    out = None
    defs = []
    for a in args:
        if a.startswith("--out="):
            out = a.split("=", 1)[1]
        elif a.startswith("-D"):
            defs.append(a[2:])
    print(build(force="--force" in args, verbose="--verbose" in args, out=out, defines=defs))
