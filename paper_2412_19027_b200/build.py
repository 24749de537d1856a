"""Build the native library ``lib/libcipm.so`` in-tree for sm_100a.

    python -m paper_2412_19027_b200.build [--force]

Every CUDA translation unit is compiled with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` (cross-compiles
without a GPU); the host symbolic analysis is plain C++17.  Objects are built in
parallel and linked into one shared library whose C ABI is ``include/cipm.h``.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libcipm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CU_SOURCES = ["capi.cu", "ldl.cu", "dense.cu", "cones.cu", "vec.cu", "batch.cu", "setup.cu"]
CPP_SOURCES = ["symbolic.cpp"]
NO_FMAD = {"cones.cu", "batch.cu", "setup.cu"}


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".hpp", ".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "cipm.h"))
    return hs


def _stale(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(h) > t for h in [src] + _headers())


def _compile(src, force):
    path = os.path.join(CSRC, src)
    obj = os.path.join(LIBDIR, "obj", src + ".o")
    if not force and not _stale(obj, path):
        return obj
    if src.endswith(".cu"):
        # cone kernels: no FMA contraction, so the barrier / BFGS / conjugate-point
        # arithmetic rounds like the reference's numpy (exp/pow status parity)
        extra = ["-fmad=false"] if src in NO_FMAD else []
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", *extra, "-Xcompiler", "-fPIC",
               "-Xptxas", "-warn-spills", "-I", os.path.join(ROOT, "include"), "-c", path, "-o", obj]
    else:
        cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-I", os.path.join(ROOT, "include"),
               "-c", path, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    if res.stderr.strip():
        sys.stderr.write(res.stderr)
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(os.path.join(LIBDIR, "obj"), exist_ok=True)
    srcs = CU_SOURCES + CPP_SOURCES
    with ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if force or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        if verbose:
            print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
