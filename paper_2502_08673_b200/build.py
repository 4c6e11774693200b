"""Builds the sm_100a library ``libsatgrad_b200.so`` in-tree with nvcc.

The product is one shared object exporting the C-ABI declared in
``include/satgrad_b200.h``; Python reaches it through ctypes
(``paper_2502_08673_b200/_lib.py``).  No torch extension machinery: the
boundary is plain C so the reference's C++ host can link it directly
(INTEGRATION.md).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsatgrad_b200.so")
SOURCES = ["sgx_kernels.cu", "sgx_format.cu", "sgx_api.cpp", "sgx_layout.cpp", "sgx_layout_io.cpp", "sgx_drain.cpp", "sgx_extract.cpp", "sgx_verify.cu", "sgx_jit.cpp", "sgx_exchange.cpp"]
HEADERS = ["sgx_kernels.cuh", "sgx_launch.hpp", "sgx_layout.hpp", "sgx_drain.hpp", "sgx_extract.hpp", "sgx_jit.hpp"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-Xptxas", "-O3",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def host_cxx() -> str:
    # The image's CXX=/opt/gcc/bin/g++ wrapper links libstdc++ statically.
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else (shutil.which("g++") or "g++")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "satgrad_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    """Compiles every source to an object in parallel (objects under build/,
    rebuilt when the source or any header is newer), then links the .so."""
    if not force and not _stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    hdr_t = max(os.path.getmtime(os.path.join(CSRC, h)) for h in HEADERS)
    hdr_t = max(hdr_t, os.path.getmtime(os.path.join(ROOT, "include", "satgrad_b200.h")))

    def compile_one(f: str) -> str:
        src = os.path.join(CSRC, f)
        obj = os.path.join(objdir, f + ".o")
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(src), hdr_t)):
            return obj
        cmd = [nvcc(), "-ccbin", host_cxx(), *NVCC_FLAGS, "-c", "-o", obj + ".tmp", src]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {f} ({r.returncode}):\n{r.stdout}\n{r.stderr}")
        os.replace(obj + ".tmp", obj)
        return obj

    # the big kernel file first: it bounds the wall time
    order = sorted(SOURCES, key=lambda f: -os.path.getsize(os.path.join(CSRC, f)))
    with ThreadPoolExecutor(max_workers=min(len(order), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, order))
    cmd = [nvcc(), "-ccbin", host_cxx(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
           "-o", LIB + ".tmp", *objs, "-ldl"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed ({r.returncode}):\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    return LIB


def ptxas_report() -> str:
    """Registers / spills / shared memory per kernel (-Xptxas -v)."""
    cmd = [nvcc(), "-ccbin", host_cxx(), *NVCC_FLAGS, "-Xptxas", "-v", "-c", "-o", os.devnull,
           os.path.join(CSRC, "sgx_kernels.cu")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return r.stdout + r.stderr


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    if "--ptxas" in sys.argv:
        print(ptxas_report())
    print(LIB)
