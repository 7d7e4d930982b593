"""Build the sm_100a shared library in-tree: paper_2110_03423_b200/_lib/librsvd_b200.so.

Explicit nvcc invocations (no JIT cache): every .cu/.cpp in csrc/ is compiled with
`-gencode arch=compute_100a,code=sm_100a -lineinfo -O3` and linked into one C-ABI
library (include/rsvd_b200.h) plus the C++ drop-in (include/randsvd/*.hpp).
Run `python -m paper_2110_03423_b200.build [-v]`.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
OBJDIR = os.path.join(LIBDIR, "obj")
LIB = os.path.join(LIBDIR, "librsvd_b200.so")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC",
          "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]
CU_FLAGS = ARCH + COMMON + ["-Xptxas", "-warn-spills", "--expt-relaxed-constexpr"]

SOURCES = ["gemm_f64.cu", "gemm_tf32.cu", "gemm_oz.cu", "omega.cu", "linalg_small.cu", "linalg_blocked.cu", "householder.cu",
           "comm.cu", "rsvd_b200.cpp", "randsvd_dropin.cpp", "dmat.cpp"]
CLI = os.path.join(LIBDIR, "randsvd_b200")


def _newer(src_files, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(f) > t for f in src_files)


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    inc = os.path.join(ROOT, "include")
    for dp, _, fs in os.walk(inc):
        hs += [os.path.join(dp, f) for f in fs if f.endswith((".h", ".hpp"))]
    return hs


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJDIR, os.path.splitext(src)[0] + ".o")
    srcp = os.path.join(CSRC, src)
    if not _newer([srcp] + _headers(), obj):
        return obj
    flags = CU_FLAGS if src.endswith(".cu") else ARCH + COMMON
    cmd = [NVCC] + flags + ["-c", srcp, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and (r.stderr.strip() or r.stdout.strip()):
        print(r.stdout + r.stderr, flush=True)
    return obj


def build(verbose: bool = False) -> str:
    os.makedirs(OBJDIR, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    if _newer(objs, LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    # the reference CLI's hot-path subcommands, built against the C++ drop-in headers
    cli_src = os.path.join(CSRC, "cli_rsvd.cpp")
    if _newer([cli_src, LIB] + _headers(), CLI):
        cmd = [NVCC, "-O2", "-std=c++20", "-I" + os.path.join(ROOT, "include"), cli_src, "-o", CLI,
               "-L" + LIBDIR, "-lrsvd_b200", "-Xlinker", "-rpath=$ORIGIN"]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"CLI build failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
