"""Build libbk.so (sm_100a) in-tree with nvcc.  Invoked by __graft_entry__.build().

Usage: python -m paper_2504_02117_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIB = os.path.join(HERE, "lib", "libbk.so")
SOURCES = ["spmm.cu", "blas.cu", "gram_mma.cu", "stream.cu", "dense.cu", "dense_warp.cu", "abi.cpp", "solve.cpp", "comm.cpp", "window.cpp", "dirk.cpp", "wide.cu", "nonlin.cu", "alg1.cpp", "flat.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    site = sysconfig.get_paths()["purelib"]
    base = os.path.join(site, "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return None, None


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    inc, libdir = nccl_dirs()
    common = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
              "-I", CSRC] + ARCH
    if inc:
        common += ["-I", inc]
    else:
        common += ["-DBK_NO_NCCL"]
    headers = [os.path.join(CSRC, "bk_internal.h"), os.path.join(CSRC, "ptx.cuh"), os.path.join(CSRC, "dense_dev.cuh"), os.path.join(CSRC, "reduce.cuh"), os.path.join(ROOT, "include", "bk.h")]
    hdr_mtime = max(os.path.getmtime(h) for h in headers)
    nvcc = _nvcc()

    def compile_one(src):
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        if not force and os.path.exists(o) and os.path.getmtime(o) >= max(os.path.getmtime(s), hdr_mtime):
            return o
        cmd = [nvcc] + common + ["-Xptxas", "-v"] * verbose + ["-c", s, "-o", o]
        if src.endswith(".cpp"):
            cmd = [nvcc] + common + ["-x", "cu", "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        if verbose and r.stderr:
            sys.stderr.write(r.stderr)
        return o

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        # static cudart (nvcc 12.9) so the library does not depend on the
        # runtime version torch ships; both share the device's primary context
        link = [nvcc, "-shared", "-cudart", "static"] + ARCH + ["-o", LIB] + objs
        if libdir:
            link += ["-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath,{libdir}"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
