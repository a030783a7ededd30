"""Builds paper_1810_06825_b200/lib/libfrpca_b200.so for sm_100a (in-tree).

Every .cu is compiled by nvcc with `-gencode arch=compute_100a,code=sm_100a
-lineinfo`; rng_host.cpp is compiled by g++ with the reference's arithmetic
flags (-O3, no -march, -ffp-contract=off) so the host Omega stream is the
identical libstdc++ stream. Incremental by mtime; objects go to build/.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "build")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libfrpca_b200.so")
SYNTH_SRC = os.path.join(HERE, "synth", "synth.cpp")
SYNTH_LIB = os.path.join(LIBDIR, "libfrpca_synth.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
                  "-Xcompiler", "-fPIC,-O3,-ffp-contract=off", "-I" + os.path.join(ROOT, "include")]
CXXFLAGS = ["-std=c++17", "-O3", "-ffp-contract=off", "-fPIC"]
LDFLAGS = ["-L" + os.path.join(CUDA, "lib64"), "-lcusolver", "-lcublas", "-ldl",
           "-Xlinker", "-rpath=" + os.path.join(CUDA, "lib64")]


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _headers_mtime():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    hs.append(os.path.join(ROOT, "include", "frpca_b200.h"))
    return max(os.path.getmtime(h) for h in hs)


def _compile(src: str, force: bool) -> str:
    base = os.path.splitext(src)[0]
    obj = os.path.join(OBJ, base + ".o")
    s = os.path.join(CSRC, src)
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
            os.path.getmtime(s), _headers_mtime()):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC] + NVFLAGS + ["-c", s, "-o", obj]
    else:
        cmd = ["g++"] + CXXFLAGS + ["-c", s, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + LDFLAGS
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if force or not os.path.exists(SYNTH_LIB) or os.path.getmtime(SYNTH_LIB) < os.path.getmtime(SYNTH_SRC):
        cmd = ["g++", "-std=c++17", "-O3", "-fPIC", "-shared", "-pthread", SYNTH_SRC, "-o", SYNTH_LIB]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"synth build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    # the drop-in C++ API test program (tests/cpp), linked against the library
    src = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
    exe = os.path.join(ROOT, "tests", "cpp", "_build", "test_dropin")
    if os.path.exists(src) and (force or not os.path.exists(exe) or
                                os.path.getmtime(exe) < max(os.path.getmtime(src), os.path.getmtime(LIB),
                                                            os.path.getmtime(os.path.join(ROOT, "include", "frpca", "frpca.hpp")))):
        os.makedirs(os.path.dirname(exe), exist_ok=True)
        cmd = ["g++", "-std=c++20", "-O2", "-I" + os.path.join(ROOT, "include"), src, "-o", exe,
               "-L" + LIBDIR, "-lfrpca_b200", "-Wl,-rpath," + LIBDIR]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"drop-in test build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(LIB)
        print(SYNTH_LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
