"""In-tree build of the sm_100a engine: csrc/*.cu -> paper_2509_21963_b200/libitercur_b200.so.

Explicit nvcc (no torch JIT cache): the built .so lives next to this file so it travels
to the GPU box with the repository snapshot. Objects are rebuilt only when a source or
header is newer than the object.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libitercur_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
EXTRA = os.environ.get("ITERCUR_NVCC_EXTRA", "").split()  # experiments: e.g. -DITERCUR_ARGMAX_SHFL
FLAGS = EXTRA + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-I" + INCLUDE, "-I" + CSRC]


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src):
    obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
    if _stale(obj, [src] + _headers()):
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj


FACADE_SRC = os.path.join(HERE, "facade", "itercur_facade.cpp")
FACADE_LIB = os.path.join(HERE, "libitercur_facade.so")
CXX = os.environ.get("CXX", "g++")


def build_facade() -> str:
    """The C++ facade (include/itercur/driver_b200.hpp -> itercur::iterative_cur & co.) over the
    C-ABI: g++, linked against libitercur_b200.so with an $ORIGIN rpath."""
    deps = [FACADE_SRC, LIB, os.path.join(INCLUDE, "itercur_b200.h"), os.path.join(INCLUDE, "itercur", "driver_b200.hpp")]
    if _stale(FACADE_LIB, deps):
        cmd = [CXX, "-O2", "-std=c++17", "-fPIC", "-shared", "-fvisibility=hidden", "-Wall", "-Wextra",
               "-I" + INCLUDE, FACADE_SRC, "-L" + HERE, "-litercur_b200", "-Wl,-rpath,$ORIGIN", "-o", FACADE_LIB]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"facade build failed:\n{r.stdout}\n{r.stderr}")
    return FACADE_LIB


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(_compile, sources))
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    build_facade()
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
