"""In-tree build of librtn_mpc.so (sm_100a) and the CPU oracle.

The shared library is written next to this file so it travels with the repo
snapshot to the GPU box (it is git-ignored, not gpurun-ignored).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librtn_mpc.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xcompiler", "-O3,-ffp-contract=off",
    "-ccbin", "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++",
]

SOURCES = ["rtn_mpc.cu", "rtn_comm.cu", "rtn_pair_tf32.cu", "rtn_pair_3xtf32.cu", "rtn_pair_bf16x3.cu", "rtn_pair_bf16.cu", "rtn_pair_order2.cu",
           "rtn_split.cu", "rtn_pair_rev.cu", "rtn_blocks.cu", "rtn_qpsolve.cu", "rtn_synth.cpp"]
HEADERS = ["rtn_kernel.cuh", "rtn_pair.cuh", "rtn_pair_launch.cuh", "rtn_launch.h", "rtn_blocks.h", "rtn_quad.cuh",
           "rtn_qpsolve.h", "rtn_rows.cuh", "rtn_split.cuh", "rtn_rowsb.cuh", "rtn_reverse.cuh", "rtn_internal.h"]
DEPS = SOURCES + HEADERS


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Compiles each translation unit in parallel (the per-precision pair
    kernels are the slow ones), then links librtn_mpc.so."""
    deps = [os.path.join(CSRC, s) for s in DEPS] + [os.path.join(ROOT, "include", "rtn_mpc.h")]
    if not (force or _stale(LIB, deps)):
        return LIB
    objdir = os.path.join(HERE, "build", "obj")
    os.makedirs(objdir, exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    procs, objs = [], []
    for src in SOURCES:
        obj = os.path.join(objdir, os.path.splitext(src)[0] + ".o")
        objs.append(obj)
        cmd = [_nvcc(), *compile_flags, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd)))
    failed = [src for src, p in procs if p.wait() != 0]
    if failed:
        raise RuntimeError(f"nvcc failed for {failed}")
    link = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-ccbin", NVCC_FLAGS[-1], *objs, "-ldl",
            "-o", LIB]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    return LIB


def build_oracle(force: bool = False) -> str:
    odir = os.path.join(ROOT, "oracle")
    if force:
        subprocess.run(["make", "-C", odir, "clean"], check=True, stdout=subprocess.DEVNULL)
    subprocess.run(["make", "-C", odir, "-j4", "all"], check=True, stdout=subprocess.DEVNULL)
    return os.path.join(odir, "build", "liboracle.so")


if __name__ == "__main__":
    build_library(force="--force" in sys.argv, verbose=True)
    build_oracle()
    print(LIB)
