"""Build libnf.so (the C-ABI library) in-tree with nvcc for sm_100a.

Usage: python -m paper_2408_12757_b200.build  (or build() from __graft_entry__)
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libnf.so")
SOURCES = ["gemm.cu", "moe.cu", "attention.cu", "misc.cu", "api.cu", "comm.cu", "planner.cpp", "profile.cu", "decode_tc.cu", "decode_ws.cu", "decode_stream.cu", "peer.cu", "prefill_tc.cu", "green.cpp", "sched.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include() -> str:
    for base in sysconfig.get_paths()["purelib"], "/usr":
        for cand in (os.path.join(base, "nvidia", "nccl", "include"), os.path.join(base, "include")):
            if os.path.exists(os.path.join(cand, "nccl.h")):
                return cand
    raise RuntimeError("nccl.h not found")


def nvcc() -> str:
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    return os.path.join(cuda, "bin", "nvcc")


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    inc = ["-I", os.path.join(os.path.dirname(HERE), "include"), "-I", _nccl_include()]
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr"] + ARCH + inc
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(os.path.dirname(HERE), "include", "nf.h")]
    newest_dep = max(os.path.getmtime(d) for d in deps)

    def compile_one(src: str) -> str:
        obj = os.path.join(BUILD, src + ".o")
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep:
            return obj
        cmd = [nvcc()] + flags + ["-c", os.path.join(CSRC, src), "-o", obj]
        if src.endswith(".cpp"):
            cmd = [nvcc(), "-x", "cu"] + flags + ["-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
