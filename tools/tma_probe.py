#!/usr/bin/env python
"""Per-SM TMA streaming ceiling (see tma_probe.cu).  Prints GB/s per SM budget."""
import ctypes as C
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "_tma_probe.so")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(os.path.join(HERE, "tma_probe.cu")):
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    os.path.join(HERE, "tma_probe.cu"), "-o", so], check=True)
lib = C.CDLL(so)
n_pages = 400000   # 3.3 GB of 8 KB pages
pool = torch.empty(n_pages * 2 * 16 * 128, dtype=torch.bfloat16, device="cuda")
perm = torch.randperm(n_pages, device="cuda").to(torch.int32)
for warps, ns in [(8, 3), (4, 6), (8, 1)]:
    for grid in [8, 16, 32, 48, 64, 148]:
        ppw = 3000 if grid <= 16 else 800
        ms = C.c_float()
        rc = lib.probe_run(C.c_void_p(pool.data_ptr()), C.c_longlong(n_pages), C.c_void_p(perm.data_ptr()), n_pages,
                           grid, warps, ns, ppw, C.byref(ms))
        byts = grid * warps * ppw * 8192
        print(f"warps={warps} stages={ns} sm={grid:3d}: {byts / ms.value / 1e6:7.0f} GB/s  "
              f"({byts / ms.value / 1e6 / grid:6.1f} GB/s/SM) rc={rc}", flush=True)
