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
cfgs = [(8, 3, 0), (4, 6, 0), (8, 1, 0), (8, 2, 0), (12, 2, 0), (13, 2, 0), (24, 1, 0), (4, 2, 0),
        (8, 3, 1), (12, 2, 1), (8, 1, 1), (8, 3, 2)]
if len(sys.argv) > 1 and sys.argv[1]:
    cfgs = [tuple(int(v) for v in c.split(":")) for c in sys.argv[1].split(",")]
grids = [int(g) for g in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 16, 32, 48, 64, 148]
for warps, ns, mode in cfgs:
    for grid in grids:
        ppw = 3000 if grid <= 16 else 800
        ms = C.c_float()
        rc = lib.probe_run(C.c_void_p(pool.data_ptr()), C.c_longlong(n_pages), C.c_void_p(perm.data_ptr()), n_pages,
                           grid, warps, ns, ppw, C.byref(ms), mode)
        byts = grid * warps * ppw * 8192
        print(f"mode={mode} warps={warps} stages={ns} inflight={warps*ns*8}KB sm={grid:3d}: {byts / ms.value / 1e6:7.0f} GB/s  "
              f"({byts / ms.value / 1e6 / grid:6.1f} GB/s/SM) rc={rc}", flush=True)
