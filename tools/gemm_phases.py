#!/usr/bin/env python
"""Where a GEMM launch's time goes: phase timestamps of CTA 0 (globaltimer) from the
-DNF_GEMM_TS build of the GEMM (NF_LIB=paper_2408_12757_b200/_ts/libnf.so):
entry -> prologue done -> first A/B stage landed -> last MMA issued -> epilogue done ->
teardown done, plus the gap from the previous launch's CTA-0 exit to this entry (two
back-to-back launches in a CUDA graph).  Usage: gemm_phases.py [budget]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_12757_b200 import nf  # noqa: E402

budget = int(sys.argv[1]) if len(sys.argv) > 1 else 148
SHAPES = [(128, 256, 1024), (128, 256, 8192), (2048, 1280, 8192), (1024, 1280, 8192), (2048, 8192, 1024),
          (1024, 7168, 8192)]
ts = (C.c_ulonglong * 8)()
names = ["prologue", "first stage", "mainloop", "epilogue tail", "teardown"]
for M, N, K in SHAPES:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
    Cm = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ws = torch.zeros(nf.gemm_workspace_bytes(M, N), dtype=torch.uint8, device="cuda")  # NF_GEMM_NOZERO=1 needs it zeroed once

    def f():
        nf.gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, Cm.data_ptr(), N, M, N, K, budget,
                     torch.cuda.current_stream().cuda_stream, ws.data_ptr(), ws.numel())
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        f()
        f()
    rows = []
    for _ in range(5):
        g.replay()
        torch.cuda.synchronize()
        nf.lib.nf_debug_gemm_ts(ts)
        t = [ts[i] for i in range(8)]
        rows.append([(t[i + 1] - t[i]) / 1e3 for i in range(5)] + [(t[0] - t[6]) / 1e3, (t[5] - t[0]) / 1e3])
    med = [sorted(r[i] for r in rows)[len(rows) // 2] for i in range(7)]
    print(f"M={M:5d} N={N:5d} K={K:5d}  " + "  ".join(f"{n} {v:6.2f}" for n, v in zip(names, med[:5])) +
          f"  | CTA0 entry->exit {med[6]:6.2f} us, gap after previous launch {med[5]:6.2f} us", flush=True)
