#!/usr/bin/env python
"""TFLOP/s of the tcgen05 GEMM on the decoder's shapes at given SM budgets
(set NF_STREAMK=1 for the stream-K tail).  Usage: gemm_micro.py [budgets...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_12757_b200 import nf, runtime as rt  # noqa: E402

SHAPES = {  # name: (N, K)
    "8b.kqv": (6144, 4096), "8b.o": (4096, 4096), "8b.ug": (28672, 4096), "8b.down": (4096, 14336),
    "70r.kqv": (1280, 8192), "70r.o": (8192, 1024), "70r.ocol": (1024, 8192), "70r.ug": (7168, 8192), "70r.down": (8192, 3584),
}
budgets = [int(x) for x in sys.argv[1:]] or [148, 108]
st = rt.stream_handle()
only = os.environ.get("ONLY")
for name, (N, K) in SHAPES.items():
    if only and not name.startswith(only):
        continue
    for M in [int(x) for x in os.environ.get("MS", "1024,2048").split(",")]:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ws = torch.empty(nf.gemm_workspace_bytes(M, N), dtype=torch.uint8, device="cuda")
        res = []
        for u in budgets:
            f = lambda: nf.gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, u, st,
                                     ws.data_ptr(), ws.numel())
            for _ in range(3):
                f()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                f()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 10 / 1e3
            res.append(f"sm{u}: {2 * M * N * K / t / 1e12:6.0f}")
        print(f"{name:9s} M={M:5d} " + "  ".join(res), flush=True)
