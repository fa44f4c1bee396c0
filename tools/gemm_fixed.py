#!/usr/bin/env python
"""Fixed (per-launch) vs per-k-block cost of the tcgen05 GEMM: times shapes at several K
with CUDA events (10 launches back to back, and the same 10 captured in a CUDA graph)
and fits t = t0 + K * slope per shape.  Usage: gemm_fixed.py [budget]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2408_12757_b200 import nf, runtime as rt  # noqa: E402

budget = int(sys.argv[1]) if len(sys.argv) > 1 else 148
SHAPES = [(128, 256), (256, 256), (2048, 1280), (1024, 1280), (2048, 8192), (2048, 7168)]
KS = [1024, 2048, 4096, 8192]
st = rt.stream_handle()



def time_us(f, graph):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                f()
        g.replay()
        torch.cuda.synchronize()
        run = g.replay
    else:
        def run():
            for _ in range(10):
                f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10 * 1e3


for M, N in SHAPES:
    rows = []
    for K in KS:
        A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        B = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ws = torch.zeros(nf.gemm_workspace_bytes(M, N), dtype=torch.uint8, device="cuda")  # zeroed once (NF_GEMM_NOZERO=1)

        def f():
            nf.gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, budget,
                         torch.cuda.current_stream().cuda_stream, ws.data_ptr(), ws.numel())
        t_s = time_us(f, False)
        t_g = time_us(f, True)
        rows.append((K, t_s, t_g))
        print(f"M={M:5d} N={N:5d} K={K:5d}  stream {t_s:8.2f} us  graph {t_g:8.2f} us  "
              f"{2 * M * N * K / t_g / 1e6:7.0f} TF/s", flush=True)
    # least-squares fit of the graph times
    n = len(rows)
    mx = sum(r[0] for r in rows) / n
    my = sum(r[2] for r in rows) / n
    sl = sum((r[0] - mx) * (r[2] - my) for r in rows) / sum((r[0] - mx) ** 2 for r in rows)
    print(f"   fit: t0 = {my - sl * mx:7.2f} us, {sl * 64:6.3f} us per 64-wide k-block", flush=True)
