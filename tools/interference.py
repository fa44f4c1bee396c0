#!/usr/bin/env python
"""GEMM / decode-attention interference on one B200: each kernel alone on its SM
share, then both at once on two streams (GEMM on G SMs, decode on D SMs).
Usage: interference.py G D   (NF_GEMM_STAGES=3 forces the 3-stage GEMM ring)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2408_12757_b200 import nf, runtime as rt  # noqa: E402

G, Dsm = int(sys.argv[1]), int(sys.argv[2])
shape = synth.SHAPES["llama3-8b"]
full = synth.workload_batch(2048, 1024, 512)
n = int((full.q_len == 1).sum())
b = synth.make_batch([1] * n, full.kv_prefix[:n], seed=3)
nb = nf.Batch.from_any(b)
cfg = rt.cfg_from_shape(shape)
pool = torch.randn((b.n_pages_pool, 2, shape.n_kv_heads, 16, 128), device="cuda").to(torch.bfloat16)
q = torch.randn((n, shape.n_q_heads, 128), device="cuda").to(torch.bfloat16)
o = torch.empty((n, shape.n_q_heads * 128), device="cuda", dtype=torch.bfloat16)
ws = rt.workspace(cfg, nb)
dec_bytes = int((b.kv_prefix + 1).sum()) * 8 * 128 * 4
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
import threading  # noqa: E402

import pynvml  # noqa: E402

pynvml.nvmlInit()
_h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())


class Clock:
    """Median SM clock (MHz) and power (W) sampled every 5 ms while active."""

    def __enter__(self):
        self.s, self.p, self.on = [], [], True
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def _run(self):
        import time
        while self.on:
            self.s.append(pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM))
            self.p.append(pynvml.nvmlDeviceGetPowerUsage(_h) / 1000)
            time.sleep(0.005)

    def __exit__(self, *a):
        self.on = False
        self.t.join()

    def summary(self):
        import statistics
        return f"{statistics.median(self.s) if self.s else 0:.0f}MHz/{statistics.median(self.p) if self.p else 0:.0f}W"




def dec(st):
    nf.attention(cfg, nb, q.data_ptr(), pool.data_ptr(), o.data_ptr(), ws.data_ptr(), ws.numel(), Dsm, Dsm,
                 int(st.cuda_stream))


for name, (M, N, K) in {"ug": (1280, 28672, 4096), "down": (1280, 4096, 14336), "kqv": (1280, 6144, 4096)}.items():
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
    Cm = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    gws = torch.empty(nf.gemm_workspace_bytes(M, N), dtype=torch.uint8, device="cuda")

    def gemm(st):
        nf.gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, Cm.data_ptr(), N, M, N, K, G, int(st.cuda_stream),
                     gws.data_ptr(), gws.numel())

    def timed(fn, st, reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            fn(st)
        e1.record(st)
        return e0, e1

    for _ in range(3):
        gemm(sa)
        dec(sb)
    torch.cuda.synchronize()
    with Clock() as ck_g:
        g0, g1 = timed(gemm, sa, 200)
        torch.cuda.synchronize()
    t_g = g0.elapsed_time(g1) / 200
    with Clock() as ck_d:
        d0, d1 = timed(dec, sb, 30)
        torch.cuda.synchronize()
    t_d = d0.elapsed_time(d1) / 30
    # concurrent: decode loop long enough to cover the GEMM loop
    nd = max(3, int(200 * t_g / t_d) + 3)
    torch.cuda.synchronize()
    with Clock() as ck_c:
        d0, d1 = timed(dec, sb, nd)
        g0, g1 = timed(gemm, sa, 200)
        torch.cuda.synchronize()
    t_gc = g0.elapsed_time(g1) / 200
    t_dc = d0.elapsed_time(d1) / nd
    fl = 2 * M * N * K
    print(f"{name}: G={G} D={Dsm} stages={os.environ.get('NF_GEMM_STAGES', '4')}  gemm alone {t_g*1e3:.0f} us "
          f"({fl/t_g/1e9:.0f} TF/s)  with decode {t_gc*1e3:.0f} us ({fl/t_gc/1e9:.0f} TF/s, x{t_gc/t_g:.2f})  | "
          f"decode alone {dec_bytes/t_d/1e6:.0f} GB/s  concurrent {dec_bytes/t_dc/1e6:.0f} GB/s | clocks gemm-alone "
          f"{ck_g.summary()} decode-alone {ck_d.summary()} both {ck_c.summary()}", flush=True)
