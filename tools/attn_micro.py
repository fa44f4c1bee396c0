#!/usr/bin/env python
"""Decode attention over the 8B steady-state decode batch at a fixed SM budget
(for ncu / quick A-B of kernel variants).  Usage: attn_micro.py SMS[,SMS...] [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2408_12757_b200 import nf, runtime as rt  # noqa: E402

sms = [int(x) for x in sys.argv[1].split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if os.environ.get("SHAPE") == "c3rank":  # one 70B TP8 rank: 8 query heads over 1 KV head, 512/1024 workload
    shape = synth.shape_with(synth.SHAPES["llama2-70b"], n_q_heads=8, n_kv_heads=1, d_ffn=3584)
    full = synth.workload_batch(2048, 512, 1024)
else:
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
keys = int((b.kv_prefix + 1).sum())
for sm in sms:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(reps + 1):
        if i == 1:
            e0.record()
        nf.attention(cfg, nb, q.data_ptr(), pool.data_ptr(), o.data_ptr(), ws.data_ptr(), ws.numel(), sm, sm,
                     rt.stream_handle())
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    print(f"impl={os.environ.get('NF_DECODE_IMPL', 'stream')} sm={sm}: {t*1e6:.1f} us {keys*shape.n_kv_heads*128*4/t/1e9:.0f} GB/s "
          f"({keys*shape.n_kv_heads*128*4/t/1e9/sm:.1f} GB/s/SM)", flush=True)
