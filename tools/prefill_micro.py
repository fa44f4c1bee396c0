#!/usr/bin/env python
"""Prefill attention of the 8B bench batch's prefill part (a 341-token chunk over
a 683-token prefix + a 1024-token prompt, 32 query / 8 KV heads) at given SM
budgets; causal TFLOP/s.  NF_PREFILL_IMPL=mma selects the mma.sync kernel.
Usage: prefill_micro.py SMS[,SMS...] [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2408_12757_b200 import nf, runtime as rt  # noqa: E402

sms = [int(x) for x in sys.argv[1].split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
shape = synth.SHAPES["llama3-8b"]
q_len, prefix = [341, 1024], [683, 0]
b = synth.make_batch(q_len, prefix, seed=3)
nb = nf.Batch.from_any(b)
cfg = rt.cfg_from_shape(shape)
pool = torch.randn((b.n_pages_pool, 2, shape.n_kv_heads, 16, 128), device="cuda").to(torch.bfloat16)
T = b.n_tokens
q = torch.randn((T, shape.n_q_heads, 128), device="cuda").to(torch.bfloat16)
o = torch.empty((T, shape.n_q_heads * 128), device="cuda", dtype=torch.bfloat16)
ws = rt.workspace(cfg, nb)
flops = sum(4 * 128 * shape.n_q_heads * (p0 + i + 1) for n, p0 in zip(q_len, prefix) for i in range(n))
for sm in sms:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(reps + 2):
        if i == 2:
            e0.record()
        nf.attention(cfg, nb, q.data_ptr(), pool.data_ptr(), o.data_ptr(), ws.data_ptr(), ws.numel(), sm, sm,
                     rt.stream_handle())
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    print(f"prefill impl={os.environ.get('NF_PREFILL_IMPL', 'tc')} sm={sm}: {t*1e6:.1f} us "
          f"{flops/t/1e12:.0f} TFLOP/s (causal, {flops/1e9:.2f} GFLOP)", flush=True)
