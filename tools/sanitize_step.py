#!/usr/bin/env python
"""A small model step and layers in every mode, for compute-sanitizer (memcheck /
racecheck / synccheck): C1-shape 2-layer model step (SEQUENTIAL, NANO_ONLY, OVERLAP
with CUDA graph), an emulated-TP2 layer in the 4/2 pipeline, a MoE layer."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2408_12757_b200 import nf, runtime as rt  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda().to(torch.bfloat16)


shape = synth.shape_with(synth.SHAPES["c1"], n_layers=2, vocab=4096)
b = synth.c1_batch()
W = synth.model_weights(shape)
cfg = rt.cfg_from_shape(shape)
model = rt.Model(cfg, dev(W["embed"]), [rt.pack_layer(cfg, {k: dev(v) for k, v in W["layers"][l].items()})
                                        for l in range(2)], rt.pack_lm_head(cfg, dev(W["lm_head"]), dev(W["final_norm"])))
nb = nf.Batch.from_any(b)
ws = rt.workspace(cfg, nb)
pools = [dev(synth.kv_pool(shape, b, layer=l)) for l in range(2)]
tok = torch.from_numpy(synth.token_ids(b.n_tokens, shape.vocab)).cuda()
for plan in (nf.Plan.explicit(cfg, nf.SEQUENTIAL), nf.Plan.explicit(cfg, nf.NANO_ONLY, shares=(1, 1), balance=2),
             nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1), balance=2, graph=True)):
    for _ in range(2):
        model.step(plan, pools, nb, tok, ws)
torch.cuda.synchronize()
print("model steps ok")
# emulated TP2 layer, 4 attention / 2 dense nano-batches
s2 = synth.shape_with(synth.SHAPES["c1"], n_q_heads=16, n_kv_heads=8, head_dim=64, d_ffn=2048, vocab=4096)
w = {k: dev(v) for k, v in synth.layer_weights(s2, 0).items()}
x = dev(synth.activations(s2, b.n_tokens))
pool = dev(synth.kv_pool(s2, b))
comms = nf.comm_create_local(2)


def rank(r):
    torch.cuda.set_device(0)
    c = rt.cfg_from_shape(s2, tp_size=2, tp_rank=r)
    pk = rt.pack_layer(c, rt.shard_layer(w, 16, 8, 64, 2, r))
    pl = nf.Plan.explicit(c, nf.OVERLAP, shares=(1, 1, 1, 1), n_dense=2, sm=[116, 16, 116, 116, 116, 116, 16])
    rt.layer_forward(pl, c, pk, rt.shard_pool(pool, 2, r), nb, x, comm=comms[r])
    torch.cuda.synchronize()


th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
[t.start() for t in th]
[t.join() for t in th]
print("tp2 layer ok")
sm = synth.SHAPES["c1-moe"]
cm = rt.cfg_from_shape(sm)
rt.layer_forward(nf.Plan.explicit(cm, nf.OVERLAP, shares=(1, 1)), cm,
                 rt.pack_layer(cm, {k: dev(v) for k, v in synth.layer_weights(sm, 0).items()}), dev(synth.kv_pool(sm, b)),
                 nb, dev(synth.activations(sm, b.n_tokens)))
torch.cuda.synchronize()
print("moe layer ok")
