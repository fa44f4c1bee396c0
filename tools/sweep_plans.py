#!/usr/bin/env python
"""Time nf_model_step for many explicit plans in one process (weights and KV
allocated once).  Usage: sweep_plans.py [--config c2|c3rank|c4rank] [--steps N]
Prints ms/step per plan, best first."""
import argparse
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--shares", default="1:1,5:3", help="comma list of a:b nano-batch shares")
    ap.add_argument("--splits", default="148/148,116/32,108/40,100/48", help="comma list of dense/decode SMs")
    ap.add_argument("--bal", default="2")
    ap.add_argument("--colocate", default="", help="comma list of a:b shares for co-located plans")
    args = ap.parse_args()
    import torch

    import synth
    from paper_2408_12757_b200 import nf, runtime as rt
    if args.config == "c3rank":
        shape = synth.shape_with(synth.SHAPES["llama2-70b"], n_q_heads=8, n_kv_heads=1, d_ffn=3584)
        p_in, d_out = 512, 1024
    elif args.config == "c4rank":
        shape = synth.shape_with(synth.SHAPES["mixtral-8x7b"], n_q_heads=4, n_kv_heads=1, d_ffn=1792)
        p_in, d_out = 512, 1024
    else:
        shape = synth.SHAPES["llama3-8b"]
        p_in, d_out = 1024, 512
    if args.layers:
        shape = synth.shape_with(shape, n_layers=args.layers)
    b = synth.workload_batch(2048, p_in, d_out)
    nb = nf.Batch.from_any(b)
    cfg = rt.cfg_from_shape(shape)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)

    def randn(s, std=1.0, mean=0.0):
        t = torch.empty(s, dtype=torch.bfloat16, device="cuda")
        t.normal_(mean, std, generator=g)
        return t

    D, F, hd, Hq, Hk = shape.d_model, shape.d_ffn, shape.head_dim, shape.n_q_heads, shape.n_kv_heads
    layers = []
    for _ in range(shape.n_layers):
        w = {"attn_norm": randn((D,), 0.1, 1.0), "w_q": randn((Hq * hd, D), D ** -0.5),
             "w_k": randn((Hk * hd, D), D ** -0.5), "w_v": randn((Hk * hd, D), D ** -0.5),
             "w_o": randn((D, Hq * hd), (Hq * hd) ** -0.5), "ffn_norm": randn((D,), 0.1, 1.0),
             "w_gate": randn((F, D), D ** -0.5), "w_up": randn((F, D), D ** -0.5), "w_down": randn((D, F), F ** -0.5)}
        if shape.n_experts:
            E = shape.n_experts
            w.update(w_router=randn((E, D), D ** -0.5), w_gate=randn((E, F, D), D ** -0.5),
                     w_up=randn((E, F, D), D ** -0.5), w_down=randn((E, D, F), F ** -0.5))
        layers.append(rt.pack_layer(cfg, w))
    model = rt.Model(cfg, randn((shape.vocab, D)), layers,
                     rt.pack_lm_head(cfg, randn((shape.vocab, D), D ** -0.5), randn((D,), 0.1, 1.0)))
    pools = [randn((b.n_pages_pool, 2, Hk, 16, hd)) for _ in range(shape.n_layers)]
    tok = torch.randint(0, shape.vocab, (b.n_tokens,), dtype=torch.int32, device="cuda", generator=g)
    ws = rt.workspace(cfg, nb)
    ids = torch.empty(b.n_req, dtype=torch.int32, device="cuda")

    def run(plan):
        for _ in range(2):
            model.step(plan, pools, nb, tok, ws, ids)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            model.step(plan, pools, nb, tok, ws, ids)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps

    # build every plan first, then time them in a forward and a reverse pass (power / thermal
    # drift of the 1 kW part would otherwise favour whichever plan runs first); mean of passes
    plans = [("sequential", nf.Plan.explicit(cfg, nf.SEQUENTIAL)),
             ("nano_only bal=2", nf.Plan.explicit(cfg, nf.NANO_ONLY, shares=(1, 1), balance=2))]
    for sh in args.shares.split(","):
        shares = tuple(int(x) for x in sh.split(":"))
        for bal in [int(x) for x in args.bal.split(",")]:
            for sp in args.splits.split(","):
                dense, dec = (int(x) for x in sp.split("/"))
                sm = [dense, dec, dense, dense, dense, dense, 8]
                plans.append((f"overlap shares={shares} bal={bal} dense={dense} dec={dec}",
                              nf.Plan.explicit(cfg, nf.OVERLAP, shares=shares, sm=sm, balance=bal)))
    for shares in ([tuple(int(x) for x in sh.split(":")) for sh in args.colocate.split(",")] if args.colocate else []):
        plans.append((f"colocate shares={shares}", nf.Plan.explicit(cfg, nf.OVERLAP, shares=shares, sm=[148] * 7,
                                                                     balance=True, colocate=True)))
    acc = {n: [] for n, _ in plans}
    for order in (plans, plans[::-1]):
        for name, pl in order:
            acc[name].append(run(pl))
    results = []
    for name, pl in plans:
        results.append((name, sum(acc[name]) / len(acc[name])))
        print((name, round(results[-1][1], 3), [round(x, 3) for x in acc[name]]), pl.runtime_note(), flush=True)
    print("---- best first")
    for n, t in sorted(results, key=lambda x: x[1])[:12]:
        print(f"{t:8.2f} ms  {n}")


if __name__ == "__main__":
    main()
