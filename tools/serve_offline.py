#!/usr/bin/env python
"""Offline serving throughput: a synthetic
trace of requests served to completion by the native scheduler + nf_model_step
on one B200 (paper_2408_12757_b200.serving.OfflineServer).

Usage: serve_offline.py [--workload splitwise|lmsys|sharegpt|const:P:D] [--n-req N]
         [--config c2|c4rank] [--pages P] [--mode overlap|sequential]
Prints one JSON line: total (input + output) tokens/s over the whole trace and in
the steady state (steps launched while requests still wait for admission, i.e.
the system at capacity, excluding the drain of the last long requests), output
tokens/s, steps, mean dense batch, scheduler host time share, useless tokens."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="splitwise")
    ap.add_argument("--n-req", type=int, default=2000)
    ap.add_argument("--config", default="c2", choices=["c2", "c4rank"])
    ap.add_argument("--pages", type=int, default=60000)
    ap.add_argument("--mode", default="overlap", choices=["overlap", "sequential"])
    ap.add_argument("--bdense", default="2048,1792,1536,1280,1024,768,512,256")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--max-len", type=int, default=4096)
    args = ap.parse_args()
    import numpy as np
    import torch

    import synth
    import synth.workloads as W
    from paper_2408_12757_b200 import nf, runtime as rt
    from paper_2408_12757_b200.serving import OfflineServer

    if args.config == "c4rank":
        shape = synth.shape_with(synth.SHAPES["mixtral-8x7b"], n_q_heads=4, n_kv_heads=1, d_ffn=1792)
    else:
        shape = synth.SHAPES["llama3-8b"]
    if args.layers:
        shape = synth.shape_with(shape, n_layers=args.layers)
    if args.workload.startswith("const:"):
        _, p, d = args.workload.split(":")
        inp = np.full(args.n_req, int(p))
        out = np.full(args.n_req, int(d))
    else:
        inp, out = W.sample_lengths(args.workload, args.n_req, seed=6, max_len=args.max_len)
    cfg = rt.cfg_from_shape(shape)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)

    def randn(s, std=1.0, mean=0.0):
        t = torch.empty(s, dtype=torch.bfloat16, device="cuda")
        t.normal_(mean, std, generator=g)
        return t

    D, F, hd, Hq, Hk, E = (shape.d_model, shape.d_ffn, shape.head_dim, shape.n_q_heads, shape.n_kv_heads,
                           shape.n_experts)
    ex = (E,) if E else ()
    layers = []
    for _ in range(shape.n_layers):
        w = {"attn_norm": randn((D,), 0.1, 1.0), "w_q": randn((Hq * hd, D), D ** -0.5),
             "w_k": randn((Hk * hd, D), D ** -0.5), "w_v": randn((Hk * hd, D), D ** -0.5),
             "w_o": randn((D, Hq * hd), (Hq * hd) ** -0.5), "ffn_norm": randn((D,), 0.1, 1.0),
             "w_gate": randn(ex + (F, D), D ** -0.5), "w_up": randn(ex + (F, D), D ** -0.5),
             "w_down": randn(ex + (D, F), F ** -0.5)}
        if E:
            w["w_router"] = randn((E, D), D ** -0.5)
        layers.append(rt.pack_layer(cfg, w))
        del w
    model = rt.Model(cfg, randn((shape.vocab, D)), layers,
                     rt.pack_lm_head(cfg, randn((shape.vocab, D), D ** -0.5), randn((D,), 0.1, 1.0)))
    pools = [torch.empty((args.pages, 2, Hk, 16, hd), dtype=torch.bfloat16, device="cuda")
             for _ in range(shape.n_layers)]
    bdense = [int(x) for x in args.bdense.split(",")]
    sched = nf.Scheduler(args.pages, 16, bdense, max(1, int(np.mean(out))))
    rng = np.random.default_rng(7)
    for i in range(args.n_req):
        sched.submit(i, rng.integers(0, shape.vocab, size=int(inp[i])).astype(np.int32), int(out[i]))
    if args.mode == "overlap":
        dense, dec = (116, 32) if args.config == "c2" else (132, 16)
        plan = nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1), sm=[dense, dec, dense, dense, dense, dense, 8],
                                balance=2)
    else:
        plan = nf.Plan.explicit(cfg, nf.SEQUENTIAL)
    srv = OfflineServer(model, plan, pools, sched, args.pages, max_tokens=max(bdense), max_reqs=max(bdense))
    n0 = nf.kernel_launches()
    st = srv.run()
    launches = nf.kernel_launches() - n0
    total_tokens = int(inp.sum() + out.sum())
    line = {"tool": "serve_offline", "model": shape.name, "n_layers": shape.n_layers, "workload": args.workload,
            "n_req": args.n_req, "mode": args.mode, "pages": args.pages, "bdense": bdense,
            "mean_input": float(inp.mean()), "mean_output": float(out.mean()),
            "throughput_tokens_per_s": total_tokens / st["wall_s"],
            "output_tokens_per_s": float(out.sum()) / st["wall_s"],
            "steady_tokens_per_s": (st["steady_tokens"] / st["steady_s"]) if st.get("steady_s") else None,
            "steady_steps": st.get("steady_steps"),
            "steady_mean_step_tokens": (st["steady_tokens"] / st["steady_steps"]) if st.get("steady_steps") else None,
            "wall_s": st["wall_s"], "device_s": st["device_s"], "steps": st["gpu_steps"],
            "mean_step_tokens": st["step_tokens"] / max(1, st["gpu_steps"]),
            "ms_per_step": 1e3 * st["wall_s"] / max(1, st["gpu_steps"]),
            "host_sched_share": st["host_sched_s"] / st["wall_s"], "useless_tokens": st["useless"],
            "evictions": st["evictions"], "peak_pages_used": st["peak_pages_used"], "finished": st["finished"],
            "gpu_launches": launches, "data": "synthetic (random-init weights, lognormal Table 3 lengths, A-19)"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
