#!/usr/bin/env python
"""NEXT-1: the hot path on Table 3-like workloads
with the nano-batch plan re-searched per workload.

For each workload (Splitwise / LMSYS-Chat / ShareGPT-like length distributions,
synth/workloads.py) a steady-state dense batch of 2048 tokens is taken from the
continuous-batching snapshot, and one model step is timed under
  * SEQUENTIAL (the non-overlapped baseline, same kernels),
  * the fixed OVERLAP plan tuned on the constant-length workload (bench default),
  * the OVERLAP plan found by nf_plan_create (autosearch) for this
    workload's batch shape on the given kernel curves,
  * the best of a small measured grid (shares x partition splits) re-searched per workload,
in interleaved rounds (power/thermal drift).  Prints one JSON line per workload.

Usage: workload_sweep.py [--config c2|c3rank] [--curves profiles/curves_b200_r1b.csv] [--steps N]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=["c2", "c3rank", "c3loop"],
                    help="c3loop: rank 0 of a 70B TP8 group with loopback collectives, the TP pipeline, "
                         "plans searched with nf_plan_create at tp 8 over --curves (c3rank curves + NET model) "
                         "and refined by measurement (paper_2408_12757_b200/refine.py)")
    ap.add_argument("--curves", default="profiles/curves_b200_r1b.csv")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--workloads", default="splitwise,lmsys,sharegpt")
    ap.add_argument("--net-model", default="", choices=["", "nvlink"],
                    help="c3loop: model the collectives' link time (ring bytes / 725 GB/s, bench.py --net-model)")
    args = ap.parse_args()
    import torch

    import synth
    from synth import workloads as W
    from paper_2408_12757_b200 import nf, runtime as rt

    tp = 8 if args.config == "c3loop" else 1
    if args.config == "c3loop":
        shape = synth.SHAPES["llama2-70b"]
        dense, dec = 148, 148
    elif args.config == "c3rank":
        shape = synth.shape_with(synth.SHAPES["llama2-70b"], n_q_heads=8, n_kv_heads=1, d_ffn=3584)
        dense, dec = 132, 16
    else:
        shape = synth.SHAPES["llama3-8b"]
        dense, dec = 116, 32
    if args.layers:
        shape = synth.shape_with(shape, n_layers=args.layers)
    D, F, hd, Hq, Hk, L = shape.d_model, shape.d_ffn, shape.head_dim, shape.n_q_heads, shape.n_kv_heads, shape.n_layers
    # KV capacity of one B200 for this shape: HBM left after weights and workspace (~20 GB reserve)
    kv_token_bytes = L * 2 * (Hk // tp) * hd * 2
    kv_cap = int((180e9 - 2 * (L * (D * (Hq + 2 * Hk) * hd + (2 if tp > 1 else 1) * Hq * hd * D + 3 * D * F)
                               + 2 * shape.vocab * D) / tp - 20e9) / kv_token_bytes)
    snaps = {}
    for name in args.workloads.split(","):
        ql, kp, st = W.snapshot(name, b_dense=2048, kv_cap_tokens=kv_cap)
        snaps[name] = (ql, kp, st)
    need = {n: int(((kp.astype("int64") + ql + 15) // 16).sum()) for n, (ql, kp, _) in snaps.items()}
    pool_pages = max(need.values())
    cfg = rt.cfg_from_shape(shape, tp_size=tp, tp_rank=0)
    comm = nf.comm_create_loopback(tp, 0) if tp > 1 else None
    if comm is not None and args.net_model == "nvlink":
        nf.comm_loopback_set_link(comm, 725.0)   # bench.py NVLINK_BUS_GBS (a model, not a measurement)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)

    def randn(s, std=1.0, mean=0.0):
        t = torch.empty(s, dtype=torch.bfloat16, device="cuda")
        t.normal_(mean, std, generator=g)
        return t

    layers = []
    qs, ks, Fl = Hq // tp * hd, Hk // tp * hd, F // tp
    for _ in range(L):
        w = {"attn_norm": randn((D,), 0.1, 1.0), "w_q": randn((qs, D), D ** -0.5),
             "w_k": randn((ks, D), D ** -0.5), "w_v": randn((ks, D), D ** -0.5), "ffn_norm": randn((D,), 0.1, 1.0),
             "w_gate": randn((Fl, D), D ** -0.5), "w_up": randn((Fl, D), D ** -0.5), "w_down": randn((D, Fl), F ** -0.5)}
        if tp > 1:   # rank 0's shards
            w["w_o_col"] = randn((D // tp, Hq * hd), (Hq * hd) ** -0.5)
            w["w_o_row"] = randn((D, qs), (Hq * hd) ** -0.5)
        else:
            w["w_o"] = randn((D, Hq * hd), (Hq * hd) ** -0.5)
        layers.append(rt.pack_layer(cfg, w))
    model = rt.Model(cfg, randn((shape.vocab, D)), layers,
                     rt.pack_lm_head(cfg, randn((shape.vocab // tp, D), D ** -0.5), randn((D,), 0.1, 1.0)))
    pools = [randn((pool_pages, 2, Hk // tp, 16, hd)) for _ in range(L)]
    rows = [l.split(",") for l in open(os.path.join(ROOT, args.curves)).read().splitlines()[1:] if l.strip()]
    pts = [(int(k), int(u), float(w), float(t)) for k, _, u, w, t in rows]

    for name, (ql, kp, st) in snaps.items():
        b = synth.make_batch(ql, kp, seed=3, pool_slack=pool_pages - need[name])
        nb = nf.Batch.from_any(b)
        ws = rt.workspace(cfg, nb)
        tok = torch.randint(0, shape.vocab, (b.n_tokens,), dtype=torch.int32, device="cuda", generator=g)
        ids = torch.empty(b.n_req, dtype=torch.int32, device="cuda")
        auto = nf.Plan.search(cfg, nb, pts, mode=nf.OVERLAP, n_nano=4 if tp > 1 else 2)
        fixed_sm = [dense, dec, dense, dense, dense, dense, 16 if tp > 1 else 8]
        plans = [("sequential", nf.Plan.explicit(cfg, nf.SEQUENTIAL)),
                 ("overlap_fixed", nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1), sm=fixed_sm, balance=2,
                                                    n_dense=2 if tp > 1 else 0)),
                 ("overlap_autosearch", auto)]
        grid = []
        if tp > 1:
            # measured re-search per workload: the autosearched plan refined by interleaved A/B moves
            from paper_2408_12757_b200 import refine as R

            def run(pl, n):
                for _ in range(n):
                    model.step(pl, pools, nb, tok, ws, ids, comm=comm)

            def ab(cand, inc, pairs=2, n=2):
                run(cand, 1)
                run(inc, 1)
                tc, ti = [], []
                for _ in range(pairs):
                    for pl, acc in ((cand, tc), (inc, ti)):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        torch.cuda.synchronize()
                        e0.record()
                        run(pl, n)
                        e1.record()
                        torch.cuda.synchronize()
                        acc.append(e0.elapsed_time(e1) / n)
                return statistics.median(tc) / statistics.median(ti), statistics.median(tc)

            refined, rlog = R.refine(cfg, auto, ab, tp)
            grid.append(("refined " + json.dumps({k: v for k, v in rlog[-1].items() if k != "ms"}), refined))
        else:
            # measured re-search per workload: a small grid of shares x partition splits
            for sh in ((1, 1), (3, 5), (5, 3)):
                for dd, de in ((dense - 8, dec + 8), (dense, dec), (dense + 8, dec - 8)):
                    if de >= 8:
                        grid.append((f"grid shares={sh[0]}:{sh[1]} dense={dd} dec={de}",
                                     nf.Plan.explicit(cfg, nf.OVERLAP, shares=sh, sm=[dd, de, dd, dd, dd, dd, 8],
                                                      balance=2)))
        plans += grid
        for _, pl in plans:
            for _ in range(2):
                model.step(pl, pools, nb, tok, ws, ids, comm=comm)
        times = {n: [] for n, _ in plans}
        for _r in range(args.rounds):
            for pn, pl in plans:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record()
                for _ in range(args.steps):
                    model.step(pl, pools, nb, tok, ws, ids, comm=comm)
                e1.record()
                torch.cuda.synchronize()
                times[pn].append(e0.elapsed_time(e1) / args.steps)
        sp = auto.spec()
        res = {"workload": name, "config": args.config, "batch": st,
               "autosearch_plan": {"sm": list(sp.sm), "shares": list(sp.share)[:sp.n_nano], "note": auto.runtime_note()}}
        for pn, _ in plans[:3]:
            ms = statistics.median(times[pn])
            res[pn] = {"ms_per_step": ms, "tokens_per_s": b.n_tokens / (ms / 1e3),
                       "tokens_per_s_per_gpu": b.n_tokens / (ms / 1e3) / tp}
        gbest = min((statistics.median(times[pn]), pn) for pn, _ in grid)
        res["overlap_measured_search"] = {"ms_per_step": gbest[0], "tokens_per_s": b.n_tokens / (gbest[0] / 1e3),
                                          "tokens_per_s_per_gpu": b.n_tokens / (gbest[0] / 1e3) / tp, "plan": gbest[1]}
        print(json.dumps(res), flush=True)
        del ws


if __name__ == "__main__":
    main()
