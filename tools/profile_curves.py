#!/usr/bin/env python
"""Offline kernel profiling vs SM budget ("estimates the kernel
performance based on offline profiling"; Fig. 5 / SPEC S:237-269).

Times each hot-path kernel of the 8B-shape step at SM budgets
{8, 16, ..., 144, 148} with CUDA events and writes the SPEC curve CSV
`op_kind,resource_class,units,work,latency_s` (op_kind = NF_OP_* index), the
input of nf_plan_create.  Work: tokens for dense ops, KV keys for attention.

With --corun every point is measured next to a co-runner on the complementary
SMs (GEMM points next to decode attention on 148-u SMs, decode points next to the
Up/Gate GEMM on 148-u SMs): the co-run-calibrated curves SURVEY.md §7 asks for
("isolated curves are optimistic": HBM, L2 and power are shared).

Usage: python tools/profile_curves.py [--out profiles/curves_b200.csv] [--quick] [--corun]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "curves_b200.csv"))
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--corun", action="store_true", help="measure each point next to a co-runner on 148-u SMs")
    ap.add_argument("--shape", default="8b", choices=["8b", "c3rank"],
                    help="c3rank: one LLaMA-2-70B TP8 rank's shards (8/1 heads, F 3584) on the 512/1024 workload, "
                         "plus NET points of an NVLink model (see --net-gbs)")
    ap.add_argument("--net-gbs", type=float, default=770.0,
                    help="c3rank NET model: per-direction NVLink GB/s reached with >= 16 SMs (B200_PROFILING.md)")
    args = ap.parse_args()
    import numpy as np
    import torch

    import synth
    from paper_2408_12757_b200 import nf, runtime as rt

    dev = torch.device("cuda")
    if args.shape == "c3rank":
        shape = synth.shape_with(synth.SHAPES["llama2-70b"], n_q_heads=8, n_kv_heads=1, d_ffn=3584)
        p_in, d_out = 512, 1024
    else:
        shape = synth.SHAPES["llama3-8b"]
        p_in, d_out = 1024, 512
    D, F, hd, Hq, Hk = shape.d_model, shape.d_ffn, shape.head_dim, shape.n_q_heads, shape.n_kv_heads
    units = [8, 16, 32, 48, 64, 80, 96, 112, 128, 148] if args.quick else list(range(8, 145, 8)) + [148]
    rows = []
    st = rt.stream_handle()

    side = torch.cuda.Stream()
    side_h = int(side.cuda_stream)
    corunner = {"fn": None}  # fn(sm_budget, stream) launching one co-runner kernel

    def timeit(fn, u=148):
        for _ in range(2):
            fn()
        cr = corunner["fn"] if args.corun and u < 148 else None
        if cr is not None:
            # keep the complementary SMs busy for the whole measurement
            torch.cuda.synchronize()
            c0 = torch.cuda.Event(enable_timing=True)
            c0.record(side)
            cr(148 - u, side_h)
            c0.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if cr is not None:
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(side)
            cr(148 - u, side_h)
            f1.record(side)
            torch.cuda.synchronize()
            per = max(f0.elapsed_time(f1), 1e-3)
            e0.record()
            for _ in range(args.reps):
                fn()
            e1.record()
            # enough co-runner launches to outlast the timed loop (estimated from the isolated run)
            e1.synchronize()
            est = e0.elapsed_time(e1)
            torch.cuda.synchronize()
            for _ in range(int(est / per) + 3):
                cr(148 - u, side_h)
            e0.record()
            for _ in range(args.reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / args.reps / 1e3
        e0.record()
        for _ in range(args.reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.reps / 1e3

    # co-runners: decode attention over the steady-state decode batch (next to GEMMs / prefill),
    # the Up/Gate GEMM at M=1024 (next to decode attention)
    full0 = synth.workload_batch(2048, p_in, d_out)
    n0 = int((full0.q_len == 1).sum())
    b_cr = synth.make_batch([1] * n0, full0.kv_prefix[:n0], seed=5)
    nb_cr = nf.Batch.from_any(b_cr)
    cfg_cr = rt.cfg_from_shape(shape)
    pool_cr = torch.randn((b_cr.n_pages_pool, 2, Hk, 16, hd), device=dev).to(torch.bfloat16) if args.corun else None
    q_cr = torch.randn((n0, Hq, hd), device=dev).to(torch.bfloat16)
    o_cr = torch.empty((n0, Hq * hd), device=dev, dtype=torch.bfloat16)
    ws_cr = rt.workspace(cfg_cr, nb_cr)
    A_cr = torch.randn(1024, D, device=dev).to(torch.bfloat16)
    B_cr = (torch.randn(2 * F, D, device=dev) * D ** -0.5).to(torch.bfloat16)
    C_cr = torch.empty(1024, 2 * F, device=dev, dtype=torch.bfloat16)

    def cr_decode(sm, sth):
        nf.attention(cfg_cr, nb_cr, q_cr.data_ptr(), pool_cr.data_ptr(), o_cr.data_ptr(), ws_cr.data_ptr(),
                     ws_cr.numel(), sm, sm, sth)

    def cr_gemm(sm, sth):
        nf.gemm_bf16(A_cr.data_ptr(), D, B_cr.data_ptr(), D, C_cr.data_ptr(), 2 * F, 1024, 2 * F, D, sm, sth)

    # dense GEMMs at the nano-batch size (1024 tokens) and the full batch
    gemms = {nf.OP_KQV: ((Hq + 2 * Hk) * hd, D), nf.OP_O: (D, Hq * hd), nf.OP_UG: (2 * F, D), nf.OP_DOWN: (D, F)}
    # (c3rank: O is the rank's row-parallel O2 [M, D] x [D, D/8]^T; its column-parallel O1 has the same FLOPs)
    corunner["fn"] = cr_decode
    for M in (512, 1024, 2048):
        A = torch.randn(M, max(D, F), device=dev).to(torch.bfloat16)
        for op, (N, K) in gemms.items():
            B = (torch.randn(N, K, device=dev) * K ** -0.5).to(torch.bfloat16)
            C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
            gws = torch.empty(nf.gemm_workspace_bytes(M, N), dtype=torch.uint8, device=dev)
            for u in units:
                t = timeit(lambda: nf.gemm_bf16(A.data_ptr(), A.shape[1], B.data_ptr(), K, C.data_ptr(), N, M, N, K,
                                                u, st, gws.data_ptr(), gws.numel()), u)
                rows.append((op, "compute", u, M, t))
            del B, C
        del A
    # decode attention over the steady-state decode requests (683, contexts 1024..1535)
    corunner["fn"] = cr_gemm
    full = synth.workload_batch(2048, p_in, d_out)
    n_dec = int((full.q_len == 1).sum())
    for frac in (0.5, 1.0):
        n = int(n_dec * frac)
        b = synth.make_batch([1] * n, full.kv_prefix[:n], seed=3)
        nb = nf.Batch.from_any(b)
        cfg = rt.cfg_from_shape(shape)
        pool = torch.randn((b.n_pages_pool, 2, Hk, 16, hd), device=dev).to(torch.bfloat16)
        q = torch.randn((n, Hq, hd), device=dev).to(torch.bfloat16)
        o = torch.empty((n, Hq * hd), device=dev, dtype=torch.bfloat16)
        ws = rt.workspace(cfg, nb)
        keys = int((b.kv_prefix + 1).sum())
        for u in units:
            t = timeit(lambda: nf.attention(cfg, nb, q.data_ptr(), pool.data_ptr(), o.data_ptr(), ws.data_ptr(),
                                            ws.numel(), u, u, st), u)
            rows.append((nf.OP_DECODE_ATTN, "memory", u, keys, t))
            print(f"decode n={n} sm={u}: {t*1e6:.1f} us  {keys*Hk*hd*4/t/1e9:.0f} GB/s", flush=True)
        del pool
    # prefill attention: the chunk (341, prefix 683) + prompt (1024)
    corunner["fn"] = cr_decode
    b = synth.make_batch([341, 1024], [683, 0], seed=3) if args.shape == "8b" else \
        synth.make_batch([171, 512], [341, 0], seed=3)
    nb = nf.Batch.from_any(b)
    pool = torch.randn((b.n_pages_pool, 2, Hk, 16, hd), device=dev).to(torch.bfloat16)
    q = torch.randn((b.n_tokens, Hq, hd), device=dev).to(torch.bfloat16)
    o = torch.empty((b.n_tokens, Hq * hd), device=dev, dtype=torch.bfloat16)
    ws = rt.workspace(cfg, nb)
    keys = int(sum(p + (i + 1) for p, ql in zip(b.kv_prefix, b.q_len) for i in range(ql)))
    for u in units:
        t = timeit(lambda: nf.attention(cfg, nb, q.data_ptr(), pool.data_ptr(), o.data_ptr(), ws.data_ptr(),
                                        ws.numel(), u, u, st), u)
        rows.append((nf.OP_PREFILL_ATTN, "compute", u, keys, t))
    if args.shape == "c3rank":
        # NET: NO measurement is possible on one GPU.  Model (reading P-8 / §7a): an
        # AllGather-equivalent token moves (N-1)/N * D * 2 bytes per rank at N = 8; NCCL reaches
        # the measured per-direction NVLink bandwidth with >= 16 CTAs (PAPER.md:614 reports 92 % of
        # peak with 35 of 108 A100 SMs), proportionally less below; 10 us launch + sync latency.
        per_tok = 7 / 8 * D * 2
        for u in units:
            for w in (256.0, 1024.0, 2048.0, 4096.0):
                bw = args.net_gbs * 1e9 * min(1.0, u / 16.0)
                rows.append((nf.OP_NET, "network", u, w, 10e-6 + w * per_tok / bw))
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        f.write("op_kind,resource_class,units,work,latency_s\n")
        for r in rows:
            f.write(f"{r[0]},{r[1]},{r[2]},{r[3]},{r[4]:.9g}\n")
    print(f"wrote {len(rows)} rows to {args.out}")


if __name__ == "__main__":
    main()
