#!/usr/bin/env python
"""Benchmark of the NanoFlow hot path on B200 (one JSON line on rank 0).

N = 1 (default, --config c2): BASELINE.json configs[1], the largest config that
fits one GPU (the metric's configs[2] 70B-TP8 does not): a LLaMA-3-8B-shape model
(32 layers, D 4096, 32/8 heads, hd 128, F 14336, V 128256), random-init bf16
weights, serving step over the B_dense = 2048 steady state of the constant
1024-in / 512-out workload: 683 decode requests (contexts
1024..1535) + a 341-token chunk (prefix 683) + one 1024-token prompt, paged KV
(page 16).  A "step" = one nf_model_step: embedding -> 32 decoder layers
(KQV+RoPE+KV append, paged decode/prefill attention, O, RMSNorm, SwiGLU, Down)
-> final norm -> LM head -> argmax, through the C ABI, replayed as a CUDA graph.
Inputs are resident in HBM (KV 115 GB + weights 15 GB per step, far above the
126 MB L2: no flush needed).

N > 1 (torchrun; default --config c3): the metric's configs[2], LLaMA-2-70B
shape (80 layers) tensor-parallel over all N ranks with NCCL (B_dense 768 at
TP2, 2048 at TP4/8), the paper's TP pipeline (4 attention / 2 dense
nano-batches, collectives on a network partition); value = the job's
tokens/s, tokens_per_s_per_gpu = value / N.  Rank 0 checks layer 0 against the
oracle in the run (sampled requests) and every rank's hidden states agree.
--config c3loop: rank 0 of a TP8 group on one GPU with loopback collectives
(per-rank performance proxy).  --impl reference: the CPU oracle (oracle/,
float64 numpy) as the reference arm, on a bounded sample.
--plan refine: the autosearched plan refined by interleaved measured A/B moves.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s/GPU and % of compute-bound optimal, LLaMA-2-70B-shape TP8"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def p_active(shape):
    """Matmul weights touched per token: L*(D*(Hq+2Hkv)*hd + Hq*hd*D + 3*D*F) + V*D;
    MoE: the FFN term is top_k*3*D*F + E*D (router), SURVEY §8d (Mixtral 12.75e9)."""
    s = shape
    ffn = (s.top_k * 3 * s.d_model * s.d_ffn + s.n_experts * s.d_model) if s.n_experts else 3 * s.d_model * s.d_ffn
    return s.n_layers * (s.d_model * (s.n_q_heads + 2 * s.n_kv_heads) * s.head_dim +
                         s.n_q_heads * s.head_dim * s.d_model + ffn) + s.vocab * s.d_model


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-lms", "100", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi needs ~0.1-0.5 s to start: wait for its first sample so that the
            # sampler is already running when the timed region begins (short runs included)
            t_end = time.time() + 3.0
            while not self.lines and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons, pw = [], 0, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
                pw.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w": statistics.median(pw) if pw else None}


# ---------------------------------------------------------------------------- oracle sample
def config_shape(config, tp=1):
    """(shape, p_in, d_out) of a bench config (SURVEY.md §8 shape key)."""
    import synth
    if config == "c3rank":
        return (synth.shape_with(synth.SHAPES["llama2-70b"], name="llama2-70b-tp8-rank", n_q_heads=8, n_kv_heads=1,
                                 d_ffn=28672 // 8), 512, 1024)
    if config in ("c3", "c3loop"):
        return synth.SHAPES["llama2-70b"], 512, 1024
    if config == "c4rank":
        return mixtral_rank_shape(), 512, 1024
    if config == "c4":
        return synth.SHAPES["mixtral-8x7b"], 512, 1024
    return synth.SHAPES["llama3-8b"], 1024, 512


def mixtral_rank_shape():
    """One Mixtral-8x7B TP8 rank's shards: 4/1 heads, 8 experts x F 1792 (configs[3] proxy)."""
    import synth
    return synth.shape_with(synth.SHAPES["mixtral-8x7b"], name="mixtral-8x7b-tp8-rank", n_q_heads=4, n_kv_heads=1,
                            d_ffn=14336 // 8)


def workload_desc(config, L, tp=1, b_dense=2048):
    if config == "c2":
        return (f"configs[1]: LLaMA-3-8B-shape {L}-layer serving step, B_dense 2048 "
                f"(683 decode ctx 1024-1535 + 341-token chunk + 1024-token prompt), page 16")
    if config == "c3rank":
        return (f"configs[2] rank-local proxy: one LLaMA-2-70B TP8 rank's shards (D 8192, 8/1 heads, "
                f"F 3584), {L} layers, B_dense 2048 (1365 decode ctx 512-1535 + 171 chunk + 512 prompt), "
                f"no collectives")
    if config == "c3loop":
        return (f"configs[2] rank proxy: rank 0 of a LLaMA-2-70B TP8 group on one GPU ({L} layers, its head / FFN / "
                f"vocab shards, B_dense 2048 = 1365 decode ctx 512-1535 + 171 chunk + 512 prompt) running the TP "
                f"pipeline with loopback collectives (local copies of the AllGather / AllReduce bytes, no peers); "
                f"value = 2048 / (T_step x 8) tokens/s/GPU")
    if config == "c4rank":
        return (f"configs[3] rank-local proxy: one Mixtral-8x7B TP8 rank's shards (D 4096, 4/1 heads, 8 experts "
                f"x F 1792, top-2), {L} layers, B_dense 2048 (1365 decode ctx 512-1535 + 171 chunk + 512 prompt), "
                f"no collectives")
    if config == "c4":
        return (f"configs[3]: Mixtral-8x7B-shape {L}-layer serving step (8 experts, top-2), TP={tp} over NCCL, "
                f"B_dense {b_dense} (constant 512 in / 1024 out steady state), page 16")
    return (f"configs[2]: LLaMA-2-70B-shape {L}-layer serving step, TP={tp} over NCCL, B_dense {b_dense} "
            f"(constant 512 in / 1024 out steady state), page 16")


def oracle_sample(shape, n_dec=64, chunk=64, p_in=1024, d_out=512):
    """Bounded sample of the same workload for the CPU oracle: n_dec decode
    requests drawn from the steady state (contexts p_in..p_in+d_out-1) plus one
    prefill chunk of `chunk` tokens (prefix 0), one decoder layer."""
    import numpy as np
    import synth
    full = synth.workload_batch(2048, p_in, d_out)
    q_len = [1] * n_dec + [chunk]
    prefix = list(full.kv_prefix[:n_dec]) + [0]
    b = synth.make_batch(q_len, prefix, seed=3)
    w = synth.layer_weights(shape, 0, seed=0)
    x = synth.activations(shape, b.n_tokens, seed=1)
    pool = synth.kv_pool(shape, b, seed=2)
    return b, w, x, pool


def time_oracle_layer(shape, b, w, x, pool, reps=1):
    import numpy as np
    from oracle import layer as OL
    from oracle import moe as OM
    layer = OM.moe_decoder_layer if shape.n_experts else OL.decoder_layer
    ts = []
    for _ in range(reps):
        p = OL.as_pool(pool)
        t0 = time.perf_counter()
        layer(x, w, p, b, shape)
        ts.append(time.perf_counter() - t0)
    return ts


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 0) for i in threadpool_info()), default=None)
    except Exception:
        return None


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The oracle as it stands (float64 numpy) on the host cores: each timed step is
    one oracle decoder layer over a bounded sample of the workload (64 decode
    requests with the steady-state contexts + one 64-token prefill chunk); value =
    the sample's tokens per second of a whole L-layer step (t_layer x L)."""
    if rank != 0:
        return
    args.config = args.config or ("c2" if max(1, args.gpus) == 1 else "c3")
    shape, p_in, d_out = config_shape(args.config)
    b, w, x, pool = oracle_sample(shape, p_in=p_in, d_out=d_out)
    T = b.n_tokens
    for _ in range(args.warmup):
        time_oracle_layer(shape, b, w, x, pool)
    ts = []
    for _ in range(args.steps):
        ts += time_oracle_layer(shape, b, w, x, pool)
    t_layer = statistics.median(ts)
    value = T / (t_layer * shape.n_layers)
    sample = (f"one float64 oracle decoder layer (numpy/BLAS) of the {shape.name} shape over {T} tokens "
              f"(64 decode requests with the steady-state contexts + one 64-token prefill chunk) per timed step "
              f"(median {t_layer:.2f} s); value = {T} tokens / ({shape.n_layers} x t_layer)")
    cores = blas_threads() or cpu_cores()
    tp = max(1, args.gpus) if args.config in ("c3", "c4") else 1
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_layer * 1e3, "higher_is_better": True,
            "scaling": "strong" if tp > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": bench_config(args.config, shape, tp, 768 if (args.config == "c3" and tp == 2) else 2048),
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


NVLINK_BUS_GBS = 725.0   # B200_PROFILING.md: measured 8-rank all-reduce bus bandwidth at 1 GiB


def bench_config(config, shape, tp, b_dense):
    """The `config` object of both arms (identical for the same workload)."""
    return {"workload": workload_desc(config, shape.n_layers, tp=tp, b_dense=b_dense), "b_dense": b_dense,
            "n_layers": shape.n_layers, "tp": tp,
            "l2": "no flush: per-step inputs (KV + weights, tens of GB) >> 126 MB L2"}


# ---------------------------------------------------------------------------- in-run parity
PARITY_REQS = {"c2": [0, 1, 2, 341, 682, 683], "c3": [0, 1, 700, 1364, 1365], "c3_768": [0, 1, 300, 511, 512]}


def compact_from_pool(b, reqs, pool_dev):
    """Sub-batch of requests `reqs` with a compact float64 host pool holding their cached
    K/V pages copied from the device pool (before the step appends to it)."""
    import numpy as np
    import synth
    sub = synth.make_batch(b.q_len[reqs], b.kv_prefix[reqs], permute=False)
    pool = np.zeros((sub.n_pages_pool,) + tuple(pool_dev.shape[1:]), dtype=np.float64)
    for i, r in enumerate(reqs):
        src = b.page_ids[b.page_indptr[r]:b.page_indptr[r + 1]]
        dst = sub.page_ids[sub.page_indptr[i]:sub.page_indptr[i + 1]]
        n = min(len(src), len(dst))
        idx = __import__("torch").as_tensor(src[:n].astype(np.int64), device=pool_dev.device)
        pool[dst[:n]] = pool_dev[idx].float().cpu().numpy()
    return sub, pool


def oracle_parity(shape, b, reqs, w_full, x_in, y_out, pool_sub, sub):
    """Oracle layer on the GPU's own bf16 layer input for sampled requests
    (teacher-forced) vs the GPU's layer output on those rows."""
    import numpy as np
    from oracle import layer as OL
    ind = np.concatenate([[0], np.cumsum(b.q_len)])
    rows = np.concatenate([np.arange(ind[r], ind[r + 1]) for r in reqs])
    ref = OL.decoder_layer(x_in[rows], w_full, pool_sub, sub, shape)
    out = y_out[rows]
    err = out - ref
    return {"layer": 0, "requests": list(map(int, reqs)), "rows": int(len(rows)),
            "rel_l2": float(np.linalg.norm(err) / np.linalg.norm(ref)), "max_abs": float(np.abs(err).max()),
            "tolerance": {"rel_l2": 1e-2, "max_abs": 5e-2}}


# ---------------------------------------------------------------------------- nf arm
def run_nf(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2408_12757_b200 import nf, runtime as rt

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    tp = 1
    comm = None
    loop = args.config == "c3loop"
    if loop:
        tp = 8   # rank 0 of a TP8 group, loopback collectives
    if args.config in ("c3", "c4"):
        # configs[2] / [3]: tensor parallel over all ranks (NCCL over NVLink)
        if world < 2:
            raise SystemExit(f"--config {args.config} needs torchrun with >= 2 GPUs (weights + KV do not fit one B200)")
        tp = world
    shape, p_in, d_out = config_shape(args.config)
    if args.layers:
        shape = synth.shape_with(shape, n_layers=args.layers)
    L = shape.n_layers
    b_dense = 768 if (args.config == "c3" and tp == 2) else 2048   # TP2: memory cap
    if args.b_dense:
        b_dense = args.b_dense   # (dev) e.g. 2049 for the batch-size cliff
    b = synth.workload_batch(b_dense, p_in, d_out)
    T = b.n_tokens
    nb = nf.Batch.from_any(b)
    cfg = rt.cfg_from_shape(shape, tp_size=tp, tp_rank=rank if (tp > 1 and not loop) else 0)

    # ---------------- plan (chosen before the communicator: its network SM budget caps NCCL's CTAs)
    sm = [int(x) for x in args.sm.split(",")] if args.sm else None
    if args.mode == "auto":
        # per-config default = the fastest plan measured on B200 (interleaved ablations,
        # profiles/r1c_bench_*_final.log, r1c_sweep_c4rank.log): the rank proxies of the
        # 70B and Mixtral TP8 configs on the constant 512/1024 workload run best SEQUENTIAL;
        # configs[1] and the TP configs run the OVERLAP pipeline
        args.mode = "sequential" if args.config in ("c3rank", "c4rank") else "overlap"
    n_dense = 0
    if args.mode == "overlap":
        if args.plan in ("auto", "refine") and not (tp > 1 and not os.path.exists(os.path.join(ROOT, args.curves_tp))):
            cpath = os.path.join(ROOT, args.curves_tp if tp > 1 else args.curves)
            rows = [l.split(",") for l in open(cpath).read().splitlines()[1:] if l.strip()]
            pts = [(int(k), int(u), float(w), float(t)) for k, _, u, w, t in rows]
            sp = nf.Plan.search(cfg, nb, pts, mode=nf.OVERLAP, n_nano=4 if tp > 1 else 2).spec()
            sp.graph = int(not args.no_graph)
            plan = nf.Plan.from_spec(cfg, sp)
        elif args.colocate:
            plan = nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1), sm=sm or [148] * 7, balance=True,
                                    colocate=True)
        else:
            # defaults = best of tools/sweep_plans.py on B200 (profiles/r1_sweep_*.log); TP: the
            # paper's 4-way KQV/attention, 2-way O/UGD/network split with a network
            # partition for the collectives
            # TP (c3 / c4 / c3loop): two dense nano-batches on per-group compute streams with decode
            # attention on them (no memory partition) and the collectives on a 16-SM network
            # partition -- the best TP8-rank plan measured on one GPU (profiles/r2_tp8_rank_plans.md)
            dense, dec, net, dshares = {"c2": (116, 32, 8, "1,1"), "c4rank": (132, 16, 8, "3,5"),
                                        "c3": (148, 148, 16, "1,1"), "c4": (148, 148, 16, "1,1"),
                                        "c3loop": (148, 148, 16, "1,1")}.get(
                args.config, (132, 16, 8, "1,1"))
            shares = tuple(int(x) for x in (args.shares or dshares).split(","))
            n_dense = 2 if (tp > 1 and len(shares) in (2, 4)) else 0
            plan = nf.Plan.explicit(cfg, nf.OVERLAP, shares=shares, sm=sm or [dense, dec, dense, dense, dense, dense, net],
                                    balance=args.balance, n_dense=n_dense, graph=not args.no_graph)
    elif args.mode == "nano":
        plan = nf.Plan.explicit(cfg, nf.NANO_ONLY, shares=tuple(int(x) for x in (args.shares or "1,1").split(",")), sm=sm,
                                balance=args.balance, graph=not args.no_graph)
    else:
        plan = nf.Plan.explicit(cfg, nf.SEQUENTIAL, sm=sm, graph=not args.no_graph)
    if loop:
        comm = nf.comm_create_loopback(tp, 0)
        if args.net_model == "nvlink":
            # link-time model (not a measurement): every collective lasts >= its ring bytes per
            # GPU / 725 GB/s, the 8-rank all-reduce bus bandwidth B200_PROFILING.md measured at 1 GiB
            nf.comm_loopback_set_link(comm, NVLINK_BUS_GBS)
    elif tp > 1:
        uid = [nf.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = nf.comm_create(tp, rank, uid[0], max_ctas=plan.spec().sm[nf.OP_NET])
    fused_note = None
    if comm is not None and args.fused_ar:
        # NEXT-3: row-parallel GEMM -> AllReduce over peer memory (CUDA IPC handles exchanged
        # through the process group; a loopback rank runs its sites as a group of one)
        h = nf.comm_sym_alloc(comm, cfg, T)
        hs = [h]
        if not loop:
            hs = [None] * world
            dist.all_gather_object(hs, h)
        nf.comm_sym_open(comm, None if loop else hs)
        fused_note = ("fused over peer memory: row-parallel GEMM->AllReduce (EPI_PEER + owner reduce) and the O "
                      "column-parallel GEMM->AllGather (epilogue stores to every rank); NCCL for the attention AllGather")

    # ---------------- weights: replicated tensors (embedding, norms) and layer 0 (in-run parity)
    # from a generator seeded identically on every rank; every other layer's shards from a
    # per-rank stream (random init either way)
    g_rep = torch.Generator(device=dev)
    g_rep.manual_seed(1234)
    g_loc = torch.Generator(device=dev)
    g_loc.manual_seed(4321 + rank)

    def randn(shape_, std=1.0, mean=0.0, gen=None):
        t = torch.empty(shape_, dtype=torch.bfloat16, device=dev)
        t.normal_(mean, std, generator=gen or g_loc)
        return t

    D, F, hd, Hq, Hk = shape.d_model, shape.d_ffn, shape.head_dim, shape.n_q_heads, shape.n_kv_heads
    E = shape.n_experts
    ex = (E,) if E else ()                     # MoE: expert-major [E, F/N, D] / [E, D, F/N]
    qs, ks, Dl, Fl = Hq // tp * hd, Hk // tp * hd, D // tp, F // tp

    def full_layer(gen):
        w = {"attn_norm": randn((D,), 0.1, 1.0, gen=g_rep), "w_q": randn((Hq * hd, D), D ** -0.5, gen=gen),
             "w_k": randn((Hk * hd, D), D ** -0.5, gen=gen), "w_v": randn((Hk * hd, D), D ** -0.5, gen=gen),
             "w_o": randn((D, Hq * hd), (Hq * hd) ** -0.5, gen=gen), "ffn_norm": randn((D,), 0.1, 1.0, gen=g_rep),
             "w_gate": randn(ex + (F, D), D ** -0.5, gen=gen), "w_up": randn(ex + (F, D), D ** -0.5, gen=gen),
             "w_down": randn(ex + (D, F), F ** -0.5, gen=gen)}
        if E:
            w["w_router"] = randn((E, D), D ** -0.5, gen=g_rep)
        return w

    srank = 0 if loop else rank

    def shard_of(w):
        return w if tp == 1 else rt.shard_layer(w, Hq, Hk, hd, tp, srank)

    layers = []
    w0_full = None
    for l in range(L):
        if l == 0 or tp == 1:
            w = full_layer(g_rep if l == 0 else g_loc)
            if l == 0:
                w0_full = w
            layers.append(rt.pack_layer(cfg, shard_of(w)))
        else:  # this rank's shards only
            w = {"attn_norm": randn((D,), 0.1, 1.0, gen=g_rep), "w_q": randn((qs, D), D ** -0.5),
                 "w_k": randn((ks, D), D ** -0.5), "w_v": randn((ks, D), D ** -0.5),
                 "w_o_col": randn((Dl, Hq * hd), (Hq * hd) ** -0.5), "w_o_row": randn((D, qs), (Hq * hd) ** -0.5),
                 "ffn_norm": randn((D,), 0.1, 1.0, gen=g_rep), "w_gate": randn(ex + (Fl, D), D ** -0.5),
                 "w_up": randn(ex + (Fl, D), D ** -0.5), "w_down": randn(ex + (D, Fl), F ** -0.5)}
            if E:
                w["w_router"] = randn((E, D), D ** -0.5, gen=g_rep)
            layers.append(rt.pack_layer(cfg, w))
        del w
    embed = randn((shape.vocab, D), gen=g_rep)
    lm_full = randn((shape.vocab, D), D ** -0.5, gen=g_rep)
    lm = rt.pack_lm_head(cfg, rt.shard_vocab(lm_full, tp, srank) if tp > 1 else lm_full, randn((D,), 0.1, 1.0, gen=g_rep))
    del lm_full
    model = rt.Model(cfg, embed, layers, lm)
    # KV pools: layer 0 full (replicated seed) then this rank's heads; the rest per rank
    pool0_full = randn((b.n_pages_pool, 2, Hk, 16, hd), gen=g_rep)
    pools = [rt.shard_pool(pool0_full, tp, srank) if tp > 1 else pool0_full.clone()]
    pools += [randn((b.n_pages_pool, 2, Hk // tp, 16, hd)) for _ in range(1, L)]
    tok = torch.randint(0, shape.vocab, (T,), dtype=torch.int32, device=dev, generator=g_rep)
    ws = rt.workspace(cfg, nb, dev)
    next_ids = torch.empty(b.n_req, dtype=torch.int32, device=dev)
    torch.cuda.synchronize()

    # ---------------- in-run parity (before timing; its step rewrites the same KV slots the timed steps do)
    parity = None
    if loop:
        parity = {"skipped": "loopback collectives do not reduce: the proxy's values are not the model's"}
    elif not args.no_parity and not E:
        key = "c3_768" if (args.config == "c3" and tp == 2) else ("c3" if args.config in ("c3", "c3rank") else "c2")
        reqs = [r for r in PARITY_REQS[key] if r < b.n_req]
        if rank == 0:
            sub, pool_sub = compact_from_pool(b, reqs, pool0_full)
            w_host = {k: v.float().cpu().numpy() for k, v in w0_full.items()}
        ids, _, hid = model.step_inspect(plan, pools, nb, tok, ws, comm=comm, logits=False, hidden=True)
        torch.cuda.synchronize()
        h0 = hid[0].float().cpu().numpy()
        h1 = hid[1].float().cpu().numpy()
        same = True
        if tp > 1:
            ck = torch.tensor([float(hid[1].float().sum()), float(hid[L].float().abs().sum())], dtype=torch.float64,
                              device=dev)
            allck = [torch.empty_like(ck) for _ in range(world)]
            dist.all_gather(allck, ck)
            same = all(torch.equal(allck[0], c) for c in allck)
        if rank == 0:
            parity = oracle_parity(shape, b, reqs, w_host, h0, h1, pool_sub, sub)
            parity["ranks_identical"] = bool(same)
            parity["ok"] = bool(parity["rel_l2"] <= 1e-2 and parity["max_abs"] <= 5e-2 and same)
        del hid
    del w0_full, pool0_full
    torch.cuda.empty_cache()
    stream = torch.cuda.current_stream()

    # ---------------- measured refinement of the (searched) plan: coordinate moves of the memory
    # partition (+-8 / +-16 SMs) and the nano-batch token shares (+-1/8), kept while the measured
    # step time (max over ranks) improves by > 0.3 %; the network partition is held fixed
    refine_log = []
    if args.plan == "refine" and plan.spec().mode == nf.OVERLAP and not plan.spec().colocate:
        def run_steps(pl, n):
            for _ in range(n):
                model.step(pl, pools, nb, tok, ws, next_ids, comm=comm)

        def ab(cand, inc, pairs=3, n=2):
            """Median step-time ratio cand / incumbent over interleaved runs (the GPU's power
            state drifts between runs; interleaving cancels it); max over ranks."""
            run_steps(cand, 2)
            run_steps(inc, 2)
            tc, ti = [], []
            for _ in range(pairs):
                for pl, acc in ((cand, tc), (inc, ti)):
                    torch.cuda.synchronize()
                    if world > 1:
                        dist.barrier()
                    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a0.record(stream)
                    run_steps(pl, n)
                    a1.record(stream)
                    torch.cuda.synchronize()
                    t = torch.tensor([a0.elapsed_time(a1) / n], dtype=torch.float64, device=dev)
                    if world > 1:
                        dist.all_reduce(t, op=dist.ReduceOp.MAX)
                    acc.append(float(t.item()))
            return statistics.median(tc) / statistics.median(ti), statistics.median(tc)

        from paper_2408_12757_b200 import refine as R
        plan, refine_log = R.refine(cfg, plan, ab, tp)
    if world > 1:   # every rank must hold the same plan: same collectives in the same order
        hs = [None] * world
        dist.all_gather_object(hs, plan.hash())
        if len(set(hs)) != 1:
            raise SystemExit(f"plan hashes differ across ranks: {hs}")

    def step(pl=plan):
        model.step(pl, pools, nb, tok, ws, next_ids, comm=comm)

    # ---------------- timed region: the plan alone, no per-launch instrumentation
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = nf.kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    graph_launches = (nf.kernel_launches() - launches0) / args.steps
    ms = e0.elapsed_time(e1)
    t_max = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms_max = float(t_max.item())
    ms_step = ms_max / args.steps
    replicas = world // tp if not loop else 1.0 / tp           # independent model copies (1 under TP)
    value = replicas * T * args.steps / (ms_max / 1e3)

    # ---------------- per-op times: a separate instrumented pass (eager launches, CUDA events per kernel)
    prof_steps = max(2, min(args.steps, 5))
    nf.profile_enable(True)
    nf.profile_read()
    l0 = nf.kernel_launches()
    for _ in range(prof_steps):
        step()
    torch.cuda.synchronize()
    nf.profile_enable(False)
    kernels_per_step = (nf.kernel_launches() - l0) / prof_steps
    prof = nf.profile_read()
    if args.timeline:
        nf.profile_enable(True)
        nf.profile_read()
        step()
        torch.cuda.synchronize()
        spans = nf.profile_timeline()
        nf.profile_enable(False)
        nf.profile_read()
        with open(args.timeline if world == 1 else f"{args.timeline}.rank{rank}", "w") as f:
            f.write("op,stream,start_ms,end_ms\n")
            for sp in spans:
                f.write(f"{sp[0]},{sp[1]},{sp[2]:.4f},{sp[3]:.4f}\n")
    if args.ncu:
        return
    n_dec = int((b.q_len == 1).sum())
    kv_keys = sum(int(b.kv_prefix[r]) + 1 for r in range(b.n_req) if b.q_len[r] == 1)
    Hq_l, Hk_l, F_l = Hq // tp, Hk // tp, F // tp      # this rank's share under TP
    dec_bytes_step = L * (kv_keys * Hk_l * hd * 2 * 2 + n_dec * Hq_l * hd * 2 * 2)  # K+V read + q read + o write
    # ---------------- F7 ablation with the same kernels: sequential and nano-batch-only,
    # timed in interleaved rounds (seq, nano, timed mode, seq, ...) so that the GPU's power / thermal
    # state (1 kW cap) drifts equally over all of them; medians of the rounds.
    ablation = {}
    if not args.no_ablation:
        sp = plan.spec()
        nano_shares = tuple(sp.share[:sp.n_nano]) if sp.n_nano > 1 else (1, 1)
        plans = [("sequential", nf.Plan.explicit(cfg, nf.SEQUENTIAL, graph=not args.no_graph)),
                 ("nano_only", nf.Plan.explicit(cfg, nf.NANO_ONLY, shares=nano_shares, balance=args.balance,
                                                n_dense=sp.n_dense if tp > 1 else 0, graph=not args.no_graph)),
                 ("timed_mode", plan)]
        rounds = 3
        per_round = max(2, args.steps // 2)
        times = {n: [] for n, _ in plans}
        for _, pl in plans:
            for _ in range(2):
                step(pl)
        for _r in range(rounds):
            for name, pl in plans:
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                a0.record(stream)
                for _ in range(per_round):
                    step(pl)
                a1.record(stream)
                torch.cuda.synchronize()
                t_ab = torch.tensor([a0.elapsed_time(a1) / per_round], dtype=torch.float64, device=dev)
                if world > 1:
                    dist.all_reduce(t_ab, op=dist.ReduceOp.MAX)
                times[name].append(float(t_ab.item()))
        # per-op times of the sequential plan (instrumented, separate)
        nf.profile_enable(True)
        nf.profile_read()
        for _ in range(2):
            step(plans[0][1])
        torch.cuda.synchronize()
        nf.profile_enable(False)
        seq_prof = {k: v[0] / 2 for k, v in nf.profile_read().items() if v[1]}
        for name, _ in plans:
            ablation[name + "_ms_per_step"] = statistics.median(times[name])
            ablation[name + "_rounds_ms"] = times[name]
        ablation["sequential_per_op_ms"] = seq_prof
        ablation["timed_mode"] = args.mode
        ablation["interleaving"] = f"{rounds} rounds x {per_round} steps per plan, medians, max over ranks"
        ablation["speedup_vs_sequential"] = ablation["sequential_ms_per_step"] / ablation["timed_mode_ms_per_step"]
        ablation["overlap_beats_sequential_p90_p10"] = bool(max(times["timed_mode"]) < min(times["sequential"]))
        seq_dec = seq_prof.get("decode_attn")
        if seq_dec:
            ablation["sequential_decode_attn_hbm_gbs"] = dec_bytes_step / (seq_dec / 1e3) / 1e9
    # ---------------- end to end through the public API with host buffers
    tok_host = tok.cpu().pin_memory()
    ids_host = torch.empty(b.n_req, dtype=torch.int32).pin_memory()
    tok_dev2 = torch.empty_like(tok)
    for _ in range(2):
        tok_dev2.copy_(tok_host, non_blocking=True)
        model.step(plan, pools, nb, tok_dev2, ws, next_ids, comm=comm)
        ids_host.copy_(next_ids, non_blocking=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record(stream)
    for _ in range(args.steps):
        tok_dev2.copy_(tok_host, non_blocking=True)
        model.step(plan, pools, nb, tok_dev2, ws, next_ids, comm=comm)
        ids_host.copy_(next_ids, non_blocking=True)
        stream.synchronize()
    f1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_value = replicas * T * args.steps / (float(e2e_ms.item()) / 1e3)
    pf_items = sum(((int(q) + 63) // 64) * Hq_l for q in b.q_len if q > 1)
    meta_words = 3 * T + int(b.page_indptr[-1]) + 4 * n_dec * Hk_l + 8 * pf_items + 3 * b.n_req
    h2d = T * 4 + meta_words * 4
    d2h = b.n_req * 4

    if rank != 0:
        return

    # ---------------- roofline of the dominant kernel (per-op CUDA-event times of the instrumented pass)
    peaks, peak_src = load_peaks()
    qkv_n = (Hq_l + 2 * Hk_l) * hd
    rows_ffn = T * (shape.top_k if E else 1)          # MoE: top_k expert rows per token (padding excluded)
    flops = {"kqv": 2 * T * qkv_n * D * L, "o_proj": 2 * T * D * Hq_l * hd * L,
             "up_gate": 2 * rows_ffn * 2 * F_l * D * L, "down": 2 * rows_ffn * D * F_l * L,
             "lm_head": 2 * b.n_req * (shape.vocab // tp) * D}
    per_op = {k: {"ms_per_step": v[0] / prof_steps, "launches_per_step": v[1] / prof_steps}
              for k, v in prof.items() if v[1]}
    comp = {k: v for k, v in per_op.items() if k != "net"}
    dom = max(comp, key=lambda k: comp[k]["ms_per_step"])
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"{args.config}:{dom}") or json.load(open(tpath)).get(dom)
    if dom == "decode_attn":
        achieved = dec_bytes_step / (per_op[dom]["ms_per_step"] / 1e3) / 1e9
        roof = {"kernel": "decode_attn", "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": traffic, "peak_source": peak_src,
                "algorithmic": "K+V bytes of every decode request's context + q/o rows, per launch"}
    else:
        achieved = flops.get(dom, 0) / (per_op[dom]["ms_per_step"] / 1e3) / 1e12
        pk = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
        roof = {"kernel": dom, "bound": "tensor", "achieved": achieved, "peak": pk, "unit": "TFLOP/s",
                "frac": achieved / pk, "traffic": traffic, "peak_source": peak_src + " sustained",
                "algorithmic": "2*M*N*K per launch"}
    pf_flops = L * sum(4 * hd * Hq_l * (int(b.kv_prefix[r]) + i + 1)
                       for r in range(b.n_req) if b.q_len[r] > 1 for i in range(int(b.q_len[r])))
    flops["prefill_attn"] = pf_flops  # causal: each row attends to its prefix + itself
    for k in per_op:
        if k in flops:
            per_op[k]["tflops"] = flops[k] / (per_op[k]["ms_per_step"] / 1e3) / 1e12
    if "decode_attn" in per_op:
        per_op["decode_attn"]["hbm_gbs"] = dec_bytes_step / (per_op["decode_attn"]["ms_per_step"] / 1e3) / 1e9
    if "net" in per_op and tp > 1:
        # bytes this rank sends per step (ring): AG (N-1)/N of the gathered bytes, AR 2 (N-1)/N of the buffer
        half = T // 2
        qd_full = Hq * hd
        ag = (half * qd_full * 2 + half * D * 2) * (tp - 1) / tp
        ar = (half * D * 2 + T * D * 2) * 2 * (tp - 1) / tp
        per_op["net"]["bytes_per_step"] = L * (ag + ar)
        per_op["net"]["bus_gbs"] = L * (ag + ar) / (per_op["net"]["ms_per_step"] / 1e3) / 1e9
    pk_s = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    roof_all = {}
    for k, v in per_op.items():
        if k == "decode_attn":
            roof_all[k] = {"bound": "hbm", "achieved_gbs": v["hbm_gbs"], "frac": v["hbm_gbs"] / peaks["hbm_gbs"],
                           "sms": plan.spec().sm[1] if args.mode == "overlap" else 148}
        elif "tflops" in v:
            roof_all[k] = {"bound": "tensor", "achieved_tflops": v["tflops"], "frac": v["tflops"] / pk_s}
        elif k == "net" and "bus_gbs" in v:
            roof_all[k] = {"bound": "nvlink", "achieved_gbs": v["bus_gbs"], "frac": v["bus_gbs"] / 770.0,
                           "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction"}
    seq_dec = ablation.get("sequential_per_op_ms", {}).get("decode_attn")
    if seq_dec:
        gbs = dec_bytes_step / (seq_dec / 1e3) / 1e9
        roof_all["decode_attn_sequential_148sm"] = {"bound": "hbm", "achieved_gbs": gbs, "frac": gbs / peaks["hbm_gbs"]}

    optimal = peaks["bf16_tflops"] * 1e12 / (2 * p_active(shape))
    cfg_line = bench_config(args.config, shape, tp, T)
    if loop and args.net_model == "nvlink":
        cfg_line["net_model"] = (f"modeled: each loopback collective lasts >= ring bytes per GPU / {NVLINK_BUS_GBS:g} GB/s "
                                 f"(measured 8-rank all-reduce bus bandwidth at 1 GiB, B200_PROFILING.md); NVLink "
                                 f"itself not measured")
    plan_line = {"mode": args.mode, "colocate": bool(plan.spec().colocate),
                 "parallelism": (f"tp{tp}" if tp > 1 else ("replicas" if world > 1 else "single-gpu")),
                 "sm": list(plan.spec().sm), "shares": list(plan.spec().share)[:plan.spec().n_nano],
                 "n_dense": int(plan.spec().n_dense), "cuda_graph": bool(plan.spec().graph),
                 "source": {"explicit": "measured default", "auto": "nf_plan_create",
                            "refine": "nf_plan_create + measured refinement"}[args.plan],
                 "refinement": refine_log, "hash": f"{plan.hash():016x}", "partitions": plan.runtime_note()}
    if fused_note:
        timeouts, n_sites = nf.comm_sym_status(comm, with_sites=True)
        plan_line["collectives"] = {"allreduce": fused_note, "fused_sites_issued": n_sites,
                                    "peer_wait_timeouts": timeouts}
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if tp > 1 else "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, seeded torch RNG on device)",
            "config": cfg_line,
            "plan": plan_line,
            "tokens_per_s_per_gpu": value / world,
            "pct_of_optimal": 100.0 * (value / world) / optimal,
            "optimal_tokens_per_s_per_gpu": optimal,
            "gpu_launches": kernels_per_step,
            "gpu_launch_note": (f"{kernels_per_step:.0f} libnf kernels per step (instrumented pass); the timed "
                                f"region issued {graph_launches:.0f} libnf launch call(s) per step "
                                f"({'CUDA graph replay' if plan.spec().graph else 'eager'})"),
            "clocks": clk.summary(),
            "parity": parity,
            "roofline": roof,
            "roofline_by_kernel": roof_all,
            "per_op": per_op,
            "ablation": ablation,
            "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_full_layer(shape, b, p_in, d_out, args.cpu_tokens)
    print(json.dumps(line), flush=True)


def cpu_baseline_full_layer(shape, b, p_in, d_out, max_tokens):
    """The oracle as it stands, on the host cores: one float64 decoder layer of the
    benched workload -- the full B_dense batch when max_tokens >= B_dense,
    else the first requests of it up to max_tokens tokens -- x L layers."""
    import numpy as np
    import synth
    reqs, tok = [], 0
    for r in range(b.n_req):
        if tok + int(b.q_len[r]) > max_tokens:
            break
        reqs.append(r)
        tok += int(b.q_len[r])
    sub = synth.make_batch(b.q_len[reqs], b.kv_prefix[reqs], seed=3)
    w = synth.layer_weights(shape, 0, seed=0)
    x = synth.activations(shape, sub.n_tokens, seed=1)
    pool = synth.kv_pool(shape, sub, seed=2)
    ts = time_oracle_layer(shape, sub, w, x, pool, reps=1)
    t_step = ts[0] * shape.n_layers
    full = sub.n_tokens == b.n_tokens
    return {"value": sub.n_tokens / t_step, "unit": "tokens/s", "cores": blas_threads() or cpu_cores(), "kind": "oracle",
            "sample": (f"float64 oracle, one {shape.name} decoder layer over "
                       f"{'the full' if full else 'a'} {sub.n_tokens}-token batch "
                       f"({int((sub.q_len == 1).sum())} decode + {int((sub.q_len > 1).sum())} prefill requests of the "
                       f"benched steady state) in {ts[0]:.1f} s, x{shape.n_layers} layers")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="nf", choices=["nf", "reference"])
    ap.add_argument("--mode", default="auto", choices=["auto", "overlap", "nano", "sequential"],
                    help="auto: the measured-best plan kind per config (OVERLAP except the c3rank/c4rank proxies)")
    ap.add_argument("--plan", default="", choices=["", "explicit", "auto", "refine"],
                    help="auto: nf_plan_create autosearch over --curves (overlap mode); refine: the searched plan "
                         "(or the explicit default when no curves exist) refined by measured coordinate moves")
    ap.add_argument("--curves", default="profiles/curves_b200_quick.csv")
    ap.add_argument("--curves-tp", default="profiles/curves_b200_tp8.csv",
                    help="curves with NET points for the TP autosearch")
    ap.add_argument("--shares", default="", help="nano-batch token shares (overlap / nano modes; default per config)")
    ap.add_argument("--balance", type=int, default=2, help="0 request order, 1 balanced, 2 exact shares + KV")
    ap.add_argument("--colocate", action="store_true", help="attention CTAs co-resident with GEMM CTAs")
    ap.add_argument("--sm", default="", help="comma-separated SM budget per op kind (7 values)")
    ap.add_argument("--config", default="", choices=["", "c2", "c3", "c3rank", "c3loop", "c4", "c4rank"],
                    help="default: c2 at N=1, c3 at N>1.  c2: configs[1] 8B 1 GPU (replicas for N>1); c3: configs[2] "
                         "70B TP=N over NCCL (the metric's config); c3rank: 1-GPU proxy of one TP8 rank; "
                         "c4: configs[3] Mixtral-8x7B TP=N; c4rank: its 1-GPU TP8-rank proxy")
    ap.add_argument("--net-model", default="", choices=["", "nvlink"],
                    help="c3loop only: model the collectives' link time (ring bytes / 725 GB/s) on the loopback rank")
    ap.add_argument("--no-graph", action="store_true", help="eager launches instead of CUDA-graph replay")
    ap.add_argument("--fused-ar", action="store_true",
                    help="TP: fuse the row-parallel GEMMs with their AllReduce over peer memory (NEXT-3)")
    ap.add_argument("--no-parity", action="store_true", help="skip the in-run oracle parity check")
    ap.add_argument("--cpu-tokens", type=int, default=2048, help="tokens of the cpu_baseline oracle layer")
    ap.add_argument("--layers", type=int, default=0, help="(dev only) override layer count")
    ap.add_argument("--b-dense", type=int, default=0, help="(dev only) override the dense batch size (tokens)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ablation", action="store_true", help="skip the sequential / nano-only comparison runs")
    ap.add_argument("--timeline", default="", help="write one step's kernel spans (CSV) to this path (per rank at N>1)")
    ap.add_argument("--ncu", action="store_true", help="profiling run: timed steps only, no e2e / JSON")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if not args.config:
        args.config = "c2" if world == 1 else "c3"   # N > 1: the metric's configs[2] (70B TP=N), never replicas
    if not args.plan:   # TP on a multi-GPU box: the default plan refined by measurement on that box
        args.plan = "refine" if (world > 1 and args.config in ("c3", "c4")) else "explicit"
    if world > 1:   # NCCL's init log (ranks, nranks, channels, NVLS) for the run's record
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ["NCCL_DEBUG_SUBSYS"] = "INIT"
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_nf(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
