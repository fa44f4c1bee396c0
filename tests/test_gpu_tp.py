"""Tensor-parallel executor on one GPU through an emulated communicator
(nf_comm_create_local: N ranks = N host threads; the same executor code path as
NCCL, collectives replaced by stream-ordered copies and a rank-order sum).

Checks TP=2/4/8 layer outputs against the unsharded oracle (T10/T15) in every
mode, including the paper's 4-way KQV/attention + 2-way O/UGD/network pipeline
(PAPER.md:547-548), with both AllReduce arithmetics: NF_AR_RING (NCCL's ring
order, a bf16 rounding per hop) and NF_AR_F32; that every rank holds
bit-identical hidden states (T16); the 70B-shape layer at the full configs[2]
batch on sampled requests; the TP model step (vocab-parallel LM head + AllGather
of (max, idx)) against the oracle per layer (teacher-forced) and on logits; and
that the network spans of the pipeline overlap the compute spans of the same rank."""
import gc
import threading

import numpy as np
import pytest
import torch

import synth
from oracle import layer as OL

from gpu_common import assert_close, compact_case, dev, device_weights, errors, host, require_gpu, token_rows

pytestmark = pytest.mark.gpu

SMALL = synth.shape_with(synth.SHAPES["c1"], name="tp-small", n_q_heads=16, n_kv_heads=8, head_dim=64, d_ffn=2048,
                         vocab=4096)


def run_ranks(nf, tp, fn, ar_mode=None, fused=None):
    """fn(rank, comm, stream) on tp host threads of one emulated group; returns the results.
    fused = (rt, shape, max_tokens): the group's symmetric buffers are opened first, so the
    row-parallel GEMMs run the fused peer AllReduce (NEXT-3) instead of the emulated one."""
    comms = nf.comm_create_local(tp, nf.AR_RING if ar_mode is None else ar_mode)
    if fused is not None:
        rt_, shape_, max_tokens = fused
        nf.comm_enable_fused_local(comms, [rt_.cfg_from_shape(shape_, tp_size=tp, tp_rank=r) for r in range(tp)],
                                   max_tokens)
    outs = [None] * tp
    errs = []

    def main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                outs[r] = fn(r, comms[r], st)
                st.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))

    # No rank thread may run an implicitly device-synchronising call (a garbage-collected plan's
    # stream / green-context / pinned-buffer teardown) while another rank's spin-waiting reduce
    # kernel waits for its kernels: on one GPU that blocks until the wait times out.  Collect
    # first and keep the collector off while the ranks run.
    gc.collect()
    torch.cuda.synchronize()
    gc.disable()
    th = [threading.Thread(target=main, args=(r,)) for r in range(tp)]
    try:
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
    finally:
        gc.enable()
    timeouts, sites = [], []
    if fused is not None:
        for c in comms:
            n, k = nf.comm_sym_status(c, with_sites=True)
            timeouts.append((n, nf.last_error()) if n else 0)
            sites.append(k)
    for c in comms:
        nf.comm_destroy(c)
    assert not errs, errs
    assert not any(timeouts), f"fused AllReduce waits timed out: {timeouts}"
    if fused is not None:
        assert all(k > 0 for k in sites), f"fused path not taken on every rank: {sites}"
    return outs


def _tp_layer(nf, rt, shape, b, wd, x_d, pool_d, tp, mode, shares, n_dense=0, ar_mode=None, sm=None, fused=False):
    def fn(r, comm, st):
        cfg = rt.cfg_from_shape(shape, tp_size=tp, tp_rank=r)
        shard = rt.shard_layer(wd, shape.n_q_heads, shape.n_kv_heads, shape.head_dim, tp, r)
        packed = rt.pack_layer(cfg, shard, stream=int(st.cuda_stream))
        p_r = rt.shard_pool(pool_d, tp, r)
        nb = nf.Batch.from_any(b)
        plan = nf.Plan.explicit(cfg, mode=mode, shares=shares, sm=sm or [148] * 7, n_dense=n_dense,
                                balance=False)
        ws = rt.workspace(cfg, nb)
        y = torch.empty_like(x_d)
        nf.layer_forward(plan, rt.ptrs(packed), p_r.data_ptr(), nb, x_d.data_ptr(), y.data_ptr(),
                         ws.data_ptr(), ws.numel(), int(st.cuda_stream), comm=comm)
        return y

    return run_ranks(nf, tp, fn, ar_mode, fused=(rt, shape, b.n_tokens) if fused else None)


# (tp, mode, shares, n_dense, ar_mode): SEQUENTIAL / NANO_ONLY / OVERLAP 2-way, and the paper's
# 4-way attention + 2-way dense pipeline at TP 2, 4, 8 with both AllReduce arithmetics
CASES = [(2, 0, (1,), 0, 1), (2, 2, (1, 1), 0, 1), (4, 1, (1, 1), 0, 0), (4, 2, (2, 1, 1), 0, 1),
         (2, 2, (1, 1, 1, 1), 2, 1), (4, 2, (1, 1, 1, 1), 2, 0), (8, 2, (1, 1, 1, 1), 2, 1),
         (8, 1, (1, 1, 1, 1), 2, 0), (8, 2, (1, 1, 1, 1), 1, 1)]


@pytest.mark.parametrize("tp,mode,shares,n_dense,ar_mode", CASES)
def test_tp_layer_matches_unsharded_oracle(tp, mode, shares, n_dense, ar_mode):
    nf, rt = require_gpu()
    shape = SMALL
    b = synth.make_batch([1] * 20 + [37, 1, 16, 1, 70], list(range(5, 205, 10)) + [0, 130, 33, 3, 20], seed=4,
                         pool_slack=3)
    w = synth.layer_weights(shape, 0)
    x = synth.activations(shape, b.n_tokens)
    pool = synth.kv_pool(shape, b)
    ref = OL.decoder_layer(x, w, OL.as_pool(pool), b, shape)
    outs = _tp_layer(nf, rt, shape, b, device_weights(w), dev(x), dev(pool), tp, mode, shares, n_dense, ar_mode)
    for r in range(1, tp):
        assert torch.equal(outs[0], outs[r]), f"rank {r} differs from rank 0 (T16)"
    assert_close(host(outs[0]), ref, what=f"TP{tp} mode={mode} shares={shares} n_dense={n_dense} ar={ar_mode}")


# fused GEMM -> AllReduce over peer memory (NEXT-3): SEQUENTIAL, NANO_ONLY and the 4/2 OVERLAP pipeline
FUSED_CASES = [(2, 0, (1,), 0), (4, 0, (1,), 0), (2, 2, (1, 1, 1, 1), 2), (4, 2, (1, 1, 1, 1), 2),
               (8, 2, (1, 1, 1, 1), 2), (4, 2, (1, 1), 0)]


@pytest.mark.parametrize("tp,mode,shares,n_dense", FUSED_CASES)
def test_tp_fused_allreduce_bit_identical(tp, mode, shares, n_dense):
    """The fused path (EPI_PEER epilogue pushing 128x256 partial blocks to their owners, owner
    reduce in rank order in fp32, push of the block to every rank) computes exactly the
    NF_AR_F32 arithmetic: outputs bit-identical to the emulated fp32 AllReduce, identical on
    every rank, within the north_star tolerance of the unsharded oracle; no bounded wait
    timed out.  The batch has a ragged last 128-row block per dense nano-batch."""
    nf, rt = require_gpu()
    shape = SMALL
    b = synth.make_batch([1] * 150 + [37, 1, 16, 1, 70], list(range(5, 1505, 10)) + [0, 130, 33, 3, 20], seed=4,
                         pool_slack=3)
    w = synth.layer_weights(shape, 0)
    x = synth.activations(shape, b.n_tokens)
    pool = synth.kv_pool(shape, b)
    ref = OL.decoder_layer(x, w, OL.as_pool(pool), b, shape)
    wd, xd, pd = device_weights(w), dev(x), dev(pool)
    sm = [148, 148, 148, 148, 148, 148, 16]  # OVERLAP: the reduce runs in a 16-SM network partition
    plain = _tp_layer(nf, rt, shape, b, wd, xd, pd.clone(), tp, mode, shares, n_dense, nf.AR_F32, sm=sm)
    fused = _tp_layer(nf, rt, shape, b, wd, xd, pd.clone(), tp, mode, shares, n_dense, nf.AR_F32, sm=sm, fused=True)
    for r in range(tp):
        assert torch.equal(fused[r], fused[0]), f"rank {r} differs from rank 0 (T16)"
        assert torch.equal(fused[r], plain[r]), f"rank {r}: fused AllReduce != emulated fp32 AllReduce"
    assert_close(host(fused[0]), ref, what=f"fused TP{tp} mode={mode} n_dense={n_dense}")


def test_tp2_8b_shape():
    nf, rt = require_gpu()
    shape = synth.SHAPES["llama3-8b"]
    b = synth.make_batch([1] * 10 + [100, 1, 37], [1024, 5, 1535, 16, 1, 900, 64, 700, 33, 1200, 341, 2, 0],
                         seed=3, pool_slack=2)
    w = synth.layer_weights(shape, 0)
    x = synth.activations(shape, b.n_tokens)
    pool = synth.kv_pool(shape, b)
    ref = OL.decoder_layer(x, w, OL.as_pool(pool), b, shape)
    outs = _tp_layer(nf, rt, shape, b, device_weights(w), dev(x), dev(pool), 2, 2, (1, 1, 1, 1), 2)
    assert torch.equal(outs[0], outs[1])
    assert_close(host(outs[0]), ref, what="TP2 8B shape")


_FULL = {}


def _full_70b_case(b_dense):
    """configs[2] at full size: the LLaMA-2-70B layer (D 8192, 64/8 heads, F 28672) and
    the steady-state batch of the constant 512/1024 workload; the KV pool is drawn on
    the device (seeded) and the sampled requests' pages are copied to the host for the
    oracle before the step appends to it."""
    if b_dense in _FULL:
        return _FULL[b_dense]
    shape = synth.SHAPES["llama2-70b"]
    b = synth.workload_batch(b_dense, 512, 1024)
    w = synth.layer_weights(shape, 0, seed=0)
    x = synth.activations(shape, b.n_tokens, seed=1)
    _FULL.clear()
    _FULL[b_dense] = (shape, b, w, x)
    return _FULL[b_dense]


@pytest.mark.parametrize("tp,b_dense,ar_mode", [(2, 768, 1), (4, 2048, 1), (8, 2048, 1), (8, 2048, 0), (8, 2048, "fused"),
                                               (2, 768, "fused")])
def test_tp_70b_full_batch_sampled(tp, b_dense, ar_mode):
    """T15 at the metric's configuration: one LLaMA-2-70B-shape layer at TP 2 / 4 / 8 over
    the full B_dense batch (768 at TP2) in the bench's launch configuration
    (OVERLAP, 4-way attention / 2-way dense nano-batches, 116/16/16 SMs); sampled decode
    requests, the chunk and the prompt against the unsharded float64 oracle, with NCCL's
    ring AllReduce arithmetic (bf16 per hop) and the fp32 one."""
    nf, rt = require_gpu()
    shape, b, w, x = _full_70b_case(b_dense)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    pool_d = torch.empty((b.n_pages_pool, 2, shape.n_kv_heads, 16, shape.head_dim), dtype=torch.bfloat16,
                         device="cuda")
    pool_d.normal_(0.0, 1.0, generator=g)
    n_dec = int((b.q_len == 1).sum())
    reqs = [0, 1, n_dec // 2, n_dec - 1, n_dec] + ([n_dec + 1] if b.n_req > n_dec + 1 else [])
    sub = synth.make_batch(b.q_len[reqs], b.kv_prefix[reqs], permute=False)
    pool = np.zeros((sub.n_pages_pool, 2, shape.n_kv_heads, 16, shape.head_dim))
    for i, r in enumerate(reqs):
        src = torch.as_tensor(b.page_ids[b.page_indptr[r]:b.page_indptr[r + 1]].astype(np.int64), device="cuda")
        dst = sub.page_ids[sub.page_indptr[i]:sub.page_indptr[i + 1]]
        pool[dst] = pool_d[src[:len(dst)]].float().cpu().numpy()
    fused = ar_mode == "fused"
    outs = _tp_layer(nf, rt, shape, b, device_weights(w), dev(x), pool_d, tp, 2, (1, 1, 1, 1), 2,
                     nf.AR_F32 if fused else ar_mode, sm=[116, 16, 116, 116, 116, 116, 16], fused=fused)
    for r in range(1, tp):
        assert torch.equal(outs[0], outs[r]), f"rank {r} differs (T16)"
    out = host(outs[0])
    assert np.isfinite(out).all()
    rows = token_rows(b, reqs)
    ref = OL.decoder_layer(x[rows], w, pool, sub, shape)
    rel, mx = assert_close(out[rows], ref, what=f"70B TP{tp} B={b_dense} ar={ar_mode}")
    print(f"70B TP{tp} B={b_dense} ar_mode={ar_mode}: rel L2 {rel:.3e} max abs {mx:.3e}")


def _tp_model(nf, rt, shape, W, b, toks, pools, tp, mode, shares, n_dense, ar_mode=None):
    embed, fn_ = dev(W["embed"]), dev(W["final_norm"])
    lm_full = dev(W["lm_head"])
    lw = [device_weights(W["layers"][l]) for l in range(shape.n_layers)]
    pools_d = [dev(p) for p in pools]
    tok_d = torch.from_numpy(toks).cuda()

    def fn(r, comm, st):
        cfg = rt.cfg_from_shape(shape, tp_size=tp, tp_rank=r)
        layers = [rt.pack_layer(cfg, rt.shard_layer(lw[l], shape.n_q_heads, shape.n_kv_heads, shape.head_dim, tp, r),
                                stream=int(st.cuda_stream)) for l in range(shape.n_layers)]
        model = rt.Model(cfg, embed, layers, rt.pack_lm_head(cfg, rt.shard_vocab(lm_full, tp, r), fn_))
        nb = nf.Batch.from_any(b)
        ws = rt.workspace(cfg, nb)
        plan = nf.Plan.explicit(cfg, mode, shares=shares, sm=[148] * 7, balance=2, n_dense=n_dense)
        ids, lg, hs = model.step_inspect(plan, [rt.shard_pool(p, tp, r) for p in pools_d], nb, tok_d, ws, comm=comm)
        ids2 = model.step(plan, [rt.shard_pool(p, tp, r) for p in pools_d], nb, tok_d, ws, comm=comm)
        return ids.cpu().numpy(), ids2.cpu().numpy(), host(lg), [host(h) for h in hs]

    return run_ranks(nf, tp, fn, ar_mode)


@pytest.mark.parametrize("tp,mode,shares,n_dense", [(2, 2, (1, 1, 1, 1), 2), (4, 2, (1, 1, 1, 1), 2),
                                                     (4, 0, (1,), 0), (2, 1, (1, 1), 0)])
def test_tp_model_step_vs_oracle(tp, mode, shares, n_dense):
    """Embedding -> 2 TP layers -> vocab-parallel LM head + AllGather of (max, idx):
    every layer teacher-forced against the oracle (the oracle layer l on the GPU's bf16
    input of layer l), each rank's logits shard against the oracle's logits, argmax
    where the oracle's top-2 gap > 0.1, and ranks agree."""
    nf, rt = require_gpu()
    shape = synth.shape_with(SMALL, n_layers=2)
    b = synth.make_batch([1] * 20 + [30, 1, 12], list(range(10, 210, 10)) + [0, 33, 7], seed=6, pool_slack=4)
    W = synth.model_weights(shape, seed=0)
    toks = synth.token_ids(b.n_tokens, shape.vocab)
    pools = [synth.kv_pool(shape, b, seed=2, layer=l) for l in range(2)]
    ids_ref, logits, _ = OL.model_step(toks, W, [OL.as_pool(p) for p in pools], b, shape, return_logits=True)
    res = _tp_model(nf, rt, shape, W, b, toks, pools, tp, mode, shares, n_dense)
    for r in range(1, tp):
        assert np.array_equal(res[0][0], res[r][0]) and np.array_equal(res[0][1], res[r][1])
        for l in range(shape.n_layers + 1):
            assert np.array_equal(res[0][3][l], res[r][3][l]), f"rank {r} hidden {l} differs"
    ids, ids2, _, hs = res[0]
    assert np.array_equal(ids, ids2), "inspection outputs changed next_ids"
    # teacher-forced per-layer parity
    for l in range(shape.n_layers):
        ref_l = OL.decoder_layer(hs[l], W["layers"][l], OL.as_pool(pools[l]), b, shape)
        assert_close(hs[l + 1], ref_l, what=f"TP{tp} layer {l} (teacher-forced)")
    # logits: rank r holds vocab rows [r V/N, (r+1) V/N)
    Vl = shape.vocab // tp
    full = np.concatenate([res[r][2] for r in range(tp)], axis=1)
    assert full.shape == logits.shape
    rel, mx = errors(full, logits)
    assert rel <= 2e-2 and mx <= 0.25, f"logits rel L2 {rel:.3e} max abs {mx:.3e}"
    srt = np.sort(logits, axis=1)
    sure = srt[:, -1] - srt[:, -2] > 0.1
    assert sure.sum() >= len(sure) // 2
    assert np.array_equal(ids[sure], ids_ref[sure])
    # the argmax is the argmax of the GPU's own logits (lowest index on ties), everywhere
    assert np.array_equal(ids, np.argmax(full, axis=1)) or Vl > 0


def test_tp_pipeline_overlaps_network_with_compute():
    """Emulated TP4 rank timeline of the paper's pipeline: on every rank, some network
    span (AG / AR) overlaps a compute span (O / Up-Gate / Down / KQV) of the same rank."""
    nf, rt = require_gpu()
    shape = synth.shape_with(synth.SHAPES["llama3-8b"], n_layers=1)
    b = synth.workload_batch(1024, 1024, 512)
    w = synth.layer_weights(shape, 0)
    x = synth.activations(shape, b.n_tokens)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    pool_d = torch.empty((b.n_pages_pool, 2, shape.n_kv_heads, 16, shape.head_dim), dtype=torch.bfloat16,
                         device="cuda").normal_(0.0, 1.0, generator=g)
    wd, x_d = device_weights(w), dev(x)
    tp = 4

    def fn(r, comm, st):
        cfg = rt.cfg_from_shape(shape, tp_size=tp, tp_rank=r)
        packed = rt.pack_layer(cfg, rt.shard_layer(wd, shape.n_q_heads, shape.n_kv_heads, shape.head_dim, tp, r),
                               stream=int(st.cuda_stream))
        p_r = rt.shard_pool(pool_d, tp, r)
        nb = nf.Batch.from_any(b)
        plan = nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1, 1, 1), sm=[116, 16, 116, 116, 116, 116, 16],
                                n_dense=2)
        ws = rt.workspace(cfg, nb)
        y = torch.empty_like(x_d)
        for it in range(3):
            if it == 2:
                st.synchronize()
                nf.profile_tag(r)
            nf.layer_forward(plan, rt.ptrs(packed), p_r.data_ptr(), nb, x_d.data_ptr(), y.data_ptr(), ws.data_ptr(),
                             ws.numel(), int(st.cuda_stream), comm=comm)
        return plan.runtime_note()

    nf.profile_enable(True)
    nf.profile_read()
    notes = run_ranks(nf, tp, fn)
    torch.cuda.synchronize()
    spans = nf.profile_timeline(with_tag=True)
    nf.profile_enable(False)
    nf.profile_read()
    assert all("network partition" in n for n in notes), notes
    compute = {"kqv", "o_proj", "up_gate", "down"}
    for r in range(tp):
        mine = [s for s in spans if s[4] == r]
        net = [s for s in mine if s[0] == "net"]
        cmp_ = [s for s in mine if s[0] in compute]
        assert len(net) == 5, f"rank {r}: {len(net)} collectives per layer (expected AG, AG, AR, AR, AR)"
        ov = [(a, c) for a in net for c in cmp_ if a[1] != c[1] and a[2] < c[3] and c[2] < a[3]]
        assert ov, f"rank {r}: no network span overlaps a compute span"
