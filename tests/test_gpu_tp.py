"""Tensor-parallel executor on one GPU through an emulated communicator
(nf_comm_create_local: N ranks = N host threads; same executor code path as
NCCL, collectives replaced by stream-ordered copies and a rank-order sum).
Checks TP=2/4 layer outputs against the unsharded oracle (T10/T15) and that
every rank holds bit-identical hidden states (T16)."""
import threading

import numpy as np
import pytest
import torch

import synth
from oracle import layer as OL

from gpu_common import assert_close, dev, device_weights, host, require_gpu

pytestmark = pytest.mark.gpu


def _run_tp_layer(nf, rt, shape, b, w, x, pool, tp, mode, shares):
    comms = nf.comm_create_local(tp)
    outs = [None] * tp
    errs = []
    wd = device_weights(w)
    pool_d = dev(pool)
    x_d = dev(x)

    def rank_main(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                cfg = rt.cfg_from_shape(shape, tp_size=tp, tp_rank=r)
                shard = rt.shard_layer(wd, shape.n_q_heads, shape.n_kv_heads, shape.head_dim, tp, r)
                packed = rt.pack_layer(cfg, shard, stream=int(st.cuda_stream))
                p_r = rt.shard_pool(pool_d, tp, r)
                nb = nf.Batch.from_any(b)
                plan = nf.Plan.explicit(cfg, mode=mode, shares=shares, sm=[148] * 7)
                ws = rt.workspace(cfg, nb)
                y = torch.empty_like(x_d)
                nf.layer_forward(plan, rt.ptrs(packed), p_r.data_ptr(), nb, x_d.data_ptr(), y.data_ptr(),
                                 ws.data_ptr(), ws.numel(), int(st.cuda_stream), comm=comms[r])
                st.synchronize()
                outs[r] = y
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(tp)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for c in comms:
        nf.comm_destroy(c)
    assert not errs, errs
    return outs


@pytest.mark.parametrize("tp,mode,shares", [(2, 0, (1,)), (2, 2, (1, 1)), (4, 1, (1, 1)), (4, 2, (2, 1, 1))])
def test_tp_layer_matches_unsharded_oracle(tp, mode, shares):
    nf, rt = require_gpu()
    shape = synth.shape_with(synth.SHAPES["c1"], n_kv_heads=4, d_ffn=1408)
    b = synth.make_batch([1] * 20 + [37, 1, 16], list(range(5, 205, 10)) + [0, 130, 33], seed=4, pool_slack=3)
    w = synth.layer_weights(shape, 0)
    x = synth.activations(shape, b.n_tokens)
    pool = synth.kv_pool(shape, b)
    ref = OL.decoder_layer(x, w, OL.as_pool(pool), b, shape)
    outs = _run_tp_layer(nf, rt, shape, b, w, x, pool, tp, mode, shares)
    for r in range(1, tp):
        assert torch.equal(outs[0], outs[r]), f"rank {r} differs from rank 0 (T16)"
    assert_close(host(outs[0]), ref, what=f"TP{tp} mode={mode}")


def test_tp2_8b_shape():
    nf, rt = require_gpu()
    shape = synth.SHAPES["llama3-8b"]
    b = synth.make_batch([1] * 10 + [100, 1, 37], [1024, 5, 1535, 16, 1, 900, 64, 700, 33, 1200, 341, 2, 0],
                         seed=3, pool_slack=2)
    w = synth.layer_weights(shape, 0)
    x = synth.activations(shape, b.n_tokens)
    pool = synth.kv_pool(shape, b)
    ref = OL.decoder_layer(x, w, OL.as_pool(pool), b, shape)
    outs = _run_tp_layer(nf, rt, shape, b, w, x, pool, 2, 2, (1, 1))
    assert torch.equal(outs[0], outs[1])
    assert_close(host(outs[0]), ref, what="TP2 8B shape")


def test_tp_model_step_matches_oracle():
    """Embedding -> 2 TP layers (emulated TP=2, OVERLAP) -> replicated LM head + argmax."""
    nf, rt = require_gpu()
    shape = synth.shape_with(synth.SHAPES["c1"], n_kv_heads=4, d_ffn=1408, n_layers=2, vocab=4096)
    b = synth.make_batch([1] * 20 + [30, 1, 12], list(range(10, 210, 10)) + [0, 33, 7], seed=6, pool_slack=4)
    W = synth.model_weights(shape, seed=0)
    toks = synth.token_ids(b.n_tokens, shape.vocab)
    pools = [synth.kv_pool(shape, b, seed=2, layer=l) for l in range(2)]
    ids_ref, logits, _ = OL.model_step(toks, W, [OL.as_pool(p) for p in pools], b, shape, return_logits=True)
    tp = 2
    comms = nf.comm_create_local(tp)
    outs, errs = [None] * tp, []
    embed, lm, fn = dev(W["embed"]), dev(W["lm_head"]), dev(W["final_norm"])
    lw = [device_weights(W["layers"][l]) for l in range(2)]
    pools_d = [dev(p) for p in pools]
    tok_d = torch.from_numpy(toks).cuda()

    def rank_main(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                cfg = rt.cfg_from_shape(shape, tp_size=tp, tp_rank=r)
                layers = [rt.pack_layer(cfg, rt.shard_layer(lw[l], shape.n_q_heads, shape.n_kv_heads, shape.head_dim,
                                                            tp, r), stream=int(st.cuda_stream)) for l in range(2)]
                model = rt.Model(cfg, embed, layers, rt.pack_lm_head(cfg, lm, fn))
                nb = nf.Batch.from_any(b)
                ws = rt.workspace(cfg, nb)
                plan = nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1), sm=[148] * 7, balance=True)
                ids = model.step(plan, [rt.shard_pool(p, tp, r) for p in pools_d], nb, tok_d, ws, comm=comms[r])
                st.synchronize()
                outs[r] = ids.cpu().numpy()
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(tp)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for c in comms:
        nf.comm_destroy(c)
    assert not errs, errs
    assert np.array_equal(outs[0], outs[1])
    srt = np.sort(logits, axis=1)
    sure = (srt[:, -1] - srt[:, -2]) > 0.1
    assert sure.sum() >= len(sure) // 2
    assert np.array_equal(outs[0][sure], ids_ref[sure])


@pytest.mark.parametrize("tp", [2, 4, 8])
def test_tp_70b_layer_vs_oracle(tp):
    """T15: one LLaMA-2-70B-shape layer (D 8192, 64/8 heads, F 28672) at TP 2 / 4 / 8
    on the C3 steady-state mix (p=512, d=1024) scaled to B_dense 256, vs the
    unsharded float64 oracle."""
    nf, rt = require_gpu()
    shape = synth.SHAPES["llama2-70b"]
    b = synth.workload_batch(256, 512, 1024, pool_slack=3)
    w = synth.layer_weights(shape, 0)
    x = synth.activations(shape, b.n_tokens)
    pool = synth.kv_pool(shape, b)
    ref = OL.decoder_layer(x, w, OL.as_pool(pool), b, shape)
    outs = _run_tp_layer(nf, rt, shape, b, w, x, pool, tp, 2, (1, 1))
    for r in range(1, tp):
        assert torch.equal(outs[0], outs[r])
    assert_close(host(outs[0]), ref, what=f"70B TP{tp}")
