"""End-to-end offline serving loop on the GPU: the
native scheduler (nf_sched_*), nf_assemble_tokens and nf_model_step driven
by paper_2408_12757_b200.serving.OfflineServer with the asynchronous
one-step-late EOS protocol.  Every step is replayed on
the float64 oracle with the same batches (page tables reused across steps
as the scheduler allocates them) and teacher-forced tokens; sampled ids must
agree wherever the oracle's top-2 logit gap exceeds 0.1 (A-15)."""
import numpy as np
import pytest
import torch

import synth
from oracle import layer as OL

from gpu_common import dev, device_weights, require_gpu

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode,shares", [(0, (1,)), (2, (1, 1))])
def test_offline_serving_matches_oracle(mode, shares):
    nf, rt = require_gpu()
    from paper_2408_12757_b200.serving import OfflineServer
    shape = synth.shape_with(synth.SHAPES["c1"], n_layers=2, vocab=4096)
    n_pages = 48
    W = synth.model_weights(shape, seed=0)
    cfg = rt.cfg_from_shape(shape)
    layers = [rt.pack_layer(cfg, device_weights(W["layers"][l])) for l in range(shape.n_layers)]
    model = rt.Model(cfg, dev(W["embed"]), layers, rt.pack_lm_head(cfg, dev(W["lm_head"]), dev(W["final_norm"])))
    pools = [torch.zeros((n_pages, 2, shape.n_kv_heads, 16, shape.head_dim), dtype=torch.bfloat16, device="cuda")
             for _ in range(shape.n_layers)]
    rng = np.random.default_rng(1)
    lens = [(40, 5), (7, 3), (64, 8), (1, 4), (23, 2), (90, 6), (16, 9), (33, 1)]
    prompts = {i: rng.integers(0, shape.vocab, size=p).astype(np.int32) for i, (p, _) in enumerate(lens)}
    sched = nf.Scheduler(n_pages, 16, [64, 32], 4)
    for i, (p, o) in enumerate(lens):
        sched.submit(i, prompts[i], o)
    plan = nf.Plan.explicit(cfg, mode=mode, shares=shares)
    steps = []
    srv = OfflineServer(model, plan, pools, sched, n_pages, max_tokens=256, max_reqs=64)
    stats = srv.run(on_step=lambda st, ids: steps.append((st, ids)))
    assert stats["finished"] == len(lens) and stats["useless"] == len(lens)
    assert stats["generated"] == sum(o + 1 for _, o in lens)
    # replay on the oracle, teacher-forced with the GPU's tokens
    opools = [np.zeros((n_pages, 2, shape.n_kv_heads, 16, shape.head_dim)) for _ in range(shape.n_layers)]
    prev_ids = None
    checked = agreed = 0
    for st, ids in steps:
        src = st["tok_src"]
        toks = np.where(src >= 0, src, prev_ids[np.maximum(-(1 + src), 0)] if prev_ids is not None else 0)
        b = synth.Batch(st["q_len"], st["kv_prefix"], st["page_indptr"], st["page_ids"], n_pages)
        ref, logits, _ = OL.model_step(toks, W, opools, b, shape, emit=st["emit"], return_logits=True)
        em = st["emit"] != 0
        assert np.array_equal(ids[~em], np.full((~em).sum(), -1))
        srt = np.sort(logits, axis=1)
        sure = srt[:, -1] - srt[:, -2] > 0.1
        checked += int(sure.sum())
        agreed += int((ids[em][sure] == ref[em][sure]).sum())
        assert np.array_equal(ids[em][sure], ref[em][sure]), st["step"]
        prev_ids = ids
    assert checked >= stats["generated"] // 2
