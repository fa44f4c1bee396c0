"""Pins of the MoE FFN oracle (oracle/moe.py, readings A-20..A-23).
CPU only.  Each pin is fixed by something other than the oracle itself:
reduction to the (independently pinned) dense layer, library routines
(torch.softmax / torch.topk), closed forms, invariances and brute force."""
import numpy as np
import pytest
import torch

import synth
from oracle import layer as L
from oracle import moe as M

SH = synth.shape_with(synth.SHAPES["c1-moe"], d_model=64, n_q_heads=8, n_kv_heads=4, head_dim=16, d_ffn=48,
                      n_experts=6, top_k=2)


def _h1(shape, T, seed=1):
    return synth.activations(shape, T, seed=seed, name="h1").astype(np.float64)


def test_single_expert_top1_is_dense_ffn():
    """E = 1, k = 1: the gate weight is exactly 1 and the layer is the dense
    decoder layer of oracle.layer (pinned by tests/test_oracle_layer.py)."""
    sh = synth.shape_with(SH, n_experts=1, top_k=1)
    b = synth.make_batch([1, 1, 5], [7, 20, 0], seed=3, pool_slack=2)
    w = synth.layer_weights(sh, 0)
    dense = {k: v for k, v in w.items() if k != "w_router"}
    dense.update(w_gate=w["w_gate"][0], w_up=w["w_up"][0], w_down=w["w_down"][0])
    x = synth.activations(sh, b.n_tokens)
    p1 = L.as_pool(synth.kv_pool(sh, b))
    p2 = p1.copy()
    out = M.moe_decoder_layer(x, w, p1, b, sh)
    ref = L.decoder_layer(x, dense, p2, b, sh)
    np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_identical_experts_equal_dense(k):
    """All experts equal: the renormalised weights sum to 1, so any routing
    gives the dense FFN h1 + y(h2)."""
    sh = synth.shape_with(SH, top_k=k)
    w = synth.layer_weights(sh, 0)
    for name in ("w_gate", "w_up", "w_down"):
        w[name] = np.repeat(w[name][:1], sh.n_experts, axis=0)
    h1 = _h1(sh, 37)
    h2 = L.rmsnorm(h1, w["ffn_norm"], sh.rms_eps)
    ref = h1 + M.expert_ffn(h2, w["w_gate"][0], w["w_up"][0], w["w_down"][0])
    np.testing.assert_allclose(M.moe_ffn(h1, w, sh), ref, rtol=0, atol=1e-12)


def test_router_matches_library_softmax_topk():
    """Mixtral's gating: softmax over all E logits (torch.softmax), top-k
    (torch.topk), renormalised — equals the oracle's softmax over the
    selected logits; ids and weights sorted descending."""
    sh = synth.shape_with(SH, n_experts=8, top_k=2)
    w = synth.layer_weights(sh, 0)
    h2 = _h1(sh, 200, seed=7)
    ids, wts, logits = M.router_topk(h2, w["w_router"], 2)
    lt = torch.tensor(h2) @ torch.tensor(w["w_router"], dtype=torch.float64).T
    probs = torch.softmax(lt, dim=-1)
    tv, ti = torch.topk(probs, 2, dim=-1)
    assert np.array_equal(ids, ti.numpy())
    np.testing.assert_allclose(wts, (tv / tv.sum(-1, keepdim=True)).numpy(), rtol=1e-13, atol=0)
    np.testing.assert_allclose(wts.sum(1), 1.0, rtol=0, atol=1e-15)
    assert (wts[:, 0] >= wts[:, 1]).all()


def test_router_ties_lowest_index():
    """Equal logits order by lower expert index (reading A-21)."""
    E, D = 5, 4
    wr = np.zeros((E, D))
    wr[1, 0] = wr[3, 0] = 1.0       # experts 1 and 3 tie at the top
    wr[4, 0] = 0.5
    h2 = np.array([[2.0, 0, 0, 0], [0.0, 0, 0, 0]])
    ids, wts, _ = M.router_topk(h2, wr, 3)
    assert ids[0].tolist() == [1, 3, 4]
    assert ids[1].tolist() == [0, 1, 2]           # all equal -> 0, 1, 2
    np.testing.assert_allclose(wts[1], 1.0 / 3, rtol=0, atol=1e-15)
    e1 = np.exp(-1.0)                            # logits 2, 2, 1
    np.testing.assert_allclose(wts[0], np.array([1, 1, e1]) / (2 + e1), rtol=1e-15)


def test_all_experts_selected_is_dense_mixture():
    """k = E: out = h1 + sum_e softmax(logits)_e y_e (brute force over experts,
    library softmax)."""
    sh = synth.shape_with(SH, n_experts=4, top_k=4)
    w = synth.layer_weights(sh, 0)
    h1 = _h1(sh, 19)
    h2 = L.rmsnorm(h1, w["ffn_norm"], sh.rms_eps)
    p = torch.softmax(torch.tensor(h2 @ w["w_router"].astype(np.float64).T), -1).numpy()
    ref = h1.copy()
    for e in range(4):
        ref += p[:, e:e + 1] * M.expert_ffn(h2, w["w_gate"][e], w["w_up"][e], w["w_down"][e])
    np.testing.assert_allclose(M.moe_ffn(h1, w, sh), ref, rtol=0, atol=1e-12)


def test_zero_down_is_identity_and_linear_in_down():
    sh = SH
    w = synth.layer_weights(sh, 0)
    h1 = _h1(sh, 23)
    w0 = dict(w, w_down=np.zeros_like(w["w_down"]))
    np.testing.assert_array_equal(M.moe_ffn(h1, w0, sh), h1)
    w2 = dict(w, w_down=2.0 * w["w_down"])
    np.testing.assert_allclose(M.moe_ffn(h1, w2, sh) - h1, 2.0 * (M.moe_ffn(h1, w, sh) - h1), rtol=1e-12,
                               atol=1e-12)


def test_expert_relabeling_invariance():
    sh = SH
    w = synth.layer_weights(sh, 0)
    perm = np.random.default_rng(0).permutation(sh.n_experts)
    wp = dict(w)
    for name in ("w_router", "w_gate", "w_up", "w_down"):
        wp[name] = w[name][perm]
    h1 = _h1(sh, 41)
    np.testing.assert_allclose(M.moe_ffn(h1, wp, sh), M.moe_ffn(h1, w, sh), rtol=0, atol=1e-12)


def test_token_permutation_and_split_invariance():
    sh = SH
    w = synth.layer_weights(sh, 0)
    h1 = _h1(sh, 50)
    out = M.moe_ffn(h1, w, sh)
    perm = np.random.default_rng(1).permutation(50)
    np.testing.assert_allclose(M.moe_ffn(h1[perm], w, sh), out[perm], rtol=0, atol=1e-12)
    parts = np.concatenate([M.moe_ffn(h1[a:b], w, sh) for a, b in [(0, 13), (13, 14), (14, 50)]])
    np.testing.assert_allclose(parts, out, rtol=0, atol=1e-12)


@pytest.mark.parametrize("N", [2, 4, 8])
def test_tp_sharded_equals_unsharded(N):
    sh = synth.shape_with(SH, d_ffn=64)
    w = synth.layer_weights(sh, 0)
    h1 = _h1(sh, 29)
    np.testing.assert_allclose(M.moe_ffn_tp(h1, w, sh, N), M.moe_ffn(h1, w, sh), rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("T,E,k,tile", [(300, 8, 2, 128), (5, 8, 2, 128), (1000, 3, 1, 16), (64, 8, 8, 128)])
def test_group_rows_invariants(T, E, k, tile):
    """A-23: brute force against a stable argsort construction, plus the
    segment invariants (aligned, tight, every assignment once, token order)."""
    rng = np.random.default_rng(T + E)
    ids = np.stack([rng.choice(E, size=k, replace=False) for _ in range(T)])
    off, cnt, dst, row_tok = M.group_rows(ids, E, tile)
    flat = ids.reshape(-1)
    order = np.argsort(flat, kind="stable")                 # assignments by expert, then a
    assert np.array_equal(cnt, np.bincount(flat, minlength=E))
    assert (off % tile == 0).all() and (np.diff(off) - cnt >= 0).all() and (np.diff(off) - cnt < tile).all()
    seg_start = np.repeat(off[:-1], cnt)
    rank_in_seg = np.arange(T * k) - np.repeat(np.concatenate([[0], np.cumsum(cnt)[:-1]]), cnt)
    expect = np.empty(T * k, dtype=np.int64)
    expect[order] = seg_start + rank_in_seg
    assert np.array_equal(dst.reshape(-1), expect)
    assert len(set(dst.reshape(-1).tolist())) == T * k
    assert np.array_equal(row_tok[dst.reshape(-1)], np.repeat(np.arange(T), k))
    assert (row_tok >= 0).sum() == T * k
    for e in range(E):
        seg = row_tok[off[e]:off[e] + cnt[e]]
        assert (np.diff(seg) > 0).all()                     # token-major order, one row per token
        assert (row_tok[off[e] + cnt[e]:off[e + 1]] == -1).all()


def test_moe_model_step_single_expert_is_dense_model_step():
    """oracle.layer.model_step on an MoE shape with E = 1, k = 1 equals the dense
    model step on the same weights (the MoE branch of the model step)."""
    sh = synth.shape_with(SH, n_experts=1, top_k=1, n_layers=2, vocab=97)
    dsh = synth.shape_with(sh, n_experts=0)
    W = synth.model_weights(sh)
    Wd = dict(W, layers=[{k: (v[0] if k in ("w_gate", "w_up", "w_down") else v) for k, v in w.items()
                          if k != "w_router"} for w in W["layers"]])
    b = synth.make_batch([1, 1, 6], [9, 30, 0], seed=3, pool_slack=2)
    toks = synth.token_ids(b.n_tokens, sh.vocab)
    pools = [L.as_pool(synth.kv_pool(sh, b, layer=l)) for l in range(2)]
    routes = []
    ids, lg, x = L.model_step(toks, W, [p.copy() for p in pools], b, sh, return_logits=True, route_logits=routes)
    ids_d, lg_d, x_d = L.model_step(toks, Wd, [p.copy() for p in pools], b, dsh, return_logits=True)
    assert len(routes) == 2 and np.array_equal(ids, ids_d)
    np.testing.assert_allclose(lg, lg_d, rtol=0, atol=1e-10)


def test_forced_ids_reduce_to_topk_and_tie_rule():
    """moe_ffn(forced_ids=the router's own top-k) == moe_ffn (same weights, A-21); a
    forced swap of the two selected experts gives the same output (the weights follow
    the experts); forcing another pair uses the softmax over those two logits."""
    shape = synth.SHAPES["c1-moe"]
    w = synth.layer_weights(shape, 0)
    h1 = synth.activations(shape, 40, seed=9)
    out, ids, wts, logits = M.moe_ffn(h1, w, shape, return_route=True)
    out2, ids2, wts2, _ = M.moe_ffn(h1, w, shape, return_route=True, forced_ids=ids)
    assert np.array_equal(ids, ids2) and np.allclose(wts, wts2, rtol=0, atol=1e-15)
    assert np.allclose(out, out2, rtol=0, atol=1e-12)
    out3 = M.moe_ffn(h1, w, shape, forced_ids=ids[:, ::-1])
    assert np.allclose(out, out3, rtol=1e-12, atol=1e-12)
    alt = np.stack([ids[:, 0], (ids[:, 1] + 1) % shape.n_experts], axis=1)
    alt[alt[:, 1] == alt[:, 0], 1] = (alt[alt[:, 1] == alt[:, 0], 1] + 1) % shape.n_experts
    _, _, wa, _ = M.moe_ffn(h1, w, shape, return_route=True, forced_ids=alt)
    sel = np.take_along_axis(logits, alt, axis=1)
    assert np.allclose(wa[:, 0], 1.0 / (1.0 + np.exp(sel[:, 1] - sel[:, 0])), rtol=1e-12)
