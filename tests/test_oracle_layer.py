"""Pins of the oracle's decoder layer, TP algebra, nano-batch split
invariance, KV write map, metadata and model step (SURVEY.md §8c T10-T14,
T17).  CPU only."""
from fractions import Fraction

import numpy as np
import pytest
import torch

import synth
from oracle import layer as L
from oracle import metadata as md

SH = synth.shape_with(synth.SHAPES["c1"], d_model=64, n_q_heads=8, n_kv_heads=4, head_dim=16,
                      d_ffn=96, vocab=211, n_layers=2)


def _case(q_len, prefix, shape=SH, seed=0, fill=0.0):
    b = synth.make_batch(q_len, prefix, seed=3 + seed, pool_slack=4)
    pool = L.as_pool(synth.kv_pool(shape, b, seed=2 + seed, fill=fill))
    x = synth.activations(shape, b.n_tokens, seed=1 + seed)
    w = synth.layer_weights(shape, 0, seed=seed)
    return b, pool, x, w


def _torch_layer(x, w, K_prefix, V_prefix, q_len, prefix, shape):
    """Independent float64 implementation with torch library routines and
    contiguous per-request K/V (no page table); RoPE via complex rotation."""
    D, hd, qh, kh = shape.d_model, shape.head_dim, shape.n_q_heads, shape.n_kv_heads
    t = lambda a: torch.tensor(np.asarray(a, dtype=np.float64))
    X = t(x)
    h = torch.nn.functional.rms_norm(X, (D,), t(w["attn_norm"]), shape.rms_eps)
    q = torch.nn.functional.linear(h, t(w["w_q"])).view(-1, qh, hd)
    k = torch.nn.functional.linear(h, t(w["w_k"])).view(-1, kh, hd)
    v = torch.nn.functional.linear(h, t(w["w_v"])).view(-1, kh, hd)
    pos = torch.tensor([p + i for n, p in zip(q_len, prefix) for i in range(n)], dtype=torch.float64)
    half = hd // 2
    freq = shape.rope_theta ** (-torch.arange(half, dtype=torch.float64) * 2 / hd)
    rot = torch.polar(torch.ones(len(pos), half, dtype=torch.float64), pos[:, None] * freq[None])

    def rope(a):
        z = torch.complex(a[..., :half], a[..., half:]) * rot[:, None, :]
        return torch.cat([z.real, z.imag], dim=-1)

    q, k = rope(q), rope(k)
    outs = []
    t0 = 0
    for r, (n, p) in enumerate(zip(q_len, prefix)):
        Kr = torch.cat([t(K_prefix[r]), k[t0:t0 + n]], 0)   # [p+n, kh, hd]
        Vr = torch.cat([t(V_prefix[r]), v[t0:t0 + n]], 0)
        R = qh // kh
        mask = torch.arange(p + n)[None, :] <= (p + torch.arange(n))[:, None]
        o = torch.nn.functional.scaled_dot_product_attention(
            q[t0:t0 + n].permute(1, 0, 2), Kr.repeat_interleave(R, 1).permute(1, 0, 2),
            Vr.repeat_interleave(R, 1).permute(1, 0, 2), attn_mask=mask)
        outs.append(o.permute(1, 0, 2).reshape(n, qh * hd))
        t0 += n
    o = torch.cat(outs, 0)
    h1 = X + torch.nn.functional.linear(o, t(w["w_o"]))
    h2 = torch.nn.functional.rms_norm(h1, (D,), t(w["ffn_norm"]), shape.rms_eps)
    m = torch.nn.functional.silu(torch.nn.functional.linear(h2, t(w["w_gate"]))) * \
        torch.nn.functional.linear(h2, t(w["w_up"]))
    return (h1 + torch.nn.functional.linear(m, t(w["w_down"]))).numpy()


def test_layer_matches_independent_torch_implementation():
    q_len, prefix = [1, 1, 9, 1, 20], [40, 3, 0, 17, 5]
    b, pool, x, w = _case(q_len, prefix)
    # prefix K/V read element by element from the pool, as contiguous arrays
    Kp, Vp = [], []
    for r in range(b.n_req):
        K = np.zeros((prefix[r], SH.n_kv_heads, SH.head_dim))
        V = np.zeros_like(K)
        for j in range(prefix[r]):
            pg = b.page_ids[b.page_indptr[r] + j // 16]
            K[j], V[j] = pool[pg, 0, :, j % 16], pool[pg, 1, :, j % 16]
        Kp.append(K)
        Vp.append(V)
    ref = _torch_layer(x, w, Kp, Vp, q_len, prefix, SH)
    out = L.decoder_layer(x, w, pool.copy(), b, SH)
    np.testing.assert_allclose(out, ref, rtol=1e-10, atol=1e-10)


@pytest.mark.parametrize("N", [2, 4])
def test_t10_tp_algebra_equals_unsharded(N):
    q_len, prefix = [1, 1, 1, 6, 1, 11], [30, 2, 17, 0, 9, 4]
    b, pool, x, w = _case(q_len, prefix, seed=1)
    ref = L.decoder_layer(x, w, pool.copy(), b, SH)
    kh = SH.n_kv_heads // N
    pools = [pool[:, :, r * kh:(r + 1) * kh].copy() for r in range(N)]
    for cut in (0, 3, 6):
        out = L.decoder_layer_tp(x, w, [p.copy() for p in pools], b, SH, N, cut)
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)


def test_t11_nano_batch_split_invariance():
    q_len, prefix = [1, 1, 1, 1, 7, 1, 12, 1], [5, 33, 16, 0, 3, 15, 0, 47]
    b, pool, x, w = _case(q_len, prefix, seed=2)
    ref = L.decoder_layer(x, w, pool.copy(), b, SH)
    for cuts in ([0, 8], [0, 4, 8], [0, 2, 4, 6, 8], [0, 1, 5, 7, 8], [0, 0, 3, 8]):
        out = L.decoder_layer_nano(x, w, pool.copy(), b, SH, cuts)
        np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)


def test_t12_request_permutation_equivariance():
    q_len, prefix = [1, 4, 1, 9, 1], [21, 0, 6, 2, 40]
    b, pool, x, w = _case(q_len, prefix, seed=3)
    ref = L.decoder_layer(x, w, pool.copy(), b, SH)
    perm = [3, 0, 4, 2, 1]
    ind = md.qo_indptr(b.q_len)
    rows = np.concatenate([np.arange(ind[r], ind[r + 1]) for r in perm])
    pages = [b.page_ids[b.page_indptr[r]:b.page_indptr[r + 1]] for r in perm]
    bp = synth.Batch(b.q_len[perm], b.kv_prefix[perm],
                     np.concatenate([[0], np.cumsum([len(p) for p in pages])]).astype(np.int32),
                     np.concatenate(pages).astype(np.int32), b.n_pages_pool)
    out = L.decoder_layer(x[rows], w, pool.copy(), bp, SH)
    np.testing.assert_allclose(out, ref[rows], rtol=1e-12, atol=1e-12)


def test_t13_kv_write_map_nan_sentinel():
    q_len, prefix = [1, 5, 1, 17, 1], [15, 0, 16, 31, 0]
    b, pool, x, w = _case(q_len, prefix, seed=4, fill=np.nan)
    before = pool.copy()
    L.decoder_layer(x, w, pool, b, SH)
    changed = ~((pool == before) | (np.isnan(pool) & np.isnan(before)))
    # brute-force expected slot set
    exp = np.zeros_like(changed)
    for r in range(b.n_req):
        for i in range(q_len[r]):
            p = prefix[r] + i
            exp[b.page_ids[b.page_indptr[r] + p // 16], :, :, p % 16, :] = True
    assert np.array_equal(changed, exp)
    assert not np.isnan(pool[exp]).any()


def test_t14_metadata_brute_force_and_snapping():
    b = synth.c1_batch()
    assert b.n_tokens == 128 and b.n_req == 65 and int(b.page_indptr[-1]) == 580
    pos = md.positions(b.q_len, b.kv_prefix)
    assert (pos[:64] == 128).all() and np.array_equal(pos[64:], np.arange(64))
    pages, offs = md.write_slots(b.q_len, b.kv_prefix, b.page_indptr, b.page_ids)
    # A-8: the decode token at position 128 opens logical page 8 (the 9th) at slot 0
    assert (offs[:64] == 0).all()
    assert all(pages[r] == b.page_ids[b.page_indptr[r] + 8] for r in range(64))
    assert len(set(zip(pages.tolist(), offs.tolist()))) == 128
    # C1 halves: [0,64) [64,128) -> request cut 64
    assert md.snap_cuts(b.q_len, [Fraction(1, 2)] * 2) == [0, 64, 65]
    # ties go to the lower boundary: boundaries at 0,2,4 target 1 -> 0; target 3 -> 2
    assert md.snap_cuts([2, 2], [Fraction(1, 4), Fraction(3, 4)]) == [0, 0, 2]
    assert md.snap_cuts([2, 2], [Fraction(3, 4), Fraction(1, 4)]) == [0, 1, 2]
    # C2 steady state: 683 decode + chunk 341 + prompt 1024 -> halves cut at request 684
    c2 = synth.workload_batch(2048, 1024, 512)
    assert c2.n_req == 685 and c2.n_tokens == 2048
    assert md.snap_cuts(c2.q_len, [Fraction(1, 2)] * 2) == [0, 684, 685]


def test_steady_state_composition_matches_survey():
    # C2 683 + 341 + 1024; C3 1365 + 171 + 512; 4096 -> 2731 + 341 + 2x512
    assert synth.steady_state_composition(2048, 1024, 512) == (683, 341, 1)
    assert synth.steady_state_composition(2048, 512, 1024) == (1365, 171, 1)
    assert synth.steady_state_composition(4096, 512, 1024) == (2731, 341, 2)


def test_t17_model_step_argmax_lowest_index_on_ties():
    sh = SH
    b = synth.make_batch([1, 3, 1], [4, 0, 9], seed=1, pool_slack=2)
    W = synth.model_weights(sh, seed=0, n_layers=1)
    W["lm_head"][:] = 0.0
    W["lm_head"][[5, 9, 150]] = 1.0      # rows 5, 9 and 150 tie for every input
    pools = [L.as_pool(synth.kv_pool(sh, b, seed=2))]
    ids = L.model_step(synth.token_ids(b.n_tokens, sh.vocab), W, pools, b, sh)
    # all-positive logits tie -> lowest index; (sum of normalised h could be
    # negative, then the zero rows win with the lowest zero row = 0)
    _, logits, _ = L.model_step(synth.token_ids(b.n_tokens, sh.vocab), W,
                                [L.as_pool(synth.kv_pool(sh, b, seed=2))], b, sh, return_logits=True)
    for i in range(3):
        exp = 5 if logits[i, 5] > 0 else 0
        assert ids[i] == exp
    # emit mask
    ids2 = L.model_step(synth.token_ids(b.n_tokens, sh.vocab), W, [L.as_pool(synth.kv_pool(sh, b, seed=2))], b, sh,
                        emit=np.array([1, 0, 1]))
    assert ids2[1] == -1 and ids2[0] == ids[0] and ids2[2] == ids[2]


def test_model_step_layers_compose():
    sh = SH
    b = synth.make_batch([1, 2], [5, 0], seed=1)
    W = synth.model_weights(sh, seed=0, n_layers=2)
    toks = synth.token_ids(b.n_tokens, sh.vocab)
    pools = [L.as_pool(synth.kv_pool(sh, b, seed=2, layer=l)) for l in range(2)]
    ids, logits, xL = L.model_step(toks, W, [p.copy() for p in pools], b, sh, return_logits=True)
    x = W["embed"][toks].astype(np.float64)
    for l in range(2):
        x = L.decoder_layer(x, W["layers"][l], pools[l], b, sh)
    np.testing.assert_array_equal(x, xL)
    lg = L.rmsnorm(x[[0, 2]], W["final_norm"], sh.rms_eps) @ W["lm_head"].astype(np.float64).T
    np.testing.assert_allclose(lg, logits, rtol=1e-12)
    assert list(ids) == list(np.argmax(lg, axis=1))
