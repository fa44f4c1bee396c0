"""Pins of the oracle's paged attention, RoPE, RMSNorm and SwiGLU against
closed forms, invariants, brute force and library routines (SURVEY.md §8c
T1-T9).  CPU only."""
import numpy as np
import pytest
import scipy.special
import torch

import synth
from oracle import layer as L
from oracle import metadata as md

SH = synth.shape_with(synth.SHAPES["c1"], d_model=64, n_q_heads=4, n_kv_heads=2, head_dim=16,
                      d_ffn=96, vocab=101)


def _setup(q_len, prefix, seed=0, shape=SH, permute=True):
    b = synth.make_batch(q_len, prefix, seed=3 + seed, pool_slack=3, permute=permute)
    pool = L.as_pool(synth.kv_pool(shape, b, seed=2 + seed))
    T = b.n_tokens
    q = synth.randn_bf16((T, shape.n_q_heads, shape.head_dim), 7 + seed, "q")
    k = synth.randn_bf16((T, shape.n_kv_heads, shape.head_dim), 7 + seed, "k")
    v = synth.randn_bf16((T, shape.n_kv_heads, shape.head_dim), 7 + seed, "v")
    L.kv_append(pool, k, v, b)
    return b, pool, q, k, v


def test_t1_single_key_returns_v():
    # kv_prefix = 0, q_len = 1: softmax over one key is exactly 1 -> o = v
    b, pool, q, k, v = _setup([1, 1], [0, 0])
    o = L.paged_attention(q, pool, b)
    R = SH.n_q_heads // SH.n_kv_heads
    for t in range(2):
        for h in range(SH.n_q_heads):
            assert np.array_equal(o[t, h], v[t, h // R].astype(np.float64))


def test_t2_softmax_rows_sum_to_one():
    b, pool, q, k, v = _setup([1, 5, 1, 3], [17, 0, 40, 9])
    _, probs = L.paged_attention(q, pool, b, return_probs=True)
    for p in probs:
        assert np.allclose(p.sum(axis=1), 1.0, atol=1e-12)
        assert (p >= 0).all()


def test_t3_constant_keys_give_mean_v():
    b, pool, q, k, v = _setup([1, 4], [30, 5])
    pool[:, 0] = 0.5  # every key equal -> uniform weights
    o = L.paged_attention(q, pool, b)
    pos = md.positions(b.q_len, b.kv_prefix)
    R = SH.n_q_heads // SH.n_kv_heads
    for t, r in enumerate(md.token_request(b.q_len)):
        _, V = L.gather_kv(pool, b, r, int(pos[t]) + 1)
        for h in range(SH.n_q_heads):
            np.testing.assert_allclose(o[t, h], V[:, h // R].mean(axis=0), rtol=1e-12, atol=1e-12)


def test_t4_page_permutation_invariance():
    q_len, prefix = [1, 3, 1, 7], [33, 20, 0, 48]
    b1 = synth.make_batch(q_len, prefix, seed=11, pool_slack=5)
    b2 = synth.make_batch(q_len, prefix, seed=12, pool_slack=5)
    assert not np.array_equal(b1.page_ids, b2.page_ids)
    rng = np.random.default_rng(0)
    T = sum(q_len)
    q = rng.standard_normal((T, SH.n_q_heads, SH.head_dim))
    k = rng.standard_normal((T, SH.n_kv_heads, SH.head_dim))
    v = rng.standard_normal((T, SH.n_kv_heads, SH.head_dim))
    # same logical prefix contents in both layouts
    outs = []
    for b in (b1, b2):
        pool = np.zeros((b.n_pages_pool, 2, SH.n_kv_heads, 16, SH.head_dim))
        for r in range(b.n_req):
            for j in range(prefix[r]):
                pg = b.page_ids[b.page_indptr[r] + j // 16]
                pool[pg, :, :, j % 16, :] = np.sin(np.arange(2 * SH.n_kv_heads * SH.head_dim) * (r + 1) + j
                                                   ).reshape(2, SH.n_kv_heads, SH.head_dim)
        L.kv_append(pool, k, v, b)
        outs.append(L.paged_attention(q, pool, b))
    assert np.array_equal(outs[0], outs[1])


def _dense_reference_torch(q, K, V, pos):
    """Library routine on contiguous K/V: torch SDPA with an explicit boolean
    mask (key j visible iff j <= pos[t]), float64, GQA by repeat."""
    qt = torch.tensor(q).permute(1, 0, 2)[None]           # [1, qh, T, hd]
    R = q.shape[1] // K.shape[1]
    Kt = torch.tensor(K).repeat_interleave(R, dim=1).permute(1, 0, 2)[None]
    Vt = torch.tensor(V).repeat_interleave(R, dim=1).permute(1, 0, 2)[None]
    mask = torch.arange(K.shape[0])[None, :] <= torch.tensor(pos)[:, None]
    o = torch.nn.functional.scaled_dot_product_attention(qt, Kt, Vt, attn_mask=mask)
    return o[0].permute(1, 0, 2).numpy()


def test_t5_brute_force_dense_attention_matches_paged():
    rng = np.random.default_rng(5)
    for trial in range(4):
        n_req = int(rng.integers(1, 4))
        q_len = rng.integers(1, 6, n_req).tolist()
        prefix = rng.integers(0, 35, n_req).tolist()
        b, pool, q, k, v = _setup(q_len, prefix, seed=trial)
        o = L.paged_attention(q, pool, b)
        ind = md.qo_indptr(b.q_len)
        pos = md.positions(b.q_len, b.kv_prefix)
        for r in range(n_req):
            n = prefix[r] + q_len[r]
            # contiguous K/V reconstructed element by element (no page math shared)
            K = np.zeros((n, SH.n_kv_heads, SH.head_dim))
            V = np.zeros_like(K)
            for j in range(n):
                page = b.page_ids[b.page_indptr[r] + j // 16]
                K[j] = pool[page, 0, :, j % 16]
                V[j] = pool[page, 1, :, j % 16]
            ref = _dense_reference_torch(q[ind[r]:ind[r + 1]].astype(np.float64), K, V,
                                         pos[ind[r]:ind[r + 1]])
            np.testing.assert_allclose(o[ind[r]:ind[r + 1]], ref, rtol=1e-10, atol=1e-12)


def test_t5b_explicit_loop_softmax_tiny():
    # fully explicit scalar loops with scipy softmax for one tiny request
    b, pool, q, k, v = _setup([2], [3], seed=9)
    o = L.paged_attention(q, pool, b)
    hd = SH.head_dim
    R = SH.n_q_heads // SH.n_kv_heads
    for i in range(2):
        P = 3 + i
        for h in range(SH.n_q_heads):
            keys, vals = [], []
            for j in range(P + 1):
                page = b.page_ids[j // 16]
                keys.append(pool[page, 0, h // R, j % 16].astype(np.float64))
                vals.append(pool[page, 1, h // R, j % 16].astype(np.float64))
            s = [sum(float(q[i, h, d]) * keys[j][d] for d in range(hd)) / hd ** 0.5 for j in range(P + 1)]
            p = scipy.special.softmax(np.array(s))
            ref = sum(p[j] * vals[j] for j in range(P + 1))
            np.testing.assert_allclose(o[i, h], ref, rtol=1e-12, atol=1e-13)


def test_t6_decode_equals_last_prefill_row():
    rng = np.random.default_rng(6)
    n = 21
    qs = rng.standard_normal((n + 1, SH.n_q_heads, SH.head_dim))
    ks = rng.standard_normal((n + 1, SH.n_kv_heads, SH.head_dim))
    vs = rng.standard_normal((n + 1, SH.n_kv_heads, SH.head_dim))
    # prefill all n+1 tokens
    bp = synth.make_batch([n + 1], [0], seed=1)
    pp = np.zeros((bp.n_pages_pool, 2, SH.n_kv_heads, 16, SH.head_dim))
    L.kv_append(pp, ks, vs, bp)
    op = L.paged_attention(qs, pp, bp)
    # decode: first n cached, then one token
    bd = synth.make_batch([1], [n], seed=2)
    pd = np.zeros((bd.n_pages_pool, 2, SH.n_kv_heads, 16, SH.head_dim))
    b0 = synth.Batch(np.array([n], np.int32), np.array([0], np.int32), bd.page_indptr, bd.page_ids, bd.n_pages_pool)
    L.kv_append(pd, ks[:n], vs[:n], b0)
    L.kv_append(pd, ks[n:], vs[n:], bd)
    od = L.paged_attention(qs[n:], pd, bd)
    np.testing.assert_allclose(od[0], op[n], rtol=1e-12, atol=1e-14)


def test_t7_chunked_prefill_equals_whole():
    rng = np.random.default_rng(7)
    n = 64
    qs = rng.standard_normal((n, SH.n_q_heads, SH.head_dim))
    ks = rng.standard_normal((n, SH.n_kv_heads, SH.head_dim))
    vs = rng.standard_normal((n, SH.n_kv_heads, SH.head_dim))
    bw = synth.make_batch([n], [0], seed=1)
    pw = np.zeros((bw.n_pages_pool, 2, SH.n_kv_heads, 16, SH.head_dim))
    L.kv_append(pw, ks, vs, bw)
    ow = L.paged_attention(qs, pw, bw)
    # two chunks of 32 sharing one page table
    full = synth.make_batch([n], [0], seed=4)
    pc = np.zeros((full.n_pages_pool, 2, SH.n_kv_heads, 16, SH.head_dim))
    c1 = synth.Batch(np.array([32], np.int32), np.array([0], np.int32), full.page_indptr, full.page_ids, full.n_pages_pool)
    c2 = synth.Batch(np.array([32], np.int32), np.array([32], np.int32), full.page_indptr, full.page_ids, full.n_pages_pool)
    L.kv_append(pc, ks[:32], vs[:32], c1)
    o1 = L.paged_attention(qs[:32], pc, c1)
    L.kv_append(pc, ks[32:], vs[32:], c2)
    o2 = L.paged_attention(qs[32:], pc, c2)
    np.testing.assert_allclose(np.concatenate([o1, o2]), ow, rtol=1e-12, atol=1e-14)


def test_mha_special_case_r1():
    # R = 1 reduces to plain multi-head attention: compare against torch SDPA is_causal
    sh = synth.shape_with(SH, n_kv_heads=SH.n_q_heads)
    rng = np.random.default_rng(8)
    n = 19
    qs = rng.standard_normal((n, sh.n_q_heads, sh.head_dim))
    ks = rng.standard_normal((n, sh.n_kv_heads, sh.head_dim))
    vs = rng.standard_normal((n, sh.n_kv_heads, sh.head_dim))
    b = synth.make_batch([n], [0], seed=1)
    pool = np.zeros((b.n_pages_pool, 2, sh.n_kv_heads, 16, sh.head_dim))
    L.kv_append(pool, ks, vs, b)
    o = L.paged_attention(qs, pool, b)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.tensor(qs).permute(1, 0, 2), torch.tensor(ks).permute(1, 0, 2),
        torch.tensor(vs).permute(1, 0, 2), is_causal=True).permute(1, 0, 2).numpy()
    np.testing.assert_allclose(o, ref, rtol=1e-10, atol=1e-12)


# ------------------------------------------------------------------ RoPE
def test_t8_rope_relative_position_invariance():
    rng = np.random.default_rng(8)
    hd = 128
    q = rng.standard_normal((5, 1, hd))
    k = rng.standard_normal((5, 1, hd))
    pos_q = np.array([3, 10, 77, 500, 1200])
    pos_k = np.array([0, 9, 70, 400, 1199])
    base = np.einsum("thd,thd->t", L.rope(q, pos_q, 1e4), L.rope(k, pos_k, 1e4))
    for c in (1, 100, 1000):
        s = np.einsum("thd,thd->t", L.rope(q, pos_q + c, 1e4), L.rope(k, pos_k + c, 1e4))
        np.testing.assert_allclose(s, base, rtol=1e-10, atol=1e-10)


def test_rope_equals_complex_rotation_and_identity_at_zero():
    rng = np.random.default_rng(9)
    hd, theta = 64, 5e5
    x = rng.standard_normal((7, 3, hd))
    pos = np.array([0, 1, 2, 15, 16, 1023, 1535])
    y = L.rope(x, pos, theta)
    assert np.array_equal(y[0], x[0])  # pos 0 is the identity
    half = hd // 2
    z = x[..., :half] + 1j * x[..., half:]
    ang = pos[:, None, None] * theta ** (-np.arange(half) * 2.0 / hd)[None, None, :]
    zr = z * np.exp(1j * ang)
    np.testing.assert_allclose(y[..., :half], zr.real, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(y[..., half:], zr.imag, rtol=1e-12, atol=1e-12)
    # per-pair norm preservation
    np.testing.assert_allclose(y[..., :half] ** 2 + y[..., half:] ** 2,
                               x[..., :half] ** 2 + x[..., half:] ** 2, rtol=1e-12)


# ------------------------------------------------------------------ RMSNorm / SiLU
def test_t9_rmsnorm_closed_form():
    rng = np.random.default_rng(10)
    x = rng.standard_normal((6, 512)) * np.array([1e-3, 0.1, 1, 3, 10, 100])[:, None]
    eps = 1e-5
    y = L.rmsnorm(x, np.ones(512), eps)
    m = np.mean(x * x, axis=1)
    np.testing.assert_allclose(np.sqrt(np.mean(y * y, axis=1)), np.sqrt(m / (m + eps)), rtol=1e-12)
    # scale invariance for c >> sqrt(eps)
    np.testing.assert_allclose(L.rmsnorm(7.0 * x[2:], np.ones(512), eps), y[2:], rtol=1e-5)
    # library routine
    ref = torch.nn.functional.rms_norm(torch.tensor(x), (512,), torch.ones(512, dtype=torch.float64), eps)
    np.testing.assert_allclose(y, ref.numpy(), rtol=1e-12)


def test_silu_closed_form():
    z = np.linspace(-30, 30, 1001)
    assert L.silu(np.array([0.0]))[0] == 0.0
    np.testing.assert_allclose(L.silu(z), z * scipy.special.expit(z), rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(L.silu(z), torch.nn.functional.silu(torch.tensor(z)).numpy(), rtol=1e-12)
