"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle.

Every test is @pytest.mark.gpu and runs on a B200.  Inputs are seeded and
synthetic (synth), the oracle runs on the same bf16 values in float64.
Tolerances: integer/index work bit-exact; floating point per BASELINE.json
north_star (rel L2 <= 1e-2, max abs <= 5e-2) unless stated."""
import numpy as np
import pytest
import torch

import synth
from oracle import layer as OL
from oracle import metadata as md

from gpu_common import (assert_close, compact_case, dev, dev_bits, device_weights, errors, host, require_gpu,
                        token_rows)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    return require_gpu()


# ------------------------------------------------------------------ GEMM
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (1, 32, 64), (200, 768, 512), (77, 2816, 1376),
                                   (1000, 6144, 4096), (2048, 4096, 14336), (513, 32000, 512)])
def test_gemm_vs_oracle(env, M, N, K):
    nf, rt = env
    rng = np.random.default_rng(M * 7 + N + K)
    A = synth.round_bf16(rng.standard_normal((M, K), dtype=np.float32))
    B = synth.round_bf16(rng.standard_normal((N, K), dtype=np.float32) / np.float32(np.sqrt(K)))
    Ad, Bd = dev(A), dev(B)
    C = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
    nf.gemm_bf16(Ad.data_ptr(), K, Bd.data_ptr(), K, C.data_ptr(), N, M, N, K, 148, rt.stream_handle())
    torch.cuda.synchronize()
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    # bf16 output rounding (2^-9 relative) + fp32 accumulation
    rel, mx = errors(host(C), ref)
    assert rel < 4e-3 and mx < 2e-2 * max(1.0, np.abs(ref).max()), (rel, mx)


@pytest.mark.parametrize("M,N,K,sm", [(1024, 4096, 4096, 108), (1024, 6144, 4096, 100), (2048, 4096, 14336, 148),
                                      (333, 2816, 1376, 37), (77, 768, 512, 148), (1024, 28672, 4096, 96)])
def test_gemm_stream_k_vs_oracle(env, M, N, K, sm, monkeypatch):
    """Split-K tail schedule (the partial last wave's tiles split 2-4 ways in K,
    fp32 partials reduced in split order; NF_STREAMK=1 forces it on, read at the
    first GEMM launch -- exercised in a subprocess): oracle values, bit-identical
    on repeat."""
    import subprocess
    import sys
    code = f"""
import sys, numpy as np, torch
sys.path.insert(0, {repr(str(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))})
sys.path.insert(0, {repr(str(__import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__)))))})
import test_gpu_parity as T
T._stream_k_case({M}, {N}, {K}, {sm})
print("OK")
"""
    env2 = dict(__import__('os').environ, NF_STREAMK="1")
    r = subprocess.run([sys.executable, "-c", code], env=env2, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr


def _stream_k_case(M, N, K, sm):
    nf, rt = require_gpu()
    rng = np.random.default_rng(M + N + K + sm)
    A = synth.round_bf16(rng.standard_normal((M, K), dtype=np.float32))
    B = synth.round_bf16(rng.standard_normal((N, K), dtype=np.float32) / np.float32(np.sqrt(K)))
    Ad, Bd = dev(A), dev(B)
    ws = torch.empty(nf.gemm_workspace_bytes(M, N), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(2):
        C = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        nf.gemm_bf16(Ad.data_ptr(), K, Bd.data_ptr(), K, C.data_ptr(), N, M, N, K, sm, rt.stream_handle(),
                     ws.data_ptr(), ws.numel())
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    rel, mx = errors(host(outs[0]), ref)
    assert rel < 4e-3 and mx < 2e-2 * max(1.0, np.abs(ref).max()), (rel, mx)


@pytest.mark.parametrize("M,N,K,sm", [(2048, 1280, 8192, 148), (1024, 1280, 8192, 132), (512, 6144, 4096, 148),
                                      (128, 2048, 14336, 148), (300, 768, 2048, 100), (1000, 1280, 8192, 116)])
def test_gemm_stream_k_subwave_vs_oracle(env, M, N, K, sm):
    """Stream-K schedule of sub-wave GEMMs (fewer 128x256 tiles than SMs, e.g.
    the 70B TP8 rank's KQV: 80 tiles on 148 SMs): CTA c runs k-blocks
    [c U/G, (c+1) U/G) of the (tile, k-block) space, owners add the later CTAs'
    fp32 partials in CTA order.  Oracle values, bit-identical on repeat."""
    nf, rt = env
    rng = np.random.default_rng(M + N + K)
    A = synth.round_bf16(rng.standard_normal((M, K), dtype=np.float32))
    B = synth.round_bf16(rng.standard_normal((N, K), dtype=np.float32) / np.float32(np.sqrt(K)))
    Ad, Bd = dev(A), dev(B)
    ws = torch.empty(nf.gemm_workspace_bytes(M, N), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(2):
        C = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        nf.gemm_bf16(Ad.data_ptr(), K, Bd.data_ptr(), K, C.data_ptr(), N, M, N, K, sm, rt.stream_handle(),
                     ws.data_ptr(), ws.numel())
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    rel, mx = errors(host(outs[0]), ref)
    assert rel < 4e-3 and mx < 2e-2 * max(1.0, np.abs(ref).max()), (rel, mx)


@pytest.mark.parametrize("M,N,K,sm", [(1024, 4096, 14336, 116), (1024, 4096, 4096, 116), (768, 28672, 4096, 116),
                                      (2048, 6144, 4096, 148), (1280, 4096, 14336, 148), (333, 4096, 4096, 20)])
def test_gemm_cta_pair_vs_oracle(env, M, N, K, sm):
    """CTA-pair (cta_group::2) schedules picked by the launcher for these shapes:
    256-row pair tiles, data-parallel and with a split-K tail over pairs, ragged
    M (333): oracle values, bit-identical on repeat."""
    _stream_k_case(M, N, K, sm)


@pytest.mark.parametrize("M,N,K,sm", [(1280, 4096, 14336, 108), (768, 4096, 4096, 108), (1280, 6144, 4096, 100),
                                      (300, 1024, 8192, 37)])
def test_gemm_split_k2_vs_oracle(env, M, N, K, sm):
    """Split-K=2 schedule (chosen when it lowers the tile rounds of nano-batch
    GEMMs): both K-halves reduced in fixed order; oracle values, bit-identical on repeat."""
    _stream_k_case(M, N, K, sm)


@pytest.mark.parametrize("sm", [1, 7, 64, 148])
def test_gemm_sm_budget_bit_identical(env, sm):
    """The SM budget only changes which CTA computes a tile, never the math."""
    nf, rt = env
    rng = np.random.default_rng(3)
    M, N, K = 600, 1024, 1024
    A, B = dev(synth.round_bf16(rng.standard_normal((M, K), dtype=np.float32))), \
        dev(synth.round_bf16(rng.standard_normal((N, K), dtype=np.float32) * 0.03))
    outs = []
    for budget in (148, sm):
        C = torch.empty((M, N), dtype=torch.bfloat16, device="cuda")
        nf.gemm_bf16(A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), N, M, N, K, budget, rt.stream_handle())
        outs.append(C)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


# ------------------------------------------------------------------ attention
def _attn_case(shape, q_len, prefix, seed=0, fill=0.0):
    b = synth.make_batch(q_len, prefix, seed=3 + seed, pool_slack=5)
    pool = synth.kv_pool(shape, b, seed=2 + seed, fill=fill)
    T = b.n_tokens
    q = synth.randn_bf16((T, shape.n_q_heads, shape.head_dim), 7 + seed, "q")
    k = synth.randn_bf16((T, shape.n_kv_heads, shape.head_dim), 7 + seed, "k")
    v = synth.randn_bf16((T, shape.n_kv_heads, shape.head_dim), 7 + seed, "v")
    opool = OL.as_pool(pool)
    OL.kv_append(opool, k, v, b)
    return b, opool, q


def _run_attn(env, shape, b, pool64, q, sm_dec=148, sm_pf=148):
    nf, rt = env
    cfg = rt.cfg_from_shape(shape)
    nb = nf.Batch.from_any(b)
    pool_d = dev(pool64)
    q_d = dev(q)
    o = torch.full((b.n_tokens, shape.n_q_heads * shape.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    ws = rt.workspace(cfg, nb)
    nf.attention(cfg, nb, q_d.data_ptr(), pool_d.data_ptr(), o.data_ptr(), ws.data_ptr(), ws.numel(), sm_dec, sm_pf,
                 rt.stream_handle())
    torch.cuda.synchronize()
    return host(o).reshape(b.n_tokens, shape.n_q_heads, shape.head_dim)


@pytest.mark.parametrize("shape_name", ["c1", "llama3-8b"])
def test_attention_vs_oracle(env, shape_name):
    shape = synth.SHAPES[shape_name]
    rng = np.random.default_rng(11)
    n_dec = 40
    q_len = [1] * n_dec + [150, 200, 64, 65, 2]
    prefix = list(rng.integers(0, 1500, n_dec)) + [300, 0, 17, 0, 1000]
    b, pool, q = _attn_case(shape, q_len, prefix)
    out = _run_attn(env, shape, b, pool, q)
    ref = OL.paged_attention(q, pool, b)
    assert_close(out, ref, what="attention")


def test_prefill_attention_bench_composition(env):
    """a5 at the bench's prefill shapes (8B: a 341-token chunk over a 683-token
    prefix + a 1024-token prompt, i.e. many 128-key blocks, ragged last tiles and
    diagonal blocks) with NaN in every unused pool slot, at several SM budgets
    (the tcgen05 kernel is persistent: the budget only changes which CTA runs
    an item, so outputs are bit-identical across budgets)."""
    shape = synth.SHAPES["llama3-8b"]
    q_len, prefix = [1, 1, 341, 1024, 129], [100, 2000, 683, 0, 255]
    b, pool, q = _attn_case(shape, q_len, prefix, seed=5, fill=np.nan)
    ref = OL.paged_attention(q, np.nan_to_num(pool), b)
    outs = [_run_attn(env, shape, b, pool, q, 148, sm) for sm in (148, 37, 1)]
    assert np.isfinite(outs[0]).all()
    assert_close(outs[0], ref, what="prefill attention (bench composition)")
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])


def test_attention_c1_config(env):
    shape = synth.SHAPES["c1"]
    b = synth.c1_batch()
    pool = OL.as_pool(synth.kv_pool(shape, b))
    T = b.n_tokens
    q = synth.randn_bf16((T, shape.n_q_heads, shape.head_dim), 7, "q")
    k = synth.randn_bf16((T, shape.n_kv_heads, shape.head_dim), 7, "k")
    v = synth.randn_bf16((T, shape.n_kv_heads, shape.head_dim), 7, "v")
    OL.kv_append(pool, k, v, b)
    for sm in (148, 5, 1):
        out = _run_attn(env, shape, b, pool, q, sm, sm)
        assert_close(out, OL.paged_attention(q, pool, b), what=f"attention C1 sm={sm}")


def test_attention_single_key_bit_exact(env):
    """T1: a request with one key returns V exactly (p = 1)."""
    shape = synth.SHAPES["llama3-8b"]
    b, pool, q = _attn_case(shape, [1, 1, 1], [0, 0, 0])
    out = _run_attn(env, shape, b, pool, q)
    ref = OL.paged_attention(q, pool, b)
    assert np.array_equal(out, ref)


def test_attention_page_permutation_bit_exact(env):
    """T4: relabelling physical pages leaves the output bit-identical."""
    shape = synth.SHAPES["llama3-8b"]
    q_len, prefix = [1] * 9 + [70], [5, 16, 17, 100, 255, 256, 1023, 1024, 1500, 33]
    outs = []
    for seed_pages in (3, 4):
        b = synth.make_batch(q_len, prefix, seed=seed_pages, pool_slack=7)
        pool = OL.as_pool(synth.kv_pool(shape, b, seed=2))
        T = b.n_tokens
        q = synth.randn_bf16((T, shape.n_q_heads, shape.head_dim), 7, "q")
        k = synth.randn_bf16((T, shape.n_kv_heads, shape.head_dim), 7, "k")
        v = synth.randn_bf16((T, shape.n_kv_heads, shape.head_dim), 7, "v")
        OL.kv_append(pool, k, v, b)
        outs.append(_run_attn(env, shape, b, pool, q))
    assert np.array_equal(outs[0], outs[1])


def test_attention_nan_outside_context_is_ignored(env):
    """Slots past kv_len hold NaN: masked keys and zeroed V rows must not leak."""
    shape = synth.SHAPES["llama3-8b"]
    b, pool, q = _attn_case(shape, [1, 1, 37, 1], [3, 40, 5, 16], fill=np.nan)
    out = _run_attn(env, shape, b, pool, q)
    assert np.isfinite(out).all()
    assert_close(out, OL.paged_attention(q, np.nan_to_num(pool), b), what="attention NaN sentinel")


# ------------------------------------------------------------------ decoder layer
def _layer_case(shape, b, seed=0, fill=0.0):
    w = synth.layer_weights(shape, 0, seed=seed)
    x = synth.activations(shape, b.n_tokens, seed=1 + seed)
    pool = synth.kv_pool(shape, b, seed=2 + seed, fill=fill)
    return w, x, pool


def _gpu_layer(env, shape, b, w, x, pool, mode, shares=(1,), sm=None, balance=False, colocate=False):
    nf, rt = env
    cfg = rt.cfg_from_shape(shape)
    nb = nf.Batch.from_any(b)
    wd = device_weights(w)
    packed = rt.pack_layer(cfg, wd)
    pool_d = dev(pool)
    plan = nf.Plan.explicit(cfg, mode=mode, shares=shares, sm=sm, balance=balance, colocate=colocate)
    out = rt.layer_forward(plan, cfg, packed, pool_d, nb, dev(x))
    torch.cuda.synchronize()
    return host(out), pool_d


@pytest.mark.parametrize("mode,shares", [(0, (1,)), (1, (1, 1)), (2, (1, 1)), (2, (1, 2, 1)), (1, (3, 1, 1, 2))])
def test_layer_c1_vs_oracle(env, mode, shares):
    shape = synth.SHAPES["c1"]
    b = synth.c1_batch()
    w, x, pool = _layer_case(shape, b)
    ref = OL.decoder_layer(x, w, OL.as_pool(pool), b, shape)
    out, _ = _gpu_layer(env, shape, b, w, x, pool, mode, shares)
    assert_close(out, ref, what=f"C1 layer mode={mode} shares={shares}")


def test_layer_kv_write_map_bit_exact(env):
    """T13: only this step's slots change (set identical to the oracle's);
    written K/V match the oracle's post-RoPE K and V within tolerance."""
    shape = synth.SHAPES["c1"]
    b = synth.make_batch([1, 5, 1, 17, 1, 40], [15, 0, 16, 31, 0, 100], seed=5, pool_slack=9)
    w, x, pool = _layer_case(shape, b, fill=np.nan)
    opool = OL.as_pool(pool)
    OL.decoder_layer(x, w, opool, b, shape)
    _, pool_d = _gpu_layer(env, shape, b, w, x, pool, 2, (1, 1))
    g = host(pool_d)
    changed = ~(np.isnan(g) & np.isnan(pool)) & ~(g == pool)
    exp = ~(np.isnan(opool) & np.isnan(pool)) & ~(opool == pool)
    assert np.array_equal(changed, exp)
    assert_close(g[exp], opool[exp], what="written K/V")


def test_layer_split_invariance_and_modes_agree(env):
    """T11: 1, 2, 3 nano-batches and the three pipeline modes give the same
    layer output (within the bf16 tolerance; bit-identical for the same
    row partition since every kernel's math is per-row)."""
    shape = synth.SHAPES["c1"]
    b = synth.make_batch([1] * 30 + [33, 1, 1, 20], list(range(3, 93, 3)) + [0, 7, 300, 50], seed=4, pool_slack=3)
    w, x, pool = _layer_case(shape, b, seed=3)
    ref = OL.decoder_layer(x, w, OL.as_pool(pool), b, shape)
    outs = {}
    for mode, shares in [(0, (1,)), (1, (1, 1)), (2, (1, 1)), (2, (2, 1, 1))]:
        out, _ = _gpu_layer(env, shape, b, w, x, pool, mode, shares)
        assert_close(out, ref, what=f"mode={mode} shares={shares}")
        outs[(mode, shares)] = out
    assert np.array_equal(outs[(1, (1, 1))], outs[(2, (1, 1))])


@pytest.mark.parametrize("shape_name", ["c1", "llama3-8b"])
def test_layer_colocated_plan(env, shape_name):
    """3-stage GEMM ring + 4-warp decode CTAs sharing SMs: same numbers."""
    shape = synth.SHAPES[shape_name]
    b = synth.make_batch([1] * 12 + [100, 1, 37], [1024, 5, 1535, 16, 1, 900, 64, 700, 33, 1200, 1300, 100, 341, 2, 0],
                         seed=3, pool_slack=2)
    w, x, pool = _layer_case(shape, b)
    ref = OL.decoder_layer(x, w, OL.as_pool(pool), b, shape)
    out, _ = _gpu_layer(env, shape, b, w, x, pool, 2, (1, 1), sm=[148] * 7, colocate=True)
    assert_close(out, ref, what="colocated layer")


def test_layer_8b_shape_small_batch(env):
    shape = synth.SHAPES["llama3-8b"]
    b = synth.make_batch([1] * 12 + [100, 1, 37], [1024, 5, 1535, 16, 1, 900, 64, 700, 33, 1200, 1300, 100, 341, 2, 0],
                         seed=3, pool_slack=2)
    w, x, pool = _layer_case(shape, b)
    ref = OL.decoder_layer(x, w, OL.as_pool(pool), b, shape)
    out, _ = _gpu_layer(env, shape, b, w, x, pool, 2, (1, 1))
    assert_close(out, ref, what="8B-shape layer")


def test_layer_8b_full_batch_sampled(env):
    """configs[1] at full size: one LLaMA-3-8B-shape layer over the B_dense=2048
    steady-state batch (683 decode + chunk 341 + prompt 1024), in the bench's
    OVERLAP launch configuration; sampled requests checked against the oracle
    (decode requests and both prefill requests in full)."""
    nf, rt = env
    shape = synth.SHAPES["llama3-8b"]
    b = synth.workload_batch(2048, 1024, 512)
    w = synth.layer_weights(shape, 0, seed=0)
    x = synth.activations(shape, b.n_tokens, seed=1)
    cfg = rt.cfg_from_shape(shape)
    nb = nf.Batch.from_any(b)
    packed = rt.pack_layer(cfg, device_weights(w))
    pool_d = dev_bits(synth.kv_pool_bits(shape, b, seed=2))
    plan = nf.Plan.explicit(cfg, mode=nf.OVERLAP, shares=(1, 1))
    out = host(rt.layer_forward(plan, cfg, packed, pool_d, nb, dev(x)))
    torch.cuda.synchronize()
    reqs = [0, 1, 2, 100, 341, 500, 682, 683, 684]
    sub, pool = compact_case(shape, b, reqs)
    rows = token_rows(b, reqs)
    ref = OL.decoder_layer(x[rows], w, pool, sub, shape)
    assert_close(out[rows], ref, what="8B full batch sampled")
    assert np.isfinite(out).all()


# ------------------------------------------------------------------ model step
def test_model_step_vs_oracle(env):
    nf, rt = env
    shape = synth.shape_with(synth.SHAPES["c1"], n_layers=2, vocab=4096)
    b = synth.make_batch([1] * 20 + [30, 1, 12], list(range(10, 210, 10)) + [0, 33, 7], seed=6, pool_slack=4)
    W = synth.model_weights(shape, seed=0)
    toks = synth.token_ids(b.n_tokens, shape.vocab)
    pools = [synth.kv_pool(shape, b, seed=2, layer=l) for l in range(2)]
    ids_ref, logits, _ = OL.model_step(toks, W, [OL.as_pool(p) for p in pools], b, shape, return_logits=True)
    cfg = rt.cfg_from_shape(shape)
    layers = [rt.pack_layer(cfg, device_weights(W["layers"][l])) for l in range(2)]
    model = rt.Model(cfg, dev(W["embed"]), layers, rt.pack_lm_head(cfg, dev(W["lm_head"]), dev(W["final_norm"])))
    nb = nf.Batch.from_any(b)
    ws = rt.workspace(cfg, nb)
    tok_d = torch.from_numpy(toks).cuda()
    for mode, shares, bal, col in [(0, (1,), False, False), (2, (1, 1), False, False), (2, (1, 1), True, False),
                                   (1, (1, 2), True, False), (2, (1, 1), True, True), (2, (1, 1), 2, False),
                                   (1, (1, 1, 1), 2, False), (2, (3, 1), 2, False)]:
        pools_d = [dev(p) for p in pools]
        plan = nf.Plan.explicit(cfg, mode=mode, shares=shares, balance=bal, colocate=col)
        ids = model.step(plan, pools_d, nb, tok_d, ws).cpu().numpy()
        srt = np.sort(logits, axis=1)
        gap = srt[:, -1] - srt[:, -2]
        sure = gap > 0.1
        assert sure.sum() >= len(gap) // 2
        assert np.array_equal(ids[sure], ids_ref[sure]), (mode, shares, bal)
        # every emitted row's logits (not only the clear argmax rows) within tolerance of the
        # oracle's, through nf_model_step_ex on a fresh copy of the KV pools
        ids2, lg, _ = model.step_inspect(plan, [dev(p) for p in pools], nb, tok_d, ws, hidden=False)
        assert np.array_equal(ids2.cpu().numpy(), ids), (mode, shares, bal)
        assert host(lg).shape == logits.shape
        assert_close(host(lg), logits, max_abs=0.25, what=f"C1 model-step logits {mode} {shares} {bal} {col}")


def test_model_step_emit_mask(env):
    nf, rt = env
    shape = synth.shape_with(synth.SHAPES["c1"], n_layers=1, vocab=2048)
    b = synth.make_batch([1, 4, 1], [9, 0, 3], seed=1)
    W = synth.model_weights(shape, seed=0)
    cfg = rt.cfg_from_shape(shape)
    model = rt.Model(cfg, dev(W["embed"]), [rt.pack_layer(cfg, device_weights(W["layers"][0]))],
                     rt.pack_lm_head(cfg, dev(W["lm_head"]), dev(W["final_norm"])))
    nb = nf.Batch.from_any(b, emit=[1, 0, 1])
    ws = rt.workspace(cfg, nb)
    ids = model.step(nf.Plan.explicit(cfg), [dev(synth.kv_pool(shape, b))], nb,
                     torch.from_numpy(synth.token_ids(b.n_tokens, shape.vocab)).cuda(), ws).cpu().numpy()
    assert ids[1] == -1 and ids[0] >= 0 and ids[2] >= 0


def test_layer_70b_rank_full_batch_sampled(env):
    """configs[2] at full size on one GPU: one LLaMA-2-70B TP8 rank's shards
    (8/1 heads, F 3584, D 8192) over the B_dense=2048 steady-state batch
    (1365 decode + 171-token chunk + 512 prompt) in the bench's c3rank OVERLAP
    launch configuration (132/16 SMs, shares 1:1); sampled requests (decode and
    both prefill requests) against the oracle."""
    nf, rt = env
    shape = synth.shape_with(synth.SHAPES["llama2-70b"], n_q_heads=8, n_kv_heads=1, d_ffn=28672 // 8)
    b = synth.workload_batch(2048, 512, 1024)
    w = synth.layer_weights(shape, 0, seed=0)
    x = synth.activations(shape, b.n_tokens, seed=1)
    cfg = rt.cfg_from_shape(shape)
    nb = nf.Batch.from_any(b)
    packed = rt.pack_layer(cfg, device_weights(w))
    pool_d = dev_bits(synth.kv_pool_bits(shape, b, seed=2))
    plan = nf.Plan.explicit(cfg, mode=nf.OVERLAP, shares=(1, 1), sm=[132, 16, 132, 132, 132, 132, 8])
    out = host(rt.layer_forward(plan, cfg, packed, pool_d, nb, dev(x)))
    torch.cuda.synchronize()
    assert np.isfinite(out).all()
    reqs = [0, 3, 500, 1000, 1364, 1365, 1366]
    sub, pool = compact_case(shape, b, reqs)
    rows = token_rows(b, reqs)
    ref = OL.decoder_layer(x[rows], w, pool, sub, shape)
    assert_close(out[rows], ref, what="70B TP8 rank full batch sampled")


@pytest.mark.parametrize("q_len,prefix", [([1], [0]), ([1], [511]), ([77], [0]), ([1, 1, 1], [15, 16, 17]),
                                          ([40, 24], [0, 100])])
def test_model_step_degenerate_batches(env, q_len, prefix):
    """Degenerate compositions through nf_model_step in every mode: a single
    decode request (empty second nano-batch), a first token (single-key
    context), prefill only, decode only."""
    nf, rt = env
    shape = synth.shape_with(synth.SHAPES["c1"], n_layers=2, vocab=4096)
    b = synth.make_batch(q_len, prefix, seed=6, pool_slack=2)
    W = synth.model_weights(shape, seed=0)
    toks = synth.token_ids(b.n_tokens, shape.vocab)
    pools = [synth.kv_pool(shape, b, seed=2, layer=l) for l in range(2)]
    ids_ref, logits, _ = OL.model_step(toks, W, [OL.as_pool(p) for p in pools], b, shape, return_logits=True)
    cfg = rt.cfg_from_shape(shape)
    layers = [rt.pack_layer(cfg, device_weights(W["layers"][l])) for l in range(2)]
    model = rt.Model(cfg, dev(W["embed"]), layers, rt.pack_lm_head(cfg, dev(W["lm_head"]), dev(W["final_norm"])))
    nb = nf.Batch.from_any(b)
    ws = rt.workspace(cfg, nb)
    srt = np.sort(logits, axis=1)
    sure = srt[:, -1] - srt[:, -2] > 0.1
    for mode, shares, bal in [(0, (1,), 0), (1, (1, 1), 2), (2, (1, 1), 2), (2, (1, 3), 0)]:
        ids = model.step(nf.Plan.explicit(cfg, mode=mode, shares=shares, balance=bal), [dev(p) for p in pools], nb,
                         torch.from_numpy(toks).cuda(), ws).cpu().numpy()
        assert ids.shape == (b.n_req,) and ((ids >= 0) & (ids < shape.vocab)).all()
        assert np.array_equal(ids[sure], ids_ref[sure]), (mode, shares, bal)


def _device_pages_to_compact(b, reqs, pool_d):
    """Sub-batch of `reqs` with a float64 host pool holding their cached pages copied
    from the device pool (taken before the step appends this step's K/V)."""
    sub = synth.make_batch(b.q_len[reqs], b.kv_prefix[reqs], permute=False)
    pool = np.zeros((sub.n_pages_pool,) + tuple(pool_d.shape[1:]))
    for i, r in enumerate(reqs):
        src = torch.as_tensor(b.page_ids[b.page_indptr[r]:b.page_indptr[r + 1]].astype(np.int64), device="cuda")
        dst = sub.page_ids[sub.page_indptr[i]:sub.page_indptr[i + 1]]
        pool[dst] = pool_d[src[:len(dst)]].float().cpu().numpy()
    return sub, pool


def test_model_step_8b_full_teacher_forced(env):
    """The benched step itself (configs[1]: LLaMA-3-8B shape, 32 layers, B_dense 2048,
    OVERLAP plan of the bench, CUDA graph off because of the inspection outputs):
    teacher-forced per-layer parity on layers {0, 1, 15, 31} -- the oracle
    layer l on the GPU's own bf16 input of layer l, sampled requests -- and the
    LM-head logits of sampled requests against the oracle head on the GPU's final
    hidden state, plus argmax agreement with the GPU's own logits.  Weights and KV
    are drawn on the device (seeded) and copied to the host for the oracle."""
    nf, rt = env
    shape = synth.SHAPES["llama3-8b"]
    L, D, F, hd, Hq, Hk, V = (shape.n_layers, shape.d_model, shape.d_ffn, shape.head_dim, shape.n_q_heads,
                              shape.n_kv_heads, shape.vocab)
    b = synth.workload_batch(2048, 1024, 512)
    g = torch.Generator(device="cuda")
    g.manual_seed(11)

    def randn(s, std=1.0, mean=0.0):
        return torch.empty(s, dtype=torch.bfloat16, device="cuda").normal_(mean, std, generator=g)

    check = [0, 1, 15, 31]
    cfg = rt.cfg_from_shape(shape)
    layers, kept = [], {}
    for l in range(L):
        w = {"attn_norm": randn((D,), 0.1, 1.0), "w_q": randn((Hq * hd, D), D ** -0.5),
             "w_k": randn((Hk * hd, D), D ** -0.5), "w_v": randn((Hk * hd, D), D ** -0.5),
             "w_o": randn((D, Hq * hd), (Hq * hd) ** -0.5), "ffn_norm": randn((D,), 0.1, 1.0),
             "w_gate": randn((F, D), D ** -0.5), "w_up": randn((F, D), D ** -0.5), "w_down": randn((D, F), F ** -0.5)}
        layers.append(rt.pack_layer(cfg, w))
        if l in check:
            kept[l] = {k: host(v) for k, v in w.items()}
        del w
    embed, lm, fnorm = randn((V, D)), randn((V, D), D ** -0.5), randn((D,), 0.1, 1.0)
    model = rt.Model(cfg, embed, layers, rt.pack_lm_head(cfg, lm, fnorm))
    pools = [randn((b.n_pages_pool, 2, Hk, 16, hd)) for _ in range(L)]
    n_dec = int((b.q_len == 1).sum())
    reqs = [0, 1, n_dec // 2, n_dec - 1, n_dec, n_dec + 1]
    compact = {l: _device_pages_to_compact(b, reqs, pools[l]) for l in check}
    tok = torch.randint(0, V, (b.n_tokens,), dtype=torch.int32, device="cuda", generator=g)
    nb = nf.Batch.from_any(b)
    ws = rt.workspace(cfg, nb)
    plan = nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1), sm=[116, 32, 116, 116, 116, 116, 8], balance=2)
    ids, lg, hs = model.step_inspect(plan, pools, nb, tok, ws)
    torch.cuda.synchronize()
    rows = token_rows(b, reqs)
    for l in check:
        sub, pool = compact[l]
        x_in = host(hs[l][torch.as_tensor(rows, device="cuda")])
        ref = OL.decoder_layer(x_in, kept[l], pool, sub, shape)
        out = host(hs[l + 1][torch.as_tensor(rows, device="cuda")])
        rms = float(np.sqrt(np.mean(ref ** 2)))
        rel, mx = assert_close(out, ref, what=f"8B step layer {l} (teacher-forced, output RMS {rms:.2f})", scale_rms=True)
        print(f"layer {l}: output RMS {rms:.2f}, rel L2 {rel:.3e} max abs {mx:.3e}")
    # logits of the sampled requests (all requests emit: logits row i = request i)
    last = np.concatenate([[0], np.cumsum(b.q_len)])[1:] - 1
    xf = host(hs[L][torch.as_tensor(last[reqs], device="cuda")])
    ref_lg = OL.rmsnorm(xf, host(fnorm), shape.rms_eps) @ host(lm).T
    out_lg = host(lg[torch.as_tensor(reqs, device="cuda")])
    rel, mx = errors(out_lg, ref_lg)
    assert rel <= 1e-2 and mx <= 0.25, f"logits rel L2 {rel:.3e} max abs {mx:.3e}"
    ids_h = ids.cpu().numpy()
    full = host(lg)
    top = np.sort(full, axis=1)
    clear = top[:, -1] - top[:, -2] > 0.05
    assert np.array_equal(ids_h[clear], np.argmax(full, axis=1)[clear])
    # the inspection pass did not change the result of the plain step
    ids2 = model.step(plan, pools, nb, tok, ws).cpu().numpy()
    assert np.array_equal(ids_h, ids2)


@pytest.mark.parametrize("impl", ["stream", "fused", "ws"])
def test_decode_impl_variants_vs_oracle(env, impl, monkeypatch):
    """Every decode kernel (stream = default, fused = item-walking, ws = warp-specialised;
    NF_DECODE_IMPL) against the oracle on the 8B
    shape (GQA 4) and a 70B TP8 rank (GQA 8, one KV head): mixed lengths incl. partial last
    pages, SM budgets 1 / 7 / 148; bit-identical across SM budgets (same per-item order)."""
    monkeypatch.setenv("NF_DECODE_IMPL", impl)
    for shape in (synth.SHAPES["llama3-8b"], synth.shape_with(synth.SHAPES["llama2-70b"], n_q_heads=8, n_kv_heads=1,
                                                             d_ffn=3584)):
        q_len = [1] * 37
        prefix = [0, 1, 15, 16, 17, 31, 32, 33, 100, 255, 256, 257, 1000, 1535] + list(range(40, 40 + 23 * 37, 37))
        b, pool, q = _attn_case(shape, q_len, prefix, seed=5)
        ref = OL.paged_attention(q, pool, b)
        outs = []
        for sm in (1, 7, 148):
            out = _run_attn(env, shape, b, pool, q, sm_dec=sm)
            assert_close(out.reshape(ref.shape), ref, what=f"decode {impl} sm={sm} {shape.name}")
            outs.append(out)
        assert all(np.array_equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("dec,net,tp", [(32, 8, 1), (16, 16, 8), (148, 16, 8)])
def test_overlap_partitions_are_sm_disjoint(env, dec, net, tp):
    """Execution-unit scheduling evidence (SURVEY §5 %smid check): probe CTAs
    launched on an OVERLAP plan's memory / compute / network partition streams run on
    pairwise disjoint SM sets of the planned sizes (green contexts), covering the GPU."""
    nf, rt = env
    shape = synth.SHAPES["llama2-70b"] if tp > 1 else synth.SHAPES["llama3-8b"]
    cfg = rt.cfg_from_shape(shape, tp_size=tp)
    comm = nf.comm_create_loopback(tp, 0) if tp > 1 else None
    plan = nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1), sm=[148, dec, 148, 148, 148, 148, net],
                            n_dense=2 if tp > 1 else 0)
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    cnt = plan.probe_partitions(rt.stream_handle(), comm, n_sm)
    sets = [set(np.nonzero(c)[0].tolist()) for c in cnt]
    if comm:
        nf.comm_destroy(comm)
    note = plan.runtime_note()
    mem, cmp_, netp = sets
    assert not (mem & cmp_) and not (mem & netp) and not (cmp_ & netp), note
    if dec < n_sm:
        assert len(mem) == (dec + 7) // 8 * 8, (len(mem), note)
    else:
        assert not mem and "no memory partition" in note
    if tp > 1:
        assert len(netp) == (net + 7) // 8 * 8, (len(netp), note)
    assert len(mem | cmp_ | netp) == n_sm
    print(note, {k: len(v) for k, v in zip(("memory", "compute", "network"), sets)})


def test_decode_row_stream_loader_bit_exact(env, monkeypatch):
    """The item-walking kernel's two loaders (NF_DECODE_IMPL=fused; row stream NF_DEC_ROWS=1
    vs item walk NF_DEC_ROWS=0) feed the same pages in the same order to the same math:
    bit-identical outputs, at several SM budgets and through a full OVERLAP layer (the rows
    are built once per step and reused)."""
    monkeypatch.setenv("NF_DECODE_IMPL", "fused")
    shape = synth.SHAPES["llama3-8b"]
    q_len = [1] * 41
    prefix = [0, 1, 15, 16, 17, 31, 32, 33, 100, 255, 256, 257, 1000, 1535, 511, 512] + list(range(40, 40 + 25 * 29, 29))
    b, pool, q = _attn_case(shape, q_len, prefix, seed=9)
    for sm in (3, 32, 148):
        monkeypatch.setenv("NF_DEC_ROWS", "0")
        ref = _run_attn(env, shape, b, pool, q, sm_dec=sm)
        monkeypatch.setenv("NF_DEC_ROWS", "1")
        out = _run_attn(env, shape, b, pool, q, sm_dec=sm)
        assert np.array_equal(ref, out), sm
    nf, rt = env
    sh = synth.shape_with(synth.SHAPES["llama3-8b"], n_layers=3)
    bb = synth.workload_batch(512, 1024, 512)
    w, x, pl = _layer_case(sh, bb)
    outs = []
    for rows in ("0", "1"):
        monkeypatch.setenv("NF_DEC_ROWS", rows)
        o, _ = _gpu_layer(env, sh, bb, w, x, pl, 2, (1, 1))
        outs.append(o)
    assert np.array_equal(outs[0], outs[1])
