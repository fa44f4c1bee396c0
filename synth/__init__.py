"""Seeded synthetic workload generators shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no norm, no RoPE, no
attention, no projection).  It only produces inputs:

* model shape tables for the BASELINE.json configs (SURVEY.md §8 shape key),
* the steady-state batch composition of a constant-length workload
  (Eq. ``eq:dense-batch-size``; recipe in SURVEY.md §8d),
* paged-KV page tables (random physical page permutation),
* seeded random tensors rounded to bf16 (values the GPU stores exactly).

Both ``oracle/`` and the tests import it; the product package does not need
it (bench.py generates its large tensors on the device with torch RNG using
the same distributions).
"""
from __future__ import annotations

import dataclasses
import zlib
from typing import Dict, List, Optional, Sequence

import numpy as np

PAGE_SIZE = 16  # tokens per KV page, PAPER.md:663 ("e.g., 16 tokens")


# --------------------------------------------------------------------------
# Model shapes (SURVEY.md §8 shape key; BASELINE.json configs)
# --------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class ModelShape:
    name: str
    d_model: int
    n_layers: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    d_ffn: int
    vocab: int
    rope_theta: float
    rms_eps: float = 1e-5          # reading A-2
    page_size: int = PAGE_SIZE
    n_experts: int = 0             # 0 = dense FFN; > 0: MoE FFN (readings A-20..A-23)
    top_k: int = 2

    @property
    def qkv_out(self) -> int:
        return (self.n_q_heads + 2 * self.n_kv_heads) * self.head_dim


SHAPES: Dict[str, ModelShape] = {
    # BASELINE.json configs[0]: D=512, 8 Q / 2 KV heads, FFN 1376, one layer (A-9: hd = D/Hq)
    "c1": ModelShape("c1-tiny", 512, 1, 8, 2, 64, 1376, 32000, 1e4),
    # configs[1]: LLaMA-3-8B shape
    "llama3-8b": ModelShape("llama3-8b", 4096, 32, 32, 8, 128, 14336, 128256, 5e5),
    # configs[2]: LLaMA-2-70B shape (F = 28672 implied by Table 2)
    "llama2-70b": ModelShape("llama2-70b", 8192, 80, 64, 8, 128, 28672, 32000, 1e4),
    # configs[3]: Mixtral-8x7B shape (public config: 8 experts, top-2, F 14336 per expert, theta 1e6)
    "mixtral-8x7b": ModelShape("mixtral-8x7b", 4096, 32, 32, 8, 128, 14336, 32000, 1e6, n_experts=8, top_k=2),
    # tiny MoE layer for parity tests (configs[0] attention shape, 8 experts, ragged F)
    "c1-moe": ModelShape("c1-moe", 512, 1, 8, 2, 64, 704, 32000, 1e4, n_experts=8, top_k=2),
}


def shape_with(base: ModelShape, **kw) -> ModelShape:
    return dataclasses.replace(base, **kw)


# --------------------------------------------------------------------------
# Batch description (request-major token rows)
# --------------------------------------------------------------------------
@dataclasses.dataclass
class Batch:
    q_len: np.ndarray        # int32 [n_req]  1 = decode, >1 = prefill chunk
    kv_prefix: np.ndarray    # int32 [n_req]  tokens cached before this step
    page_indptr: np.ndarray  # int32 [n_req+1]
    page_ids: np.ndarray     # int32 [page_indptr[-1]]
    n_pages_pool: int

    @property
    def n_req(self) -> int:
        return int(self.q_len.shape[0])

    @property
    def n_tokens(self) -> int:
        return int(self.q_len.sum())


def steady_state_composition(b_dense: int, p: int, d: int):
    """Steady state of a constant p-in / d-out workload at dense batch b_dense.

    B_req = B_dense (d+1)/(p+d)  (Eq. dense-batch-size);
    n_dec = floor(B_req d/(d+1) + 1/2); prefill tokens = B_dense - n_dec are
    packed as whole prompts of p tokens plus one tail chunk.
    Returns (n_dec, tail_chunk_len, n_full_prompts).
    """
    # exact rational arithmetic: B_req * d/(d+1) = b_dense * d / (p + d)
    n_dec = (2 * b_dense * d + (p + d)) // (2 * (p + d))
    n_pre = b_dense - n_dec
    if p == 0:
        raise ValueError("p must be > 0")
    n_full, tail = divmod(n_pre, p)
    return int(n_dec), int(tail), int(n_full)


def make_batch(q_len: Sequence[int], kv_prefix: Sequence[int], *, seed: int = 3,
               pool_slack: int = 0, page_size: int = PAGE_SIZE,
               permute: bool = True) -> Batch:
    """Allocate ceil((prefix+q_len)/page) pages per request from a randomly
    permuted pool (seed 3)."""
    q_len = np.asarray(q_len, dtype=np.int32)
    kv_prefix = np.asarray(kv_prefix, dtype=np.int32)
    need = (kv_prefix.astype(np.int64) + q_len + page_size - 1) // page_size
    indptr = np.zeros(len(q_len) + 1, dtype=np.int32)
    indptr[1:] = np.cumsum(need)
    total = int(indptr[-1])
    pool = total + pool_slack
    if permute:
        perm = np.random.default_rng(seed).permutation(pool).astype(np.int32)
    else:
        perm = np.arange(pool, dtype=np.int32)
    return Batch(q_len, kv_prefix, indptr, perm[:total].copy(), pool)


def workload_batch(b_dense: int, p: int, d: int, *, seed_ctx: int = 4, seed_pages: int = 3,
                   pool_slack: int = 0) -> Batch:
    """Token order [decode...][tail chunk][full prompts...].
    Decode contexts c_i = p + floor(i d / n_dec), shuffled with seed 4."""
    n_dec, tail, n_full = steady_state_composition(b_dense, p, d)
    ctx = np.array([p + (i * d) // n_dec for i in range(n_dec)], dtype=np.int64)
    np.random.default_rng(seed_ctx).shuffle(ctx)
    q_len: List[int] = [1] * n_dec
    prefix: List[int] = list(ctx)
    if tail:
        q_len.append(tail)
        prefix.append(p - tail)
    q_len += [p] * n_full
    prefix += [0] * n_full
    return make_batch(q_len, prefix, seed=seed_pages, pool_slack=pool_slack)


def c1_batch(seed_pages: int = 3) -> Batch:
    """BASELINE.json configs[0]: 64 decode requests with 128 cached tokens each
    (reading A-8) plus one 64-token prompt; pool of 640 pages."""
    q_len = [1] * 64 + [64]
    prefix = [128] * 64 + [0]
    b = make_batch(q_len, prefix, seed=seed_pages, pool_slack=640 - 580)
    return b


# --------------------------------------------------------------------------
# bf16 helpers (storage format only)
# --------------------------------------------------------------------------
def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even float32 -> bf16 bit pattern (uint16)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = np.isnan(a)
    if nan.any():
        r[nan] = 0x7FC0
    return r


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    b = np.ascontiguousarray(b, dtype=np.uint16)
    return (b.astype(np.uint32) << 16).view(np.float32)


def round_bf16(a: np.ndarray) -> np.ndarray:
    return bf16_bits_to_f32(f32_to_bf16_bits(a))


def _rng(seed: int, name: str) -> np.random.Generator:
    return np.random.default_rng([seed, zlib.crc32(name.encode())])


def randn_bf16(shape, seed: int, name: str, scale: float = 1.0, mean: float = 0.0) -> np.ndarray:
    """N(mean, scale^2) rounded to bf16, returned as float32 holding bf16 values."""
    x = _rng(seed, name).standard_normal(size=shape, dtype=np.float32)
    if scale != 1.0:
        x *= np.float32(scale)
    if mean != 0.0:
        x += np.float32(mean)
    return round_bf16(x)


# --------------------------------------------------------------------------
# Weights / activations / KV (SURVEY.md §8d value distributions)
# --------------------------------------------------------------------------
def layer_weights(shape: ModelShape, layer: int, seed: int = 0) -> Dict[str, np.ndarray]:
    """Unsharded, unpacked weights of one decoder layer, [out, in] row-major.
    W ~ N(0, 1/fan_in); gamma = 1 + 0.1 N(0,1)."""
    D, F, hd = shape.d_model, shape.d_ffn, shape.head_dim
    Hq, Hk = shape.n_q_heads, shape.n_kv_heads
    p = f"L{layer}."
    if shape.n_experts:
        E = shape.n_experts
        return {
            "attn_norm": randn_bf16((D,), seed, p + "attn_norm", 0.1, 1.0),
            "w_q": randn_bf16((Hq * hd, D), seed, p + "w_q", D ** -0.5),
            "w_k": randn_bf16((Hk * hd, D), seed, p + "w_k", D ** -0.5),
            "w_v": randn_bf16((Hk * hd, D), seed, p + "w_v", D ** -0.5),
            "w_o": randn_bf16((D, Hq * hd), seed, p + "w_o", (Hq * hd) ** -0.5),
            "ffn_norm": randn_bf16((D,), seed, p + "ffn_norm", 0.1, 1.0),
            "w_router": randn_bf16((E, D), seed, p + "w_router", D ** -0.5),
            "w_gate": randn_bf16((E, F, D), seed, p + "w_gate", D ** -0.5),
            "w_up": randn_bf16((E, F, D), seed, p + "w_up", D ** -0.5),
            "w_down": randn_bf16((E, D, F), seed, p + "w_down", F ** -0.5),
        }
    return {
        "attn_norm": randn_bf16((D,), seed, p + "attn_norm", 0.1, 1.0),
        "w_q": randn_bf16((Hq * hd, D), seed, p + "w_q", D ** -0.5),
        "w_k": randn_bf16((Hk * hd, D), seed, p + "w_k", D ** -0.5),
        "w_v": randn_bf16((Hk * hd, D), seed, p + "w_v", D ** -0.5),
        "w_o": randn_bf16((D, Hq * hd), seed, p + "w_o", (Hq * hd) ** -0.5),
        "ffn_norm": randn_bf16((D,), seed, p + "ffn_norm", 0.1, 1.0),
        "w_gate": randn_bf16((F, D), seed, p + "w_gate", D ** -0.5),
        "w_up": randn_bf16((F, D), seed, p + "w_up", D ** -0.5),
        "w_down": randn_bf16((D, F), seed, p + "w_down", F ** -0.5),
    }


def model_weights(shape: ModelShape, seed: int = 0, n_layers: Optional[int] = None):
    L = shape.n_layers if n_layers is None else n_layers
    return {
        "embed": randn_bf16((shape.vocab, shape.d_model), 1, "embed"),
        "layers": [layer_weights(shape, l, seed) for l in range(L)],
        "final_norm": randn_bf16((shape.d_model,), seed, "final_norm", 0.1, 1.0),
        "lm_head": randn_bf16((shape.vocab, shape.d_model), seed, "lm_head", shape.d_model ** -0.5),
    }


def activations(shape: ModelShape, n_tokens: int, seed: int = 1, name: str = "x") -> np.ndarray:
    """Unit-RMS layer input x ~ N(0,1) (seed 1)."""
    return randn_bf16((n_tokens, shape.d_model), seed, name)


def kv_pool(shape: ModelShape, batch: Batch, seed: int = 2, layer: int = 0,
            fill: float = 0.0, n_kv_heads: Optional[int] = None) -> np.ndarray:
    """Paged KV pool [n_pages][2][kv_heads][page][head_dim].
    Slots of the cached prefix hold N(0,1) bf16 values (seed 2); every other
    slot holds `fill` (use NaN as a sentinel for write-map tests)."""
    hk = shape.n_kv_heads if n_kv_heads is None else n_kv_heads
    P, hd = shape.page_size, shape.head_dim
    pool = np.full((batch.n_pages_pool, 2, hk, P, hd), fill, dtype=np.float32)
    for r in range(batch.n_req):
        n = int(batch.kv_prefix[r])
        if n:
            j = np.arange(n)
            pages = batch.page_ids[batch.page_indptr[r] + j // P]
            pool[pages, :, :, j % P, :] = request_kv(shape, r, n, seed, layer, hk)
    return pool


def request_kv(shape: ModelShape, r: int, n: int, seed: int = 2, layer: int = 0,
               n_kv_heads: Optional[int] = None) -> np.ndarray:
    """Cached K/V of request r's first n positions: [n, 2, kv_heads, head_dim]
    (its own RNG stream, so a subset of requests can be regenerated alone)."""
    hk = shape.n_kv_heads if n_kv_heads is None else n_kv_heads
    return randn_bf16((n, 2, hk, shape.head_dim), seed, f"kv{layer}.r{r}")


def kv_pool_bits(shape: ModelShape, batch: Batch, seed: int = 2, layer: int = 0, fill_bits: int = 0,
                 n_kv_heads: Optional[int] = None) -> np.ndarray:
    """Same values as kv_pool, as a bf16 bit-pattern array (uint16) — half the
    host memory, for full-size pools uploaded to the GPU."""
    hk = shape.n_kv_heads if n_kv_heads is None else n_kv_heads
    P, hd = shape.page_size, shape.head_dim
    pool = np.full((batch.n_pages_pool, 2, hk, P, hd), fill_bits, dtype=np.uint16)
    for r in range(batch.n_req):
        n = int(batch.kv_prefix[r])
        if n:
            j = np.arange(n)
            pages = batch.page_ids[batch.page_indptr[r] + j // P]
            pool[pages, :, :, j % P, :] = f32_to_bf16_bits(request_kv(shape, r, n, seed, layer, hk))
    return pool


def cached_slots(batch: Batch, page_size: int = PAGE_SIZE):
    """(page, offset) of every token cached BEFORE the step, request-major."""
    n = batch.kv_prefix.astype(np.int64)
    tot = int(n.sum())
    req = np.repeat(np.arange(batch.n_req), n)
    start = np.concatenate([[0], np.cumsum(n)[:-1]]).astype(np.int64)
    j = np.arange(tot, dtype=np.int64) - np.repeat(start, n)
    pages = batch.page_ids[batch.page_indptr[req] + j // page_size]
    return pages.astype(np.int64), (j % page_size).astype(np.int64)


def token_ids(n_tokens: int, vocab: int, seed: int = 5) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, vocab, size=n_tokens, dtype=np.int64).astype(np.int32)
