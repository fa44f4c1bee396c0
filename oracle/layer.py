"""Float64 oracle of the decoder layer over a mixed, paged batch — test infrastructure only.

Follows PAPER.md:141 (inference workflow), :161 (attention), :183 and
:577-579 (head-parallel TP), :547-548 (nano-batch O1-col / O2-row), :663
(paged KV), with the readings of SURVEY.md §8c (A-1 .. A-15, restated in
DESIGN.md "Readings of the paper").

Inputs are bf16-valued float32 arrays from ``synth``; everything is upcast to
float64 here.  Products use numpy matmul (a library primitive for the
definition y = x W^T); there is no blocking, fusion or reordering beyond the
definitions.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import numpy as np

from . import metadata as md


def f64(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64)


# ---------------------------------------------------------------- norm / rope
def rmsnorm(x, gamma, eps: float) -> np.ndarray:
    """Pre-RMSNorm (reading A-1, eps A-2): x / sqrt(mean(x^2) + eps) * gamma."""
    x = f64(x)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * f64(gamma)


def rope(x, pos, theta: float) -> np.ndarray:
    """Rotary embedding, rotate-half convention (reading A-4; PAPER.md:630 names RoPE).

    x: [T, H, hd]; for i < hd/2, f_i = theta^(-2i/hd), a = pos * f_i,
    (x_i, x_{i+hd/2}) <- (x_i cos a - x_{i+hd/2} sin a, x_{i+hd/2} cos a + x_i sin a).
    """
    x = f64(x)
    hd = x.shape[-1]
    half = hd // 2
    i = np.arange(half, dtype=np.float64)
    f = float(theta) ** (-2.0 * i / hd)
    a = f64(pos)[:, None] * f[None, :]
    c, s = np.cos(a)[:, None, :], np.sin(a)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(z) -> np.ndarray:
    """SiLU(z) = z / (1 + e^-z) (reading A-3)."""
    z = f64(z)
    return z / (1.0 + np.exp(-z))


# ---------------------------------------------------------------- paged KV
def as_pool(pool) -> np.ndarray:
    """float64 copy of a (bf16-valued) KV pool for the oracle."""
    return np.array(pool, dtype=np.float64)


def kv_append(pool: np.ndarray, k, v, batch, page_size: int = 16) -> None:
    """Write the new tokens' (post-RoPE) K and V into their page slots,
    before attention (reading A-6; "concatenated into the
    existing KV-cache"; page layout PAPER.md:663 / A-7).
    pool: [n_pages, 2, kv_heads, page, hd] (modified in place)."""
    if pool.dtype != np.float64:
        raise TypeError("oracle KV pool must be float64 (use oracle.layer.as_pool)")
    pages, offs = md.write_slots(batch.q_len, batch.kv_prefix, batch.page_indptr,
                                 batch.page_ids, page_size)
    pool[pages, 0, :, offs, :] = k
    pool[pages, 1, :, offs, :] = v


def gather_kv(pool: np.ndarray, batch, r: int, n: int, page_size: int = 16):
    """K_r, V_r for logical positions 0..n-1 of request r through the page table."""
    j = np.arange(n)
    pages = batch.page_ids[batch.page_indptr[r] + j // page_size]
    K = pool[pages, 0, :, j % page_size, :]   # [n, kh, hd]
    V = pool[pages, 1, :, j % page_size, :]
    return f64(K), f64(V)


def paged_attention(q, pool, batch, page_size: int = 16, return_probs: bool = False):
    """Causal GQA attention through the page table (GQA).

    For token t of request r at position P and query head h:
      logits_j = q[t,h] . K_r[j, g(h)] / sqrt(hd),  j = 0..P
      o[t,h]   = sum_j softmax(logits)_j V_r[j, g(h)]
    with g(h) = floor(h / R), R = qh/kh (reading A-5).  Softmax subtracts the
    row max.  q: [T, qh, hd] -> o [T, qh, hd].
    """
    q = f64(q)
    T, qh, hd = q.shape
    kh = pool.shape[2]
    R = qh // kh
    pos = md.positions(batch.q_len, batch.kv_prefix)
    ind = md.qo_indptr(batch.q_len)
    out = np.zeros_like(q)
    probs = [] if return_probs else None
    g = np.arange(qh) // R
    for r in range(batch.n_req):
        t0, t1 = int(ind[r]), int(ind[r + 1])
        if t1 == t0:
            continue
        n = int(batch.kv_prefix[r]) + (t1 - t0)
        K, V = gather_kv(pool, batch, r, n, page_size)
        Kh = K[:, g, :]   # [n, qh, hd] key of each query head's group
        Vh = V[:, g, :]
        for t in range(t0, t1):
            P = int(pos[t])
            logits = np.einsum("hd,jhd->hj", q[t], Kh[:P + 1]) / np.sqrt(hd)
            logits -= logits.max(axis=1, keepdims=True)
            p = np.exp(logits)
            p /= p.sum(axis=1, keepdims=True)
            out[t] = np.einsum("hj,jhd->hd", p, Vh[:P + 1])
            if return_probs:
                probs.append(p)
    return (out, probs) if return_probs else out


# ---------------------------------------------------------------- layer
def qkv(h, w):
    return h @ f64(w["w_q"]).T, h @ f64(w["w_k"]).T, h @ f64(w["w_v"]).T


def attention_block(x, w: Dict[str, np.ndarray], pool: np.ndarray, batch, shape,
                    page_size: int = 16) -> np.ndarray:
    """Steps 1-6 of ``decoder_layer``: h1 = x + Attn(RMSNorm(x) * g_attn) W_o^T
    (readings A-1, A-4..A-6); appends the step's K/V to ``pool``."""
    x = f64(x)
    T = x.shape[0]
    hd, qh, kh = shape.head_dim, shape.n_q_heads, shape.n_kv_heads
    pos = md.positions(batch.q_len, batch.kv_prefix)
    h = rmsnorm(x, w["attn_norm"], shape.rms_eps)
    q, k, v = qkv(h, w)
    q = rope(q.reshape(T, qh, hd), pos, shape.rope_theta)
    k = rope(k.reshape(T, kh, hd), pos, shape.rope_theta)
    v = v.reshape(T, kh, hd)
    kv_append(pool, k, v, batch, page_size)
    o = paged_attention(q, pool, batch, page_size).reshape(T, qh * hd)
    return x + o @ f64(w["w_o"]).T


def decoder_layer(x, w: Dict[str, np.ndarray], pool: np.ndarray, batch, shape,
                  page_size: int = 16) -> np.ndarray:
    """One LLaMA-style decoder layer (readings A-1..A-6).

    1. h = RMSNorm(x) * g_attn
    2. q, k, v = h W_q^T, h W_k^T, h W_v^T
    3. RoPE on q, k at pos
    4. KV append (before attention)
    5. o = paged causal GQA attention
    6. h1 = x + o W_o^T
    7. m = SiLU(h2 W_g^T) * (h2 W_u^T), h2 = RMSNorm(h1) * g_ffn
    8. out = h1 + m W_d^T
    ``pool`` is updated in place (the appended K/V).
    """
    h1 = attention_block(x, w, pool, batch, shape, page_size)
    h2 = rmsnorm(h1, w["ffn_norm"], shape.rms_eps)
    m = silu(h2 @ f64(w["w_gate"]).T) * (h2 @ f64(w["w_up"]).T)
    return h1 + m @ f64(w["w_down"]).T


def sub_batch(batch, r0: int, r1: int):
    """Requests [r0, r1) of a batch sharing the same pool and page ids."""
    import synth
    return synth.Batch(batch.q_len[r0:r1].copy(), batch.kv_prefix[r0:r1].copy(),
                       (batch.page_indptr[r0:r1 + 1] - batch.page_indptr[r0]).copy(),
                       batch.page_ids[batch.page_indptr[r0]:batch.page_indptr[r1]].copy(),
                       batch.n_pages_pool)


def decoder_layer_nano(x, w, pool, batch, shape, req_cuts: Sequence[int], page_size: int = 16):
    """The same layer run nano-batch by nano-batch over request ranges
    [req_cuts[i], req_cuts[i+1]) in order (nano-batches of
    user requests; within a nano-batch operations are sequential).  Must equal
    ``decoder_layer`` (split invariance)."""
    ind = md.qo_indptr(batch.q_len)
    out = np.zeros(f64(x).shape)
    for a, b in zip(req_cuts[:-1], req_cuts[1:]):
        if b <= a:
            continue
        t0, t1 = int(ind[a]), int(ind[b])
        out[t0:t1] = decoder_layer(f64(x)[t0:t1], w, pool, sub_batch(batch, a, b), shape, page_size)
    return out


# ---------------------------------------------------------------- TP algebra
def shard_weights(w, shape, N: int, rank: int):
    """Rank `rank`'s shards under head-parallel TP:
    column W_q/W_k/W_v by heads, column O (rows of W_o), row O (columns of
    W_o), column gate/up, row down."""
    hd, qh, kh, D, F = shape.head_dim, shape.n_q_heads, shape.n_kv_heads, shape.d_model, shape.d_ffn
    qs, ks, ds, fs = qh // N * hd, kh // N * hd, D // N, F // N
    return {
        "attn_norm": w["attn_norm"], "ffn_norm": w["ffn_norm"],
        "w_q": w["w_q"][rank * qs:(rank + 1) * qs],
        "w_k": w["w_k"][rank * ks:(rank + 1) * ks],
        "w_v": w["w_v"][rank * ks:(rank + 1) * ks],
        "w_o_col": w["w_o"][rank * ds:(rank + 1) * ds, :],      # [D/N, D]   output columns
        "w_o_row": w["w_o"][:, rank * qs:(rank + 1) * qs],      # [D, D/N]   input rows (heads)
        "w_gate": w["w_gate"][rank * fs:(rank + 1) * fs],
        "w_up": w["w_up"][rank * fs:(rank + 1) * fs],
        "w_down": w["w_down"][:, rank * fs:(rank + 1) * fs],
    }


def decoder_layer_tp(x, w, pools: List[np.ndarray], batch, shape, N: int, half_cut_req: int,
                     page_size: int = 16):
    """Sharded-mode oracle (fp64): every rank computes its heads;
    H1 (requests [0, half_cut_req)) uses AG(attn) -> O1-col -> AG;
    H2 uses O2-row -> AR; FFN: column gate/up, row down, AR.
    AG = concatenation, AR = sum.  pools[r] holds rank r's KV heads.
    Must equal ``decoder_layer``."""
    x = f64(x)
    T = x.shape[0]
    hd, qh, kh, D = shape.head_dim, shape.n_q_heads, shape.n_kv_heads, shape.d_model
    ind = md.qo_indptr(batch.q_len)
    cut = int(ind[half_cut_req])
    pos = md.positions(batch.q_len, batch.kv_prefix)
    shards = [shard_weights(w, shape, N, r) for r in range(N)]
    h = rmsnorm(x, w["attn_norm"], shape.rms_eps)
    o_local = []
    for r in range(N):
        s = shards[r]
        q = rope((h @ f64(s["w_q"]).T).reshape(T, qh // N, hd), pos, shape.rope_theta)
        k = rope((h @ f64(s["w_k"]).T).reshape(T, kh // N, hd), pos, shape.rope_theta)
        v = (h @ f64(s["w_v"]).T).reshape(T, kh // N, hd)
        kv_append(pools[r], k, v, batch, page_size)
        o_local.append(paged_attention(q, pools[r], batch, page_size).reshape(T, qh // N * hd))
    h1 = np.zeros_like(x)
    # H1: AG of attention outputs, column-parallel O, AG of O outputs
    o_full = np.concatenate([o[:cut] for o in o_local], axis=1)              # AG
    h1[:cut] = x[:cut] + np.concatenate([o_full @ f64(s["w_o_col"]).T for s in shards], axis=1)  # O1-col + AG
    # H2: row-parallel O with AllReduce
    h1[cut:] = x[cut:] + sum(o_local[r][cut:] @ f64(shards[r]["w_o_row"]).T for r in range(N))
    h2 = rmsnorm(h1, w["ffn_norm"], shape.rms_eps)
    out = h1.copy()
    for r in range(N):
        s = shards[r]
        m = silu(h2 @ f64(s["w_gate"]).T) * (h2 @ f64(s["w_up"]).T)
        out += m @ f64(s["w_down"]).T                                        # AR (sum)
    return out


# ---------------------------------------------------------------- model step
def emit_rows(batch, emit: Optional[np.ndarray] = None) -> np.ndarray:
    """Row of the last token of each request (the one whose logits are
    sampled; reading A-15 / C8).  -1 where the request does not emit."""
    ind = md.qo_indptr(batch.q_len)
    rows = ind[1:] - 1
    if emit is not None:
        rows = np.where(np.asarray(emit) != 0, rows, -1)
    return rows


def model_step(token_ids, weights, pools: List[np.ndarray], batch, shape, emit=None,
               page_size: int = 16, return_logits: bool = False, route_logits: Optional[list] = None):
    """x0 = E[token_ids] -> L decoder layers -> RMSNorm * g_final -> logits of
    each emitting request's last row -> greedy argmax, lowest index on ties
    (reading A-15; LM head is our addition C8).  Returns next ids [n_req]
    (-1 where not emitted).  MoE shapes use oracle.moe's layer; their router
    logits per layer are appended to ``route_logits`` when given."""
    x = f64(weights["embed"])[np.asarray(token_ids)]
    for l, w in enumerate(weights["layers"]):
        if getattr(shape, "n_experts", 0):       # Mixtral-shape MoE layer (oracle.moe)
            from . import moe
            x, _, _, lg = moe.moe_decoder_layer(x, w, pools[l], batch, shape, page_size, return_route=True)
            if route_logits is not None:
                route_logits.append(lg)
        else:
            x = decoder_layer(x, w, pools[l], batch, shape, page_size)
    rows = emit_rows(batch, emit)
    sel = rows[rows >= 0]
    hN = rmsnorm(x[sel], weights["final_norm"], shape.rms_eps)
    logits = hN @ f64(weights["lm_head"]).T
    ids = np.full(batch.n_req, -1, dtype=np.int64)
    ids[rows >= 0] = np.argmax(logits, axis=1)
    if return_logits:
        return ids, logits, x
    return ids
