"""Float64 oracle of the MoE (Mixtral-8x7B-shape) FFN — test infrastructure only.

PAPER.md:689: "Mixtral is an MoE model, for which the gating operation is
required for expert selection.  We inserted gating into the original
pipeline ... and changed the dimensions of FFN layers."  The paper says
nothing else about the MoE layer, so the operation follows the public
Mixtral-8x7B definition the paper names (readings A-20 .. A-23 in DESIGN.md):

* A-20 gating input: the FFN-normalised hidden state h2 = RMSNorm(h1) * g_ffn
  (the same input the dense FFN of PAPER.md:141 gets);
* A-21 router: logits = h2 W_r^T (W_r [E, D]); top-k experts (k = 2) by logit,
  ties to the lowest expert index; weights = softmax over all E logits
  renormalised over the k selected ones (= softmax over the k selected logits);
* A-22 expert e is the SwiGLU FFN of PAPER.md:141 with its own weights:
  y_e = (SiLU(h2 W_g[e]^T) * (h2 W_u[e]^T)) W_d[e]^T;
  out = h1 + sum_k w_k y_{e_k};  no capacity limit, no token dropping;
* A-23 token grouping (the integer layout the grouped GEMMs consume, our
  design, bit-exact contract with the CUDA path): assignments (t, j) in
  token-major order; expert e's segment starts at a multiple of `tile` rows.

Everything in float64; products by numpy matmul (a library primitive for
y = x W^T).  The TP-sharded form splits every expert's F columns across ranks
(column gate/up, row down + AllReduce as a sum; PAPER.md:183 applied per
expert).
"""
from __future__ import annotations

from typing import Dict, List

import numpy as np

from .layer import f64, rmsnorm, silu


def router_topk(h2, w_router, k: int):
    """Reading A-21.  Returns (ids [T, k] int64, weights [T, k] float64, logits [T, E]).

    ids[t] are the k largest logits in descending order, equal logits ordered
    by lower expert index; weights[t, j] = exp(l_j) / sum_{j' < k} exp(l_j')
    over the selected logits."""
    logits = f64(h2) @ f64(w_router).T
    T, E = logits.shape
    if not 1 <= k <= E:
        raise ValueError("need 1 <= k <= n_experts")
    ids = np.zeros((T, k), dtype=np.int64)
    for t in range(T):
        # stable sort of -logit: equal logits keep ascending expert order
        order = sorted(range(E), key=lambda e: (-logits[t, e], e))
        ids[t] = order[:k]
    sel = np.take_along_axis(logits, ids, axis=1)
    p = np.exp(sel - sel[:, :1])
    return ids, p / p.sum(axis=1, keepdims=True), logits


def expert_ffn(h2, w_gate_e, w_up_e, w_down_e):
    """SwiGLU FFN of one expert (reading A-3, A-22)."""
    h2 = f64(h2)
    return (silu(h2 @ f64(w_gate_e).T) * (h2 @ f64(w_up_e).T)) @ f64(w_down_e).T


def forced_weights(logits, ids):
    """Reading A-21 weights for a given selection: softmax over the selected logits."""
    sel = np.take_along_axis(f64(logits), np.asarray(ids, dtype=np.int64), axis=1)
    p = np.exp(sel - sel.max(axis=1, keepdims=True))
    return p / p.sum(axis=1, keepdims=True)


def moe_ffn(h1, w: Dict[str, np.ndarray], shape, return_route: bool = False, forced_ids=None):
    """out = h1 + sum_j w_j * expert_{e_j}(h2), h2 = RMSNorm(h1) * g_ffn (A-20..A-22).

    w: ffn_norm [D], w_router [E, D], w_gate / w_up [E, F, D], w_down [E, D, F].
    forced_ids [T, k] (optional): use this expert selection instead of the top-k (the
    weights are still A-21's softmax over the selected logits) -- for comparing rows
    whose top-k is a near-tie with the selection another implementation made."""
    h1 = f64(h1)
    h2 = rmsnorm(h1, w["ffn_norm"], shape.rms_eps)
    ids, wts, logits = router_topk(h2, w["w_router"], shape.top_k)
    if forced_ids is not None:
        ids = np.asarray(forced_ids, dtype=np.int64).reshape(ids.shape)
        wts = forced_weights(logits, ids)
    out = h1.copy()
    for e in range(shape.n_experts):
        rows, slot = np.nonzero(ids == e)
        if rows.size == 0:
            continue
        y = expert_ffn(h2[rows], w["w_gate"][e], w["w_up"][e], w["w_down"][e])
        out[rows] += wts[rows, slot][:, None] * y
    if return_route:
        return out, ids, wts, logits
    return out


def moe_ffn_tp(h1, w, shape, N: int):
    """Sharded mode: rank r holds columns [r F/N, (r+1) F/N) of every expert's
    gate/up and the matching columns of down; the per-rank partial sums are
    AllReduced (a plain sum) and the residual added once.  Must equal moe_ffn."""
    h1 = f64(h1)
    F = shape.d_ffn
    fs = F // N
    h2 = rmsnorm(h1, w["ffn_norm"], shape.rms_eps)
    ids, wts, _ = router_topk(h2, w["w_router"], shape.top_k)
    partials = []
    for r in range(N):
        cols = slice(r * fs, (r + 1) * fs)
        part = np.zeros_like(h1)
        for e in range(shape.n_experts):
            rows, slot = np.nonzero(ids == e)
            if rows.size:
                y = expert_ffn(h2[rows], w["w_gate"][e][cols], w["w_up"][e][cols], w["w_down"][e][:, cols])
                part[rows] += wts[rows, slot][:, None] * y
        partials.append(part)
    return h1 + sum(partials)


def group_rows(ids, n_experts: int, tile: int = 128):
    """Token grouping of reading A-23 (integer, bit-exact contract).

    ids [T, k].  Assignments a = t*k + j are visited in increasing a; expert e
    receives them in that order.  cnt[e] = assignments of e;
    off[0] = 0, off[e+1] = off[e] + ceil(cnt[e] / tile) * tile;
    dst[t, j] = off[e] + (number of earlier assignments to e);
    row_tok[p] = t for p = dst[t, j], -1 for padding rows p < off[E].
    Returns (off [E+1], cnt [E], dst [T, k], row_tok [off[E]])."""
    ids = np.asarray(ids, dtype=np.int64)
    T, k = ids.shape
    cnt = np.zeros(n_experts, dtype=np.int64)
    for a in range(T * k):
        cnt[ids[a // k, a % k]] += 1
    off = np.zeros(n_experts + 1, dtype=np.int64)
    for e in range(n_experts):
        off[e + 1] = off[e] + (cnt[e] + tile - 1) // tile * tile
    dst = np.zeros((T, k), dtype=np.int64)
    row_tok = np.full(int(off[-1]), -1, dtype=np.int64)
    seen = np.zeros(n_experts, dtype=np.int64)
    for a in range(T * k):
        t, j = divmod(a, k)
        e = ids[t, j]
        dst[t, j] = off[e] + seen[e]
        seen[e] += 1
        row_tok[dst[t, j]] = t
    return off, cnt, dst, row_tok


def moe_decoder_layer(x, w: Dict[str, np.ndarray], pool: np.ndarray, batch, shape, page_size: int = 16,
                      return_route: bool = False, forced_ids=None):
    """Decoder layer with the MoE FFN: steps 1-6 of
    ``oracle.layer.decoder_layer`` (attention block unchanged), then moe_ffn."""
    from . import layer as OL
    h1 = OL.attention_block(x, w, pool, batch, shape, page_size)
    return moe_ffn(h1, w, shape, return_route=return_route, forced_ids=forced_ids)


def moe_model_layers(x, layers: List[Dict[str, np.ndarray]], pools, batch, shape, page_size: int = 16):
    for l, w in enumerate(layers):
        x = moe_decoder_layer(x, w, pools[l], batch, shape, page_size)
    return x
