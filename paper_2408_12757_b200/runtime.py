"""PyTorch plumbing around the C ABI: device memory (weights, packed weights,
KV pools, workspace) and streams.  No compute happens here: every step of the
path runs inside libnf.so (see nf.py)."""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import torch

from . import nf

BF16 = torch.bfloat16


def cfg_from_shape(shape, tp_size: int = 1, tp_rank: int = 0, n_layers: Optional[int] = None) -> nf.ModelCfg:
    """nf_model_cfg from any object with the synth.ModelShape attributes."""
    return nf.model_cfg(shape.d_model, shape.n_layers if n_layers is None else n_layers, shape.n_q_heads,
                        shape.n_kv_heads, shape.head_dim, shape.d_ffn, shape.vocab, shape.rms_eps,
                        shape.rope_theta, shape.page_size, tp_size, tp_rank, getattr(shape, "n_experts", 0),
                        getattr(shape, "top_k", 2))


def stream_handle(stream: Optional[torch.cuda.Stream] = None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def alloc_packed_layer(cfg: nf.ModelCfg, device="cuda") -> Dict[str, torch.Tensor]:
    sizes = nf.packed_layer_bytes(cfg)
    names = ["w_qkv", "w_o", "w_o_row", "w_gate_up", "w_down", "w_router"]
    return {n: torch.empty(max(s, 2) // 2, dtype=BF16, device=device) for n, s in zip(names, sizes) if s > 0}


def ptrs(d: Dict[str, torch.Tensor]) -> Dict[str, int]:
    return {k: v.data_ptr() for k, v in d.items()}


def pack_layer(cfg: nf.ModelCfg, w: Dict[str, torch.Tensor], stream: Optional[int] = None) -> Dict[str, torch.Tensor]:
    """w: canonical device bf16 weights (nf_layer_weights names)."""
    packed = alloc_packed_layer(cfg, next(iter(w.values())).device)
    nf.pack_layer(cfg, ptrs(w), ptrs(packed), stream_handle() if stream is None else stream)
    return packed


def pack_lm_head(cfg: nf.ModelCfg, lm_head: torch.Tensor, final_norm: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(lm_head)
    nf.pack_lm_head(cfg, lm_head.data_ptr(), final_norm.data_ptr(), out.data_ptr(), stream_handle())
    return out


def kv_pool(cfg: nf.ModelCfg, n_pages: int, device="cuda") -> torch.Tensor:
    kh = cfg.n_kv_heads // cfg.tp_size
    return torch.empty((n_pages, 2, kh, cfg.page_size, cfg.head_dim), dtype=BF16, device=device)


def workspace(cfg: nf.ModelCfg, b: nf.Batch, device="cuda") -> torch.Tensor:
    n = nf.workspace_size(cfg, b)
    return torch.empty(n, dtype=torch.uint8, device=device)


def layer_forward(plan: nf.Plan, cfg: nf.ModelCfg, packed: Dict[str, torch.Tensor], pool: torch.Tensor, b: nf.Batch,
                  x_in: torch.Tensor, ws: Optional[torch.Tensor] = None, x_out: Optional[torch.Tensor] = None,
                  comm: Optional[int] = None) -> torch.Tensor:
    if ws is None:
        ws = workspace(cfg, b, x_in.device)
    if x_out is None:
        x_out = torch.empty_like(x_in)
    nf.layer_forward(plan, ptrs(packed), pool.data_ptr(), b, x_in.data_ptr(), x_out.data_ptr(), ws.data_ptr(),
                     ws.numel(), stream_handle(), comm)
    return x_out


class Model:
    """Packed model weights on the device plus the nf_model_weights view."""

    def __init__(self, cfg: nf.ModelCfg, embed: torch.Tensor, packed_layers: Sequence[Dict[str, torch.Tensor]],
                 lm_head_packed: torch.Tensor):
        self.cfg = cfg
        self.embed = embed
        self.layers = list(packed_layers)
        self.lm_head_packed = lm_head_packed
        self.handle = nf.ModelHandle(embed.data_ptr(), [ptrs(d) for d in self.layers], lm_head_packed.data_ptr())

    def step(self, plan: nf.Plan, pools: Sequence[torch.Tensor], b: nf.Batch, token_ids: torch.Tensor,
             ws: torch.Tensor, next_ids: Optional[torch.Tensor] = None, comm: Optional[int] = None) -> torch.Tensor:
        if next_ids is None:
            next_ids = torch.empty(len(b.q_len), dtype=torch.int32, device=token_ids.device)
        nf.model_step(plan, self.handle, [p.data_ptr() for p in pools], b, token_ids.data_ptr(), next_ids.data_ptr(),
                      ws.data_ptr(), ws.numel(), stream_handle(), comm)
        return next_ids

    def step_inspect(self, plan: nf.Plan, pools: Sequence[torch.Tensor], b: nf.Batch, token_ids: torch.Tensor,
                     ws: torch.Tensor, comm: Optional[int] = None, logits: bool = True, hidden: bool = True):
        """nf_model_step_ex: (next_ids, logits [n_emit, V/N] or None, [L+1] hidden [T, D] or None)."""
        dev = token_ids.device
        T, D = b.n_tokens, self.cfg.d_model
        next_ids = torch.empty(len(b.q_len), dtype=torch.int32, device=dev)
        n_emit = len(b.q_len) if b.emit is None else int((b.emit != 0).sum())
        lg = torch.empty((n_emit, self.cfg.vocab // self.cfg.tp_size), dtype=BF16, device=dev) if logits else None
        hs = [torch.empty((T, D), dtype=BF16, device=dev) for _ in range(self.cfg.n_layers + 1)] if hidden else None
        nf.model_step_ex(plan, self.handle, [p.data_ptr() for p in pools], b, token_ids.data_ptr(),
                         next_ids.data_ptr(), ws.data_ptr(), ws.numel(), stream_handle(), comm,
                         logits=lg.data_ptr() if lg is not None else 0,
                         hidden=[h.data_ptr() for h in hs] if hs is not None else None)
        return next_ids, lg, hs


def shard_layer(w: Dict[str, torch.Tensor], n_q_heads: int, n_kv_heads: int, head_dim: int, tp: int,
                rank: int) -> Dict[str, torch.Tensor]:
    """Rank `rank`'s canonical shards for head-parallel TP:
    column W_q/W_k/W_v by heads, column O (rows of W_o) and row O (columns of
    W_o), column gate/up, row down.  Slicing only (views made contiguous)."""
    D = w["w_o"].shape[0]
    F = w["w_gate"].shape[-2]
    qs, ks = n_q_heads // tp * head_dim, n_kv_heads // tp * head_dim
    ds, fs = D // tp, F // tp
    c = lambda t: t.contiguous()
    return {
        "attn_norm": w["attn_norm"], "ffn_norm": w["ffn_norm"],
        "w_q": c(w["w_q"][rank * qs:(rank + 1) * qs]),
        "w_k": c(w["w_k"][rank * ks:(rank + 1) * ks]),
        "w_v": c(w["w_v"][rank * ks:(rank + 1) * ks]),
        "w_o_col": c(w["w_o"][rank * ds:(rank + 1) * ds, :]),
        "w_o_row": c(w["w_o"][:, rank * qs:(rank + 1) * qs]),
        # dense [F, D] / [D, F]; MoE [E, F, D] / [E, D, F]: every expert's F columns are split
        "w_gate": c(w["w_gate"][..., rank * fs:(rank + 1) * fs, :]),
        "w_up": c(w["w_up"][..., rank * fs:(rank + 1) * fs, :]),
        "w_down": c(w["w_down"][..., rank * fs:(rank + 1) * fs]),
        **({"w_router": w["w_router"]} if "w_router" in w else {}),
    }


def shard_vocab(lm_head: torch.Tensor, tp: int, rank: int) -> torch.Tensor:
    """Rank's rows of a [V, D] LM head (vocab-parallel head)."""
    v = lm_head.shape[0] // tp
    return lm_head[rank * v:(rank + 1) * v].contiguous()


def shard_pool(pool: torch.Tensor, tp: int, rank: int) -> torch.Tensor:
    """Rank's KV heads of a [n_pages, 2, kh, page, hd] pool (head-parallel KV)."""
    kh = pool.shape[2] // tp
    return pool[:, :, rank * kh:(rank + 1) * kh].contiguous()
