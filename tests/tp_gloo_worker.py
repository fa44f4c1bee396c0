"""Worker of test_tp_gloo: one process per TP rank (gloo), executing the TP
executor's dataflow (csrc/api.cu run_dense_tail_tp) with float64 oracle
primitives and real torch.distributed collectives."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from oracle import layer as OL  # noqa: E402
from oracle import metadata as md  # noqa: E402


def shard(w, shape, N, r):
    # same slicing as paper_2408_12757_b200.runtime.shard_layer (checked below against it)
    from paper_2408_12757_b200.runtime import shard_layer
    t = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in w.items()}
    s = shard_layer(t, shape.n_q_heads, shape.n_kv_heads, shape.head_dim, N, r)
    return {k: v.numpy().astype(np.float64) for k, v in s.items()}


def all_gather_rank_major(x):
    """Executor AG: recv = [rank0 | rank1 | ...] of equal-sized row blocks."""
    parts = [torch.empty_like(x) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, x)
    return torch.stack(parts)              # [N, M, C]


def interleave(g):
    """launch_interleave: [N, M, C] -> [M, N*C]."""
    N, M, C = g.shape
    return g.permute(1, 0, 2).reshape(M, N * C)


def worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = synth.shape_with(synth.SHAPES["c1"], n_kv_heads=4, d_ffn=1408, d_model=256, n_q_heads=8, head_dim=32)
    b = synth.make_batch([1] * 6 + [9, 1, 5], [3, 17, 40, 0, 21, 8, 0, 30, 12], seed=2, pool_slack=1)
    w = synth.layer_weights(shape, 0)
    x = synth.activations(shape, b.n_tokens).astype(np.float64)
    pool = OL.as_pool(synth.kv_pool(shape, b))
    ref = OL.decoder_layer(x, w, pool.copy(), b, shape)
    N, r = world, rank
    s = shard(w, shape, N, r)
    hd, qh, kh, D = shape.head_dim, shape.n_q_heads // N, shape.n_kv_heads // N, shape.d_model
    T = b.n_tokens
    pos = md.positions(b.q_len, b.kv_prefix)
    my_pool = pool[:, :, r * kh:(r + 1) * kh].copy()
    # column-parallel KQV on this rank's heads, local attention
    h = OL.rmsnorm(x, w["attn_norm"], shape.rms_eps)
    q = OL.rope((h @ s["w_q"].T).reshape(T, qh, hd), pos, shape.rope_theta)
    k = OL.rope((h @ s["w_k"].T).reshape(T, kh, hd), pos, shape.rope_theta)
    v = (h @ s["w_v"].T).reshape(T, kh, hd)
    OL.kv_append(my_pool, k, v, b)
    o_local = OL.paged_attention(q, my_pool, b).reshape(T, qh * hd)
    cut = int(md.qo_indptr(b.q_len)[4])     # nano-batch 0 = requests [0, 4): column O; rest: row O
    h1 = np.zeros_like(x)
    # nano 0: AG(o) -> interleave -> O_col (+ x columns) -> AG -> interleave
    o_cat = interleave(all_gather_rank_major(torch.from_numpy(o_local[:cut]))).numpy()
    Dl = D // N
    hcol = x[:cut, r * Dl:(r + 1) * Dl] + o_cat @ s["w_o_col"].T
    h1[:cut] = interleave(all_gather_rank_major(torch.from_numpy(hcol))).numpy()
    # nano 1: O_row partial (+ x on rank 0) -> AR
    part = o_local[cut:] @ s["w_o_row"].T + (x[cut:] if r == 0 else 0.0)
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    h1[cut:] = t.numpy()
    # column Up/Gate + SiLU, row Down partial (+ h1 on rank 0) -> AR
    h2 = OL.rmsnorm(h1, w["ffn_norm"], shape.rms_eps)
    m = OL.silu(h2 @ s["w_gate"].T) * (h2 @ s["w_up"].T)
    part = m @ s["w_down"].T + (h1 if r == 0 else 0.0)
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    out = t.numpy()
    err = float(np.abs(out - ref).max() / np.abs(ref).max())
    gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(N)]
    dist.all_gather(gathered, torch.tensor([err], dtype=torch.float64))
    if r == 0:
        np.save(out_path, np.array([g.item() for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()


def worker_moe(rank, world, port, out_path):
    """MoE FFN dataflow of run_dense_tail_tp (PAPER.md:689 + :183 per expert): the
    router on the replicated h1 (identical on every rank), this rank's column
    shard of every expert's gate/up and row shard of its down (runtime.shard_layer),
    weighted partial sums -> AllReduce -> + h1."""
    from oracle import moe as OM
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shape = synth.shape_with(synth.SHAPES["c1-moe"], d_model=256, n_q_heads=8, n_kv_heads=4, head_dim=32,
                             d_ffn=512, n_experts=6, top_k=2)
    w = synth.layer_weights(shape, 0)
    h1 = synth.activations(shape, 37, seed=3, name="h1").astype(np.float64)
    ref = OM.moe_ffn(h1, w, shape)
    N, r = world, rank
    s = shard(w, shape, N, r)
    assert np.array_equal(s["w_router"], w["w_router"].astype(np.float64))
    h2 = OL.rmsnorm(h1, w["ffn_norm"], shape.rms_eps)
    ids, wts, _ = OM.router_topk(h2, w["w_router"], shape.top_k)
    part = np.zeros_like(h1)
    for e in range(shape.n_experts):
        rows, slot = np.nonzero(ids == e)
        if rows.size:
            y = OM.expert_ffn(h2[rows], s["w_gate"][e], s["w_up"][e], s["w_down"][e])
            part[rows] += wts[rows, slot][:, None] * y
    t = torch.from_numpy(part)
    dist.all_reduce(t)
    out = h1 + t.numpy()
    err = float(np.abs(out - ref).max() / np.abs(ref).max())
    gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(N)]
    dist.all_gather(gathered, torch.tensor([err], dtype=torch.float64))
    if r == 0:
        np.save(out_path, np.array([g.item() for g in gathered]))
    dist.barrier()
    dist.destroy_process_group()
