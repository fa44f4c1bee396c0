"""Helpers for the -m gpu parity tests: seeded host inputs (synth) -> device,
the oracle on the same values, and the tolerance of BASELINE.json north_star
(bf16 layer outputs vs the fp32+ oracle: relative L2 <= 1e-2, max abs <= 5e-2
at unit-RMS activations)."""
import numpy as np
import torch

import synth
from oracle import layer as OL

REL_L2 = 1e-2
MAX_ABS = 5e-2


def require_gpu():
    assert torch.cuda.is_available(), "GPU tests need a B200; the product has no CPU fallback"
    from paper_2408_12757_b200 import build
    build.build()
    from paper_2408_12757_b200 import nf, runtime
    return nf, runtime


def dev(a, dtype=torch.bfloat16):
    """Host float32 array holding bf16-representable values -> exact device bf16."""
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to("cuda").to(dtype)


def dev_bits(bits: np.ndarray):
    t = torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).to("cuda")
    return t.view(torch.bfloat16)


def host(t) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def errors(out, ref):
    out = np.asarray(out, np.float64)
    ref = np.asarray(ref, np.float64)
    err = out - ref
    return float(np.linalg.norm(err) / max(np.linalg.norm(ref), 1e-30)), float(np.abs(err).max())


def assert_close(out, ref, rel_l2=REL_L2, max_abs=MAX_ABS, what="", scale_rms=False):
    """north_star tolerance.  scale_rms (reading A-31): the max-abs bound is stated "at
    unit-RMS activations"; deep layers of a model step carry a residual stream whose RMS
    grows with depth, so there the bound is max_abs x max(1, RMS(ref))."""
    rel, mx = errors(out, ref)
    if scale_rms:
        max_abs = max_abs * max(1.0, float(np.sqrt(np.mean(np.asarray(ref, np.float64) ** 2))))
    assert np.isfinite(out).all(), f"{what}: non-finite output"
    assert rel <= rel_l2 and mx <= max_abs, f"{what}: rel L2 {rel:.3e} (<= {rel_l2}), max abs {mx:.3e} (<= {max_abs})"
    return rel, mx


def device_weights(w: dict):
    return {k: dev(v) for k, v in w.items()}


def compact_case(shape, batch, reqs, seed_kv=2, layer=0):
    """Sub-batch of requests `reqs` with a compact float64 pool regenerated from
    the per-request RNG streams (so the oracle can check sampled requests of a
    full-size batch without materialising the whole pool)."""
    P = shape.page_size
    q_len = batch.q_len[reqs]
    prefix = batch.kv_prefix[reqs]
    sub = synth.make_batch(q_len, prefix, permute=False)
    pool = np.zeros((sub.n_pages_pool, 2, shape.n_kv_heads, P, shape.head_dim), dtype=np.float64)
    for i, r in enumerate(reqs):
        n = int(batch.kv_prefix[r])
        if n:
            j = np.arange(n)
            pool[sub.page_ids[sub.page_indptr[i] + j // P], :, :, j % P, :] = synth.request_kv(shape, int(r), n, seed_kv, layer)
    return sub, pool


def token_rows(batch, reqs):
    ind = np.concatenate([[0], np.cumsum(batch.q_len)])
    return np.concatenate([np.arange(ind[r], ind[r + 1]) for r in reqs])
