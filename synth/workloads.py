"""Length-distribution workloads and steady-state batch snapshots (SURVEY.md
§8f NEXT-1) -- input generation only, no arithmetic of the method.

PAPER.md:726-728 (Table 3, "average input / output length ± std"):

    Splitwise    1155 ± 1109 in,  211 ± 163 out
    LMSYS-Chat    102 ±  169 in,  222 ± 210 out
    ShareGPT      246 ±  547 in,  322 ± 244 out

The traces themselves are not available (no datasets), so lengths are drawn
from a lognormal matched to each mean and std (the traces are heavy-tailed:
std > mean for the inputs), clipped to [1, max_len] (reading A-19).

A step of the serving loop is a dense batch of ``b_dense`` tokens that mixes
decode tokens and chunked prefill.  ``snapshot``
runs a small discrete-time continuous-batching simulation (offline
throughput: an unbounded queue of arrivals) and returns the composition of
one step after warm-up:

* every admitted request whose prompt is complete contributes one decode
  token per step until it has produced its output length, then leaves;
* the remaining token budget goes to prompt chunks of admitted requests in
  arrival order (a prompt may span several steps: chunked prefill);
* a request is admitted only while the KV cache can hold the peak footprint
  (input + output tokens) of every admitted request (peak-memory admission,
  PAPER.md:573-575).
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Tuple

import numpy as np

TABLE3: Dict[str, Tuple[float, float, float, float]] = {
    # name: (input mean, input std, output mean, output std)
    "splitwise": (1155.0, 1109.0, 211.0, 163.0),
    "lmsys": (102.0, 169.0, 222.0, 210.0),
    "sharegpt": (246.0, 547.0, 322.0, 244.0),
}


def lognormal_params(mean: float, std: float) -> Tuple[float, float]:
    """(mu, sigma) of the lognormal with this mean and standard deviation."""
    s2 = np.log1p((std / mean) ** 2)
    return float(np.log(mean) - s2 / 2), float(np.sqrt(s2))


def sample_lengths(name: str, n: int, seed: int = 6, max_len: int = 8192) -> Tuple[np.ndarray, np.ndarray]:
    """n (input, output) length pairs of workload ``name`` (integers >= 1)."""
    mi, si, mo, so = TABLE3[name]
    rng = np.random.default_rng(seed)
    out = []
    for mean, std in ((mi, si), (mo, so)):
        mu, sig = lognormal_params(mean, std)
        x = np.rint(rng.lognormal(mu, sig, n))
        out.append(np.clip(x, 1, max_len).astype(np.int64))
    return out[0], out[1]


@dataclasses.dataclass
class _Req:
    inp: int
    out: int
    prefilled: int = 0
    generated: int = 0


def snapshot(name: str, b_dense: int = 2048, kv_cap_tokens: int = 1_000_000, warm_steps: int = 1500,
             seed: int = 6, max_len: int = 8192) -> Tuple[np.ndarray, np.ndarray, dict]:
    """Composition (q_len, kv_prefix) of one steady-state step of workload ``name``.

    Rows are in the batch's token order: decode requests first, then prompt
    chunks in arrival order.  ``stats`` reports the step's decode / prefill
    token counts and the admitted footprint."""
    pool_in, pool_out = sample_lengths(name, 200_000, seed=seed, max_len=max_len)
    nxt = 0
    running: List[_Req] = []
    reserved = 0
    q_len: List[int] = []
    kv_prefix: List[int] = []
    for step in range(warm_steps + 1):
        # admission: peak footprint of every admitted request must fit the KV cache
        while nxt < len(pool_in) and reserved + int(pool_in[nxt] + pool_out[nxt]) <= kv_cap_tokens:
            r = _Req(int(pool_in[nxt]), int(pool_out[nxt]))
            nxt += 1
            running.append(r)
            reserved += r.inp + r.out
        budget = b_dense
        q_len, kv_prefix = [], []
        dec = [r for r in running if r.prefilled == r.inp]
        for r in dec[:budget]:
            q_len.append(1)
            kv_prefix.append(r.inp + r.generated)
        budget -= min(len(dec), budget)
        chunks = []
        for r in running:
            if budget == 0:
                break
            if r.prefilled < r.inp:
                c = min(r.inp - r.prefilled, budget)
                chunks.append((r, c))
                budget -= c
        for r, c in chunks:
            q_len.append(c)
            kv_prefix.append(r.prefilled)
        if step == warm_steps:
            break
        # advance: decodes produce a token, chunks extend the prompt's cached prefix
        for r in dec[:b_dense]:
            r.generated += 1
        for r, c in chunks:
            r.prefilled += c
        done = [r for r in running if r.prefilled == r.inp and r.generated >= r.out]
        for r in done:
            reserved -= r.inp + r.out
        running = [r for r in running if not (r.prefilled == r.inp and r.generated >= r.out)]
    ql = np.array(q_len, dtype=np.int32)
    kp = np.array(kv_prefix, dtype=np.int32)
    stats = {"workload": name, "b_dense": int(ql.sum()), "n_req": int(len(ql)), "n_decode": int((ql == 1).sum()),
             "prefill_tokens": int(ql[ql > 1].sum()), "mean_decode_ctx": float(kp[ql == 1].mean()) if (ql == 1).any() else 0.0,
             "admitted": len(running), "reserved_tokens": reserved, "kv_cap_tokens": kv_cap_tokens}
    return ql, kp, stats
