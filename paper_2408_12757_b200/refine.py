"""Measured refinement of a nano-batch plan (host orchestration; no arithmetic of the
method): coordinate moves from a searched or default OVERLAP plan, each candidate
timed against the incumbent in interleaved A/B rounds (the GPU's power and thermal
state drifts; interleaving cancels it), keeping a move while it improves the step by
more than `gain`.  Moves: the memory partition +-8 / +-16 SMs (8..72) or none (decode
on the compute streams, TP), the nano-batch token shares +-1/8, and at TP the 2- / 4-way
attention split.  The network partition is held fixed (it sizes the NCCL CTA cap).
PAPER.md:671-674 searches on offline curves; DESIGN.md §7 records why B200 needs the
measured step (co-run power / HBM effects the curves miss)."""
from __future__ import annotations

from typing import Callable, List, Tuple

from . import nf


def variant(cfg, base: nf.PlanSpec, dec: int, s8: int, nn: int, tp: int) -> nf.Plan:
    sp = nf.PlanSpec()
    for f, _ in nf.PlanSpec._fields_:
        setattr(sp, f, getattr(base, f))
    for k in range(nf.OP_COUNT):
        sp.sm[k] = base.sm[k]
    sp.sm[nf.OP_DECODE_ATTN] = dec
    for k in (nf.OP_KQV, nf.OP_PREFILL_ATTN, nf.OP_O, nf.OP_UG, nf.OP_DOWN):
        sp.sm[k] = 148
    sh = (s8, s8, 8 - s8, 8 - s8) if nn == 4 else (s8, 8 - s8)
    sp.n_nano = nn
    for i, v in enumerate(sh):
        sp.share[i] = v
    sp.n_dense = 2 if tp > 1 else 0
    return nf.Plan.from_spec(cfg, sp)


def refine(cfg, plan: nf.Plan, ab: Callable[[nf.Plan, nf.Plan], Tuple[float, float]], tp: int,
           max_moves: int = 8, gain: float = 0.997) -> Tuple[nf.Plan, List[dict]]:
    """ab(candidate, incumbent) -> (median time ratio, candidate ms)."""
    base = plan.spec()
    nn = base.n_nano if base.n_nano in (2, 4) else 2
    tot = sum(base.share[:base.n_nano])
    s8 = max(1, min(7, round(8 * base.share[0] * (2 if nn == 4 else 1) / tot)))
    dec = min(148, max(8, (base.sm[nf.OP_DECODE_ATTN] + 7) // 8 * 8))
    cur = variant(cfg, base, dec, s8, nn, tp)
    log = [{"dec_sms": dec, "share8": s8, "n_nano": nn, "ratio": 1.0}]
    seen = {(dec, s8, nn)}
    for _ in range(max_moves):
        cands = [(dec, s8 + ds, nn) for ds in (-1, 1) if 1 <= s8 + ds <= 7]
        if dec < 148:
            cands += [(dec + dd, s8, nn) for dd in (-16, -8, 8, 16) if 8 <= dec + dd <= 72]
        if tp > 1:
            cands.append((dec, s8, 6 - nn))                       # 4-way <-> 2-way attention
            cands.append((148 if dec < 148 else 24, s8, nn))      # with / without a memory partition
        cands = list(dict.fromkeys(c for c in cands if c not in seen))
        if not cands:
            break
        res = []
        for d2, s2, n2 in cands:
            seen.add((d2, s2, n2))
            pl = variant(cfg, base, d2, s2, n2, tp)
            ratio, t = ab(pl, cur)
            log.append({"dec_sms": d2, "share8": s2, "n_nano": n2, "ratio": ratio, "ms": t})
            res.append((ratio, d2, s2, n2, pl))
        ratio, d2, s2, n2, pl = min(res, key=lambda x: x[0])
        if ratio >= gain:
            break
        dec, s8, nn, cur = d2, s2, n2, pl
    return cur, log
