#!/usr/bin/env python
"""Run nf_plan_create (autosearch) for the 8B-shape B_dense=2048 workload on a
curve CSV and print the plan + predicted per-layer period vs sequential."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2408_12757_b200 import nf  # noqa: E402
from paper_2408_12757_b200.runtime import cfg_from_shape  # noqa: E402


def load(path):
    rows = [l.split(",") for l in open(path).read().splitlines()[1:] if l.strip()]
    return [(int(k), int(u), float(w), float(t)) for k, _, u, w, t in rows]


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "curves_b200_quick.csv")
    pts = load(path)
    b = nf.Batch.from_any(synth.workload_batch(2048, 1024, 512))
    cfg = cfg_from_shape(synth.SHAPES["llama3-8b"])
    plan = nf.Plan.search(cfg, b, pts, max_iters=200)
    s = plan.spec()
    rows = [l.split(",") for l in plan.csv().splitlines()[1:]]
    mk = max(float(r[5]) for r in rows)
    print("shares", list(s.share)[:s.n_nano], "sm", list(s.sm))
    print(f"predicted 3-layer makespan {mk*1e3:.3f} ms")
    return plan


if __name__ == "__main__":
    main()
