"""nf_plan_create (C++ autosearch in libnf) against the oracle planner
(oracle/planner.py) on the same curves and batch: identical split, SM units
and schedule.  Host-only: runs on CPU."""
import os

import numpy as np
import pytest

import synth
from oracle import planner as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def nf():
    from paper_2408_12757_b200 import build
    build.build()
    from paper_2408_12757_b200 import nf as _nf
    return _nf


def load_curves(path):
    rows = [l.split(",") for l in open(path).read().splitlines()[1:] if l.strip()]
    return [(int(k), int(u), float(w), float(t)) for k, _, u, w, t in rows]


def synthetic_curves():
    pts = []
    for k in range(6):
        a = 0.9 if k != P.DECODE else 0.55
        scale = {P.KQV: 1.5e-6, P.O: 1.1e-6, P.UG: 5.5e-6, P.DOWN: 3.2e-6, P.PREFILL: 1.7e-10, P.DECODE: 6.5e-10}[k]
        for u in (8, 16, 32, 48, 64, 96, 128, 148):
            for w in (512.0, 2048.0, 1e5, 1e6):
                pts.append((k, u, w, scale * w * (148 / u) ** a))
    return pts


@pytest.mark.parametrize("which", ["synthetic", "measured"])
def test_autosearch_matches_oracle(nf, which):
    from paper_2408_12757_b200.runtime import cfg_from_shape
    pts = synthetic_curves() if which == "synthetic" else load_curves(os.path.join(ROOT, "profiles", "curves_b200_quick.csv"))
    rng = np.random.default_rng(4)
    q_len = [1] * 60 + [96, 40]
    prefix = list(rng.integers(500, 1500, 60)) + [0, 300]
    b = synth.make_batch(q_len, prefix, seed=2)
    cfg = cfg_from_shape(synth.SHAPES["llama3-8b"])
    iters = 40
    best, table = P.search(q_len, prefix, P.Curves(pts), budget=148, q=8, max_iters=iters, n_layers=3)
    plan = nf.Plan.search(cfg, nf.Batch.from_any(b), pts, sm_budget=148, sm_quantum=8, mode=nf.OVERLAP, n_nano=2,
                          max_iters=iters)
    spec = plan.spec()
    assert [spec.share[0], spec.share[1]] == best[0]
    kinds = sorted({n.kind for n in best[3]})
    assert [spec.sm[k] for k in kinds] == [best[1][k] for k in kinds]
    csv = [l.split(",") for l in plan.csv().splitlines()[1:]]
    assert len(csv) == len(best[3])
    for row, n in zip(csv, best[3]):
        assert int(row[2]) == n.nano
        assert float(row[4]) == pytest.approx(best[4][n.id], rel=1e-7, abs=1e-12)
        assert float(row[5]) == pytest.approx(best[5][n.id], rel=1e-7, abs=1e-12)
    assert max(float(r[5]) for r in csv) == pytest.approx(best[2], rel=1e-9)


def test_autosearch_errors_and_sequential(nf):
    from paper_2408_12757_b200.runtime import cfg_from_shape
    cfg = cfg_from_shape(synth.SHAPES["llama3-8b"])
    b = nf.Batch.from_any(synth.make_batch([1, 1, 30], [100, 7, 0]))
    with pytest.raises(nf.NFError) as e:   # decode attention has work but no curve
        nf.Plan.search(cfg, b, [(0, 148, 512.0, 1e-4)], mode=nf.OVERLAP)
    assert e.value.status == nf.NF_EINVAL
    with pytest.raises(nf.NFError):
        nf.Plan.search(cfg, b, [], sm_budget=0)
    p = nf.Plan.search(cfg, b, [], mode=nf.SEQUENTIAL)
    assert p.spec().n_nano == 1 and list(p.spec().sm) == [148] * 7


def synthetic_curves_tp():
    pts = synthetic_curves()
    for u in (8, 16, 24, 32, 48):
        for w in (256.0, 1024.0, 4096.0):   # NET: AllGather-equivalent tokens (reading P-8)
            pts.append((P.NET, u, w, 2.5e-8 * w * min(1.0, 16 / u) ** 0.8 + 8e-6))
    return pts


def test_tp_pipeline_dag_structure():
    """Reading P-8: per layer five collectives in the fixed order
    AG_attn(H1), AG_o(H1), AR_o(H2), AR_d(H1), AR_d(H2); column O waits for the
    attention AllGather, row O for the decode attention of Q3 and Q4, Up/Gate of H1
    for AG_o, of H2 for AR_o; the next layer's KQV of a half waits for its AR_d."""
    work = [(300, 1000, 0), (300, 900, 0), (200, 800, 5000), (200, 700, 0)]
    nodes = P.build_pipeline_tp(work, n_layers=2)
    kinds = [n.kind for n in nodes]
    assert kinds.count(P.NET) == 10 and kinds.count(P.KQV) == 8 and kinds.count(P.O) == 4
    net = [n for n in nodes if n.kind == P.NET]
    assert [(n.nano, n.work) for n in net[:5]] == [(0, 600), (0, 600), (1, 800), (0, 1200), (1, 800)]
    by_id = {n.id: n for n in nodes}
    o1, o2 = [n for n in nodes if n.kind == P.O][:2]
    assert net[0].id in o1.deps
    dec = [n for n in nodes if n.kind == P.DECODE]
    assert dec[2].id in o2.deps and dec[3].id in o2.deps
    ug = [n for n in nodes if n.kind == P.UG][:2]
    assert net[1].id in ug[0].deps and net[2].id in ug[1].deps
    kqv2 = [n for n in nodes if n.kind == P.KQV][4:]
    assert net[3].id in kqv2[0].deps and net[3].id in kqv2[1].deps
    assert net[4].id in kqv2[2].deps and net[4].id in kqv2[3].deps
    for n in nodes:
        assert all(d < n.id for d in n.deps)
        for d in n.deps:
            assert d in by_id


def test_tp_autosearch_matches_oracle(nf):
    """nf_plan_create at tp_size 8 (the 70B TP8 rank) == the oracle's reading-P-8 search."""
    from paper_2408_12757_b200.runtime import cfg_from_shape
    pts = synthetic_curves_tp()
    b = synth.workload_batch(512, 512, 1024)
    q_len, prefix = list(map(int, b.q_len)), list(map(int, b.kv_prefix))
    cfg = cfg_from_shape(synth.SHAPES["llama2-70b"], tp_size=8, tp_rank=3)
    iters = 30
    best, table = P.search_tp(q_len, prefix, P.Curves(pts), budget=148, q=8, max_iters=iters, n_layers=3)
    plan = nf.Plan.search(cfg, nf.Batch.from_any(b), pts, sm_budget=148, sm_quantum=8, mode=nf.OVERLAP, n_nano=4,
                          max_iters=iters)
    spec = plan.spec()
    assert spec.n_nano == 4 and spec.n_dense == 2
    assert [spec.share[i] for i in range(4)] == best[0]
    kinds = sorted({n.kind for n in best[3]})
    assert P.NET in kinds
    assert [spec.sm[k] for k in kinds] == [best[1][k] for k in kinds]
    csv = [l.split(",") for l in plan.csv().splitlines()[1:]]
    assert len(csv) == len(best[3])
    assert max(float(r[5]) for r in csv) == pytest.approx(best[2], rel=1e-7)
    # lower bound: never worse than the whole budget per kind
    seq = P.simulate(best[3], [148] * P.N_KINDS, P.Curves(pts), 148)[0]
    assert best[2] <= seq + 1e-12
