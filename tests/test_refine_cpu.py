"""paper_2408_12757_b200.refine (the measured plan refinement bench.py runs) as host
logic: with a synthetic step-time model in place of GPU timings it walks to the model's
optimum by coordinate moves, never returns a plan slower than its start, explores the
2-/4-way attention split and the memory-partition toggle only at TP > 1, and stops."""
import pytest

import synth


@pytest.fixture(scope="module")
def nf():
    from paper_2408_12757_b200 import build
    build.build()
    from paper_2408_12757_b200 import nf as _nf
    return _nf


def _model(opt_dec, opt_s8, opt_nn=2):
    def t(plan):
        sp = plan.spec()
        dec = min(sp.sm[1], 148)
        s8 = sp.share[0] * 8 // sum(sp.share[:sp.n_nano]) * (2 if sp.n_nano == 4 else 1)
        d = (1.0 if opt_dec >= 148 else abs(dec - opt_dec) / 8.0) if (dec >= 148) != (opt_dec >= 148) \
            else abs(dec - opt_dec) / 8.0
        return 40.0 * (1.0 + 0.01 * abs(s8 - opt_s8) + 0.01 * d + (0.0 if sp.n_nano == opt_nn else 0.03))
    return t


def test_refine_walks_to_optimum_tp1(nf):
    from paper_2408_12757_b200 import refine as R
    from paper_2408_12757_b200.runtime import cfg_from_shape
    cfg = cfg_from_shape(synth.SHAPES["llama3-8b"])
    t = _model(opt_dec=40, opt_s8=5)
    start = nf.Plan.explicit(cfg, nf.OVERLAP, shares=(2, 6), sm=[148, 64, 148, 148, 148, 148, 8])
    plan, log = R.refine(cfg, start, lambda c, i: (t(c) / t(i), t(c)), tp=1, max_moves=20)
    sp = plan.spec()
    assert (sp.sm[1], sp.share[0], sp.share[1], sp.n_nano) == (40, 5, 3, 2)
    assert all(e["n_nano"] == 2 for e in log) and all(e["dec_sms"] <= 72 for e in log)
    assert t(plan) <= t(start)


def test_refine_tp_explores_split_and_partition(nf):
    from paper_2408_12757_b200 import refine as R
    from paper_2408_12757_b200.runtime import cfg_from_shape
    cfg = cfg_from_shape(synth.SHAPES["llama2-70b"], tp_size=8)
    t = _model(opt_dec=148, opt_s8=4, opt_nn=2)
    start = nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1, 1, 1), n_dense=2, sm=[116, 16, 116, 116, 116, 116, 16])
    plan, log = R.refine(cfg, start, lambda c, i: (t(c) / t(i), t(c)), tp=8, max_moves=20)
    sp = plan.spec()
    assert sp.n_nano == 2 and sp.n_dense == 2 and sp.sm[1] >= 148 and sp.sm[6] == 16
    assert any(e["n_nano"] == 2 for e in log) and any(e["dec_sms"] >= 148 for e in log)


def test_refine_stops_without_gain(nf):
    from paper_2408_12757_b200 import refine as R
    from paper_2408_12757_b200.runtime import cfg_from_shape
    cfg = cfg_from_shape(synth.SHAPES["llama3-8b"])
    start = nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1), sm=[116, 32, 116, 116, 116, 116, 8])
    plan, log = R.refine(cfg, start, lambda c, i: (1.0, 40.0), tp=1)
    assert plan.spec().sm[1] == 32 and len(log) <= 7
