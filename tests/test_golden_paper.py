"""Golden values the paper prints (tests/golden/*.json, each with its PAPER.md
citation) against the cost-model oracle (oracle/costmodel.py) and the metric
bench.py reports (pct_of_optimal uses Eq. 9 with the shapes' active params)."""
import json
import os

import pytest

from oracle import costmodel as CM

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return json.load(open(os.path.join(GOLD, name)))


def _digits(v):
    s = repr(v)
    return len(s.split(".")[1]) if "." in s else 0


def test_table2_reproduced_to_printed_precision():
    g = _load("table2_llama2_70b_8xa100.json")
    rows = CM.table2(**{k: v for k, v in g["inputs"].items() if k != "inputs_source"})
    checked = 0
    for op, cells in g["rows"].items():
        for key, printed in cells.items():
            got = rows[op][key]
            tol = 0.5 * 10 ** -_digits(printed) + 1e-9        # the paper rounds to the printed digits
            # ... or 0.25 %: GEMM-D T_mem prints 3.11 = 49.7 GB (already rounded) / 16 TB/s = 3.106,
            # the unrounded 49.66 GB gives 3.104
            assert abs(got - printed) <= max(tol, 2.5e-3 * abs(printed)), (op, key, got, printed)
            checked += 1
    assert checked == 27


def test_optimal_throughput_eq9():
    for c in _load("optimal_throughput.json")["cases"]:
        assert int(CM.optimal_throughput(c["compute_flops"], c["p_model"])) == c["tokens_per_s"], c["cite"]


def test_steady_state_eq2_and_bench_metric():
    """Eq. 2 gives Table 2's B_req = 1366.7 and n_dec = 1365.3 (SURVEY A-14: B_dense counts tokens);
    bench.py's optimum for 70B with the paper's nominal P = 70e9 and 260 TF/s is the paper's 1857."""
    b_req, n_pre, n_dec = CM.steady_state(2048, 512, 1024)
    assert round(b_req, 1) == 1366.7 and round(n_dec, 1) == 1365.3
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(GOLD), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    import synth
    pa = bench.p_active(synth.SHAPES["llama2-70b"])
    assert abs(pa - 68.713e9) / 68.713e9 < 1e-3                 # matmul weights per token
    assert int(CM.optimal_throughput(260e12, 70e9)) == 1857
    pm = bench.p_active(synth.SHAPES["mixtral-8x7b"])
    assert abs(pm - 12.75e9) / 12.75e9 < 2e-3                    # top-2 experts + router
