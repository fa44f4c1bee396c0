"""NEXT-1 workload generators (synth/workloads.py): Table 3 length statistics
 and the continuous-batching snapshot's invariants."""
import numpy as np
import pytest

from synth import workloads as W


@pytest.mark.parametrize("name", sorted(W.TABLE3))
def test_lognormal_lengths_match_table3(name):
    mi, si, mo, so = W.TABLE3[name]
    mu, sig = W.lognormal_params(mi, si)
    # closed form of the lognormal moments
    assert np.isclose(np.exp(mu + sig ** 2 / 2), mi) and np.isclose(np.sqrt(np.expm1(sig ** 2)) * mi, si)
    i, o = W.sample_lengths(name, 400_000, seed=11, max_len=1 << 20)
    assert abs(i.mean() / mi - 1) < 0.03 and abs(o.mean() / mo - 1) < 0.03
    assert abs(i.std() / si - 1) < 0.15 and abs(o.std() / so - 1) < 0.15
    assert i.min() >= 1 and o.min() >= 1


def test_lengths_deterministic_by_seed():
    a = W.sample_lengths("sharegpt", 1000, seed=3)
    b = W.sample_lengths("sharegpt", 1000, seed=3)
    c = W.sample_lengths("sharegpt", 1000, seed=4)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    assert not np.array_equal(a[0], c[0])


@pytest.mark.parametrize("name", sorted(W.TABLE3))
def test_snapshot_is_a_full_dense_step(name):
    ql, kp, st = W.snapshot(name, b_dense=2048, kv_cap_tokens=2_000_000, warm_steps=600)
    assert ql.sum() == 2048 == st["b_dense"]            # dense batch filled (offline, unbounded queue)
    assert (ql >= 1).all() and (kp >= 0).all()
    n_dec = st["n_decode"]
    assert (ql[:n_dec] == 1).all()                       # token order: decodes first, then chunks
    assert st["reserved_tokens"] <= st["kv_cap_tokens"]  # peak-memory admission
    # decode-heavy vs prefill-heavy mixes follow the output/input ratio (Little's law)
    mi, _, mo, _ = W.TABLE3[name]
    frac = n_dec / 2048
    assert abs(frac - mo / (mi + mo)) < 0.15, (frac, mo / (mi + mo))


def test_snapshot_chunks_continue_cached_prefixes():
    ql, kp, st = W.snapshot("splitwise", b_dense=512, kv_cap_tokens=200_000, warm_steps=300)
    pf = ql > 1
    # a chunk's prefix is the part of its prompt already prefilled by earlier steps
    assert (kp[pf] >= 0).all()
    assert W.snapshot("splitwise", b_dense=512, kv_cap_tokens=200_000, warm_steps=300)[0].tolist() == ql.tolist()


def test_snapshot_memory_bound_admission():
    """With a small KV cache the admitted peak footprint, not the token budget, bounds the step."""
    ql, kp, st = W.snapshot("lmsys", b_dense=2048, kv_cap_tokens=200_000, warm_steps=400)
    assert st["reserved_tokens"] <= 200_000 and st["reserved_tokens"] > 200_000 - 8192
    assert ql.sum() < 2048
