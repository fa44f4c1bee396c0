"""Serving loop:
the oracle scheduler (oracle/serving.py) pinned by a hand-worked trace,
invariants and brute force, and the native scheduler (nf_sched_*) bit-exact
against it.  CPU only (the scheduler is host code)."""
import numpy as np
import pytest

import synth.workloads as W
from oracle import serving as OS

V = 997


def fake_ids(step, req_ids):
    """Deterministic stand-in for a model step's next_ids."""
    return [int((r * 1009 + step * 7) % V) for r in req_ids]


def drive(s, max_steps=10000, as_dict=False):
    """The asynchronous protocol of PAPER.md:652-657: form step i+1, then read
    back step i's tokens (complete(i)), then form step i+2 ..."""
    steps, prev = [], None
    for _ in range(max_steps):
        st = s.next()
        st = st if as_dict else {k: getattr(st, k) for k in ("step", "req_ids", "q_len", "kv_prefix", "emit",
                                                              "page_indptr", "page_ids", "tok_src")}
        if prev is not None:
            s.complete(prev["step"], fake_ids(prev["step"], list(prev["req_ids"])))
        steps.append({k: (list(map(int, v)) if not np.isscalar(v) else int(v)) for k, v in st.items()})
        if len(st["req_ids"]) == 0 and (prev is None or len(prev["req_ids"]) == 0):
            break
        prev = st
    return steps


def trace(n, name="lmsys", seed=3, scale=0.2, max_len=600):
    inp, out = W.sample_lengths(name, n, seed=seed, max_len=max_len)
    inp = np.maximum(1, (inp * scale).astype(int))
    out = np.maximum(1, (out * scale).astype(int))
    rng = np.random.default_rng(seed)
    return [(i, rng.integers(0, V, size=int(a)).tolist(), int(b)) for i, (a, b) in enumerate(zip(inp, out))]


def test_hand_trace():
    """Worked by hand from the policy text (A-25..A-29): pool 64
    pages of 16, B_dense in {32, 16}, avg decode 8."""
    s = OS.Scheduler(64, 16, [32, 16], 8)
    s.submit(0, [5] * 20, 3)
    s.submit(1, [7] * 5, 2)
    st = drive(s)
    # step 0: both admitted (peak (20+8+15 + 5+8+15)//16 = 4 pages); 25 tokens available -> B = 16: r0's first 16
    assert (st[0]["q_len"], st[0]["kv_prefix"], st[0]["emit"], st[0]["page_ids"]) == ([16], [0], [0], [0])
    # step 1: 9 tokens < 16 -> drain: r0's last 4 (completes, emits), r1's 5
    assert (st[1]["q_len"], st[1]["kv_prefix"], st[1]["emit"], st[1]["page_ids"]) == ([4, 5], [16, 0], [1, 1], [0, 1, 2])
    # step 2: two decodes whose input tokens are still on the device (rows 0 and 1 of step 1)
    assert (st[2]["q_len"], st[2]["kv_prefix"], st[2]["tok_src"]) == ([1, 1], [20, 5], [-1, -2])
    # r1 emits its 2nd (= EOS) token in step 2, read back after step 3 is formed: step 3 still runs it
    assert (st[3]["req_ids"], st[3]["kv_prefix"]) == ([0, 1], [21, 6])
    assert (st[4]["req_ids"], st[4]["kv_prefix"]) == ([0], [22])      # r1 retired; r0 useless token
    assert st[5]["req_ids"] == []
    assert s.stats["useless"] == 2 and s.stats["finished"] == 2 and s.stats["generated"] == 7


def _check_invariants(s, reqs, steps, n_pages, bdense, eos=False):
    prompts = {r: p for r, p, _ in reqs}
    produced = {}          # rid -> tokens emitted so far (from fake_ids)
    cursor = {r: 0 for r in prompts}
    first_admit = []
    for i, st in enumerate(steps):
        T = sum(st["q_len"])
        n_dec = sum(1 for r, kv in zip(st["req_ids"], st["kv_prefix"]) if kv >= len(prompts[r]))
        assert T == 0 or T in bdense or T < min(bdense) or T == n_dec    # A-26 (decodes never wait)
        owners = {}
        src = st["tok_src"]
        row_tok0 = np.concatenate([[0], np.cumsum(st["q_len"])]).astype(int)
        ids = fake_ids(st["step"], st["req_ids"])
        for j, r in enumerate(st["req_ids"]):
            if r not in first_admit:
                first_admit.append(r)
            q, kv = st["q_len"][j], st["kv_prefix"][j]
            pages = st["page_ids"][st["page_indptr"][j]:st["page_indptr"][j + 1]]
            assert len(pages) == -(-(kv + q) // 16)
            for p in pages:
                assert 0 <= p < n_pages and owners.setdefault(p, r) == r
            toks = src[row_tok0[j]:row_tok0[j] + q]
            if kv < len(prompts[r]):              # prompt chunk: next tokens in order, exactly once
                if kv == 0 and cursor[r] > 0:          # restarted after an eviction (A-27)
                    assert s.stats["evictions"] > 0
                    cursor[r], produced[r] = 0, []
                assert kv == cursor[r] and toks == prompts[r][kv:kv + q]
                cursor[r] += q
            else:                                  # decode: input = the request's last produced token
                assert q == 1 and kv == len(prompts[r]) + len(produced[r]) - 1
                t = toks[0]
                if t < 0:
                    prev = steps[i - 1]
                    assert prev["req_ids"][-(1 + t)] == r
                    t = fake_ids(prev["step"], prev["req_ids"])[-(1 + t)]
                assert t == produced[r][-1]
            if st["emit"][j]:
                produced.setdefault(r, []).append(ids[j])
        # pages of concurrently scheduled requests are disjoint (checked via owners)
    assert all(cursor[r] == len(prompts[r]) for r in prompts)
    if not s.stats["evictions"]:
        assert first_admit == sorted(first_admit)                # FCFS
        for r, p, out in reqs:
            if not eos:
                assert len(produced[r]) == out + 1               # exactly one useless token
        if not eos:
            assert s.stats["useless"] == len(reqs)


@pytest.mark.parametrize("name,n,pages,bd,avg", [("lmsys", 60, 400, [256, 128, 64], 40),
                                                  ("splitwise", 40, 300, [512, 256], 40),
                                                  ("sharegpt", 50, 2000, [256, 192, 128, 64, 32], 64)])
def test_oracle_invariants(name, n, pages, bd, avg):
    reqs = trace(n, name)
    s = OS.Scheduler(pages, 16, bd, avg)
    for r, p, o in reqs:
        s.submit(r, p, o)
    steps = drive(s)
    assert s.idle() and s.stats["finished"] == n
    _check_invariants(s, reqs, steps, pages, bd)
    assert s.stats["peak_pages_used"] <= pages


def test_oracle_peak_estimate_bounds():
    """A-27 estimate vs brute force: with every request decoding exactly its
    predicted length, the per-request ceil page sum at each future step never
    exceeds the estimate, and the estimate is within one page per request."""
    rng = np.random.default_rng(0)
    for _ in range(50):
        s = OS.Scheduler(10 ** 6, 16, [64], int(rng.integers(1, 300)))
        reqs = []
        for i in range(int(rng.integers(1, 30))):
            r = OS._Req(i, [1] * int(rng.integers(1, 900)), 5, i)
            r.generated = int(rng.integers(0, 400))
            reqs.append(r)
        est = s._peak_pages(reqs)
        taus = [max(s.avg - r.generated, 1) for r in reqs]
        brute = max(sum(-(-(len(r.prompt) + r.generated + t) // 16) for r, tr in zip(reqs, taus) if tr >= t)
                    for t in range(1, max(taus) + 1))
        assert brute <= est <= brute + len(reqs)


def test_oracle_eviction_and_eos():
    """Tiny pool (decode lengths above the average force evictions) and an
    eos_id hit by the fake model: still every prompt token once, in order,
    and token plumbing intact."""
    reqs = trace(30, "sharegpt", seed=5, scale=0.3)
    s = OS.Scheduler(40, 16, [64, 32], 1, eos_id=3)
    for r, p, o in reqs:
        s.submit(r, p, o)
    steps = drive(s, max_steps=5000)
    assert s.idle() and s.stats["evictions"] > 0 and s.stats["finished"] == len(reqs)
    _check_invariants(s, reqs, steps, 40, [64, 32], eos=True)
    s2 = OS.Scheduler(40, 16, [64, 32], 1, eos_id=3)
    for r, p, o in reqs:
        s2.submit(r, p, o)
    assert drive(s2, max_steps=5000) == steps          # deterministic


@pytest.mark.parametrize("case", range(6))
def test_native_scheduler_bit_exact(case):
    from paper_2408_12757_b200 import nf
    cfgs = [("lmsys", 60, 400, [256, 128, 64], 40, -1, 0.2), ("splitwise", 40, 300, [512, 256], 40, -1, 0.2),
            ("lmsys", 120, 4000, [48, 24], 60, -1, 0.3, 7),  # decode count above the discrete size (A-26)
            ("sharegpt", 50, 2000, [256, 192, 128, 64, 32], 64, -1, 0.2), ("sharegpt", 30, 40, [64, 32], 1, 3, 0.3),
            ("splitwise", 25, 120, [2048, 1024, 512, 256], 30, 11, 0.5)]
    name, n, pages, bd, avg, eos, scale = cfgs[case][:7]
    reqs = trace(n, name, seed=cfgs[case][7] if len(cfgs[case]) > 7 else case + 3, scale=scale)
    a = OS.Scheduler(pages, 16, bd, avg, eos_id=eos)
    b = nf.Scheduler(pages, 16, bd, avg, eos_id=eos)
    for r, p, o in reqs:
        a.submit(r, p, o)
        b.submit(r, p, o)
    sa = drive(a, max_steps=5000)
    sb = drive(b, max_steps=5000, as_dict=True)
    assert len(sa) == len(sb)
    for x, y in zip(sa, sb):
        assert x == y
    st = b.stats()
    for k, v in a.stats.items():
        assert st[k] == v, k


def test_native_scheduler_errors():
    from paper_2408_12757_b200 import nf
    with pytest.raises(nf.NFError):
        nf.Scheduler(0, 16, [64], 8)
    s = nf.Scheduler(64, 16, [64], 8)
    s.submit(1, [1, 2], 3)
    with pytest.raises(nf.NFError):
        s.submit(1, [1], 1)                               # duplicate id
    with pytest.raises(nf.NFError):
        s.submit(2, [], 1)
    with pytest.raises(nf.NFError):
        s.complete(5, [0])                                # not pending


def test_discrete_batch_never_defers_decodes():
    """A-26: 6 decoding requests + 1 prompt token pending, allowed sizes {8, 4}:
    the largest size not above the 7 available tokens is 4 < 6 decodes, so the
    step runs all 6 decodes (up to the largest size) and no prefill."""
    s = OS.Scheduler(256, 16, [8, 4], 50)
    for r in range(7):
        q = OS._Req(r, [r + 1], 20, r)
        q.admit_seq = r
        if r < 6:
            q.prefilled, q.generated = 1, 1
        s.running.append(q)
    comp = s._compose()
    assert [(c[0].rid, c[1], c[2]) for c in comp] == [(r, 1, 1) for r in range(6)]
    s2 = OS.Scheduler(256, 16, [8, 4], 50)
    s2.running = s.running[:4] + s.running[6:]          # 4 decodes + 1 prompt token: B = 4, decodes only
    assert [(c[0].rid, c[1]) for c in s2._compose()] == [(r, 1) for r in range(4)]


def test_native_traces_exercise_the_decode_rule():
    """The bit-exact native-vs-oracle traces include steps where the decode count
    exceeds the largest allowed size not above the available tokens (A-26)."""
    hits = 0
    for (name, n, pages, bd, avg, eos, scale, seed) in [("lmsys", 120, 4000, [48, 24], 60, -1, 0.3, 7)]:
        reqs = trace(n, name, seed=seed, scale=scale)
        s = OS.Scheduler(pages, 16, bd, avg, eos_id=eos)
        for r, p, o in reqs:
            s.submit(r, p, o)
        orig = s._compose

        def spy():
            nonlocal hits
            dec = [r for r in s.running if r.prefilled == len(r.prompt)]
            avail = len(dec) + sum(len(r.prompt) - r.prefilled for r in s.running)
            fits = [b for b in s.bdense if b <= avail]
            if (fits[0] if fits else avail) < len(dec):
                hits += 1
            return orig()
        s._compose = spy
        drive(s, max_steps=5000)
    assert hits > 0
