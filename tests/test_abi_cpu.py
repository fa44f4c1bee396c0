"""C-ABI library: loads without a GPU, exports every symbol include/nf.h
declares, host-only metadata is bit-exact with the oracle, validation errors.
CPU only (no compute calls)."""
import os
import re
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import metadata as md

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def nf():
    from paper_2408_12757_b200 import build
    build.build()
    from paper_2408_12757_b200 import nf as _nf
    return _nf


def header_functions():
    src = open(os.path.join(ROOT, "include", "nf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nf_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported(nf):
    names = header_functions()
    assert len(names) >= 18
    for n in names:
        assert hasattr(nf.lib, n), f"{n} declared in nf.h but not exported"
    assert set(names) == set(nf.EXPORTED)
    assert nf.lib.nf_abi_version() == 3


def _cfg(nf, shape, **kw):
    from paper_2408_12757_b200.runtime import cfg_from_shape
    return cfg_from_shape(shape, **kw)


@pytest.mark.parametrize("case", ["c1", "c2", "random"])
def test_metadata_bit_exact_vs_oracle(nf, case):
    if case == "c1":
        b, shape = synth.c1_batch(), synth.SHAPES["c1"]
    elif case == "c2":
        b, shape = synth.workload_batch(2048, 1024, 512), synth.SHAPES["llama3-8b"]
    else:
        rng = np.random.default_rng(0)
        n = 37
        b = synth.make_batch(rng.integers(1, 40, n), rng.integers(0, 200, n), seed=9, pool_slack=11)
        shape = synth.SHAPES["c1"]
    cfg = _cfg(nf, shape)
    nb = nf.Batch.from_any(b)
    pos, slot = nf.batch_metadata(cfg, nb)
    opos = md.positions(b.q_len, b.kv_prefix)
    pages, offs = md.write_slots(b.q_len, b.kv_prefix, b.page_indptr, b.page_ids)
    assert np.array_equal(pos, opos)
    assert np.array_equal(slot, pages * 16 + offs)


def test_snap_cuts_bit_exact_vs_oracle(nf):
    rng = np.random.default_rng(1)
    for trial in range(30):
        n = int(rng.integers(1, 30))
        q = rng.integers(1, 50, n)
        b = synth.make_batch(q, np.zeros(n, int), seed=trial)
        k = int(rng.integers(1, 5))
        shares = rng.integers(1, 9, k)
        got = nf.snap_cuts(nf.Batch.from_any(b), shares)
        exp = md.snap_cuts(q, [Fraction(int(s), int(shares.sum())) for s in shares])
        assert list(got) == exp


def test_validation_errors(nf):
    cfg = _cfg(nf, synth.SHAPES["c1"])
    b = synth.make_batch([1, 3], [5, 0])
    bad = nf.Batch(b.q_len, b.kv_prefix, b.page_indptr, b.page_ids, n_pages_pool=1)  # page id out of pool
    with pytest.raises(nf.NFError) as e:
        nf.batch_metadata(cfg, bad)
    assert e.value.status == nf.NF_EINVAL and "outside pool" in str(e.value)
    few = nf.Batch([1, 3], [40, 0], b.page_indptr, b.page_ids, b.n_pages_pool)  # too few pages
    with pytest.raises(nf.NFError):
        nf.batch_metadata(cfg, few)
    neg = nf.Batch([0, 3], [5, 0], b.page_indptr, b.page_ids, b.n_pages_pool)
    with pytest.raises(nf.NFError):
        nf.workspace_size(cfg, neg)
    bad_cfg = _cfg(nf, synth.shape_with(synth.SHAPES["c1"], head_dim=96))
    with pytest.raises(nf.NFError) as e:
        nf.workspace_size(bad_cfg, nf.Batch.from_any(b))
    assert e.value.status == nf.NF_EUNSUPPORTED
    with pytest.raises(nf.NFError):
        _ = nf.workspace_size(_cfg(nf, synth.SHAPES["c1"], tp_size=4), nf.Batch.from_any(b))  # 4 does not divide kh=2
    with pytest.raises(nf.NFError):
        nf.Plan.explicit(cfg, mode=7)
    with pytest.raises(nf.NFError):
        nf.Plan.explicit(cfg, mode=nf.OVERLAP, shares=(1, 0))
    p = nf.Plan.explicit(cfg, mode=nf.SEQUENTIAL, shares=(1, 1))
    assert p.spec().n_nano == 1
    p2 = nf.Plan.explicit(cfg, mode=nf.OVERLAP, shares=(1, 1), balance=True)
    s = p2.spec()
    assert s.n_nano == 2 and s.balance == 1 and list(s.share)[:2] == [1, 1]


def test_workspace_size_monotone(nf):
    cfg = _cfg(nf, synth.SHAPES["llama3-8b"])
    small = nf.workspace_size(cfg, nf.Batch.from_any(synth.c1_batch()))
    big = nf.workspace_size(cfg, nf.Batch.from_any(synth.workload_batch(2048, 1024, 512)))
    assert 0 < small < big


def test_moe_cfg_validation_and_sizes(nf):
    """MoE fields of nf_model_cfg (A-20..A-23): validation, packed
    sizes, grouped-row capacity (segments padded to 128 rows)."""
    import ctypes
    assert ctypes.sizeof(nf.ModelCfg) == 14 * 4
    sh = synth.SHAPES["mixtral-8x7b"]
    cfg = _cfg(nf, sh, tp_size=8)
    D, F, E = sh.d_model, sh.d_ffn // 8, sh.n_experts
    sizes = nf.packed_layer_bytes(cfg)
    assert sizes[3] == E * ((F + 127) // 128) * 256 * D * 2
    assert sizes[4] == E * D * F * 2 and sizes[5] == E * D * 4
    assert nf.packed_layer_bytes(_cfg(nf, synth.SHAPES["llama3-8b"]))[5] == 0
    for T in (1, 127, 2048):
        cap = nf.moe_rows_cap(cfg, T)
        assert cap % 128 == 0 and cap >= T * 2 + E * 127
    b = nf.Batch.from_any(synth.c1_batch())
    assert nf.workspace_size(cfg, b) > nf.workspace_size(_cfg(nf, synth.shape_with(sh, n_experts=0), tp_size=8), b)
    with pytest.raises(nf.NFError) as e:
        nf.workspace_size(_cfg(nf, synth.shape_with(sh, top_k=9)), b)
    assert e.value.status == nf.NF_EINVAL
    with pytest.raises(nf.NFError) as e:
        nf.workspace_size(_cfg(nf, synth.shape_with(sh, n_experts=32)), b)
    assert e.value.status == nf.NF_EUNSUPPORTED
    with pytest.raises(nf.NFError) as e:
        nf.moe_route(_cfg(nf, synth.SHAPES["llama3-8b"]), 1, 1, 4, 1, 1, 1, 1, 1, 1, 1 << 20, 0)
    assert e.value.status == nf.NF_EINVAL


def test_forward_rejects_incomplete_packed_layers(nf):
    """nf_layer_forward / nf_model_step validate the packed-layer pointers before
    any launch: a MoE layer without its router, a NULL projection (NF_EINVAL)."""
    sh = synth.SHAPES["c1-moe"]
    cfg = _cfg(nf, sh)
    b = nf.Batch.from_any(synth.c1_batch())
    plan = nf.Plan.explicit(cfg, mode=nf.SEQUENTIAL)
    fake = {"w_qkv": 256, "w_o": 512, "w_gate_up": 768, "w_down": 1024}     # never dereferenced
    with pytest.raises(nf.NFError) as e:
        nf.layer_forward(plan, fake, 4096, b, 8192, 12288, 16384, 1 << 30, 0)
    assert e.value.status == nf.NF_EINVAL and "w_router" in str(e.value)
    with pytest.raises(nf.NFError) as e:
        nf.layer_forward(plan, dict(fake, w_router=2048, w_down=None), 4096, b, 8192, 12288, 16384, 1 << 30, 0)
    assert e.value.status == nf.NF_EINVAL and "NULL packed weight" in str(e.value)


def test_tp_plan_and_comm_validation(nf):
    """n_dense must divide n_nano (and equal it at tp_size 1); SEQUENTIAL collapses to one
    nano-batch; the emulated group's AllReduce mode, the loopback communicator and the
    vocab-parallel head's divisibility are validated; plan hashes ignore tp_rank only."""
    from paper_2408_12757_b200.runtime import cfg_from_shape
    c8 = cfg_from_shape(synth.SHAPES["llama2-70b"], tp_size=8, tp_rank=1)
    p = nf.Plan.explicit(c8, nf.OVERLAP, shares=(1, 1, 1, 1), n_dense=2)
    assert p.spec().n_dense == 2 and p.spec().n_nano == 4
    assert nf.Plan.explicit(c8, nf.OVERLAP, shares=(1, 1, 1, 1)).spec().n_dense == 4   # 0 = n_nano
    for bad in (3, 5, -1):
        with pytest.raises(nf.NFError) as e:
            nf.Plan.explicit(c8, nf.OVERLAP, shares=(1, 1, 1, 1), n_dense=bad)
        assert e.value.status == nf.NF_EINVAL
    c1 = cfg_from_shape(synth.SHAPES["llama3-8b"])
    with pytest.raises(nf.NFError):
        nf.Plan.explicit(c1, nf.OVERLAP, shares=(1, 1, 1, 1), n_dense=2)
    s = nf.Plan.explicit(c8, nf.SEQUENTIAL, n_dense=0).spec()
    assert s.n_nano == 1 and s.n_dense == 1
    # hashes: equal across ranks, different across plans
    c8b = cfg_from_shape(synth.SHAPES["llama2-70b"], tp_size=8, tp_rank=5)
    assert nf.Plan.explicit(c8b, nf.OVERLAP, shares=(1, 1, 1, 1), n_dense=2).hash() == p.hash()
    assert nf.Plan.explicit(c8, nf.OVERLAP, shares=(1, 1, 1, 1), n_dense=1).hash() != p.hash()
    with pytest.raises(nf.NFError):
        nf.lib.nf_comm_create_local  # noqa: B018  (exists)
        nf.comm_create_local(2, 7)
    with pytest.raises(nf.NFError):
        nf.comm_create_local(9)
    h = nf.comm_create_loopback(8, 3)
    assert h
    nf.comm_loopback_set_link(h, 725.0)   # link-time model on / off
    nf.comm_loopback_set_link(h, 0.0)
    for bad in (-1.0, float("nan"), 1e7):
        with pytest.raises(nf.NFError):
            nf.comm_loopback_set_link(h, bad)
    nf.comm_destroy(h)
    g = nf.comm_create_local(2)
    with pytest.raises(nf.NFError):   # only a loopback communicator has a link model
        nf.comm_loopback_set_link(g[0], 725.0)
    for c in g:
        nf.comm_destroy(c)
    with pytest.raises(nf.NFError):
        nf.comm_create_loopback(8, 8)
    # vocab-parallel head: V % N and (V/N) % 32
    for V, ok in ((32000, True), (32008, False), (8448, True), (8320, False)):
        cfg = cfg_from_shape(synth.shape_with(synth.SHAPES["llama2-70b"], vocab=V), tp_size=8)
        if ok:
            nf.packed_layer_bytes(cfg)
        else:
            with pytest.raises(nf.NFError):
                nf.packed_layer_bytes(cfg)


def test_comm_sym_bytes_layout():
    """nf_comm_sym_bytes (NEXT-3 symmetric buffer, host-only size query): it must hold, for
    each of the 8 fused sites, a result region of max_tokens x d_model bf16 and the staging of
    every 128x256 output block once, grows with the token count and the group size only
    through the per-owner rounding, and rejects d_model not a multiple of 256."""
    import ctypes as C

    from paper_2408_12757_b200 import nf
    cfg = nf.ModelCfg()
    cfg.d_model, cfg.n_layers, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim = 8192, 1, 64, 8, 128
    cfg.d_ffn, cfg.vocab, cfg.page_size, cfg.tp_rank = 28672, 32000, 16, 0
    sizes = {}
    for tp in (1, 2, 8):
        cfg.tp_size = tp
        for T in (1, 2048):
            sizes[(tp, T)] = nf.comm_sym_bytes(cfg, T)
    blocks = (2048 + 127) // 128 * (8192 // 256)
    for tp in (1, 2, 8):
        assert sizes[(tp, 2048)] >= 8 * (2048 * 8192 * 2 + blocks * 128 * 256 * 2)
        assert sizes[(tp, 2048)] > sizes[(tp, 1)]
    cfg.d_model = 8192 + 128
    with pytest.raises(nf.NFError):
        nf.comm_sym_bytes(cfg, 16)
