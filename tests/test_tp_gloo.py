"""world_size-2 (and 4) gloo test of the TP executor's dataflow on CPU:
runtime.shard_layer slicing + rank-major AllGather/interleave + residual on
rank 0 before AllReduce reproduce the unsharded oracle layer (T10)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
def test_tp_dataflow_gloo(tmp_path, world):
    from paper_2408_12757_b200 import build
    build.build()
    import tp_gloo_worker
    out = str(tmp_path / "err.npy")
    mp.start_processes(tp_gloo_worker.worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    errs = np.load(out)
    assert len(errs) == world and (errs < 1e-12).all(), errs


@pytest.mark.parametrize("world", [2, 4])
def test_tp_moe_dataflow_gloo(tmp_path, world):
    """MoE FFN under TP (every expert's F columns split across ranks,
    weighted partials AllReduced over gloo) == unsharded oracle moe_ffn."""
    import tp_gloo_worker
    out = str(tmp_path / "err_moe.npy")
    mp.start_processes(tp_gloo_worker.worker_moe, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    errs = np.load(out)
    assert len(errs) == world and (errs < 1e-12).all(), errs


@pytest.mark.parametrize("world", [2, 4])
def test_tp_plans_identical_across_ranks(tmp_path, world):
    """libnf on every rank (gloo, CPU): explicit and autosearched TP plans, their hashes,
    schedules, step metadata and workspace sizes are identical on all ranks."""
    from paper_2408_12757_b200 import build
    build.build()
    import tp_plan_worker
    out = str(tmp_path / "ok.npy")
    mp.start_processes(tp_plan_worker.worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    ok, distinct = np.load(out)
    assert ok and distinct
