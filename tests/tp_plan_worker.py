"""Worker of test_tp_gloo.test_tp_plans_identical_across_ranks: one process per TP rank
(gloo on CPU) loading libnf; every rank builds its TP plans -- explicit 4/2 pipeline
plans and the autosearch (nf_plan_create at tp_size = world) -- from the same inputs,
and the ranks' plan hashes, specs, schedule CSVs, step metadata and workspace sizes
are AllGathered and must be identical (the collective issue order depends on them)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def worker(rank, world, port, out):
    import numpy as np
    import torch.distributed as dist

    import synth
    from paper_2408_12757_b200 import nf
    from paper_2408_12757_b200.runtime import cfg_from_shape
    from test_planner_abi import synthetic_curves_tp

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    shape = synth.SHAPES["llama2-70b"]
    cfg = cfg_from_shape(shape, tp_size=world, tp_rank=rank)
    b = synth.workload_batch(512, 512, 1024)
    nb = nf.Batch.from_any(b)
    mine = []
    plans = [nf.Plan.explicit(cfg, nf.OVERLAP, shares=(1, 1, 1, 1), sm=[116, 16, 116, 116, 116, 116, 16], n_dense=2,
                              balance=2, graph=True),
             nf.Plan.explicit(cfg, nf.NANO_ONLY, shares=(3, 3, 5, 5), n_dense=2),
             nf.Plan.search(cfg, nb, synthetic_curves_tp(), mode=nf.OVERLAP, n_nano=4, max_iters=20)]
    for p in plans:
        sp = p.spec()
        mine.append((p.hash(), sp.mode, sp.n_nano, sp.n_dense, tuple(sp.share), tuple(sp.sm), p.csv()))
    pos, slot = nf.batch_metadata(cfg, nb)
    mine.append((int(pos.sum()), int(slot.astype(np.int64).sum()), nf.workspace_size(cfg, nb)))
    allp = [None] * world
    dist.all_gather_object(allp, mine)
    ok = all(a == allp[0] for a in allp)
    distinct = len({m[0] for m in mine[:3]}) == 3
    if rank == 0:
        np.save(out, np.array([ok, distinct]))
    dist.destroy_process_group()
