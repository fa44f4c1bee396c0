"""The shipped NCCL data plane on one GPU: two (and four) processes form a real NCCL
TP group on GPU 0 (NCCL_HOSTID per process -> NCCL's socket transport over
loopback; tests/nccl_tp_worker.py).  Collective performance here is meaningless;
what is checked is that the NCCL path (nf_comm_create with a CTA cap, bf16
AllGather / AllReduce issued on the network stream in the TP pipeline's order,
the vocab-parallel LM head's AllGather, CUDA-graph capture with NCCL inside)
produces oracle-matching, rank-identical results."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_tp_group_on_one_gpu(tmp_path, world):
    port = _free_port()
    procs, outs = [], []
    for r in range(world):
        out = tmp_path / f"rank{r}.json"
        outs.append(out)
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "nccl_tp_worker.py"), str(r), str(world),
                                       str(port), str(out)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                      text=True))
    logs = []
    for p in procs:
        try:
            logs.append(p.communicate(timeout=600)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for r, p in enumerate(procs):
        assert p.returncode == 0, f"rank {r} failed:\n{logs[r][-4000:]}"
    res = [json.load(open(o)) for o in outs]
    print(json.dumps(res[0], indent=1))
    for r in res:
        for name, v in r["layer"].items():
            assert v["ranks_identical"], (r["rank"], name)
            assert v["rel_l2"] <= 1e-2 and v["max_abs"] <= 5e-2, (r["rank"], name, v)
        for name, v in r["step"].items():
            assert v["argmax_ok"] and v["replays_identical"] and v["ranks_identical"], (r["rank"], name, v)
