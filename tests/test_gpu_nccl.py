"""The shipped NCCL data plane on one GPU: two (and four) processes form a real NCCL
TP group on GPU 0 (NCCL_HOSTID per process -> NCCL's socket transport over
loopback; tests/nccl_tp_worker.py).  The processes share the GPU through CUDA MPS
(a private pipe directory, started and stopped by the test); without MPS the test is
skipped: NCCL kernels of several processes wait on one another, and time-sliced
processes on one GPU are not guaranteed to run them at the same time (B200_PROFILING:
Xid 109 context-switch timeouts).  Collective performance here is meaningless;
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


@pytest.fixture(scope="module")
def mps(tmp_path_factory):
    """A private CUDA MPS daemon for the worker processes (None if unavailable)."""
    import shutil
    ctl = shutil.which("nvidia-cuda-mps-control")
    if not ctl or os.environ.get("NF_TEST_NO_MPS"):
        yield None
        return
    d = tmp_path_factory.mktemp("mps")
    env = dict(os.environ, CUDA_MPS_PIPE_DIRECTORY=str(d / "pipe"), CUDA_MPS_LOG_DIRECTORY=str(d / "log"))
    os.makedirs(env["CUDA_MPS_PIPE_DIRECTORY"])
    os.makedirs(env["CUDA_MPS_LOG_DIRECTORY"])
    r = subprocess.run([ctl, "-d"], env=env, capture_output=True, text=True, timeout=30)
    if r.returncode != 0:
        yield None
        return
    yield env
    subprocess.run([ctl], input="quit\n", env=env, capture_output=True, text=True, timeout=60)


@pytest.mark.parametrize("world", [2, 4])
def test_nccl_tp_group_on_one_gpu(tmp_path, world, mps):
    if not mps:
        pytest.skip("CUDA MPS unavailable: ranks that wait on one another must not time-slice one GPU")
    port = _free_port()
    procs, outs = [], []
    env = dict(mps)
    for r in range(world):
        out = tmp_path / f"rank{r}.json"
        outs.append(out)
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "nccl_tp_worker.py"), str(r), str(world),
                                       str(port), str(out)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                      text=True, env=env))
    logs = []
    for r, p in enumerate(procs):
        try:
            logs.append(p.communicate(timeout=420)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            dump = os.environ.get("NF_TEST_DUMP")
            if dump:
                import glob
                import shutil
                os.makedirs(dump, exist_ok=True)
                for f in glob.glob(str(tmp_path / "*.log")):
                    shutil.copy(f, dump)
            prog = "".join(open(str(o) + ".progress.log").read()[-600:] for o in outs
                           if os.path.exists(str(o) + ".progress.log"))
            raise AssertionError(f"NCCL group (world {world}, mps {bool(mps)}) timed out; progress:\n{prog}")
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
        # fused GEMM -> AllReduce through CUDA IPC peer mappings (NEXT-3)
        fz = r["fused"]
        assert "error" not in fz, (r["rank"], fz)
        assert fz["timeouts"] == 0, (r["rank"], fz)
        for name in ("sequential", "overlap42"):
            v = fz[name]
            assert v["ranks_identical"] and v["rel_l2"] <= 1e-2 and v["max_abs"] <= 5e-2, (r["rank"], name, v)
        g = fz["graph"]
        assert g["argmax_ok"] and g["replays_identical"] and g["ranks_identical"], (r["rank"], g)
