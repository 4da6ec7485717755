"""N > 1 path on CPU: world_size-2 gloo tests of the multi-rank plumbing (paper_2301_01396_b200.
parallel) and an end-to-end torchrun launch of bench.py's reference arm (rank 0 alone prints)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    from paper_2301_01396_b200 import parallel as par
    env = par.init("gloo")
    got = dict(rank=env.rank, world=env.world)
    got["max"] = par.reduce_max(10.0 + env.rank)
    got["sum"] = par.reduce_sum(1.0 + env.rank)
    got["seed"] = par.scene_seed(4, env.rank)
    got["shard"] = list(par.shard(7, env.world, env.rank))
    par.barrier()
    got["thr"] = par.job_throughput(100.0, got["max"], env.world)
    par.shutdown()
    q.put(got)


def test_gloo_world2_plumbing():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda d: d["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r["max"] for r in res] == [11.0, 11.0]          # max over ranks
    assert [r["sum"] for r in res] == [3.0, 3.0]
    assert res[0]["seed"] != res[1]["seed"]                 # independent scenes
    assert res[0]["shard"] + res[1]["shard"] == list(range(7))
    assert res[0]["thr"] == pytest.approx(2 * 100.0 / 11e-3)


def test_shard_covers_everything():
    from paper_2301_01396_b200.parallel import shard
    for n in range(0, 20):
        for w in range(1, 9):
            parts = [list(shard(n, w, r)) for r in range(w)]
            assert sum(parts, []) == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_torchrun_reference_arm_world2():
    """bench.py --impl reference under torchrun with 2 ranks: exactly one JSON line (rank 0), exit 0."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl", "reference",
           "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-n", "12"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    for k in ("metric", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling", "dtype", "data",
              "config", "vs_baseline"):
        assert k in d, k
    assert d["higher_is_better"] is True and d["e2e"]["value"] == d["value"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
