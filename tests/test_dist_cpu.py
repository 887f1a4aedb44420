"""Multi-process host logic of bench.py's N > 1 path on CPU (gloo, world size 2): the timing
reduction is the max over ranks, `bench.py --gpus N` outside torchrun re-launches itself with N
ranks through the same launcher the driver uses, WORLD_SIZE != --gpus is refused, no NCCL
communicator is created, and the reference arm runs on rank 0 only (the other ranks exit 0
without work)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        # rank r reports [p50, p90, mean, e2e] = [10 + r, 11 + r, 10.5 + 2 r, 12 - r]
        vals = bench.reduce_over_ranks([10 + rank, 11 + rank, 10.5 + 2 * rank, 12 - rank])
        out.put((rank, vals))
    finally:
        dist.destroy_process_group()


def test_reduce_over_ranks_is_max_gloo():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(ws))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(ws):
        assert res[r] == [11.0, 12.0, 12.5, 12.0]


def test_reduce_single_process_is_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.reduce_over_ranks([1, 2.5]) == [1.0, 2.5]


def test_reference_arm_rank1_exits_without_work():
    env = dict(os.environ, WORLD_SIZE="2", RANK="1", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3"], capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_bench_gpus_n_spawns_replicas_over_gloo():
    """The real launcher path: no WORLD_SIZE in the environment, --gpus 2 -> torch.distributed.run
    with 2 ranks -> gloo group -> max/min over ranks printed by rank 0 only."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    doc = json.loads(lines[0])
    assert doc["world_size"] == 2
    assert doc["max"] == [1.0, 11.0] and doc["min"] == [0.0]
    assert doc["nccl_initialized"] is False
    assert doc["staging_threads"] >= 0


def test_bench_world_size_must_match_gpus():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--launch-check"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0
    assert "WORLD_SIZE=2 but --gpus 4" in (r.stderr + r.stdout)


# ---------------------------------------------------------------- view-sharded VE orchestration
# bench.ve_shard_bench over a world of 3 gloo ranks with a fake engine (no GPU): every rank takes
# part in the same collectives whatever fails where, so a failing rank can never leave the others
# waiting; rank 0 reports the latency only when every rank succeeded.

class _FakeBufs:
    def __init__(self, base):
        self.base = base

    def as_list(self):
        return [self.base + i for i in range(6)]


class _FakeEngine:
    fail = {}  # (rank, stage) -> raise

    def __init__(self, cfg, device=0, ve_shards=0, ve_shard=0, **_):
        self.rank = ve_shard
        self._check("create")

    def _check(self, stage):
        if _FakeEngine.fail.get((self.rank, stage)):
            raise RuntimeError(f"injected {stage} failure")

    def gen_weights(self, seed):
        pass

    def ve_buffers(self):
        return _FakeBufs(1000 * (self.rank + 1))

    def set_ve_peers(self, peers):
        assert len(peers) == 2

    def run(self, *a):
        import numpy as np
        return np.zeros((63, 32))

    def run_prefix(self, *a):
        self._check("prefix")

    def replay(self, part, stream):
        self._check(f"replay{part}")

    def close(self):
        pass


class _FakeTimer:
    def time(self, fn):
        fn(None)
        return 1.0


def _ve_worker(rank, ws, port, fail, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    from paper_2510_26742_b200 import engine as E
    from paper_2510_26742_b200.config import mid_config
    E.Engine = _FakeEngine
    _FakeEngine.fail = fail
    E.ipc_export = lambda p: bytes([p % 256]) * 64
    E.ipc_open = lambda h: h[0]
    E.ipc_close = lambda p: None
    E.VeBuffers.from_list = classmethod(lambda cls, v: _FakeBufs(v[0]))
    bench.DeviceTimer = _FakeTimer
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        res = bench.ve_shard_bench(mid_config(views=2), ws, rank, 0, steps=5, warmup=2, single_p50=2.0)
        out.put((rank, res))
    finally:
        dist.destroy_process_group()


def _run_ve(fail):
    ws, port = 3, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_ve_worker, args=(r, ws, port, fail, q)) for r in range(ws)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(ws))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[1] is None and res[2] is None  # only rank 0 reports
    return res[0]


@pytest.mark.parametrize("fail,expect", [
    ({}, "ok"),
    ({(1, "create"): True}, "rank 1 setup"),
    ({(1, "replay1"): True}, "rank 1 run"),
    ({(0, "replay0"): True}, "rank 0 run"),
])
def test_ve_shard_bench_orchestration_gloo(fail, expect):
    r = _run_ve(fail)
    if expect == "ok":
        assert r["gpus"] == 2 and r["steps"] == 5 and r["p50_ms"] == 1.0 and r["lowers_latency"] is True, r
    else:
        assert "error" in r and expect in r["error"], r
