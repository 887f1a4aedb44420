"""View-sharded vision encoder (BASELINE.json north_star: "a view-sharded SigLIP
stage, where each GPU encodes one camera view and gathers the tokens over NVLink P2P").

Functional test on ONE device: `ve_shards` engines (one per view) run concurrently on their own
streams and exchange rows through the same peer-memory protocol a multi-GPU run uses (the fused
push + system-scope release kernel and the acquire wait, kernels_misc.cu) -- here the "peer"
buffers are simply other allocations on the same GPU.  Shard 0 runs the LLM and the action
expert on the gathered prefix.  The sharded result must equal the unsharded engine's (same
weights; only the GEMM tiling of the VE rows differs) and stay within the golden tolerance.
Multi-GPU latency is measured by bench.py (--gpus >= 2, "ve_shard")."""
import json
import os
import threading

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_26742_b200 import engine as E
from paper_2510_26742_b200.config import default_config, mid_config

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RUN_TO_RUN = 0.02


def _shards(cfg, n):
    engs = [E.Engine(cfg, ve_shards=n, ve_shard=g) for g in range(n)]
    for e in engs:
        e.gen_weights(1)
    bufs = [e.ve_buffers() for e in engs]
    for e in engs:
        e.set_ve_peers(bufs)
    return engs


def _sharded_run(engs, x):
    errs = []

    def peer(e):
        try:
            e.run_prefix(x["patches"], x.get("prompt"))
        except Exception as ex:  # surfaced below
            errs.append(ex)

    th = [threading.Thread(target=peer, args=(e,)) for e in engs[1:]]
    for t in th:
        t.start()
    y = engs[0].run(x["patches"], x["state"], x["noise"], x.get("prompt"))
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    return y


@pytest.mark.parametrize("views,prompt", [(2, 0), (3, 32)])
def test_ve_shard_mid_config_matches_unsharded(views, prompt):
    cfg = mid_config(views=views, prompt_tokens=prompt)
    x = O.gen_inputs(cfg, 1)
    ref, _ = O.port_forward(cfg, x)
    base = E.Engine(cfg)
    base.gen_weights(1)
    y0 = base.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
    engs = _shards(cfg, views)
    for it in range(4):  # several inferences: the per-inference sequence numbers advance
        y = _sharded_run(engs, x)
        d = float(np.abs(y - y0).max())
        print(f"{views} shards, run {it}: max |sharded - unsharded| {d:.3e}, vs oracle {np.abs(y - ref).max():.3e}")
        assert d < RUN_TO_RUN
        assert np.abs(y - ref).max() < 0.05
    # a fresh input on the same shards
    x2 = O.gen_inputs(cfg, 5)
    assert np.abs(_sharded_run(engs, x2) - base.run(x2["patches"], x2["state"], x2["noise"], x2.get("prompt"))).max() < RUN_TO_RUN


def test_ve_shard_full_scale_2v_golden():
    cfg = default_config(views=2)
    x = O.gen_inputs(cfg, 1)
    gold = np.array(json.load(open(os.path.join(GOLDEN, "full_2v.json")))["actions"]).reshape(63, 32)
    engs = _shards(cfg, 2)
    y = _sharded_run(engs, x)
    err = float(np.abs(y - gold).max())
    print(f"full 2v, 2 VE shards on one device: max |y - golden| {err:.3e}")
    assert err < 0.025


def test_ve_shard_rejects_misuse():
    cfg = mid_config(views=2)
    with pytest.raises(E.ShapeError):
        E.Engine(cfg, ve_shards=3, ve_shard=0)   # shards must divide the views
    e1 = E.Engine(cfg, ve_shards=2, ve_shard=1)
    e1.gen_weights(1)
    x = O.gen_inputs(cfg, 1)
    with pytest.raises(RuntimeError):
        e1.run_prefix(x["patches"])                # peers not set
    e1.set_ve_peers([e1.ve_buffers(), e1.ve_buffers()])
    with pytest.raises(RuntimeError):
        e1.run(x["patches"], x["state"], x["noise"])  # non-root shards serve run_prefix only
