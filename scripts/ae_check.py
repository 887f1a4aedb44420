"""Megakernel bring-up check: mid-config parity (actions + per-layer cosines vs the fp64 oracle),
full-scale golden actions, and replay / AE timing.  Run under `timeout` on the GPU box."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from _util import cosine, rel_err  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config, mid_config  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"


def report(y, ref):
    d = y - ref
    return {"max_abs": float(np.abs(d).max()), "rel": rel_err(y, ref, 0.1), "cos": cosine(y, ref)}


if what in ("all", "mid"):
    for views, prompt in [(1, 0), (2, 0), (3, 32)]:
        cfg = mid_config(views=views, prompt_tokens=prompt)
        x = O.gen_inputs(cfg, 1)
        AR = cfg.ae_layers * cfg.flow_steps
        rec = [("ae.down", i, (cfg.suffix_tokens, cfg.ae_width)) for i in range(AR)]
        rec += [("ae.head", s, (cfg.chunk_len, cfg.ae_action_dim)) for s in range(cfg.flow_steps)]
        ref, recs = O.port_forward(cfg, x, record=rec)
        eng = E.Engine(cfg, record_checkpoints=True)
        eng.gen_weights(1)
        print(eng.describe()[-3:] if views == 1 else "", flush=True)
        y = eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
        cos = {f"{n}[{i}]": cosine(eng.checkpoint(n, i, *r.shape), r) for (n, i), r in recs.items()}
        worst = sorted(cos.items(), key=lambda kv: kv[1])[:4]
        print(f"mid {views}v+{prompt}p record: {report(y, ref)} worst {worst}", flush=True)
        g = E.Engine(cfg)
        g.gen_weights(1)
        y2 = g.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
        print(f"mid {views}v+{prompt}p graph : {report(y2, ref)}  |graph-record| {np.abs(y2 - y).max():.2e}",
              flush=True)

if what in ("all", "full"):
    for views in (1, 2):
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", f"full_{views}v.json")))
        ref = np.array(gold["actions"], dtype=np.float64).reshape(63, 32)
        cfg = default_config(views=views)
        x = O.gen_inputs(cfg, 1)
        eng = E.Engine(cfg)
        eng.gen_weights(1)
        t = time.time()
        y = eng.run(x["patches"], x["state"], x["noise"])
        print(f"full {views}v: {report(y, ref)}  first run {time.time() - t:.2f}s", flush=True)
        import torch
        st = torch.cuda.Stream()
        for _ in range(3):
            eng.replay(0, st.cuda_stream)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for a, b in ev:
            a.record(st)
            eng.replay(0, st.cuda_stream)
            b.record(st)
        st.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ev)
        print(f"full {views}v replay p50 {ms[10]:.3f} ms  min {ms[0]:.3f}", flush=True)
        for part, name in ((1, "prefix"), (2, "action")):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
            for a, b in ev:
                a.record(st)
                eng.replay(part, st.cuda_stream)
                b.record(st)
            st.synchronize()
            ms = sorted(a.elapsed_time(b) for a, b in ev)
            print(f"full {views}v {name} p50 {ms[5]:.3f} ms", flush=True)
        y3 = eng.run(x["patches"], x["state"], x["noise"])
        print(f"full {views}v after replays: {report(y3, ref)}", flush=True)
