"""run() end-to-end overhead over a bare graph replay for different host staging thread counts
(PI0B_STAGING_THREADS, read at engine creation)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402
from paper_2510_26742_b200.inputs import gen_inputs  # noqa: E402

cfg = default_config(views=2)
x = gen_inputs(cfg, 1)
for n in sys.argv[1:] or ["0", "1", "3", "7"]:
    os.environ["PI0B_STAGING_THREADS"] = n
    eng = E.Engine(cfg)
    eng.gen_weights(1)
    eng.run(x["patches"], x["state"], x["noise"])
    r, g = [], []
    for i in range(40):
        t0 = time.perf_counter(); eng.replay(0); eng.sync(); g.append(time.perf_counter() - t0)
        t0 = time.perf_counter(); eng.run(x["patches"], x["state"], x["noise"]); r.append(time.perf_counter() - t0)
    print(f"staging threads {n}: run p50 {np.median(r[5:]) * 1e6:.0f} us, replay+sync p50 {np.median(g[5:]) * 1e6:.0f} us, "
          f"overhead {(np.median(r[5:]) - np.median(g[5:])) * 1e6:.0f} us")
    del eng
