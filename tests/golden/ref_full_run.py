"""One full-scale run of the UNMODIFIED reference ``rtvla::evaluate`` (compiled into
oracle/_ref/librtvla_ref.so), recording its spot values — the cross-check that pins the
full-scale restatement goldens (make_golden.py) to the reference itself, as SURVEY.md 8(c)
did for 1 and 2 views.

Single-threaded fp64 (the reference has no internal parallelism): 13 min (1v), 24 min (2v),
~40 min (3v + 32-token prompt) and 22-26 GB RSS in this container.

Usage:  PYTHONPATH=. python tests/golden/ref_full_run.py VIEWS PROMPT  -> ref_full_<tag>.json
"""
import json
import os
import resource
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main(views: int, prompt: int) -> None:
    cfg = default_config(views=views, prompt_tokens=prompt)
    t0 = time.time()
    ctx = O.RefContext(cfg)            # build_pi0_graph + gen_weights + gen_inputs (seed 1)
    t1 = time.time()
    y = ctx.evaluate()                 # rtvla::evaluate, proj/src/evaluate.cpp:365-370
    t2 = time.time()
    ctx.close()
    tag = f"{views}v" + (f"{prompt}p" if prompt else "")
    doc = {"config": cfg.as_dict(), "weight_seed": 1, "input_seed": 1,
           "source": "reference rtvla::evaluate (unmodified, -O3, single thread)",
           "setup_seconds": t1 - t0, "evaluate_seconds": t2 - t1,
           "peak_rss_gb": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20,
           "y0": float(y.ravel()[0]), "y1": float(y.ravel()[1]), "ylast": float(y.ravel()[-1]),
           "sum": float(y.sum()), "abs_sum": float(np.abs(y).sum()),
           "actions": [float(v) for v in y.ravel()]}
    path = os.path.join(HERE, f"ref_full_{tag}.json")
    with open(path, "w") as f:
        json.dump(doc, f, indent=0)
    print("wrote", path, f"evaluate {t2 - t1:.1f} s")


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]))
