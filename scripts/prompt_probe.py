"""Diagnostic: engine vs oracle error over (views, prompt) combinations, megakernel on/off."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import mid_config  # noqa: E402

for views, prompt in [(3, 7), (3, 32), (3, 39), (2, 200), (1, 300), (2, 45), (3, 0), (2, 230)]:
    cfg = mid_config(views=views, prompt_tokens=prompt)
    x = O.gen_inputs(cfg, 1)
    ref, _ = O.port_forward(cfg, x)
    out = []
    for mega in ("1", "0"):
        os.environ["PI0B_AE_MEGA"] = mega
        eng = E.Engine(cfg)
        eng.gen_weights(1)
        y = eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
        out.append(float(np.abs(y - ref).max()))
        eng.close()
    L = cfg.prefix_tokens
    print(f"views {views} prompt {prompt:4d} L {L:5d} Lp {(L + 31) // 32 * 32:5d}: mega {out[0]:.3e}  per-node {out[1]:.3e}", flush=True)
