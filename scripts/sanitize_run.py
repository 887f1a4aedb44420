"""One eager mid-config inference per engine variant, for compute-sanitizer (scripts/sanitize.sh).
argv[1] = views.  The action-expert megakernel runs as a plain cooperative launch when the
environment disables its CTA-pair tasks (PI0B_AE_PAIR=0 PI0B_AE_PAIR_FFN=0)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import mid_config  # noqa: E402

views = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prompt = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = mid_config(views=views, prompt_tokens=prompt)
x = O.gen_inputs(cfg, 1)
ref, _ = O.port_forward(cfg, x)
eng = E.Engine(cfg, use_cuda_graph=False)
eng.gen_weights(1)
y = eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
print(f"sanitize_run views={views} prompt={prompt}: max |engine - oracle| = {np.abs(y - ref).max():.3e}")
