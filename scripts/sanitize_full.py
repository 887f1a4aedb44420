"""One eager FULL-SCALE inference for compute-sanitizer memcheck: exercises the planner's
per-config tilings (llm.down bn 256 x 3 / bn 128 x 4 splits with the pull-form combine,
llm.attn key splits 2 / 4, llm.proj bn 128, ve.fc2 bn 128 x 2).  argv: views prompt."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402
from paper_2510_26742_b200.inputs import gen_inputs  # noqa: E402

views = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prompt = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = default_config(views=views, prompt_tokens=prompt)
eng = E.Engine(cfg, use_cuda_graph=False)
eng.gen_weights(1)
x = gen_inputs(cfg, 1)
y = eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
print(f"sanitize_full views={views} prompt={prompt}: finite {bool(np.isfinite(y).all())}, rms {float(np.sqrt((y ** 2).mean())):.4f}")
