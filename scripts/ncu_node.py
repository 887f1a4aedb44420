"""Launch the kernels of one node (all instances, once) on a fresh full-scale engine so that
`ncu -k regex:<kernel> -c 1` captures exactly that node's first launch."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402
from paper_2510_26742_b200.inputs import gen_inputs  # noqa: E402

node = sys.argv[1]
views = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = default_config(views=views)
eng = E.Engine(cfg, use_cuda_graph=False)
eng.gen_weights(1)
if len(sys.argv) > 3 and sys.argv[3] == "run":
    x = gen_inputs(cfg, 1)
    eng.run(x["patches"], x["state"], x["noise"])
print(node, eng.time_node(node, reps=1))
