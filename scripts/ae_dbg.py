"""Run the mid-config engine once (eager, no graph) and print the status: used for bisecting the
megakernel with PI0B_AE_LIMIT=<phases> and under compute-sanitizer."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# the per-task timestamps are compiled only into the trace variant of the library
_VAR = os.path.join(ROOT, "variants", "libpi0b_aetrace.so")
if not os.path.exists(_VAR):
    from paper_2510_26742_b200.build import build  # noqa: E402
    build(lib=_VAR, defines=["-DPI0B_AE_TRACE_CODE=1"])
os.environ.setdefault("PI0B_LIB", _VAR)
from oracle import oracle as O
from paper_2510_26742_b200 import engine as E
from paper_2510_26742_b200.config import mid_config
cfg = mid_config(views=int(sys.argv[1]) if len(sys.argv) > 1 else 1)
x = O.gen_inputs(cfg, 1)
eng = E.Engine(cfg, use_cuda_graph=False)
eng.gen_weights(1)
try:
    eng.run_prefix(x["patches"])
    print("prefix ok", flush=True)
    y = eng.run_action(x["state"], x["noise"])
    print("ok", float(abs(y).max()))
except Exception as e:
    print("FAIL", e)
