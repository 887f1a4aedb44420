"""Action-expert megakernel configuration sweep: p50 of the action-part replay (2 views) for a
list of PI0B_AE_* environment settings, one engine per setting.
    python scripts/ae_sweep.py 'PI0B_AE_DOWN_NCOL=128' 'PI0B_AE_DOWN_NCOL=128 PI0B_AE_DOWN_TASKS=144' ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402
from paper_2510_26742_b200.inputs import gen_inputs  # noqa: E402

cfg = default_config(views=2)
x = gen_inputs(cfg, 1)
for setting in [""] + sys.argv[1:]:
    keys = [kv.split("=")[0] for kv in setting.split()]
    for kv in setting.split():
        k, v = kv.split("=")
        os.environ[k] = v
    eng = E.Engine(cfg)
    eng.gen_weights(1)
    eng.run(x["patches"], x["state"], x["noise"])
    st = torch.cuda.Stream()
    for _ in range(3):
        eng.replay(2, st.cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(15)]
    for a, b in ev:
        a.record(st)
        eng.replay(2, st.cuda_stream)
        b.record(st)
    st.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    print(f"{setting or 'default':60s} action p50 {ms[7]:.3f} ms  min {ms[0]:.3f}", flush=True)
    del eng
    for k in keys:
        del os.environ[k]
