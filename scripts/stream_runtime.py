"""SURVEY 8(f) f2 on the full model: the streaming runtime (pi0b_stream_run) at the paper's 480 Hz
and at the reference simulator's predicted B200 maximum, both KV policies, 2 views, one flow step
per tick.  On the GPU box:  python scripts/stream_runtime.py [seconds] > gpurun_out/stream_runtime.json
Then (CPU) scripts/streamsim_b200.py-style comparison: see DESIGN.md."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402

seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
cfg = default_config(views=2).replace(flow_steps=1)
out = {"views": 2, "flow_steps_per_tick": 1, "seconds": seconds, "runs": []}
# the maximum comes from the reference simulator on this engine's stream numbers
# (profiles/r01_streamsim_2v.json b200_max_feasible_rate_hz; 1440 Hz at the time of writing)
max_rate = float(os.environ.get("PI0B_STREAM_MAX_HZ", "1440"))
for rate, policy in ((480.0, "most_recent"), (480.0, "frame_sticky"), (max_rate, "most_recent")):
    r = E.stream_run(cfg, seconds, ae_rate=rate, kv_policy=policy)
    r.update({"ae_rate_target": rate, "kv_policy": policy})
    out["runs"].append(r)
print(json.dumps(out, indent=1))
