"""Per-node device time of one pi0 inference (eager launches timed with CUDA events),
plus the CUDA-graph replay time; writes gpurun_out/node_times.json."""
import collections
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402
from paper_2510_26742_b200.inputs import gen_inputs  # noqa: E402

views = int(sys.argv[1]) if len(sys.argv) > 1 else 2
prompt = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = default_config(views=views, prompt_tokens=prompt)
eng = E.Engine(cfg)
t = time.time()
eng.gen_weights(1)
print(f"gen_weights {time.time() - t:.2f}s")
x = gen_inputs(cfg, 1)
y = eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
plan = eng.describe()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
open(os.path.join(ROOT, "gpurun_out", "plan.txt"), "w").write("\n".join(plan))
counts = collections.Counter(l.split()[3] for l in plan if l.split()[2] in ("gemm", "attn", "skinny"))
rows = []
for node, n in counts.items():
    ms, launches = eng.time_node(node, reps=3)
    rows.append((node, n, ms * 1e3, ms * n))
rows.sort(key=lambda r: -r[3])
tot = sum(r[3] for r in rows)
for r in rows:
    print(f"{r[0]:16s} x{r[1]:4d}  {r[2]:9.2f} us/launch  {r[3]:8.3f} ms  {100 * r[3] / tot:5.1f}%")
print(f"sum of per-node eager times: {tot:.3f} ms")
s = torch.cuda.Stream()
for _ in range(5):
    eng.replay(0, s.cuda_stream)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ms = []
for _ in range(20):
    ev[0].record(s)
    eng.replay(0, s.cuda_stream)
    ev[1].record(s)
    torch.cuda.synchronize()
    ms.append(ev[0].elapsed_time(ev[1]))
print(f"graph replay p50 {np.median(ms):.3f} ms  (kernels/inference {eng.kernel_count(0)})")
t = []
for _ in range(10):
    t0 = time.perf_counter()
    eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
    t.append((time.perf_counter() - t0) * 1e3)
print(f"run() e2e p50 {np.median(t):.3f} ms")
json.dump({"rows": rows, "replay_ms": ms, "e2e_ms": t}, open(os.path.join(ROOT, "gpurun_out", "node_times.json"), "w"))
