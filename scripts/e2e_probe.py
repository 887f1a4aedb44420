import time, ctypes, numpy as np, os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2510_26742_b200 import engine as E
from paper_2510_26742_b200.config import default_config
from paper_2510_26742_b200.inputs import gen_inputs
cfg = default_config(views=2)
x = gen_inputs(cfg, 1)
p = np.ascontiguousarray(x["patches"])
out = np.zeros(p.size, dtype=np.uint16)
L = E.lib()
ts = []
for _ in range(50):
    t0 = time.perf_counter(); L.pi0b_f64_to_bf16_host(p.ctypes.data_as(E._dp), p.size, out.ctypes.data); ts.append(time.perf_counter() - t0)
print("host f64->bf16 of the 2v patches, one thread: %.1f us" % (np.median(ts) * 1e6))
t = []
for _ in range(50):
    t0 = time.perf_counter(); q = p.copy(); t.append(time.perf_counter() - t0)
print("numpy copy of the patches: %.1f us" % (np.median(t) * 1e6))
eng = E.Engine(cfg); eng.gen_weights(1)
eng.run(x["patches"], x["state"], x["noise"])
import torch
s = torch.cuda.Stream()
for mode in ("replay+sync", "run"):
    t = []
    for i in range(60):
        t0 = time.perf_counter()
        if mode == "run":
            eng.run(x["patches"], x["state"], x["noise"])
        else:
            eng.replay(0); eng.sync()
        t.append(time.perf_counter() - t0)
    print(mode, "%.1f us" % (np.median(t[10:]) * 1e6))
t = []
for i in range(60):
    t0 = time.perf_counter(); eng.run_action(x["state"], x["noise"]); t.append(time.perf_counter() - t0)
print("run_action %.1f us" % (np.median(t[10:]) * 1e6))
# CPU cost of the graph launch call itself (no sync)
t = []
for i in range(30):
    eng.sync()
    t0 = time.perf_counter(); eng.replay(0); t.append(time.perf_counter() - t0)
eng.sync()
print("cudaGraphLaunch (replay call, CPU side) %.1f us" % (np.median(t[5:]) * 1e6))
