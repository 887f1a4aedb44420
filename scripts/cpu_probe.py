"""Host-CPU speed probe for the reference arm: the reference's own rtvla::matmul (oracle/_ref)
on the llm.ffn shape for a few rows (B = [2048, 32768] fp64 re-streamed per row, the pattern
that dominates a full-scale rtvla::evaluate), plus the tiny-config evaluate.  Prints one JSON
line; compare the container against the GPU box host before sizing the reference arm."""
import ctypes
import json
import os
import platform
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2510_26742_b200.config import tiny_config  # noqa: E402

lib = O.ref_lib()
rows, k, m = 32, 2048, 32768
a = np.random.default_rng(0).uniform(-1, 1, (rows, k))
b = np.random.default_rng(1).uniform(-1, 1, (k, m))
y = np.zeros((rows, m))
dp = ctypes.POINTER(ctypes.c_double)
best = 1e9
for _ in range(3):
    t = time.perf_counter()
    lib.ref_matmul(a.ctypes.data_as(dp), rows, k, b.ctypes.data_as(dp), m, y.ctypes.data_as(dp))
    best = min(best, time.perf_counter() - t)
cfg = tiny_config()
ctx = O.RefContext(cfg)
ts = []
for _ in range(5):
    t = time.perf_counter()
    ctx.evaluate()
    ts.append(time.perf_counter() - t)
ctx.close()
cpu = ""
try:
    cpu = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":", 1)[1].strip()
except Exception:
    pass
print(json.dumps({"matmul_llm_ffn_ms_per_row": best / rows * 1e3, "gmac_s": rows * k * m / best / 1e9,
                  "tiny_evaluate_ms": float(np.median(ts)) * 1e3, "nproc": os.cpu_count(), "cpu": cpu,
                  "libc": platform.libc_ver()}))
