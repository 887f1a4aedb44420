"""Timeline of the prefill GEMM kernel (gemm.cu) from its globaltimer stamps: builds the
-DPI0B_GEMM_TRACE variant (variants/libpi0b_gmtrace.so, PI0B_LIB), runs a full-scale engine and
traces the last instance of each listed node (eager launches of that node, back to back).
    python scripts/gemm_trace.py [views] [node ...]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PI0B_LIB"] = os.environ.get("GM_LIB", os.path.join(ROOT, "variants", "libpi0b_gmtrace.so"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402
from paper_2510_26742_b200.inputs import gen_inputs  # noqa: E402

views = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nodes = sys.argv[2:] or ["ve.qkv", "ve.proj", "ve.fc1", "ve.fc2", "llm.qkv", "llm.proj", "llm.down", "llm.ffn"]
STAMPS = ["start", "setup", "pdl(tma)", "full0(mma)", "acc_full", "parked", "cl_sync", "epi_end", "cl_sync2", "exit",
          "acc32#0", "chunk0", "loop_end"]
cfg = default_config(views=views)
eng = E.Engine(cfg, use_cuda_graph=False)
eng.gen_weights(1)
x = gen_inputs(cfg, 1)
eng.run(x["patches"], x["state"], x["noise"])
lib = E.lib()
lib.pi0b_gemm_trace_buffer.argtypes = [ctypes.c_void_p]
plan = eng.describe()
buf = torch.zeros(4096 * 16, dtype=torch.int64, device="cuda")
for node in nodes:
    grid = [l for l in plan if f" {node} " in l][:1]
    ms, n = eng.time_node(node, reps=3)
    buf.zero_()
    lib.pi0b_gemm_trace_buffer(buf.data_ptr())
    eng.time_node(node, reps=1)
    torch.cuda.synchronize()
    lib.pi0b_gemm_trace_buffer(None)
    st = buf.view(4096, 16).cpu().numpy().astype(np.float64)
    st = st[st[:, 0] > 0]
    t0 = st[:, 0].min()
    rel = np.where(st > 0, (st - t0) / 1e3, np.nan)
    print(f"{node}: {grid[0] if grid else ''}\n   {ms * 1e3:.2f} us/launch back to back; traced launch: {len(st)} CTAs, "
          f"span {np.nanmax(rel):.2f} us")
    for i, nm in enumerate(STAMPS):
        v = rel[:, i]
        v = v[np.isfinite(v)]
        if len(v):
            print(f"   {nm:12s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f}")
