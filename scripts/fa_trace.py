"""Timeline of the prefill flash-attention kernel (fattn.cu) from its globaltimer stamps.
Builds the -DPI0B_FA_TRACE variant of libpi0b (variants/libpi0b_fatrace.so, PI0B_LIB) and runs
the VE / LLM attention shapes of a full-scale config through the kernel-level C-ABI.
    python scripts/fa_trace.py [views]"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VAR = os.path.join(ROOT, "variants", "libpi0b_fatrace.so")
os.environ["PI0B_LIB"] = VAR
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_26742_b200 import engine as E  # noqa: E402

views = int(sys.argv[1]) if len(sys.argv) > 1 else 2
T = 256 * views
STAMPS = ["start", "pdl", "setup", "s_full0", "softmax_end", "o_done", "staged", "copies_issued", "combined", "exit",
          "tma_go", "mma_qk0", "bar5", "stored", "split_staged", "cluster_bar"]


def run(name, hd, q_rows, heads, kv_heads, rows0, splits, reps=20):
    dev = "cuda"
    qw, kvw = heads * hd, kv_heads * hd
    ld = qw + 2 * kvw
    X = (torch.randn(max(q_rows, rows0), ld, device=dev) * 0.5).to(torch.bfloat16)
    out = torch.zeros(q_rows, qw, dtype=torch.bfloat16, device=dev)
    d = E.AttnDesc()
    d.head_dim = hd
    d.q, d.ldq, d.q_rows, d.heads, d.kv_heads = X.data_ptr(), ld, q_rows, heads, kv_heads
    d.k0, d.v0, d.ld0, d.rows0 = X[:, qw:].data_ptr(), X[:, qw + kvw:].data_ptr(), ld, rows0
    d.out, d.ldo = out.data_ptr(), qw
    d.kv_splits = splits
    ws = torch.zeros(max(1, E.attention_ws_floats(d)), device=dev)  # key-split workspace
    d.ws = ws.data_ptr()
    grows = heads // kv_heads * q_rows
    ctas = ((grows + 127) // 128) * max(1, splits) * kv_heads
    buf = torch.zeros(ctas * 16, dtype=torch.int64, device=dev)
    lib = E.lib()
    lib.pi0b_fa_trace_buffer.argtypes = [ctypes.c_void_p]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            E.attention(d, s.cuda_stream)
        torch.cuda.synchronize()
        # back-to-back launches (as in the graph, PDL between them): time per launch
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            E.attention(d, s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        per = a.elapsed_time(b) / reps * 1e3
        lib.pi0b_fa_trace_buffer(buf.data_ptr())
        E.attention(d, s.cuda_stream)
        torch.cuda.synchronize()
        lib.pi0b_fa_trace_buffer(None)
    st = buf.view(ctas, 16).cpu().numpy().astype(np.float64)
    t0 = st[:, 0].min()
    rel = np.where(st > 0, (st - t0) / 1e3, np.nan)
    print(f"{name}: grid {ctas} CTAs (splits {splits}), back-to-back {per:.2f} us/launch; "
          f"traced launch span {np.nanmax(rel):.2f} us")
    for i, nm in enumerate(STAMPS):
        v = rel[:, i]
        v = v[np.isfinite(v)]
        if len(v):
            print(f"   {nm:12s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f}")


run(f"ve.attn {views}v", 72, T, 16, 16, T, 1)
run(f"ve.attn {views}v", 72, T, 16, 16, T, 2)
run(f"llm.attn {views}v", 256, T, 8, 1, T, 1)
run(f"llm.attn {views}v", 256, T, 8, 1, T, 2)
run(f"llm.attn {views}v", 256, T, 8, 1, T, 4)
