"""In-graph timeline of one full inference (CUDA-graph replay) from the -DPI0B_KTRACE variant
(variants/libpi0b_ktrace.so; paper_2510_26742_b200/csrc/ktrace.cuh): for every kernel launch,
when its CTAs observed the previous kernel complete (griddepcontrol.wait), when its last CTA
finished, and the gap between the previous kernel's last CTA and this kernel's release.
    python scripts/graph_timeline.py [views]"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PI0B_LIB"] = os.environ.get("KT_LIB", os.path.join(ROOT, "variants", "libpi0b_ktrace.so"))
import ctypes  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402
from paper_2510_26742_b200.inputs import gen_inputs  # noqa: E402

views = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = default_config(views=views)
eng = E.Engine(cfg)
eng.gen_weights(1)
x = gen_inputs(cfg, 1)
eng.run(x["patches"], x["state"], x["noise"])
lib = E.lib()
lib.pi0b_ktrace_buffer.argtypes = [ctypes.c_void_p]
buf = torch.zeros(8 + 4 * 262144 + 8192, dtype=torch.int64, device="cuda")
names = {}
for line in eng.describe():  # "<i> <part> gemm <node> <inst> <grid> M= N= K= ..."
    f = line.split()
    if len(f) > 8 and f[2] == "gemm":
        kv = dict(t.split("=") for t in f if "=" in t)
        names[(int(kv["N"]), int(kv["K"]))] = f[3]

for rep in range(3):
    buf.zero_()
    eng.sync()
    assert lib.pi0b_ktrace_buffer(buf.data_ptr()) == 0
    eng.replay(0)
    eng.sync()
    lib.pi0b_ktrace_buffer(None)
rec = buf.cpu().numpy()
n = int(rec[0])
r = rec[8:8 + 4 * n].reshape(n, 4).astype(np.uint64)
tag, t0, tdep, t1 = r[:, 0], r[:, 1].astype(np.int64), r[:, 2].astype(np.int64), r[:, 3].astype(np.int64)
base = t0.min()


def node_of(tg):
    kind = int(tg >> np.uint64(62))
    if kind == 1:
        N = int((tg >> np.uint64(40)) & np.uint64(0xffff))
        K = int((tg >> np.uint64(24)) & np.uint64(0xffff))
        return names.get((N, K), f"gemm N={N} K={K}")
    if kind == 2:
        return "ve.attn" if int((tg >> np.uint64(40)) & np.uint64(0xfff)) == 72 else "llm.attn"
    return "ae.mega"


# launches: CTAs of one tag whose dependency release (or start, without one) lies within 3 us
launches = []
for tg in np.unique(tag):
    idx = np.where(tag == tg)[0]
    key = np.where(tdep[idx] > 0, tdep[idx], t0[idx])
    idx = idx[np.argsort(key)]
    key = np.sort(key)
    cut = np.where(np.diff(key) > 3000)[0] + 1
    for grp in np.split(idx, cut):
        dep = tdep[grp][tdep[grp] > 0]
        launches.append(dict(node=node_of(tg), ctas=len(grp), start=t0[grp].min() - base,
                             dep=(dep.min() - base) if len(dep) else None, dep_max=(dep.max() - base) if len(dep) else None,
                             end=t1[grp].max() - base))
launches.sort(key=lambda l: l["dep"] if l["dep"] is not None else l["start"])
print(f"{n} CTA records, {len(launches)} launches, replay span {(t1.max() - base) / 1e3:.1f} us")
per = collections.defaultdict(list)
prev_end = None
gap_total = 0.0
rows = []
for l in launches:
    rel = l["dep"] if l["dep"] is not None else l["start"]
    gap = (rel - prev_end) / 1e3 if prev_end is not None else 0.0
    work = (l["end"] - rel) / 1e3
    per[l["node"]].append((gap, work, (l["dep_max"] - l["dep"]) / 1e3 if l["dep"] is not None else 0.0))
    gap_total += max(gap, 0.0)
    rows.append((l["node"], l["ctas"], rel / 1e3, l["end"] / 1e3, gap, work))
    prev_end = l["end"]
print(f"sum of gaps (previous kernel's last CTA done -> this kernel's CTAs released): {gap_total:.1f} us")
print(f"{'node':12s} {'n':>4s} {'gap us':>8s} {'work us':>8s} {'release spread':>15s}")
for k, v in sorted(per.items(), key=lambda kv: -sum(w for _, w, _ in kv[1])):
    a = np.array(v)
    print(f"{k:12s} {len(v):4d} {a[:, 0].mean():8.2f} {a[:, 1].mean():8.2f} {a[:, 2].mean():15.2f}")
print("\nfirst 24 launches (us from the first CTA start): node ctas released end gap work")
for row in rows[:24]:
    print(f"  {row[0]:12s} {row[1]:4d} {row[2]:9.2f} {row[3]:9.2f} {row[4]:7.2f} {row[5]:8.2f}")
print("...\nlast 6 launches:")
for row in rows[-6:]:
    print(f"  {row[0]:12s} {row[1]:4d} {row[2]:9.2f} {row[3]:9.2f} {row[4]:7.2f} {row[5]:8.2f}")
