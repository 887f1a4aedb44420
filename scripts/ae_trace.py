"""Per-phase timeline of the action-expert megakernel from its globaltimer trace
(PI0B_AE_TRACE=1): where the time of one AE launch goes."""
import collections
import ctypes
import os
import sys

os.environ["PI0B_AE_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
# the per-task timestamps are compiled only into the trace variant of the library
_VAR = os.path.join(ROOT, "variants", "libpi0b_aetrace.so")
if not os.path.exists(_VAR):
    from paper_2510_26742_b200.build import build  # noqa: E402
    build(lib=_VAR, defines=["-DPI0B_AE_TRACE_CODE=1"])
os.environ.setdefault("PI0B_LIB", _VAR)
import numpy as np  # noqa: E402

from paper_2510_26742_b200 import engine as E  # noqa: E402
from paper_2510_26742_b200.config import default_config  # noqa: E402
from paper_2510_26742_b200.inputs import gen_inputs  # noqa: E402

views = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = default_config(views=views)
eng = E.Engine(cfg, use_cuda_graph=False)
eng.gen_weights(1)
x = gen_inputs(cfg, 1)
for _ in range(3):
    eng.run(x["patches"], x["state"], x["noise"])
lib = E.lib()
lib.pi0b_engine_ae_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
cap = 148 * 4096
dt = np.dtype([("kind", "u1"), ("xsrc", "u1"), ("epi", "u1"), ("rowoff", "u1"), ("wmap", "<u2"), ("xmap", "<u2"),
               ("pad0", "<u2"), ("tile", "<u2"), ("kb0", "<u2"), ("nkb", "<u2"), ("wait_bar", "<u2"),
               ("wait_cnt", "<u2"), ("sig_bar", "<u2"), ("aux", "<u2"), ("step", "<u2"), ("layer", "<u2"),
               ("phase", "<u2"), ("pad1", "<u2")])
tasks = np.zeros(cap, dtype=dt)
st = np.zeros((cap + 148 * 8, 16), dtype=np.uint64)
ctas, stride = ctypes.c_int(), ctypes.c_int()
rc = lib.pi0b_engine_ae_trace(eng._h, tasks.ctypes.data, st.ctypes.data, cap, ctypes.byref(ctas), ctypes.byref(stride))
assert rc == 0, E.lib().pi0b_last_error()
n = ctas.value * stride.value
dbg = st[n:n + ctas.value * 8].reshape(ctas.value, 128).astype(np.int64)
tasks, st = tasks[:n], st[:n].astype(np.int64)
ok = (tasks["kind"] != 0) & (st[:, 3] > 0)
t0 = st[ok, 0].min()
st = np.where(st > 0, st - t0, -1)
names = {(1, 5): "INIT", (1, 3): "AP", (1, 0): "RED", (1, 1): "QKV", (1, 2): "FFN", (1, 4): "HEAD"}
ph = collections.defaultdict(list)
for i in np.nonzero(ok)[0]:
    ph[int(tasks["phase"][i])].append(i)
kind_of = {}
rows = []
for p in sorted(ph):
    idx = ph[p]
    tk = tasks[idx[0]]
    if tk["kind"] == 2:
        nm = "ATTN"
    elif tk["kind"] == 1 and tk["epi"] == 0:
        nm = {0: "AO/DOWN", 2: "PROJ"}.get(int(tk["xsrc"]), "RED")
        if tk["xsrc"] == 0 and tk["rowoff"] == 1:
            nm = "AO"
    else:
        nm = names.get((int(tk["kind"]), int(tk["epi"])), f"K{tk['kind']}")
    s = st[idx]
    rows.append((p, nm, len(idx), s[:, 0].min(), s[:, 1].max(), s[:, 3].max(),
                 np.mean(s[:, 1] - s[:, 0]), np.mean(s[:, 2] - s[:, 1]), np.mean(s[:, 3] - s[:, 2])))
tot = max(r[5] for r in rows)
print(f"AE megakernel: {len(rows)} phases, {ok.sum()} tasks, span {tot / 1e3:.1f} us")
agg = collections.defaultdict(lambda: np.zeros(6))
prev_end = 0
for r in rows:
    p, nm, cnt, smin, rmax, emax, wait, stage, epi = r
    a = agg[nm]
    a += [1, emax - prev_end, cnt, wait, stage, epi]
    prev_end = emax
print(f"{'phase':8s} {'n':>4s} {'tasks':>6s} {'us/phase(end-to-end)':>21s} {'wait':>8s} {'stage':>8s} {'mma+epi':>8s}")
for nm, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{nm:8s} {int(a[0]):4d} {a[2] / a[0]:6.0f} {a[1] / a[0] / 1e3:21.2f} {a[3] / a[0] / 1e3:8.2f} "
          f"{a[4] / a[0] / 1e3:8.2f} {a[5] / a[0] / 1e3:8.2f}")
print("first 16 phases:")
for r in rows[:16]:
    print("  %3d %-8s n=%3d start %8.2f ready(max) %8.2f end(max) %8.2f  wait %.2f stage %.2f epi %.2f" %
          (r[0], r[1], r[2], r[3] / 1e3, r[4] / 1e3, r[5] / 1e3, r[6] / 1e3, r[7] / 1e3, r[8] / 1e3))

# detail of one mid-inference layer: per phase, percentiles of each stamp relative to the
# completion of the previous phase
cta_of = np.arange(n) // stride.value
mid = [r for r in rows if r[0] >= len(rows) // 2][:6]
prev_end = 0
for r in rows:
    if r[0] == mid[0][0] - 1:
        prev_end = r[5]
print("\nlayer detail (us relative to the previous phase's last publish):")
for r in mid:
    idx = np.array(ph[r[0]])
    s8 = st[idx].astype(np.float64)
    rel = lambda c: (s8[:, c] - prev_end) / 1e3
    def q(v):
        v = v[np.isfinite(v)]
        return "%7.2f/%7.2f/%7.2f" % (np.min(v), np.median(v), np.max(v)) if len(v) else "      -"
    print(f"  {r[1]:8s} n={r[2]:3d} start {q(rel(0))} ready {q(rel(1))} staged {q(rel(2))} pub {q(rel(3))}")
    if tasks["kind"][idx[0]] == 1:
        print(f"  {'':8s}       w_first_issue {q(rel(4))} w_last_issue {q(rel(5))} w_last_full {q(rel(6))} acc {q(rel(7))}")
        print(f"  {'':8s}       acc_seen {q(rel(8))} epi_done {q(rel(9))}")
    elif tasks["kind"][idx[0]] == 2:
        print(f"  {'':8s}       qk_landed {q(rel(6))} s_full {q(rel(10))} p_full {q(rel(11))} pv_ready {q(rel(7))} o_done {q(rel(12))} stored {q(rel(13))}")
    prev_end = r[5]

# pair (2-CTA split-K) tasks of the mid layer: owner vs helper stamps
print("\npair tasks of the mid layer (us relative to the previous phase's last publish):")
prev_end = 0
for r in rows:
    if r[0] == mid[0][0] - 1:
        prev_end = r[5]
for r in mid:
    idx = np.array(ph[r[0]])
    pr = tasks["pad1"][idx]
    if (pr > 0).any():
        for role in sorted(set(int(v) for v in pr if v > 0)):
            nm = {1: "owner", 2: "helper", 3: "ffn-a", 4: "ffn-b", 5: "qkv-a", 6: "qkv-b"}.get(role, str(role))
            s8 = st[idx[pr == role]].astype(np.float64)
            rel = lambda c: np.where(s8[:, c] > 0, (s8[:, c] - prev_end) / 1e3, np.nan) if len(s8) else np.zeros(0)

            def q(v):
                v = v[np.isfinite(v)]
                return "%6.2f/%6.2f/%6.2f" % (np.min(v), np.median(v), np.max(v)) if len(v) else "     -"
            print(f"  {r[1]:6s} {nm:6s} ready {q(rel(1))} staged {q(rel(2))} acc {q(rel(7))} acc_seen {q(rel(8))} "
                  f"epi_done {q(rel(9))} pub {q(rel(3))}")
            if role == 2:
                print(f"  {'':13s} ready_ok {q(rel(10))} stores {q(rel(11))} bar {q(rel(12))} fence {q(rel(13))}")
    prev_end = r[5]

if os.environ.get("AE_TRACE_RAW"):
    print("\nraw stamps of the first phases (us from kernel start): start ready staged pub | wfirst wlast wfull acc | accseen epidone | sfull pfull odone stored | drainer_done barrier")
    for r in rows[:5]:
        for i in ph[r[0]][:4]:
            v = st[i] / 1e3
            print(f"  ph{r[0]} {r[1]:6s} cta {i // stride.value:3d} " + " ".join(f"{x:7.2f}" if x >= 0 else "      -" for x in v[:16]))

if os.environ.get("AE_TRACE_KB"):
    rows_d = [c for c in range(ctas.value) if dbg[c, 0] > 0]
    print("\nper-k-block stamps of an ae.qkv task (step 1, layer 5; us from its first stamp), CTAs", rows_d[:3])
    for c in rows_d[:3]:
        d = dbg[c].astype(np.float64)
        base = d[0]
        for k in range(16):
            w = (d[k * 4:k * 4 + 4] - base) / 1e3
            m = (d[64 + k * 4:64 + k * 4 + 4] - base) / 1e3
            print(f"  kb{k:2d} worker: start {w[0]:6.2f} f_landed {w[1]:6.2f} x_empty {w[2]:6.2f} x_full_arrive {w[3]:6.2f}   "
                  f"mma: start {m[0]:6.2f} w_full {m[1]:6.2f} x_full {m[2]:6.2f} issued {m[3]:6.2f}")

if os.environ.get("AE_TRACE_LATE"):
    print("\nlatest-ready tasks of a mid PROJ phase and their CTA's previous task:")
    pr = [r for r in rows if r[1] == "PROJ"]
    r = pr[len(pr) // 2]
    idx = sorted(ph[r[0]], key=lambda i: -st[i][1])[:6]
    for i in idx:
        c, k = divmod(i, stride.value)
        prev = i - 1 if k > 0 else None
        pt = tasks[prev] if prev is not None else None
        desc = f"prev phase {pt['phase']} kind {pt['kind']} epi {pt['epi']} start {st[prev][0]/1e3:.2f} ready {st[prev][1]/1e3:.2f} pub {st[prev][3]/1e3:.2f}" if prev is not None else "first"
        print(f"  cta {c:3d} task {k:3d} ready {st[i][1]/1e3:8.2f} pub {st[i][3]/1e3:8.2f} | {desc}")
