"""Streaming-mode measurement: the prefix is run once per camera frame
and the action expert once per control tick on the cached prefix KV.

(i)  p50 of the prefix replay and of the action-expert replay (device time, CUDA events) for a
     10-step and a 1-step flow, and of the public `run_action` call (host fp64 state/noise in,
     actions out: H2D + replay + D2H) with fresh inputs every tick;
(ii) the sustained action tick rate on one GPU while a second engine re-runs the prefix at 30 Hz
     on its own stream (two engines = two KV caches, the double-buffered layout of SURVEY 8(f)
     f2), plus the tick-latency percentiles under that interference, for 10-step and 1-step ticks;
(iii) concurrent prefix + k one-step AE passes makespans, the calibration points of the
     reference's eta interference model (scripts/streamsim_b200.py feeds them, with (i), into the
     reference's own simulate()/measure_loops()).
Writes one JSON object to stdout.   python scripts/stream_bench.py [views] [seconds]
"""
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
seconds = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0


def replay_p50(eng, part, n=30):
    st = torch.cuda.Stream()
    for _ in range(3):
        eng.replay(part, st.cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        a.record(st)
        eng.replay(part, st.cuda_stream)
        b.record(st)
    st.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    return ms[n // 2]


out = {"views": views, "data": "synthetic (gen_inputs seed 1; fresh noise/state per tick from seeds 2..)"}
for fs in (10, 1):
    cfg = default_config(views=views).replace(flow_steps=fs)
    eng = E.Engine(cfg)
    eng.gen_weights(1)
    x = gen_inputs(cfg, 1)
    eng.run(x["patches"], x["state"], x["noise"])
    row = {"prefix_replay_ms": replay_p50(eng, 1), "action_replay_ms": replay_p50(eng, 2)}
    eng.run_prefix(x["patches"])
    rng = np.random.default_rng(7)
    lat = []
    for k in range(40):
        state = rng.uniform(-1, 1, size=(1, cfg.ae_state_dim))
        noise = rng.uniform(-1, 1, size=(cfg.chunk_len, cfg.ae_action_dim))
        t0 = time.perf_counter()
        eng.run_action(state, noise)
        lat.append((time.perf_counter() - t0) * 1e3)
    row["run_action_e2e_ms"] = float(np.median(lat[5:]))
    out[f"flow_steps_{fs}"] = row
    del eng

# (ii) action ticks with a concurrent 30 Hz prefix on a second engine / stream, for 10-step ticks
# (a full action chunk per tick) and 1-step ticks (one "AE pass" of the paper's 480 Hz stream)
cfg = default_config(views=views)
eb = E.Engine(cfg)
eb.gen_weights(1)
x = gen_inputs(cfg, 1)
eb.run(x["patches"], x["state"], x["noise"])
sa, sb = torch.cuda.Stream(priority=-1), torch.cuda.Stream()
engines = {}
for fs in (10, 1):
    c = cfg.replace(flow_steps=fs)
    ea = E.Engine(c)
    ea.gen_weights(1)
    xa = gen_inputs(c, 1)
    ea.run(xa["patches"], xa["state"], xa["noise"])
    engines[fs] = ea
    ticks, frames, fev = [], 0, []
    t_start = time.perf_counter()
    t_end = t_start + seconds
    next_frame = time.perf_counter()
    while time.perf_counter() < t_end:
        now = time.perf_counter()
        if now >= next_frame:
            fa, fb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            fa.record(sb)
            eb.replay(1, sb.cuda_stream)
            fb.record(sb)
            fev.append((fa, fb))
            frames += 1
            next_frame += 1.0 / 30.0
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(sa)
        ea.replay(2, sa.cuda_stream)
        b.record(sa)
        ticks.append((a, b))
        b.synchronize()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_start  # until both streams drained
    ms = sorted(a.elapsed_time(b) for a, b in ticks)
    fms = sorted(a.elapsed_time(b) for a, b in fev)
    span = ticks[0][0].elapsed_time(max((fev[-1][1], ticks[-1][1]), key=lambda e: ticks[0][0].elapsed_time(e))) / 1e3
    out["concurrent_30hz_prefix" + ("" if fs == 10 else "_1step")] = {
        "flow_steps_per_tick": fs,
        "seconds": seconds,
        "wall_s_until_drained": wall,
        "gpu_span_s": span,
        "action_ticks": len(ticks),
        "prefix_frames": frames,
        "ticks_per_s": len(ticks) / span,
        "prefix_frames_per_s": frames / span,
        "flow_steps_per_s": fs * len(ticks) / span,
        "prefix_frame_p50_ms": fms[len(fms) // 2],
        "tick_p50_ms": ms[len(ms) // 2],
        "tick_p99_ms": ms[min(len(ms) - 1, int(0.99 * len(ms)))],
    }

# (iii) interference calibration for the reference's eta model (rtvla::calibrate_eta,
# proj/include/rtvla/streamsim.hpp:35-45; its built-in points are the 4090's VLM + 10 / 16 AE
# passes): one prefix on stream B concurrently with k one-step AE passes on stream A.
ea = engines[1]


def makespan(k, n=15):
    res = []
    for _ in range(n):
        t0 = torch.cuda.Event(enable_timing=True)
        ea_end, eb_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(sa)
        sb.wait_event(t0)
        eb.replay(1, sb.cuda_stream)
        eb_end.record(sb)
        for _ in range(k):
            ea.replay(2, sa.cuda_stream)
        ea_end.record(sa)
        torch.cuda.synchronize()
        res.append(max(t0.elapsed_time(ea_end), t0.elapsed_time(eb_end)))
    return float(np.median(res))


def alone(k, n=15):
    res = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(sa)
        for _ in range(k):
            ea.replay(2, sa.cuda_stream)
        b.record(sa)
        torch.cuda.synchronize()
        res.append(a.elapsed_time(b))
    return float(np.median(res))


t_vlm = replay_p50(eb, 1)
pts = []
for k in (10, 16):
    pts.append({"ae_passes": k, "t_vlm_ms": t_vlm, "t_ae_ms": alone(k), "measured_ms": makespan(k)})
out["eta_points"] = pts
print(json.dumps(out))
