"""the reference's full-streaming analysis redone with this engine's B200
numbers.  Reads the streaming measurement (scripts/stream_bench.py output), fits the
reference's eta interference model to the measured concurrent runs and runs the reference's own
event simulator (rtvla::simulate + measure_loops, proj/src/streamsim.cpp compiled unmodified into
oracle/_ref/streamsim_driver by `make -C oracle streamsim`) at the paper's 480 Hz target and at
the highest feasible pass rate.  CPU only (no GPU needed):

    python scripts/streamsim_b200.py profiles/r01_stream_2v.json > profiles/r01_streamsim_2v.json
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "streamsim_driver")


def sim(vlm_s, ae_s, rate, pts, policy="most_recent", horizon=2.0):
    args = [DRIVER, repr(vlm_s), repr(ae_s), repr(rate), repr(horizon), policy]
    for p in pts:
        args += [repr(p["t_vlm_ms"] / 1e3), repr(p["t_ae_ms"] / 1e3), repr(p["measured_ms"] / 1e3)]
    return json.loads(subprocess.run(args, check=True, capture_output=True, text=True).stdout)


def main():
    m = json.load(open(sys.argv[1]))
    vlm = m["flow_steps_1"]["prefix_replay_ms"] / 1e3
    ae = m["flow_steps_1"]["action_replay_ms"] / 1e3
    pts = m.get("eta_points", [])
    out = {"source": os.path.relpath(sys.argv[1], ROOT), "vlm_time_s": vlm, "ae_time_s": ae,
           "eta_points": pts, "paper_4090": {"vlm_time_s": 0.016562, "ae_time_s": 0.0011001}}
    out["ref_4090_defaults_480hz"] = sim(0.016562, 0.0011001, 480.0, [])
    out["b200_480hz"] = sim(vlm, ae, 480.0, pts)
    # highest target rate whose closed-form frame makespan still fits the 30 Hz period
    lo, hi = 480.0, 30.0 * 400
    while hi - lo > 30.0:
        mid = 30.0 * round(((lo + hi) / 2) / 30.0)
        r = sim(vlm, ae, mid, pts, horizon=0.5)
        if r["loops"]["feasible"]:
            lo = mid
        else:
            hi = mid
    out["b200_max_feasible_rate_hz"] = lo
    out["b200_max_rate"] = sim(vlm, ae, lo, pts)
    conc = m.get("concurrent_30hz_prefix_1step")
    if conc:
        out["measured_concurrent_1step_passes_per_s"] = conc["flow_steps_per_s"]
        out["measured_concurrent_prefix_frames_per_s"] = conc["prefix_frames_per_s"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
