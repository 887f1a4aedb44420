"""The reference's own stream simulator (proj/src/streamsim.cpp, compiled unmodified into
oracle/_ref/streamsim_driver) as used by scripts/streamsim_b200.py for SURVEY.md 8(d)(iii):
the driver reproduces the reference's 4090 defaults and reports a feasible schedule for B200
stream times.  CPU only; skipped where the reference was not built."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DRIVER = os.path.join(ROOT, "oracle", "_ref", "streamsim_driver")

pytestmark = pytest.mark.skipif(not os.path.exists(DRIVER), reason="reference streamsim not built here")


def _run(*args):
    out = subprocess.run([DRIVER, *map(str, args)], check=True, capture_output=True, text=True).stdout
    return json.loads(out)


def test_reference_defaults_480hz():
    # the reference's built-in 4090 calibration (streamsim.hpp:47-51): 16 AE passes per 30 Hz
    # frame fit the 33.3 ms period (the paper's full-streaming claim)
    r = _run(0.016562, 0.0011001, 480.0, 1.0, "most_recent")
    assert r["passes_per_frame"] == 16
    assert r["loops"]["feasible"]
    assert 0.030 < r["closed_form_frame_makespan_s"] < 1.0 / 30.0
    assert abs(r["loops"]["ae_per_s"] - 480) < 10


def test_eta_fit_and_b200_schedule():
    # eta fitted from concurrent-run points: measured makespan = max + (1 - eta) * min
    t_a, t_b, eta = 0.0038, 0.0069, 0.25
    meas = max(t_a, t_b) + (1 - eta) * min(t_a, t_b)
    r = _run(0.0038, 0.00072, 480.0, 1.0, "frame_sticky", t_a, t_b, meas)
    assert abs(r["eta"] - eta) < 1e-6 and r["eta_points"] == 1
    assert r["loops"]["feasible"] and r["loops"]["utilization_margin"] > 0.4
    assert r["loops"]["quick_loop"]["present"]
