"""the full-streaming runtime (include/pi0b.h pi0b_stream_run) runs camera frames
(prefix into double-buffered KV) and action-expert ticks concurrently on one GPU and reports the
reference's loop metrics (rtvla::measure_loops semantics) on what actually ran."""
import pytest

from paper_2510_26742_b200 import engine as E
from paper_2510_26742_b200.config import mid_config

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("policy", ["most_recent", "frame_sticky"])
def test_stream_runtime_mid(policy):
    cfg = mid_config(views=2).replace(flow_steps=1)
    r = E.stream_run(cfg, 1.5, ae_rate=480.0, kv_policy=policy)
    print(r)
    assert abs(r["vlm_per_s"] - 30.0) < 4.0            # every camera frame was processed
    assert r["ae_per_s"] > 400.0                         # mid config: ticks keep up with 480 Hz
    assert r["quick_count"] > 100 and 0.0 < r["quick_mean_ms"] < 10.0
    assert r["slow_count"] >= 20 and r["slow_mean_ms"] > 2 * 1000.0 / 30.0  # includes 2 frames of camera latency
    assert r["committed_slots"] > 400
