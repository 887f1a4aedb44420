"""The performance switches are schedule choices, not numerics: every setting must
produce the same actions at full scale, within the run-to-run spread of the fp32 `red.add`
residual updates, and stay within the golden tolerance.

Several switches are read once per process (static in the launchers), so each setting runs in
its own subprocess: 2 views, seed 1, actions written to an .npy file and compared here."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden", "full_2v.json")
SPREAD_MAX = 0.01      # as tests/test_gpu_stress.py: run-to-run spread of the default engine
GOLD_MAX_ABS = 0.025

_SCRIPT = """
import sys, numpy as np
sys.path.insert(0, {root!r})
from paper_2510_26742_b200 import engine as E
from paper_2510_26742_b200.config import default_config
from paper_2510_26742_b200.inputs import gen_inputs
cfg = default_config(views=2)
eng = E.Engine(cfg)
eng.gen_weights(1)
x = gen_inputs(cfg, 1)
np.save({out!r}, eng.run(x["patches"], x["state"], x["noise"]))
"""

SETTINGS = {
    "default": {},
    "gemm_no_warm_no_stage": {"PI0B_GEMM_WARM": "0", "PI0B_GEMM_STAGE_BF16": "0"},
    "fa72_two_threads_per_row": {"PI0B_FA72_NQ": "2"},
    "fa72_64_key_tiles": {"PI0B_FA72_KEYS": "64"},
    "llm_attn_unsplit_ve_proj_split": {"PI0B_ATTN_SPLITS_LLM_ATTN": "1", "PI0B_SPLIT_VE_PROJ": "2"},
    "no_pdl": {"PI0B_PDL": "0"},
}


def _actions(tmp_path, name, env):
    out = str(tmp_path / f"{name}.npy")
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, out=out)], env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(out)


def test_switch_settings_agree(tmp_path):
    gold = np.array(json.load(open(GOLDEN))["actions"]).reshape(63, 32)
    ys = {name: _actions(tmp_path, name, env) for name, env in SETTINGS.items()}
    base = ys["default"]
    for name, y in ys.items():
        d, g = float(np.abs(y - base).max()), float(np.abs(y - gold).max())
        print(f"{name:32s} max |y - default| {d:.3e}   max |y - golden| {g:.3e}")
        assert np.isfinite(y).all()
        assert d < SPREAD_MAX, name
        assert g < GOLD_MAX_ABS, name
