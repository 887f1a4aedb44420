"""CPU tests of the parity checker itself (no GPU).

1. The compiled reference reproduces its own known-answer tests (proj/tests/test_tensor.cpp)
   and the golden spot values recorded from full reference runs.
2. The fp64 restatement (oracle/pi0_oracle.cpp) is BITWISE equal to rtvla::evaluate on the
   reference's tiny twin and on the mid configs (1v, 2v, 3v + prompt), including hidden
   states of every node kind.
3. The committed golden fixtures equal what the reference computes now.
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_26742_b200.config import default_config, mid_config, tiny_config

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def _splitmix_restated(state):
    state = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    return state, z ^ (z >> 31)


# ------------------------------------------------------------------ reference KATs

@needs_ref
@pytest.mark.parametrize("seed", [0, 1, 42, 0xDEADBEEF, 2**64 - 1])
def test_rng_matches_published_splitmix64(seed):
    """proj/tests/test_tensor.cpp:37-43."""
    import ctypes
    out = (ctypes.c_uint64 * 64)()
    O.ref_lib().ref_rng_stream(seed, 64, out)
    st = seed
    for i in range(64):
        st, v = _splitmix_restated(st)
        assert out[i] == v


@needs_ref
def test_numerics_known_answers():
    L = O.ref_lib()
    # gelu / silu closed forms (test_tensor.cpp:150-169)
    assert L.ref_gelu(0.0) == 0.0 and L.ref_silu(0.0) == 0.0
    assert abs(L.ref_gelu(1.0) - 0.8411919906082768) < 1e-15
    assert abs(L.ref_silu(1.0) - 1.0 / (1.0 + np.exp(-1.0))) < 1e-15
    # softmax [0, ln3] -> [0.25, 0.75] and shift invariance (test_tensor.cpp:125-148)
    x = np.array([[0.0, np.log(3.0)], [5.0, 5.0 + np.log(3.0)]])
    y = np.zeros_like(x)
    L.ref_softmax_rows(O._ptr(x), 2, 2, O._ptr(y))
    assert np.allclose(y, [[0.25, 0.75], [0.25, 0.75]], atol=1e-15)
    # rms hand value (test_tensor.cpp:104-123): [3, 4] -> 1/sqrt(12.5 + eps)
    x = np.array([[3.0, 4.0]])
    s = np.zeros(1)
    L.ref_rms_scales(O._ptr(x), 1, 2, 1e-6, O._ptr(s))
    assert abs(s[0] - 1.0 / np.sqrt(12.5 + 1e-6)) < 1e-14
    # rope: identity at p=0, first pair rotates by angle p (test_tensor.cpp:171-203)
    x = np.random.default_rng(0).uniform(-1, 1, (3, 8))
    y = np.zeros_like(x)
    L.ref_rope(O._ptr(x), 3, 8, 8, 0, O._ptr(y))
    assert np.array_equal(y[0], x[0])
    c, s_ = np.cos(1.0), np.sin(1.0)
    assert abs(y[1, 0] - (x[1, 0] * c - x[1, 4] * s_)) < 1e-15
    # matmul vs naive triple loop (test_tensor.cpp:83-92)
    a = np.random.default_rng(1).uniform(-1, 1, (5, 7))
    b = np.random.default_rng(2).uniform(-1, 1, (7, 3))
    out = np.zeros((5, 3))
    L.ref_matmul(O._ptr(a), 5, 7, O._ptr(b), 3, O._ptr(out))
    assert np.abs(out - a @ b).max() < 1e-12
    # max_rel_deviation (test_tensor.cpp:243-251)
    p, q = np.array([1.0, 2.0]), np.array([1.0, 4.0])
    assert L.ref_max_rel_deviation(O._ptr(p), O._ptr(q), 2) == 2.0 / (4.0 + 1e-12)


@needs_ref
def test_reference_tiny_golden_spot_values():
    """Spot values printed from the reference for tiny_config, seed 1."""
    y = O.ref_evaluate(tiny_config())
    assert y.shape == (63, 2)
    assert y.ravel()[0] == 0.5210705041517647
    assert y.ravel()[-1] == -0.16544959527708591


@needs_ref
def test_reference_full_shapes():
    """The builder's full-scale shape table (proj/src/builder.cpp:170-193)."""
    rows = {r[0]: r for r in O.ref_graph_listing(default_config())}
    assert rows["llm.ffn"][3:] == (512, 2048, 32768)
    assert rows["llm.qkv"][2:] == (18, 512, 2048, 2560)
    assert rows["ae.qkv"][2:] == (180, 64, 1024, 2560)
    assert rows["ve.fc1"][3:] == (512, 1152, 4304)
    assert O.ref_lib().ref_count_gemm_instances(default_config()) == 1378


# ------------------------------------------------------------------ restatement == reference

@needs_ref
def test_restatement_inputs_bitwise():
    for cfg in (tiny_config(), mid_config(3, 32)):
        a = O.gen_inputs(cfg, 1)
        b = O.gen_inputs(cfg, 1, use_reference=True)
        for k in a:
            assert np.array_equal(a[k], b[k]), k


@needs_ref
@pytest.mark.parametrize("node,k,m,bias", [("ve.qkv", 288, 864, True), ("llm.ffn", 512, 2048, False),
                                           ("ae.head", 256, 32, True)])
def test_restatement_weights_bitwise(node, k, m, bias):
    cfg = mid_config()
    inst = 0 if node == "ae.head" else 1       # Shared binding has one instance
    w_ref, b_ref, _ = O.ref_node_weight(cfg, node, inst, k, m, bias=bias)
    w, b = O.port_weight(node, inst, k, m, bias=bias)
    assert np.array_equal(w, w_ref)
    if bias:
        assert np.array_equal(b, b_ref)


@needs_ref
@pytest.mark.parametrize("cfg", [tiny_config(), mid_config(1), mid_config(2), mid_config(3, 32)],
                         ids=["tiny", "mid1v", "mid2v", "mid3v32p"])
def test_restatement_actions_bitwise(cfg):
    x = O.gen_inputs(cfg, 1)
    ref = O.ref_evaluate(cfg)
    got, _ = O.port_forward(cfg, x)
    assert np.array_equal(got, ref)


@needs_ref
@pytest.mark.parametrize("node,inst", [("ve.fc2", 1), ("ve.attn", 0), ("llm.qkv", 2), ("llm.ffn", 1),
                                       ("llm.down", 1), ("ae.qkv", 3), ("ae.attn", 2), ("ae.down", 5),
                                       ("ae.suffix", 1), ("ae.head", 1), ("ae.action_proj", 2)])
def test_restatement_hidden_states_bitwise(node, inst):
    cfg = mid_config(2)
    x = O.gen_inputs(cfg, 1)
    ref = O.ref_node(cfg, node, inst)
    _, rec = O.port_forward(cfg, x, record=[(node, inst, ref.shape)])
    assert np.array_equal(rec[(node, inst)], ref)


# ------------------------------------------------------------------ fixtures

@pytest.mark.parametrize("name", ["tiny_1v", "mid_1v", "mid_2v", "mid_3v32p"])
def test_golden_fixtures_reproduce(name):
    """Committed fixtures (made from the reference) == the restatement now (runs anywhere)."""
    doc = json.load(open(os.path.join(GOLDEN, name + ".json")))
    from paper_2510_26742_b200.config import ModelConfig
    cfg = ModelConfig(**doc["config"])
    x = O.gen_inputs(cfg, doc["input_seed"])
    got, _ = O.port_forward(cfg, x, wseed=doc["weight_seed"])
    assert np.array_equal(got.ravel(), np.array(doc["actions"]))


@pytest.mark.parametrize("views", [1, 2])
def test_full_scale_fixture_matches_reference_spots(views):
    """The full-scale fixtures agree with the reference's own full runs."""
    path = os.path.join(GOLDEN, f"full_{views}v.json")
    if not os.path.exists(path):
        pytest.skip("full-scale fixture not generated")
    y = np.array(json.load(open(path))["actions"])
    spots = {1: (1.0286562565432205, 1.2088658830676564, 0.34389548371564982, 175.91048182764209),
             2: (0.99116682917401266, 1.2019504034525859, 0.014307136309375735, 206.67524788946236)}[views]
    assert (y[0], y[1], y[-1]) == spots[:3]
    assert abs(y.sum() - spots[3]) < 1e-10
