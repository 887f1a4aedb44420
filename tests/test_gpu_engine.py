"""End-to-end parity of the B200 engine against the fp64 oracle.

* device `gen_weights` is bit-exact (bf16 RNE of the reference's fp64 draws);
* the full forward (VE -> LLM -> AE, all flow steps) on the mid config matches the oracle:
  actions within the stated bf16 tolerance, per-layer hidden-state cosine >= 0.999
  (north star), through both weight paths (device generation and host WeightStore upload);
* the streaming split (run_prefix + run_action) equals run();
* full-scale 1-view and 2-view actions match the reference's published golden values.
"""
import json
import os

import numpy as np
import pytest

from _util import bf16_bits_from_f64, cosine, rel_err, sketch_checkpoints, sketch_take
from oracle import oracle as O
from paper_2510_26742_b200 import engine as E
from paper_2510_26742_b200.config import default_config, mid_config

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

# bf16 tolerance on the [63, 32] action chunk (north star: "a stated bf16 tolerance").
ACT_MAX_ABS = 0.05      # of actions whose rms is ~1
ACT_REL = 0.25          # max |d| / max(|ref|, 0.1*rms(ref))
LAYER_COS = 0.999
RUN_TO_RUN = 0.02      # fp32 atomic (split-K / row-stat) ordering differs between runs
# full scale (r02 measurements, profiles/r02_parity_*.json: max-abs 0.011-0.013, rel 0.13-0.16,
# rms error 0.0047-0.0048 on actions of rms 0.80; per-layer cosine >= 0.99995): ~2x margins
FULL_MAX_ABS = 0.025
FULL_REL = 0.2
FULL_RMS_ERR = 0.01


def test_device_weight_stream_bitexact():
    import torch
    k, m = 1152, 3456
    seed = E.seed_hash(1, "ve.qkv", 3, 1)
    assert seed == O.ref_lib().ref_seed_hash(1, b"ve.qkv", 3, 1)
    lim = 1.0 / np.sqrt(k)
    d64 = torch.zeros(k * m, dtype=torch.float64, device="cuda")
    E.random_f64(d64.data_ptr(), k * m, seed, -lim, lim)
    w_ref, _ = O.port_weight("ve.qkv", 3, k, m)
    assert np.array_equal(d64.cpu().numpy().reshape(k, m), w_ref)
    packed = torch.zeros(m, k, dtype=torch.int16, device="cuda")
    E.random_packed_bf16(packed.data_ptr(), k, k, m, E.PERM_NONE, seed, -lim, lim)
    got = packed.cpu().numpy().view(np.uint16)
    assert np.array_equal(got, bf16_bits_from_f64(w_ref).T)


def _record_list(cfg):
    T, L, S = cfg.image_tokens, cfg.prefix_tokens, cfg.suffix_tokens
    rec = [("ve.embed", 0, (T, cfg.ve_width))]
    rec += [("ve.fc2", i, (T, cfg.ve_width)) for i in range(cfg.ve_layers)]
    rec += [("ve.qkv", 0, (T, 3 * cfg.ve_width)), ("ve.attn", 0, (T, cfg.ve_width))]
    rec += [("llm.proj_in", 0, (T, cfg.llm_width))]
    qkv = (cfg.llm_q_heads + 2 * cfg.llm_kv_heads) * cfg.llm_head_dim
    rec += [("llm.qkv", l, (L, qkv)) for l in range(cfg.llm_layers)]
    rec += [("llm.down", l, (L, cfg.llm_width)) for l in range(cfg.llm_layers - 1)]
    AR = cfg.ae_layers * cfg.flow_steps
    rec += [("ae.down", i, (S, cfg.ae_width)) for i in range(AR)]
    rec += [("ae.head", s, (cfg.chunk_len, cfg.ae_action_dim)) for s in range(cfg.flow_steps)]
    return rec


def _compare_layers(eng, cfg, recs, lq):
    cos = {}
    for (node, inst), ref in recs.items():
        got = eng.checkpoint(node, inst, *ref.shape)
        if node == "llm.qkv" and inst == cfg.llm_layers - 1:
            got, ref = got[:, lq:], ref[:, lq:]        # dead Q of the last layer is skipped
        cos[f"{node}[{inst}]"] = cosine(got, ref)
    return cos


def _action_report(y, ref):
    d = y - ref
    return {"max_abs": float(np.abs(d).max()), "rms_err": float(np.sqrt(np.mean(d * d))),
            "rms_ref": float(np.sqrt(np.mean(ref * ref))), "rel": rel_err(y, ref, 0.1), "cos": cosine(y, ref)}


# GEMM variants forced onto every eligible prefill GEMM (default: chosen by size)
GEMM_VARIANTS = {
    "auto": {},
    "persist+pair": {"PI0B_PERSIST": "2", "PI0B_CG": "2"},       # persistent CTA-pair tcgen05
    "pair": {"PI0B_PERSIST": "0", "PI0B_CG": "2"},               # one CTA-pair tile per cluster
    "persist+mt2": {"PI0B_PERSIST": "2", "PI0B_CG": "0", "PI0B_MT": "2"},
}


@pytest.mark.parametrize("views,prompt,variant", [(1, 0, "auto"), (2, 0, "auto"), (3, 32, "auto"),
                                                  (2, 0, "persist+pair"), (2, 0, "pair"), (2, 0, "persist+mt2")])
def test_engine_mid_config_matches_oracle(views, prompt, variant, monkeypatch):
    for k, v in GEMM_VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    cfg = mid_config(views=views, prompt_tokens=prompt)
    x = O.gen_inputs(cfg, 1)
    ref, recs = O.port_forward(cfg, x, record=_record_list(cfg))
    eng = E.Engine(cfg, record_checkpoints=True)
    eng.gen_weights(1)
    y = eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
    rep = _action_report(y, ref)
    lq = cfg.llm_q_heads * cfg.llm_head_dim
    cos = _compare_layers(eng, cfg, recs, lq)
    print("actions", rep)
    print("worst layers", sorted(cos.items(), key=lambda kv: kv[1])[:6])
    assert rep["max_abs"] < ACT_MAX_ABS and rep["rel"] < ACT_REL, rep
    bad = {k: v for k, v in cos.items() if v < LAYER_COS}
    assert not bad, bad
    # graph-captured replay gives the same actions as the eager recorded run
    g = E.Engine(cfg, use_cuda_graph=True)
    g.gen_weights(1)
    y2 = g.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
    assert np.abs(y2 - y).max() < RUN_TO_RUN


def test_engine_host_weightstore_path():
    """Weights uploaded one WeightSet at a time from the reference's gen_weights."""
    cfg = mid_config()
    x = O.gen_inputs(cfg, 1)
    ref, _ = O.port_forward(cfg, x)
    eng = E.Engine(cfg)
    vw, lw, aw = cfg.ve_width, cfg.llm_width, cfg.ae_width
    lqkv = (cfg.llm_q_heads + 2 * cfg.llm_kv_heads) * 256
    aq = cfg.ae_q_heads * 256
    nodes = [("ve.embed", 1, cfg.ve_patch_in, vw, True), ("ve.qkv", cfg.ve_layers, vw, 3 * vw, True),
             ("ve.proj", cfg.ve_layers, vw, vw, True), ("ve.fc1", cfg.ve_layers, vw, cfg.ve_mlp, True),
             ("ve.fc2", cfg.ve_layers, cfg.ve_mlp, vw, True), ("llm.proj_in", 1, vw, lw, True),
             ("llm.qkv", cfg.llm_layers, lw, lqkv, False),
             ("llm.proj", cfg.llm_layers - 1, cfg.llm_q_heads * 256, lw, False),
             ("llm.ffn", cfg.llm_layers - 1, lw, 2 * cfg.llm_mlp, False),
             ("llm.down", cfg.llm_layers - 1, cfg.llm_mlp, lw, False),
             ("ae.state_proj", 1, cfg.ae_state_dim, aw, True), ("ae.action_proj", 1, cfg.ae_action_dim, aw, False),
             ("ae.action_out", 1, aw, aw, True), ("ae.qkv", cfg.ae_layers, aw, aq + 512, False),
             ("ae.proj", cfg.ae_layers, aq, aw, False), ("ae.ffn", cfg.ae_layers, aw, 2 * cfg.ae_mlp, False),
             ("ae.down", cfg.ae_layers, cfg.ae_mlp, aw, False), ("ae.head", 1, aw, cfg.ae_action_dim, True)]
    for node, n, k, m, has_b in nodes:
        for i in range(n):
            w, b = O.port_weight(node, i, k, m, bias=has_b)
            eng.set_weight(node, i, w, b)
    # bias table rows: U(+-1/sqrt(act)) seeded per flow step (proj/src/evaluate.cpp:64-71)
    lim = 1.0 / np.sqrt(cfg.ae_action_dim)
    tab = np.zeros((cfg.flow_steps, aw))
    import torch
    for s in range(cfg.flow_steps):
        t = torch.zeros(aw, dtype=torch.float64, device="cuda")
        E.random_f64(t.data_ptr(), aw, E.seed_hash(1, "ae.action_proj", s, 4), -lim, lim)
        tab[s] = t.cpu().numpy()
    eng.set_bias_table("ae.action_proj", tab)
    y = eng.run(x["patches"], x["state"], x["noise"])
    assert np.abs(y - ref).max() < ACT_MAX_ABS
    gen = E.Engine(cfg)
    gen.gen_weights(1)
    y2 = gen.run(x["patches"], x["state"], x["noise"])
    assert np.abs(y2 - y).max() < RUN_TO_RUN


def test_streaming_split_equals_full_run():
    cfg = mid_config(views=2)
    x = O.gen_inputs(cfg, 1)
    eng = E.Engine(cfg)
    eng.gen_weights(1)
    y = eng.run(x["patches"], x["state"], x["noise"])
    eng.run_prefix(x["patches"])
    y2 = eng.run_action(x["state"], x["noise"])
    assert np.abs(y2 - y).max() < RUN_TO_RUN
    # fresh noise on the cached prefix == a full run with that noise
    x2 = O.gen_inputs(cfg, 7)
    y3 = eng.run_action(x["state"], x2["noise"])
    y4 = eng.run(x["patches"], x["state"], x2["noise"])
    assert np.abs(y3 - y4).max() < RUN_TO_RUN


def test_engine_rejects_bad_inputs():
    cfg = mid_config()
    eng = E.Engine(cfg)
    x = O.gen_inputs(cfg, 1)
    with pytest.raises(E.ShapeError):
        eng.run(x["patches"][:-1], x["state"], x["noise"])
    with pytest.raises(E.ShapeError):
        E.Engine(cfg.replace(llm_head_dim=128))
    with pytest.raises(E.ShapeError):
        eng.set_weight("ve.qkv", 99, np.zeros((cfg.ve_width, 3 * cfg.ve_width)), np.zeros(3 * cfg.ve_width))


def _record_parity(tag, doc):
    """Measured errors go to $PI0B_PARITY_OUT/<tag>.json (copied under profiles/ per round)."""
    out = os.environ.get("PI0B_PARITY_OUT")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"{tag}.json"), "w") as f:
            json.dump(doc, f, indent=1)


FULL_CONFIGS = [(1, 0, "1v"), (2, 0, "2v"), (3, 32, "3v32p")]
# + an unaligned prompt (L = 273): the padded-prefix path (32-row Lp, masked padding keys) at full scale
FULL_ACTION_CONFIGS = FULL_CONFIGS + [(1, 17, "1v17p")]


@pytest.mark.parametrize("views,prompt,tag", FULL_ACTION_CONFIGS)
def test_full_scale_actions_match_reference_golden(views, prompt, tag):
    """Full-scale pi0 (seed 1) vs the reference's fp64 output (tests/golden/full_<tag>.json,
    generated by tests/golden/make_golden.py and pinned to the compiled reference's own
    full-scale run), through the default (graph-replay) engine."""
    gold = json.load(open(os.path.join(GOLDEN, f"full_{tag}.json")))
    ref = np.array(gold["actions"], dtype=np.float64).reshape(63, 32)
    cfg = default_config(views=views, prompt_tokens=prompt)
    x = O.gen_inputs(cfg, 1)
    eng = E.Engine(cfg)
    eng.gen_weights(1)
    y = eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
    rep = _action_report(y, ref)
    print(f"full {tag} actions", rep)
    _record_parity(f"actions_{tag}", rep)
    assert rep["max_abs"] < FULL_MAX_ABS and rep["rel"] < FULL_REL and rep["rms_err"] < FULL_RMS_ERR, rep
    assert rep["cos"] > 0.9999, rep


@pytest.mark.parametrize("views,prompt,tag", FULL_ACTION_CONFIGS)
def test_full_scale_per_layer_cosine(views, prompt, tag):
    """North star: per-layer hidden-state cosine >= 0.999 at FULL scale, across all 225 serial
    layers' checkpoints of SURVEY.md 8(c) (ve.fc2[0..26], llm.proj_in, the KV cache
    llm.qkv[l][:, 2048:2560], llm.down[l], ae.down of flow steps 0 and 9 and the last layer of
    every step, ae.head[s]) against the committed fp64 sketches (tests/golden/sketch_<tag>.npz:
    fixed row subsets of the bitwise-equal restatement's hidden states)."""
    sk = np.load(os.path.join(GOLDEN, f"sketch_{tag}.npz"))
    cfg = default_config(views=views, prompt_tokens=prompt)
    x = O.gen_inputs(cfg, 1)
    eng = E.Engine(cfg, record_checkpoints=True)
    eng.gen_weights(1)
    y = eng.run(x["patches"], x["state"], x["noise"], x.get("prompt"))
    cos = {}
    for node, inst, shape, cols in sketch_checkpoints(cfg):
        key = f"{node}[{inst}]"
        cos[key] = cosine(sketch_take(eng.checkpoint(node, inst, *shape), cols), sk[key])
    rep = _action_report(y, sk["actions"])
    worst = sorted(cos.items(), key=lambda kv: kv[1])[:8]
    print(f"full {tag}: {len(cos)} checkpoints, worst {worst}, actions {rep}")
    _record_parity(f"layers_{tag}", {"checkpoints": len(cos), "min_cos": min(cos.values()), "worst": worst,
                                     "cos": cos, "actions": rep})
    assert len(cos) == len(sk.files) - 1
    bad = {k: v for k, v in cos.items() if v < LAYER_COS}
    assert not bad, bad


DEMO = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "pi0b_rtvla_demo")


@pytest.mark.parametrize("views,prompt", [(1, 0), (3, 32)])
def test_rtvla_cpp_dropin(views, prompt):
    """include/pi0b_rtvla.hpp with the reference's own C++ types: pi0b::evaluate(g, w, x) and
    pi0b::Engine vs rtvla::evaluate (fp64, compiled from the reference) on the same graph,
    WeightStore and Inputs; a non-pi0 graph is rejected with rtvla::ShapeError."""
    import subprocess
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/pi0b_rtvla_demo not built (needs /root/reference at build time)")
    r = subprocess.run([DEMO, str(views), str(prompt)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("views,prompt", [(1, 0), (3, 32)])
def test_rtvla_cpp_naive_graph(views, prompt):
    """an unfused graph (rtvla::build_pi0_graph_naive: separate q/k/v, RMSNorm gamma,
    time MLP) and its WeightStore through pi0b::evaluate_naive -- fused on the host by the engine's
    own weight rules (pi0b::fuse_naive; bitwise == rtvla::apply_weight_rules, test_adaptor_cpu.py)
    -- vs rtvla::evaluate on the naive graph."""
    import subprocess
    if not os.path.exists(DEMO):
        pytest.skip("oracle/_ref/pi0b_rtvla_demo not built (needs /root/reference at build time)")
    r = subprocess.run([DEMO, "naive", str(views), str(prompt)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
