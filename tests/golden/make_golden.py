"""Generate the committed golden fixtures (run in the container that has /root/reference).

* tiny_1v.json, mid_{1v,2v,3v32p}.json — actions from the compiled UNMODIFIED reference
  (``rtvla::evaluate`` via oracle/_ref/librtvla_ref.so), seed 1 for weights and inputs.
* sketch_{1v,2v,3v32p}.npz — full-scale per-layer hidden-state "sketches": a fixed subset of
  rows (tests/_util.py sketch_rows) of every SURVEY.md 8(c) checkpoint, in fp32, from the
  bitwise-equal restatement: ve.fc2[0..26], llm.proj_in, llm.qkv[l] K|V columns [2048,2560)
  (the KV cache), llm.down[l], ae.down at every layer of flow steps 0 and 9 and the last
  layer of every step, ae.head[s].  The GPU tests assert cosine >= 0.999 on each.
* full_1v.json, full_2v.json — full-scale actions from the fp64 restatement
  (oracle/pi0_oracle.cpp, bitwise equal to the reference on every config the tests can
  afford to run through the reference), cross-checked against the reference's own
  full-scale run recorded in SURVEY.md 8(c) / BASELINE.md 3 (y[0], y[1], y[last], sum,
  sum|y| at 17 significant digits); generation aborts if they disagree.

* full_3v32p.json — restatement actions, checked element for element against the reference's
  own full-scale run (ref_full_3v32p.json from ref_full_run.py, ~40 min single-threaded).
* full_1v17p.json — the same for 1 view + a 17-token prompt (L = 273, not a multiple of 32: the
  engine's padded-prefix path at full scale), against ref_full_1v17p.json.

Usage:  PYTHONPATH=. python tests/golden/make_golden.py [tiny mid full1 full2 full3 full1p17 sketch1 sketch2 sketch3 sketch1p17]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2510_26742_b200.config import default_config, mid_config, tiny_config  # noqa: E402

sys.path.insert(0, os.path.join(ROOT, "tests"))
from _util import sketch_checkpoints, sketch_take  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# Reference full-scale outputs, seed 1 (770.4 s / 1432.5 s single-thread runs).
REFERENCE_SPOTS = {
    1: {"y0": 1.0286562565432205, "y1": 1.2088658830676564, "ylast": 0.34389548371564982,
        "sum": 175.91048182764209, "abs_sum": 1308.9780619608166},
    2: {"y0": 0.99116682917401266, "y1": 1.2019504034525859, "ylast": 0.014307136309375735,
        "sum": 206.67524788946236, "abs_sum": 1321.5203657793868},
}


def dump(name, cfg, actions, source, extra=None):
    doc = {"config": cfg.as_dict(), "weight_seed": 1, "input_seed": 1, "source": source,
           "actions": [float(v) for v in actions.ravel()],
           "sum": float(actions.sum()), "abs_sum": float(np.abs(actions).sum())}
    if extra:
        doc.update(extra)
    with open(os.path.join(HERE, name), "w") as f:
        json.dump(doc, f, indent=0)
    print("wrote", name)


def main(which):
    if "tiny" in which:
        cfg = tiny_config()
        dump("tiny_1v.json", cfg, O.ref_evaluate(cfg), "reference rtvla::evaluate")
    if "mid" in which:
        for views, prompt, tag in [(1, 0, "1v"), (2, 0, "2v"), (3, 32, "3v32p")]:
            cfg = mid_config(views=views, prompt_tokens=prompt)
            dump(f"mid_{tag}.json", cfg, O.ref_evaluate(cfg), "reference rtvla::evaluate")
    for views, key in [(1, "full1"), (2, "full2")]:
        if key not in which:
            continue
        cfg = default_config(views=views)
        x = O.gen_inputs(cfg, 1)
        t = time.time()
        y, _ = O.port_forward(cfg, x)
        dt = time.time() - t
        spots = REFERENCE_SPOTS[views]
        got = {"y0": y.ravel()[0], "y1": y.ravel()[1], "ylast": y.ravel()[-1], "sum": y.sum(),
               "abs_sum": np.abs(y).sum()}
        for k, v in spots.items():
            tol = 0.0 if k in ("y0", "y1", "ylast") else 1e-12 * abs(v)
            if abs(got[k] - v) > tol:
                raise SystemExit(f"full {views}v: {k} = {got[k]!r} != reference {v!r}")
        dump(f"full_{views}v.json", cfg, y, "pi0_oracle restatement (bitwise == reference spot values)",
             {"restatement_seconds": dt})
    if "full1p17" in which:   # unaligned prompt at full scale: L = 273 (the engine pads to 288 rows)
        cfg = default_config(views=1, prompt_tokens=17)
        x = O.gen_inputs(cfg, 1)
        t = time.time()
        y, _ = O.port_forward(cfg, x)
        dt = time.time() - t
        ref = json.load(open(os.path.join(HERE, "ref_full_1v17p.json")))
        r = np.array(ref["actions"]).reshape(y.shape)
        if not np.array_equal(r, y):
            raise SystemExit(f"full 1v17p: restatement != reference, max |d| {np.abs(r - y).max():.3e}")
        dump("full_1v17p.json", cfg, y, "pi0_oracle restatement (bitwise == reference rtvla::evaluate, "
             "ref_full_1v17p.json)", {"restatement_seconds": dt, "reference_evaluate_seconds": ref["evaluate_seconds"]})
    if "full3" in which:
        cfg = default_config(views=3, prompt_tokens=32)
        x = O.gen_inputs(cfg, 1)
        t = time.time()
        y, _ = O.port_forward(cfg, x)
        dt = time.time() - t
        ref_path = os.path.join(HERE, "ref_full_3v32p.json")
        ref = json.load(open(ref_path))
        r = np.array(ref["actions"]).reshape(y.shape)
        if not np.array_equal(r, y):
            raise SystemExit(f"full 3v32p: restatement != reference, max |d| {np.abs(r - y).max():.3e}")
        dump("full_3v32p.json", cfg, y, "pi0_oracle restatement (bitwise == reference rtvla::evaluate, "
             "ref_full_3v32p.json)", {"restatement_seconds": dt,
                                      "reference_evaluate_seconds": ref["evaluate_seconds"]})
    for views, prompt, key in [(1, 0, "sketch1"), (2, 0, "sketch2"), (3, 32, "sketch3"), (1, 17, "sketch1p17")]:
        if key not in which:
            continue
        cfg = default_config(views=views, prompt_tokens=prompt)
        x = O.gen_inputs(cfg, 1)
        cks = sketch_checkpoints(cfg)
        t = time.time()
        y, recs = O.port_forward(cfg, x, record=[(n, i, shape) for (n, i, shape, _) in cks])
        dt = time.time() - t
        arrays = {"actions": y.astype(np.float64)}
        for (node, inst, shape, cols) in cks:
            arrays[f"{node}[{inst}]"] = sketch_take(recs[(node, inst)], cols).astype(np.float32)
        tag = f"{views}v" + (f"{prompt}p" if prompt else "")
        gold = os.path.join(HERE, f"full_{tag}.json")
        if os.path.exists(gold):   # the sketch's forward must be the golden forward
            g = np.array(json.load(open(gold))["actions"]).reshape(y.shape)
            if not np.array_equal(g, y):
                raise SystemExit(f"sketch {tag}: actions differ from {gold}")
        np.savez_compressed(os.path.join(HERE, f"sketch_{tag}.npz"), **arrays)
        print(f"wrote sketch_{tag}.npz ({len(arrays) - 1} checkpoints, {dt:.0f} s)")


if __name__ == "__main__":
    main(sys.argv[1:] or ["tiny", "mid"])
