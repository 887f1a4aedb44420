"""Host-side `rtvla::gen_inputs` (proj/src/evaluate.cpp:77-85): every Source node of the fused
graph (patches, state, noise, and prompt when prompt_tokens > 0) is drawn as
random_tensor(rows, cols, -1, 1, seed_hash(seed, id, 0, 5)) — a SplitMix64 stream whose n-th
output u gives lo + (hi - lo) * u (proj/src/tensor.cpp:7-47).  Vectorised with uint64 numpy
arithmetic; bit-identical to the reference (tests/test_inputs.py)."""
from __future__ import annotations

import numpy as np

from .config import ModelConfig

_MASK = (1 << 64) - 1


def seed_hash(seed: int, label: str, a: int, b: int) -> int:
    """FNV-1a over the 8 bytes of seed, the label, and the 8 bytes of a and b
    (proj/src/tensor.cpp:24-40)."""
    h = 0xCBF29CE484222325
    for v in (seed,):
        for i in range(8):
            h = ((h ^ ((v >> (8 * i)) & 0xFF)) * 0x100000001B3) & _MASK
    for ch in label.encode():
        h = ((h ^ ch) * 0x100000001B3) & _MASK
    for v in (a, b):
        for i in range(8):
            h = ((h ^ ((v >> (8 * i)) & 0xFF)) * 0x100000001B3) & _MASK
    return h


def random_tensor(rows: int, cols: int, lo: float, hi: float, seed: int) -> np.ndarray:
    n = np.arange(1, rows * cols + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + n * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return (lo + (hi - lo) * u).reshape(rows, cols)


def gen_inputs(cfg: ModelConfig, seed: int = 1) -> dict:
    out = {
        "patches": random_tensor(cfg.image_tokens, cfg.ve_patch_in, -1.0, 1.0, seed_hash(seed, "patches", 0, 5)),
        "state": random_tensor(1, cfg.ae_state_dim, -1.0, 1.0, seed_hash(seed, "state", 0, 5)),
        "noise": random_tensor(cfg.chunk_len, cfg.ae_action_dim, -1.0, 1.0, seed_hash(seed, "noise", 0, 5)),
    }
    if cfg.prompt_tokens > 0:
        out["prompt"] = random_tensor(cfg.prompt_tokens, cfg.llm_width, -1.0, 1.0, seed_hash(seed, "prompt", 0, 5))
    return out
