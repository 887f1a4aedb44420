"""Shared helpers for the parity tests."""
import numpy as np


def bf16_bits_from_f64(x: np.ndarray) -> np.ndarray:
    """fp64 -> bf16 bit patterns with one round-to-nearest-even (the engine's rule,
    csrc/numerics.cuh f64_to_bf16_bits): truncate to fp32, sticky bit, RNE to bf16."""
    x = np.asarray(x, dtype=np.float64)
    f = x.astype(np.float32)
    over = np.abs(f.astype(np.float64)) > np.abs(x)
    f = np.where(over, np.nextafter(f, np.float32(0)), f).astype(np.float32)
    u = f.view(np.uint32).copy()
    u |= (f.astype(np.float64) != x).astype(np.uint32)
    u = u + np.uint32(0x7FFF) + ((u >> 16) & np.uint32(1))
    return (u >> 16).astype(np.uint16)


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def cosine(a, b) -> float:
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    return float(a @ b / (np.linalg.norm(a) * np.linalg.norm(b) + 1e-300))


def rel_err(a, b, floor_frac: float = 1e-2) -> float:
    """max |a-b| / max(|b|, floor) with floor = floor_frac * rms(b)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    floor = floor_frac * np.sqrt(np.mean(b * b)) + 1e-300
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)))


def sketch_rows(n_rows: int, count: int = 8) -> np.ndarray:
    """The fixed row subset a full-scale hidden-state sketch keeps: `count` rows spread evenly
    over [0, n_rows) including the first and last (row 0 = the AE state token)."""
    return np.unique(np.linspace(0, n_rows - 1, min(count, n_rows)).round().astype(np.int64))


def sketch_checkpoints(cfg) -> list:
    """SURVEY.md 8(c) parity checkpoints at full scale: [(node, instance, full shape, column
    range or None)].  llm.qkv keeps only its K|V columns (the KV cache the action expert reads;
    the last layer's Q columns are dead compute the engine skips)."""
    T, L, S = cfg.image_tokens, cfg.prefix_tokens, cfg.suffix_tokens
    lq = cfg.llm_q_heads * cfg.llm_head_dim
    qkv = lq + 2 * cfg.llm_kv_heads * cfg.llm_head_dim
    out = [("ve.fc2", i, (T, cfg.ve_width), None) for i in range(cfg.ve_layers)]
    out.append(("llm.proj_in", 0, (T, cfg.llm_width), None))
    out += [("llm.qkv", l, (L, qkv), (lq, qkv)) for l in range(cfg.llm_layers)]
    out += [("llm.down", l, (L, cfg.llm_width), None) for l in range(cfg.llm_layers - 1)]
    A, F = cfg.ae_layers, cfg.flow_steps
    ae = sorted({i for i in range(A)} | {(F - 1) * A + i for i in range(A)} | {s * A + A - 1 for s in range(F)})
    out += [("ae.down", i, (S, cfg.ae_width), None) for i in ae]
    out += [("ae.head", s, (cfg.chunk_len, cfg.ae_action_dim), None) for s in range(F)]
    return out


def sketch_take(a: np.ndarray, cols) -> np.ndarray:
    """Apply a sketch's row subset (all rows of small tensors such as ae.head) and column range."""
    rows = sketch_rows(a.shape[0]) if a.size > 4096 else np.arange(a.shape[0])
    a = a[rows]
    return a if cols is None else a[:, cols[0]:cols[1]]
