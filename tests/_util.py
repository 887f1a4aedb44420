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
