"""Algorithmic work of one pi0 inference and its roofline lower bound.

Follows the reference's own lower-bound method (proj/src/costmodel.cpp:82-92, 480-609;
PAPER.md:184-253): every GEMM instance costs max(2*K*M / BW, N*K*M / MACrate) (bf16 weight
bytes vs multiply-accumulates), self-attention costs 2*h*q*kv*d MACs, and the action
expert's cross-attention is costed as the two GEMM rows [h*q x d x kv] and [h*q x kv x d]
(proj/src/costmodel.cpp:507-528).  With the B200 peaks of MEASURED_PEAKS.json this gives
BASELINE.md's 1.699 / 2.461 / 3.323 ms (1v / 2v / 3v+32p, burst).
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass

from .config import ModelConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@dataclass
class Gemm:
    node: str
    n: int
    k: int
    m: int
    repeat: int
    stage: str

    @property
    def macs(self) -> int:
        return self.n * self.k * self.m

    @property
    def weight_bytes(self) -> int:
        return 2 * self.k * self.m


def gemms(c: ModelConfig) -> list[Gemm]:
    T, L, S, C, FS = c.image_tokens, c.prefix_tokens, c.suffix_tokens, c.chunk_len, c.flow_steps
    vw, lw, aw = c.ve_width, c.llm_width, c.ae_width
    lq, lkv = c.llm_q_heads * c.llm_head_dim, c.llm_kv_heads * c.llm_head_dim
    aq, akv = c.ae_q_heads * c.ae_head_dim, c.ae_kv_heads * c.ae_head_dim
    VL, LL, AR = c.ve_layers, c.llm_layers, c.ae_layers * FS
    return [
        Gemm("ve.embed", T, c.ve_patch_in, vw, 1, "VE"),
        Gemm("ve.qkv", T, vw, 3 * vw, VL, "VE"),
        Gemm("ve.proj", T, vw, vw, VL, "VE"),
        Gemm("ve.fc1", T, vw, c.ve_mlp, VL, "VE"),
        Gemm("ve.fc2", T, c.ve_mlp, vw, VL, "VE"),
        Gemm("llm.proj_in", T, vw, lw, 1, "LLM"),
        Gemm("llm.qkv", L, lw, lq + 2 * lkv, LL, "LLM"),
        Gemm("llm.proj", L, lq, lw, LL - 1, "LLM"),
        Gemm("llm.ffn", L, lw, 2 * c.llm_mlp, LL - 1, "LLM"),
        Gemm("llm.down", L, c.llm_mlp, lw, LL - 1, "LLM"),
        Gemm("ae.state_proj", 1, c.ae_state_dim, aw, 1, "AE"),
        Gemm("ae.action_proj", C, c.ae_action_dim, aw, FS, "AE"),
        Gemm("ae.action_out", C, aw, aw, FS, "AE"),
        Gemm("ae.qkv", S, aw, aq + 2 * akv, AR, "AE"),
        Gemm("ae.proj", S, aq, aw, AR, "AE"),
        Gemm("ae.ffn", S, aw, 2 * c.ae_mlp, AR, "AE"),
        Gemm("ae.down", S, c.ae_mlp, aw, AR, "AE"),
        Gemm("ae.head", C, aw, c.ae_action_dim, FS, "AE"),
    ]


def attention_macs(c: ModelConfig) -> dict:
    """MACs per instance and repeat of each attention node (2*h*q*kv*d)."""
    T, L, S = c.image_tokens, c.prefix_tokens, c.suffix_tokens
    return {
        "ve.attn": (2 * c.ve_heads * T * T * c.ve_head_dim, c.ve_layers),
        "llm.attn": (2 * c.llm_q_heads * L * L * c.llm_head_dim, c.llm_layers - 1),
        "ae.attn": (2 * c.ae_q_heads * S * (L + S) * c.ae_head_dim, c.ae_layers * c.flow_steps),
    }


def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    # fallback stated by /opt/skills/guides/B200_PROFILING.md
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


def lower_bound_ms(c: ModelConfig, sustained: bool = False, peaks: dict | None = None) -> dict:
    """Reference-method roofline (sum of per-kernel max(bytes/BW, MACs/MACrate)), per stage."""
    pk = peaks or measured_peaks()
    bw = pk["hbm_gbs"] * 1e9
    mac = (pk["bf16_tflops_sustained"] if sustained else pk["bf16_tflops"]) * 1e12 / 2
    out = {"VE": 0.0, "LLM": 0.0, "AE": 0.0}
    for g in gemms(c):
        out[g.stage] += g.repeat * max(g.weight_bytes / bw, g.macs / mac)
    att = attention_macs(c)
    out["VE"] += att["ve.attn"][1] * att["ve.attn"][0] / mac
    out["LLM"] += att["llm.attn"][1] * att["llm.attn"][0] / mac
    # AE cross attention as two GEMM rows: [h*S x d x kv] and [h*S x kv x d]
    hq, kv, d = c.ae_q_heads * c.suffix_tokens, c.prefix_tokens + c.suffix_tokens, c.ae_head_dim
    row = max(2 * d * kv / bw, hq * d * kv / mac) + max(2 * kv * d / bw, hq * kv * d / mac)
    out["AE"] += c.ae_layers * c.flow_steps * row
    out = {k: v * 1e3 for k, v in out.items()}
    out["total"] = out["VE"] + out["LLM"] + out["AE"]
    return out


def totals(c: ModelConfig) -> dict:
    """Algorithmic FLOPs and weight bytes of one inference."""
    flops = sum(2 * g.macs * g.repeat for g in gemms(c))
    flops += sum(2 * m * r for m, r in attention_macs(c).values())
    wbytes = sum(g.weight_bytes * g.repeat for g in gemms(c))
    unique = sum(g.weight_bytes * (1 if g.node.startswith("ae.") and g.node not in ("ae.qkv", "ae.proj",
                 "ae.ffn", "ae.down") else g.repeat) for g in gemms(c))
    return {"flops": flops, "weight_bytes_streamed": wbytes, "weight_bytes_unique": unique}


def ae_weight_bytes(c: ModelConfig) -> int:
    """bf16 bytes of every action-expert weight the megakernel streams once per flow step:
    18 x (qkv + proj + ffn + down) + action_proj + action_out + head (state_proj once per launch
    is included here too; it is 64 KB)."""
    W, A = c.ae_width, c.ae_action_dim
    nq = (c.ae_q_heads + 2 * c.ae_kv_heads) * c.ae_head_dim
    layer = W * nq + c.ae_q_heads * c.ae_head_dim * W + W * 2 * c.ae_mlp + c.ae_mlp * W
    return 2 * (c.ae_layers * layer + A * W + W * W + W * A)


def kv_cache_bytes(c: ModelConfig) -> int:
    """bf16 bytes of the LLM K and V rows the action expert attends to, per flow step."""
    return 2 * 2 * c.prefix_tokens * c.llm_kv_heads * c.llm_head_dim * c.ae_layers
