"""pi0 model configuration — a field-for-field mirror of ``rtvla::ModelConfig``
(proj/include/rtvla/graph.hpp:114-160) laid out as the C struct ``pi0b_model_config``
of include/pi0b.h, plus the reference's presets (proj/src/builder.cpp:10-22)."""
from __future__ import annotations

import ctypes

FIELDS = [
    "views", "prompt_tokens", "tokens_per_view", "chunk_len", "flow_steps",
    "ve_layers", "ve_width", "ve_heads", "ve_head_dim", "ve_mlp", "ve_patch_in",
    "llm_layers", "llm_width", "llm_q_heads", "llm_head_dim", "llm_kv_heads", "llm_mlp",
    "ae_layers", "ae_width", "ae_q_heads", "ae_head_dim", "ae_kv_heads", "ae_mlp",
    "ae_action_dim", "ae_state_dim",
]


class ModelConfig(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int) for f in FIELDS]

    # --- derived sizes (proj/include/rtvla/graph.hpp:156-158, builder.cpp:128-164)
    @property
    def image_tokens(self) -> int:
        return self.views * self.tokens_per_view

    @property
    def prefix_tokens(self) -> int:
        return self.image_tokens + self.prompt_tokens

    @property
    def suffix_tokens(self) -> int:
        return self.chunk_len + 1

    @property
    def cross_kv_tokens(self) -> int:
        return self.prefix_tokens + self.suffix_tokens

    def replace(self, **kw) -> "ModelConfig":
        c = ModelConfig(**{f: getattr(self, f) for f in FIELDS})
        for k, v in kw.items():
            setattr(c, k, v)
        return c

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f in FIELDS}

    def __repr__(self) -> str:  # pragma: no cover - debugging aid
        return "ModelConfig(" + ", ".join(f"{f}={getattr(self, f)}" for f in FIELDS) + ")"


def default_config(views: int = 2, prompt_tokens: int = 0) -> ModelConfig:
    """rtvla::default_config(): full-scale pi0 (SigLIP 27x1152, Gemma-2B 18x2048, AE 18x1024)."""
    return ModelConfig(
        views=views, prompt_tokens=prompt_tokens, tokens_per_view=256, chunk_len=63, flow_steps=10,
        ve_layers=27, ve_width=1152, ve_heads=16, ve_head_dim=72, ve_mlp=4304, ve_patch_in=588,
        llm_layers=18, llm_width=2048, llm_q_heads=8, llm_head_dim=256, llm_kv_heads=1, llm_mlp=16384,
        ae_layers=18, ae_width=1024, ae_q_heads=8, ae_head_dim=256, ae_kv_heads=1, ae_mlp=4096,
        ae_action_dim=32, ae_state_dim=32,
    )


def tiny_config() -> ModelConfig:
    """rtvla::tiny_config(): the reference's reduced twin (widths/16).  Oracle-only: its head
    dims (9, 16) are outside what the sm_100a kernels implement."""
    return ModelConfig(
        views=1, prompt_tokens=0, tokens_per_view=256, chunk_len=63, flow_steps=2,
        ve_layers=2, ve_width=72, ve_heads=8, ve_head_dim=9, ve_mlp=269, ve_patch_in=588,
        llm_layers=2, llm_width=128, llm_q_heads=8, llm_head_dim=16, llm_kv_heads=1, llm_mlp=1024,
        ae_layers=2, ae_width=64, ae_q_heads=8, ae_head_dim=16, ae_kv_heads=1, ae_mlp=256,
        ae_action_dim=2, ae_state_dim=2,
    )


def mid_config(views: int = 1, prompt_tokens: int = 0) -> ModelConfig:
    """A reduced-width twin that keeps the full-scale head geometry (VE d72, LLM/AE d256 MQA),
    awkward K tails (patch 588, VE mlp 1076) and every node kind, so the GPU kernels run their
    full-scale code paths while the fp64 oracle finishes in seconds."""
    return ModelConfig(
        views=views, prompt_tokens=prompt_tokens, tokens_per_view=256, chunk_len=63, flow_steps=3,
        ve_layers=2, ve_width=288, ve_heads=4, ve_head_dim=72, ve_mlp=1076, ve_patch_in=588,
        llm_layers=3, llm_width=512, llm_q_heads=2, llm_head_dim=256, llm_kv_heads=1, llm_mlp=1024,
        ae_layers=2, ae_width=256, ae_q_heads=2, ae_head_dim=256, ae_kv_heads=1, ae_mlp=512,
        ae_action_dim=32, ae_state_dim=32,
    )
