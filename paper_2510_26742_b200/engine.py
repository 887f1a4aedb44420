"""ctypes binding of libpi0b.so (include/pi0b.h).

Mirrors the reference's C++ inference API for the pi0 path
(proj/include/rtvla/evaluate.hpp:38-44):

    rtvla::gen_weights(g, seed)      -> Engine.gen_weights(seed)       (on device, bit-exact bf16)
    WeightStore / WeightSet          -> Engine.set_weight(node, inst, w, bias) / set_bias_table
    rtvla::evaluate(g, w, x)         -> Engine.run(patches, state, noise, prompt) -> [63, 32] fp64
    errors: ShapeError / NumericError are raised as the same-named Python exceptions.

There is no CPU fallback: if the CUDA library is missing or no sm_100 device is present the
constructor raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .config import ModelConfig

# PI0B_LIB: an alternative build of the same library (A/B experiments, scripts/variants.sh)
LIB_PATH = os.environ.get("PI0B_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libpi0b.so")

PI0B_E_INVALID = -1
PI0B_E_UNSUPPORTED = -2
PI0B_E_STATE = -3
PI0B_E_NUMERIC = -4

# GEMM epilogue modes / flags (csrc/gemm.cuh)
MODE_BF16, MODE_GATE, MODE_F32_STORE, MODE_RESID, MODE_SILU_TABLE = 0, 1, 2, 3, 4
FLAG_ROWSCALE, FLAG_BIAS, FLAG_GELU, FLAG_ROPE = 1, 2, 4, 8


class ShapeError(ValueError):
    """rtvla::ShapeError (proj/include/rtvla/tensor.hpp:15-17)."""


class NumericError(ArithmeticError):
    """rtvla::NumericError (proj/include/rtvla/tensor.hpp:18-20)."""


class UnsupportedConfig(ShapeError):
    pass


class EngineOptions(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("use_cuda_graph", ctypes.c_int), ("record_checkpoints", ctypes.c_int),
                ("ve_shards", ctypes.c_int), ("ve_shard", ctypes.c_int), ("ae_ctas", ctypes.c_int)]


class VeBuffers(ctypes.Structure):
    """pi0b_ve_buffers: device buffers a view-sharded VE engine exposes to its peers."""
    _fields_ = [("qkv", ctypes.c_void_p * 2), ("x", ctypes.c_void_p), ("xb", ctypes.c_void_p),
                ("stats", ctypes.c_void_p), ("sync", ctypes.c_void_p)]

    FIELDS = ("qkv0", "qkv1", "x", "xb", "stats", "sync")

    def as_list(self):
        return [self.qkv[0], self.qkv[1], self.x, self.xb, self.stats, self.sync]

    @classmethod
    def from_list(cls, v):
        b = cls()
        b.qkv[0], b.qkv[1], b.x, b.xb, b.stats, b.sync = v
        return b


class GemmDesc(ctypes.Structure):
    _fields_ = [
        ("a", ctypes.c_void_p), ("lda", ctypes.c_int64),
        ("w", ctypes.c_void_p), ("ldw", ctypes.c_int64),
        ("M", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int),
        ("bn", ctypes.c_int), ("splits", ctypes.c_int),
        ("mode", ctypes.c_int), ("flags", ctypes.c_int),
        ("row_stats", ctypes.c_void_p), ("inv_width", ctypes.c_float), ("eps", ctypes.c_float),
        ("bias", ctypes.c_void_p),
        ("table_row", ctypes.c_void_p),
        ("rope_cs", ctypes.c_void_p), ("rope_pos0", ctypes.c_int), ("rope_cols", ctypes.c_int),
        ("resid_scale", ctypes.c_float),
        ("out", ctypes.c_void_p), ("ldo", ctypes.c_int64),
        ("outb", ctypes.c_void_p), ("ldob", ctypes.c_int64),
        ("out_stats", ctypes.c_void_p),
        ("row0_src", ctypes.c_void_p),
        ("ws", ctypes.c_void_p), ("counters", ctypes.c_void_p),
    ]


class AttnDesc(ctypes.Structure):
    _fields_ = [
        ("head_dim", ctypes.c_int),
        ("q", ctypes.c_void_p), ("ldq", ctypes.c_int64), ("q_rows", ctypes.c_int), ("heads", ctypes.c_int),
        ("kv_heads", ctypes.c_int),
        ("k0", ctypes.c_void_p), ("v0", ctypes.c_void_p), ("ld0", ctypes.c_int64), ("rows0", ctypes.c_int),
        ("k1", ctypes.c_void_p), ("v1", ctypes.c_void_p), ("ld1", ctypes.c_int64), ("rows1", ctypes.c_int),
        ("out", ctypes.c_void_p), ("ldo", ctypes.c_int64),
        ("kv_splits", ctypes.c_int),
        ("ws", ctypes.c_void_p), ("counters", ctypes.c_void_p),
        ("rows0_valid", ctypes.c_int),
    ]


_lib = None
_dp = ctypes.POINTER(ctypes.c_double)


def lib():
    """Load libpi0b.so (raises if it was not built: there is no fallback path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        cfgp = ctypes.POINTER(ModelConfig)
        vp = ctypes.c_void_p
        L.pi0b_last_error.restype = ctypes.c_char_p
        L.pi0b_default_config.argtypes = [cfgp]
        L.pi0b_engine_create.argtypes = [cfgp, ctypes.POINTER(EngineOptions), ctypes.POINTER(vp)]
        if hasattr(L, "pi0b_engine_create_shared"):
            L.pi0b_engine_create_shared.argtypes = [cfgp, ctypes.POINTER(EngineOptions), vp, ctypes.POINTER(vp)]
        L.pi0b_engine_destroy.argtypes = [vp]
        L.pi0b_engine_destroy.restype = None
        L.pi0b_engine_gen_weights.argtypes = [vp, ctypes.c_uint64]
        L.pi0b_engine_set_weight.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64, _dp, ctypes.c_int64,
                                             ctypes.c_int64, _dp, ctypes.c_int64]
        L.pi0b_engine_set_bias_table.argtypes = [vp, ctypes.c_char_p, _dp, ctypes.c_int64, ctypes.c_int64]
        L.pi0b_engine_run.argtypes = [vp, _dp, _dp, _dp, _dp, _dp]
        L.pi0b_engine_run_prefix.argtypes = [vp, _dp, _dp]
        L.pi0b_stream_run.argtypes = [cfgp, ctypes.c_uint64, ctypes.POINTER(StreamOptions), ctypes.c_double,
                                       ctypes.POINTER(StreamReport)]
        L.pi0b_engine_run_images.argtypes = [vp, _dp, ctypes.c_int, ctypes.c_int, _dp, _dp, _dp, _dp]
        L.pi0b_image_patches.argtypes = [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, vp, vp]
        L.pi0b_engine_run_action.argtypes = [vp, _dp, _dp, _dp]
        L.pi0b_f64_to_bf16_host.argtypes = [_dp, ctypes.c_longlong, vp]
        L.pi0b_engine_replay.argtypes = [vp, ctypes.c_int, vp]
        L.pi0b_engine_sync.argtypes = [vp]
        L.pi0b_engine_kernel_count.argtypes = [vp, ctypes.c_int]
        L.pi0b_engine_read_checkpoint.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64,
                                                  ctypes.POINTER(ctypes.c_float), ctypes.c_int64, ctypes.c_int64]
        L.pi0b_engine_time_node.argtypes = [vp, ctypes.c_char_p, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                            ctypes.POINTER(ctypes.c_int)]
        L.pi0b_engine_describe.argtypes = [vp, ctypes.c_char_p, ctypes.c_int64]
        L.pi0b_gemm.argtypes = [ctypes.POINTER(GemmDesc), vp]
        L.pi0b_gemm_skinny.argtypes = [ctypes.POINTER(GemmDesc), ctypes.c_int, vp]
        L.pi0b_attention.argtypes = [ctypes.POINTER(AttnDesc), vp]
        L.pi0b_attention_ws_floats.argtypes = [ctypes.POINTER(AttnDesc)]
        L.pi0b_attention_ws_floats.restype = ctypes.c_int64
        L.pi0b_random_f64.argtypes = [vp, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_double, vp]
        L.pi0b_random_packed_bf16.argtypes = [vp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_uint64, ctypes.c_double, ctypes.c_double, vp]
        L.pi0b_seed_hash.argtypes = [ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64]
        L.pi0b_seed_hash.restype = ctypes.c_uint64
        # (entry points an older build may lack: PI0B_LIB A/B runs against earlier libraries)
        for name, args in (("pi0b_engine_ve_buffers", [vp, ctypes.POINTER(VeBuffers)]),
                           ("pi0b_engine_set_ve_peers", [vp, ctypes.POINTER(VeBuffers), ctypes.c_int]),
                           ("pi0b_ipc_export", [vp, ctypes.c_char_p]),
                           ("pi0b_ipc_open", [ctypes.c_char_p, ctypes.POINTER(vp)]),
                           ("pi0b_ipc_close", [vp]),
                           ("pi0b_rope_table_host", [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float)])):
            if hasattr(L, name):
                getattr(L, name).argtypes = args
        _lib = L
    return _lib


class StreamOptions(ctypes.Structure):
    """include/pi0b.h pi0b_stream_options"""
    _fields_ = [("frame_rate", ctypes.c_double), ("camera_latency", ctypes.c_int), ("ae_rate", ctypes.c_double),
                ("trajectory_rate", ctypes.c_double), ("kv_policy", ctypes.c_int), ("device", ctypes.c_int),
                ("prefix_sms", ctypes.c_int)]


class StreamReport(ctypes.Structure):
    """include/pi0b.h pi0b_stream_report"""
    _fields_ = [("seconds", ctypes.c_double), ("frames", ctypes.c_int64), ("ticks", ctypes.c_int64),
                ("vlm_per_s", ctypes.c_double), ("ae_per_s", ctypes.c_double),
                ("quick_mean_ms", ctypes.c_double), ("quick_best_ms", ctypes.c_double),
                ("quick_worst_ms", ctypes.c_double), ("quick_count", ctypes.c_int64),
                ("slow_mean_ms", ctypes.c_double), ("slow_best_ms", ctypes.c_double),
                ("slow_worst_ms", ctypes.c_double), ("slow_count", ctypes.c_int64),
                ("prefix_p50_ms", ctypes.c_double), ("tick_p50_ms", ctypes.c_double), ("tick_p99_ms", ctypes.c_double),
                ("committed_slots", ctypes.c_int64), ("overwritten_slots", ctypes.c_int64)]


def stream_run(cfg, seconds: float, *, weight_seed: int = 1, frame_rate: float = 30.0, camera_latency: int = 2,
               ae_rate: float = 480.0, trajectory_rate: float = 480.0, kv_policy: str = "most_recent",
               device: int = 0, prefix_sms: int = 0) -> dict:
    """The full-streaming runtime (include/pi0b.h pi0b_stream_run): `seconds` of camera frames and
    control ticks on one GPU, two engines over one weight arena (double-buffered KV).
    cfg.flow_steps = flow steps per tick; prefix_sms = SMs the ticks leave to the prefix (0: 20)."""
    o = StreamOptions(frame_rate, camera_latency, ae_rate, trajectory_rate,
                      {"most_recent": 0, "frame_sticky": 1}[kv_policy], device, prefix_sms)
    r = StreamReport()
    _raise(lib().pi0b_stream_run(ctypes.byref(cfg), weight_seed, ctypes.byref(o), seconds, ctypes.byref(r)),
           "stream_run")
    return {k: getattr(r, k) for k, _ in StreamReport._fields_}


EXPORTED_SYMBOLS = [
    "pi0b_default_config", "pi0b_engine_create", "pi0b_engine_destroy", "pi0b_engine_gen_weights",
    "pi0b_engine_set_weight", "pi0b_engine_set_bias_table", "pi0b_engine_run", "pi0b_engine_run_prefix",
    "pi0b_engine_run_action", "pi0b_engine_replay", "pi0b_engine_sync", "pi0b_engine_kernel_count",
    "pi0b_engine_read_checkpoint", "pi0b_engine_time_node", "pi0b_engine_describe", "pi0b_engine_ae_trace",
    "pi0b_last_error", "pi0b_gemm", "pi0b_gemm_skinny", "pi0b_attention",
    "pi0b_attention_ws_floats", "pi0b_random_f64", "pi0b_random_packed_bf16", "pi0b_seed_hash",
    "pi0b_engine_run_images", "pi0b_image_patches", "pi0b_stream_run", "pi0b_f64_to_bf16_host", "pi0b_rope_table_host",
    "pi0b_premultiply_rows", "pi0b_fold_time_mlp", "pi0b_time_embedding",
    "pi0b_engine_create_shared", "pi0b_engine_ve_buffers", "pi0b_engine_set_ve_peers", "pi0b_ipc_export", "pi0b_ipc_open", "pi0b_ipc_close",
]


def _raise(rc: int, what: str):
    if rc == 0:
        return
    msg = f"{what}: {lib().pi0b_last_error().decode()} (code {rc})"
    if rc == PI0B_E_UNSUPPORTED:
        raise UnsupportedConfig(msg)
    if rc == PI0B_E_INVALID:
        raise ShapeError(msg)
    if rc == PI0B_E_NUMERIC:
        raise NumericError(msg)
    raise RuntimeError(msg)


def _f64(a, shape) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if tuple(a.shape) != tuple(shape):
        raise ShapeError(f"expected shape {tuple(shape)}, got {tuple(a.shape)}")
    return a


def seed_hash(seed: int, label: str, a: int, b: int) -> int:
    return lib().pi0b_seed_hash(seed, label.encode(), a, b)


class Engine:
    """One pi0 engine on one B200 (weights, activations, KV cache, captured CUDA graphs)."""

    def __init__(self, cfg: ModelConfig, device: int = 0, use_cuda_graph: bool = True,
                 record_checkpoints: bool = False, ve_shards: int = 0, ve_shard: int = 0,
                 share_weights_with: "Engine | None" = None, ae_ctas: int = 0):
        """share_weights_with: read that engine's weight arena (include/pi0b.h
        pi0b_engine_create_shared); it must stay alive as long as this one."""
        self.cfg = cfg
        self._h = ctypes.c_void_p()
        self._donor = share_weights_with
        opt = EngineOptions(device, int(use_cuda_graph), int(record_checkpoints), ve_shards, ve_shard, ae_ctas)
        if share_weights_with is None:
            _raise(lib().pi0b_engine_create(ctypes.byref(cfg), ctypes.byref(opt), ctypes.byref(self._h)),
                   "pi0b_engine_create")
        else:
            _raise(lib().pi0b_engine_create_shared(ctypes.byref(cfg), ctypes.byref(opt), share_weights_with._h,
                                                   ctypes.byref(self._h)), "pi0b_engine_create_shared")

    def close(self):
        if self._h:
            lib().pi0b_engine_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # ---- weights
    def gen_weights(self, seed: int = 1) -> None:
        _raise(lib().pi0b_engine_gen_weights(self._h, seed), "gen_weights")

    def set_weight(self, node: str, inst: int, w: np.ndarray, bias: np.ndarray | None = None) -> None:
        w = np.ascontiguousarray(w, dtype=np.float64)
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float64)
        _raise(lib().pi0b_engine_set_weight(self._h, node.encode(), inst, w.ctypes.data_as(_dp), w.shape[0],
                                            w.shape[1], None if b is None else b.ctypes.data_as(_dp),
                                            0 if b is None else b.size), f"set_weight({node}[{inst}])")

    def set_bias_table(self, node: str, table: np.ndarray) -> None:
        t = np.ascontiguousarray(table, dtype=np.float64)
        _raise(lib().pi0b_engine_set_bias_table(self._h, node.encode(), t.ctypes.data_as(_dp), t.shape[0],
                                                t.shape[1]), "set_bias_table")

    # ---- inference
    def _inputs(self, patches=None, state=None, noise=None, prompt=None):
        c = self.cfg
        out = {}
        if patches is not None:
            out["patches"] = _f64(patches, (c.image_tokens, c.ve_patch_in))
        if state is not None:
            out["state"] = _f64(state, (1, c.ae_state_dim))
        if noise is not None:
            out["noise"] = _f64(noise, (c.chunk_len, c.ae_action_dim))
        if c.prompt_tokens > 0:
            if prompt is None and patches is not None:
                raise ShapeError("config has prompt tokens but no prompt was given")
            if prompt is not None:
                out["prompt"] = _f64(prompt, (c.prompt_tokens, c.llm_width))
        return out

    @staticmethod
    def _p(a):
        return None if a is None else a.ctypes.data_as(_dp)

    def run(self, patches, state, noise, prompt=None) -> np.ndarray:
        x = self._inputs(patches, state, noise, prompt)
        y = np.zeros((self.cfg.chunk_len, self.cfg.ae_action_dim), dtype=np.float64)
        _raise(lib().pi0b_engine_run(self._h, self._p(x["patches"]), self._p(x["state"]), self._p(x["noise"]),
                                     self._p(x.get("prompt")), self._p(y)), "run")
        return y

    def run_images(self, images, state, noise, prompt=None) -> np.ndarray:
        """run() from camera frames [views, height, width, 3] (any size >= 2x2): resize + img2col on
        the device (include/pi0b.h pi0b_engine_run_images)."""
        img = np.ascontiguousarray(images, dtype=np.float64)
        if img.ndim != 4 or img.shape[0] != self.cfg.views or img.shape[3] != 3:
            raise ShapeError(f"images must be [views={self.cfg.views}, h, w, 3], got {img.shape}")
        x = self._inputs(state=state, noise=noise, prompt=prompt)
        y = np.zeros((self.cfg.chunk_len, self.cfg.ae_action_dim), dtype=np.float64)
        _raise(lib().pi0b_engine_run_images(self._h, self._p(img), img.shape[1], img.shape[2], self._p(x["state"]),
                                            self._p(x["noise"]), self._p(x.get("prompt")), self._p(y)), "run_images")
        return y

    def run_prefix(self, patches, prompt=None) -> None:
        x = self._inputs(patches=patches, prompt=prompt)
        _raise(lib().pi0b_engine_run_prefix(self._h, self._p(x["patches"]), self._p(x.get("prompt"))),
               "run_prefix")

    def run_action(self, state, noise) -> np.ndarray:
        x = self._inputs(state=state, noise=noise)
        y = np.zeros((self.cfg.chunk_len, self.cfg.ae_action_dim), dtype=np.float64)
        _raise(lib().pi0b_engine_run_action(self._h, self._p(x["state"]), self._p(x["noise"]), self._p(y)),
               "run_action")
        return y

    # ---- view-sharded vision encoder (include/pi0b.h pi0b_ve_buffers)
    def ve_buffers(self) -> VeBuffers:
        b = VeBuffers()
        _raise(lib().pi0b_engine_ve_buffers(self._h, ctypes.byref(b)), "ve_buffers")
        return b

    def set_ve_peers(self, peers: list) -> None:
        """peers[i] = VeBuffers of shard i (this shard's own entry is ignored)."""
        arr = (VeBuffers * len(peers))(*peers)
        _raise(lib().pi0b_engine_set_ve_peers(self._h, arr, len(peers)), "set_ve_peers")

    def replay(self, part: int = 0, stream: int | None = None) -> None:
        _raise(lib().pi0b_engine_replay(self._h, part, stream), "replay")

    def sync(self) -> None:
        _raise(lib().pi0b_engine_sync(self._h), "sync")

    def kernel_count(self, part: int = 0) -> int:
        return lib().pi0b_engine_kernel_count(self._h, part)

    def time_node(self, node: str, reps: int = 5) -> tuple[float, int]:
        ms, n = ctypes.c_double(), ctypes.c_int()
        _raise(lib().pi0b_engine_time_node(self._h, node.encode(), reps, ctypes.byref(ms), ctypes.byref(n)),
               f"time_node({node})")
        return ms.value, n.value

    def describe(self) -> list[str]:
        buf = ctypes.create_string_buffer(1 << 20)
        _raise(lib().pi0b_engine_describe(self._h, buf, len(buf)), "describe")
        return buf.value.decode().splitlines()

    def checkpoint(self, node: str, inst: int, rows: int, cols: int) -> np.ndarray:
        out = np.zeros((rows, cols), dtype=np.float32)
        _raise(lib().pi0b_engine_read_checkpoint(self._h, node.encode(), inst,
                                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), rows, cols),
               f"checkpoint {node}[{inst}]")
        return out


def ipc_export(dptr: int) -> bytes:
    """64-byte CUDA IPC handle of a device allocation (cudaIpcGetMemHandle)."""
    buf = ctypes.create_string_buffer(64)
    _raise(lib().pi0b_ipc_export(dptr, buf), "ipc_export")
    return buf.raw


def ipc_open(handle: bytes) -> int:
    """Map another process's allocation into this one (cudaIpcOpenMemHandle); returns the pointer."""
    p = ctypes.c_void_p()
    _raise(lib().pi0b_ipc_open(handle, ctypes.byref(p)), "ipc_open")
    return p.value


def ipc_close(dptr: int) -> None:
    _raise(lib().pi0b_ipc_close(dptr), "ipc_close")


def evaluate(cfg: ModelConfig, weight_seed: int, inputs: dict) -> np.ndarray:
    """Drop-in for rtvla::evaluate(build_pi0_graph(cfg), gen_weights(g, seed), x)."""
    eng = Engine(cfg)
    try:
        eng.gen_weights(weight_seed)
        return eng.run(inputs["patches"], inputs["state"], inputs["noise"], inputs.get("prompt"))
    finally:
        eng.close()


# ---------------------------------------------------------------- kernel-level helpers (tests)

def gemm(desc: GemmDesc, stream: int | None = None) -> None:
    _raise(lib().pi0b_gemm(ctypes.byref(desc), stream), "pi0b_gemm")


def gemm_skinny(desc: GemmDesc, cluster: int = 1, stream: int | None = None) -> None:
    _raise(lib().pi0b_gemm_skinny(ctypes.byref(desc), cluster, stream), "pi0b_gemm_skinny")


def attention(desc: AttnDesc, stream: int | None = None) -> None:
    _raise(lib().pi0b_attention(ctypes.byref(desc), stream), "pi0b_attention")


def attention_ws_floats(desc: AttnDesc) -> int:
    return lib().pi0b_attention_ws_floats(ctypes.byref(desc))


def random_f64(ptr: int, n: int, seed: int, lo: float, hi: float, stream: int | None = None) -> None:
    _raise(lib().pi0b_random_f64(ptr, n, seed, lo, hi, stream), "pi0b_random_f64")


PERM_NONE, PERM_GATE128, PERM_GATE64, PERM_ROPE = 0, 1, 2, 3


def random_packed_bf16(ptr: int, ldk: int, k: int, m: int, perm: int, seed: int, lo: float, hi: float,
                       rope_cols: int = 0, stream: int | None = None) -> None:
    _raise(lib().pi0b_random_packed_bf16(ptr, ldk, k, m, perm, rope_cols, seed, lo, hi, stream),
           "random_packed_bf16")
