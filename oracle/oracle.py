"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module.  It loads two CPU libraries:

* ``oracle/_ref/librtvla_ref.so`` — the UNMODIFIED reference (``/root/reference/proj/src``
  tensor/graph/builder/evaluate/passes) compiled by ``oracle/Makefile`` plus an ``extern "C"``
  shim (``oracle/ref_shim.cpp``).  This is ``rtvla::evaluate`` itself.
* ``oracle/_build/libpi0_oracle.so`` — ``oracle/pi0_oracle.cpp``, a threaded fp64 restatement
  of the same forward that is bitwise identical to the reference (asserted by
  ``tests/test_oracle.py``) and fast enough for full-scale hidden-state dumps.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from paper_2510_26742_b200.config import ModelConfig

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "librtvla_ref.so")
PORT_LIB = os.path.join(HERE, "_build", "libpi0_oracle.so")
REFERENCE_SRC = "/root/reference/proj"

_dp = ctypes.POINTER(ctypes.c_double)
_ref = None
_port = None


def build(quiet: bool = True) -> None:
    """Compile the oracle libraries (reference leg only where /root/reference exists)."""
    targets = ["port"]
    if os.path.isdir(REFERENCE_SRC):
        targets.append("ref")
        # the reference's stream simulator + driver (scripts/streamsim_b200.py)
        targets.append("streamsim")
        targets.append("naive")
        targets.append("analyze")
        # the C++ drop-in demo (include/pi0b_rtvla.hpp over libpi0b.so, reference types)
        if os.path.exists(os.path.join(os.path.dirname(HERE), "paper_2510_26742_b200", "libpi0b.so")):
            targets.append("demo")
    out = subprocess.run(["make", "-C", HERE, "-j8", *targets], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + out.stdout[-4000:] + out.stderr[-4000:])


def _ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            raise FileNotFoundError(f"{REF_LIB} missing: run `make -C oracle ref` where /root/reference exists")
        lib = ctypes.CDLL(REF_LIB)
        cfgp = ctypes.POINTER(ModelConfig)
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_default_config.argtypes = [cfgp]
        lib.ref_tiny_config.argtypes = [cfgp]
        lib.ref_count_gemm_instances.argtypes = [cfgp]
        lib.ref_count_gemm_instances.restype = ctypes.c_int64
        lib.ref_graph_listing.argtypes = [cfgp, ctypes.c_char_p, ctypes.c_int64]
        lib.ref_gen_inputs.argtypes = [cfgp, ctypes.c_uint64, _dp, _dp, _dp, _dp]
        lib.ref_gen_node_weight.argtypes = [cfgp, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int64, _dp, _dp, _dp]
        lib.ref_evaluate.argtypes = [cfgp, ctypes.c_uint64, ctypes.c_uint64, _dp]
        lib.ref_evaluate_node.argtypes = [cfgp, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int64,
                                          _dp, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                                          ctypes.POINTER(ctypes.c_int64)]
        lib.ref_seed_hash.argtypes = [ctypes.c_uint64, ctypes.c_char_p, ctypes.c_uint64, ctypes.c_uint64]
        lib.ref_seed_hash.restype = ctypes.c_uint64
        lib.ref_rng_stream.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.POINTER(ctypes.c_uint64)]
        lib.ref_random_tensor.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, ctypes.c_double,
                                          ctypes.c_uint64, _dp]
        lib.ref_gelu.argtypes = [ctypes.c_double]
        lib.ref_gelu.restype = ctypes.c_double
        lib.ref_silu.argtypes = [ctypes.c_double]
        lib.ref_silu.restype = ctypes.c_double
        lib.ref_matmul.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, _dp, ctypes.c_int64, _dp]
        lib.ref_rms_scales.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double, _dp]
        lib.ref_softmax_rows.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, _dp]
        lib.ref_bilinear_resize.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
        lib.ref_rope.argtypes = [_dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _dp]
        lib.ref_rope_table.argtypes = [ctypes.c_int, ctypes.c_int, _dp, _dp]
        lib.ref_time_embedding.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _dp]
        lib.ref_max_rel_deviation.argtypes = [_dp, _dp, ctypes.c_int64]
        lib.ref_max_rel_deviation.restype = ctypes.c_double
        lib.ref_ctx_create.argtypes = [cfgp, ctypes.c_uint64, ctypes.c_uint64]
        lib.ref_ctx_create.restype = ctypes.c_void_p
        lib.ref_ctx_evaluate.argtypes = [ctypes.c_void_p, _dp]
        lib.ref_ctx_destroy.argtypes = [ctypes.c_void_p]
        _ref = lib
    return _ref


def port_lib():
    global _port
    if _port is None:
        if not os.path.exists(PORT_LIB):
            build()
        lib = ctypes.CDLL(PORT_LIB)
        cfgp = ctypes.POINTER(ModelConfig)
        lib.orc_last_error.restype = ctypes.c_char_p
        lib.orc_gen_inputs.argtypes = [cfgp, ctypes.c_uint64, _dp, _dp, _dp, _dp]
        lib.orc_forward.argtypes = [cfgp, ctypes.c_uint64, _dp, _dp, _dp, _dp, _dp, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(_dp), ctypes.POINTER(ctypes.c_int64)]
        lib.orc_weight.argtypes = [ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                   _dp, _dp]
        _port = lib
    return _port


def _check(rc: int, lib, which: str) -> None:
    if rc != 0:
        err = (lib.ref_last_error() if which == "ref" else lib.orc_last_error()).decode()
        raise RuntimeError(f"{which} oracle failed: {err}")


# ------------------------------------------------------------------ inputs / shapes

def input_shapes(cfg: ModelConfig) -> dict:
    return {
        "patches": (cfg.image_tokens, cfg.ve_patch_in),
        "state": (1, cfg.ae_state_dim),
        "noise": (cfg.chunk_len, cfg.ae_action_dim),
        "prompt": (cfg.prompt_tokens, cfg.llm_width),
    }


def gen_inputs(cfg: ModelConfig, seed: int = 1, use_reference: bool = False) -> dict:
    """rtvla::gen_inputs(build_pi0_graph(cfg), seed) as fp64 arrays."""
    sh = input_shapes(cfg)
    out = {k: np.zeros(v, dtype=np.float64) for k, v in sh.items()}
    pr = out["prompt"] if cfg.prompt_tokens > 0 else None
    if use_reference:
        lib = ref_lib()
        _check(lib.ref_gen_inputs(ctypes.byref(cfg), seed, _ptr(out["patches"]), _ptr(out["state"]),
                                  _ptr(out["noise"]), _ptr(pr)), lib, "ref")
    else:
        lib = port_lib()
        _check(lib.orc_gen_inputs(ctypes.byref(cfg), seed, _ptr(out["patches"]), _ptr(out["state"]),
                                  _ptr(out["noise"]), _ptr(pr)), lib, "port")
    return out


# ------------------------------------------------------------------ reference calls

def ref_evaluate(cfg: ModelConfig, wseed: int = 1, iseed: int = 1) -> np.ndarray:
    lib = ref_lib()
    out = np.zeros((cfg.chunk_len, cfg.ae_action_dim), dtype=np.float64)
    _check(lib.ref_evaluate(ctypes.byref(cfg), wseed, iseed, _ptr(out)), lib, "ref")
    return out


class RefContext:
    """build_pi0_graph + gen_weights + gen_inputs once; evaluate() alone is what a
    bench step times (the reference's own inference call, proj/src/evaluate.cpp:365-370)."""

    def __init__(self, cfg: ModelConfig, wseed: int = 1, iseed: int = 1):
        self.cfg = cfg
        self.lib = ref_lib()
        self.h = self.lib.ref_ctx_create(ctypes.byref(cfg), wseed, iseed)
        if not self.h:
            raise RuntimeError("ref_ctx_create: " + self.lib.ref_last_error().decode())

    def evaluate(self) -> np.ndarray:
        out = np.zeros((self.cfg.chunk_len, self.cfg.ae_action_dim), dtype=np.float64)
        _check(self.lib.ref_ctx_evaluate(self.h, _ptr(out)), self.lib, "ref")
        return out

    def close(self):
        if self.h:
            self.lib.ref_ctx_destroy(self.h)
            self.h = None


def ref_node(cfg: ModelConfig, node: str, inst: int, wseed: int = 1, iseed: int = 1,
             max_elems: int = 1 << 24) -> np.ndarray:
    lib = ref_lib()
    buf = np.zeros(max_elems, dtype=np.float64)
    r, c = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.ref_evaluate_node(ctypes.byref(cfg), wseed, iseed, node.encode(), inst, _ptr(buf), max_elems,
                                 ctypes.byref(r), ctypes.byref(c)), lib, "ref")
    return buf[: r.value * c.value].reshape(r.value, c.value).copy()


def ref_node_weight(cfg: ModelConfig, node: str, inst: int, k: int, m: int, seed: int = 1,
                    bias: bool = False, table_rows: int = 0):
    lib = ref_lib()
    w = np.zeros((k, m), dtype=np.float64)
    b = np.zeros(m, dtype=np.float64) if bias else None
    t = np.zeros((table_rows, m), dtype=np.float64) if table_rows else None
    _check(lib.ref_gen_node_weight(ctypes.byref(cfg), seed, node.encode(), inst, _ptr(w), _ptr(b), _ptr(t)),
           lib, "ref")
    return w, b, t


def ref_graph_listing(cfg: ModelConfig) -> list[tuple]:
    lib = ref_lib()
    buf = ctypes.create_string_buffer(1 << 16)
    _check(lib.ref_graph_listing(ctypes.byref(cfg), buf, len(buf)), lib, "ref")
    rows = []
    for line in buf.value.decode().strip().splitlines():
        nid, kind, rep, n, k, m = line.split()
        rows.append((nid, kind, int(rep), int(n), int(k), int(m)))
    return rows


# ------------------------------------------------------------------ restatement calls

def port_forward(cfg: ModelConfig, inputs: dict, wseed: int = 1, threads: int = 0,
                 record: list[tuple[str, int, tuple]] | None = None):
    """Full forward; `record` = [(node, inst, shape)] -> returns (actions, {(node, inst): array})."""
    lib = port_lib()
    out = np.zeros((cfg.chunk_len, cfg.ae_action_dim), dtype=np.float64)
    record = record or []
    bufs = [np.zeros(shape, dtype=np.float64) for (_, _, shape) in record]
    n = len(record)
    names = (ctypes.c_char_p * max(n, 1))(*[r[0].encode() for r in record])
    insts = (ctypes.c_int64 * max(n, 1))(*[r[1] for r in record])
    ptrs = (_dp * max(n, 1))(*[_ptr(b) for b in bufs])
    caps = (ctypes.c_int64 * max(n, 1))(*[b.size for b in bufs])
    pr = inputs.get("prompt") if cfg.prompt_tokens > 0 else None
    _check(lib.orc_forward(ctypes.byref(cfg), wseed, _ptr(inputs["patches"]), _ptr(inputs["state"]),
                           _ptr(inputs["noise"]), _ptr(pr), _ptr(out), threads, n, names, insts, ptrs, caps),
           lib, "port")
    return out, {(r[0], r[1]): b for r, b in zip(record, bufs)}


def port_weight(node: str, inst: int, k: int, m: int, seed: int = 1, bias: bool = False):
    lib = port_lib()
    w = np.zeros((k, m), dtype=np.float64)
    b = np.zeros(m, dtype=np.float64) if bias else None
    _check(lib.orc_weight(seed, node.encode(), inst, k, m, _ptr(w), _ptr(b)), lib, "port")
    return w, b
