"""CPU checks of the C-ABI boundary: libpi0b.so loads without a GPU and exports every
function include/pi0b.h declares; the Python mirror of pi0b_model_config matches the
header and the reference's presets."""
import ctypes
import os
import re

import pytest

from paper_2510_26742_b200 import config as C
from paper_2510_26742_b200 import engine as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pi0b.h")


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pi0b_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = E.lib()
    declared = _declared_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), f"libpi0b.so does not export {name}"
    assert sorted(E.EXPORTED_SYMBOLS) == declared


def test_config_struct_matches_header():
    text = open(HEADER).read()
    body = text[text.index("typedef struct pi0b_model_config"):text.index("} pi0b_model_config;")]
    fields = re.findall(r"\b([a-z_][a-z0-9_]*)\s*[,;]", body.split("{", 1)[1])
    assert fields == C.FIELDS
    assert ctypes.sizeof(C.ModelConfig) == 4 * len(C.FIELDS)


def test_default_config_matches_library_and_reference():
    c = C.ModelConfig()
    E.lib().pi0b_default_config(ctypes.byref(c))
    assert c.as_dict() == C.default_config().as_dict()
    from oracle import oracle as O
    if O.ref_available():
        r = C.ModelConfig()
        O.ref_lib().ref_default_config(ctypes.byref(r))
        assert r.as_dict() == C.default_config().as_dict()
        t = C.ModelConfig()
        O.ref_lib().ref_tiny_config(ctypes.byref(t))
        assert t.as_dict() == C.tiny_config().as_dict()


def test_seed_hash_matches_reference():
    from oracle import oracle as O
    if not O.ref_available():
        pytest.skip("reference not built")
    for label, a, b in [("ve.qkv", 3, 1), ("ae.action_proj", 9, 4), ("patches", 0, 5)]:
        assert E.seed_hash(1, label, a, b) == O.ref_lib().ref_seed_hash(1, label.encode(), a, b)


def test_engine_create_fails_loudly_without_gpu():
    """No CPU fallback: on a box without an sm_100 device, creation raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        E.Engine(C.mid_config())



def test_cpp_dropin_fails_loudly_without_gpu():
    """The C++ drop-in (include/pi0b_rtvla.hpp) over the reference's types builds and, with no
    sm_100 device, throws instead of falling back to the CPU."""
    import subprocess
    demo = os.path.join(ROOT, "oracle", "_ref", "pi0b_rtvla_demo")
    if not os.path.exists(demo):
        pytest.skip("demo not built (needs /root/reference)")
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present: covered by tests/test_gpu_engine.py::test_rtvla_cpp_dropin")
    except ImportError:
        pass
    r = subprocess.run([demo, "1", "0"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 2 and "pi0b error" in r.stdout, r.stdout + r.stderr


def _bf16_of_f32_rne(x64):
    """numpy restatement of bf16(float(x)): fp64 -> fp32 round-to-nearest-even (numpy's cast),
    then fp32 -> bf16 round-to-nearest-even on the bit pattern, NaN -> 0x7fff (cvt.rn.bf16.f32)."""
    import numpy as np
    u = x64.astype(np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r[nan] = 0x7FFF
    return r


def test_host_patch_conversion_matches_device_rounding():
    """pi0b_f64_to_bf16_host (the conversion run() applies to the patches before their DMA) is
    bf16(float(x)) with round-to-nearest-even at both steps: ties, values that round differently
    via fp32 than directly, subnormals, infinities and NaN."""
    import numpy as np
    rng = np.random.default_rng(5)
    x = np.concatenate([
        rng.normal(size=20000), rng.uniform(-1, 1, 20000) * 1e-40, rng.normal(size=2000) * 1e30,
        # exact bf16 ties (odd and even lower halves) and ties broken only by the fp64 tail
        np.array([1.0 + 2.0 ** -8, 1.0 + 3 * 2.0 ** -8, 1.0 + 2.0 ** -8 + 2.0 ** -40, -(1.0 + 2.0 ** -8 - 2.0 ** -40),
                  3.3895313892515355e38, 3.4e38, 1e39, -1e39, 0.0, -0.0, np.inf, -np.inf, np.nan, 1e-46]),
    ])
    out = np.empty(x.size, dtype=np.uint16)
    rc = E.lib().pi0b_f64_to_bf16_host(x.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), x.size,
                                       out.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0
    with np.errstate(over="ignore"):
        ref = _bf16_of_f32_rne(x)
    assert np.array_equal(out, ref)


def test_rope_table_bitexact_vs_reference():
    """The engine's RoPE table (pi0b_rope_table_host: what Engine uploads) is the reference's
    make_rope_table (proj/src/tensor.cpp:133-148) rounded once to fp32, bit for bit, over every
    position an engine uses (prefix rows and the action expert's L..L+63)."""
    import numpy as np
    from oracle import oracle as O
    npos, d = 1400, 256
    got = np.zeros(npos * d, dtype=np.float32)
    assert E.lib().pi0b_rope_table_host(npos, d, got.ctypes.data_as(ctypes.POINTER(ctypes.c_float))) == 0
    got = got.reshape(npos, d // 2, 2)
    c = np.zeros(npos * d // 2)
    s = np.zeros(npos * d // 2)
    O.ref_lib().ref_rope_table(npos, d, c.ctypes.data_as(O._dp), s.ctypes.data_as(O._dp))
    assert np.array_equal(got[:, :, 0].view(np.uint32), c.reshape(npos, d // 2).astype(np.float32).view(np.uint32))
    assert np.array_equal(got[:, :, 1].view(np.uint32), s.reshape(npos, d // 2).astype(np.float32).view(np.uint32))
