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
