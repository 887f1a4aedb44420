"""Host side of the C++ drop-in (include/pi0b_rtvla.hpp) without a GPU — SURVEY 8(f) f1 and 8(a)
a17: pi0b::fuse_naive turns the reference's naive graph + WeightStore into the fused graph's
weights with the ENGINE's own weight rules (libpi0b host code, csrc/naive.cu: PremultiplyDiag,
ConcatCols, ComposeTimeFold + time_embedding).  oracle/naive_fuse_check.cpp compares every fused
weight instance, bias and the bias table BITWISE with the reference's rtvla::pass_registry +
rtvla::apply_weight_rules (proj/src/passes.cpp:665-790), and the fp64 forward on them with the
naive graph's (reference tolerance 1e-9).  time_embedding is pinned bitwise to the reference's."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK = os.path.join(ROOT, "oracle", "_ref", "naive_fuse_check")
have_ref = pytest.mark.skipif(not os.path.exists(CHECK), reason="reference not built here")


@have_ref
@pytest.mark.parametrize("cfg,views,prompt", [("tiny", 1, 0), ("tiny", 2, 0), ("tiny", 3, 32), ("mid", 1, 0),
                                              ("mid", 3, 32)])
def test_naive_weight_rules_bitwise(cfg, views, prompt):
    r = subprocess.run([CHECK, cfg, str(views), str(prompt)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert " 0 differ" in r.stdout


def _libs():
    from oracle import oracle as O
    from paper_2510_26742_b200 import engine as E
    return E.lib(), O.ref_lib()


@have_ref
def test_time_embedding_bitwise():
    lib, ref = _libs()
    dp = ctypes.POINTER(ctypes.c_double)
    lib.pi0b_time_embedding.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, dp]
    for dim, fs in [(2, 1), (8, 3), (64, 10), (256, 10), (1024, 50)]:
        for s in range(fs + 1):
            a = np.zeros(dim)
            b = np.zeros(dim)
            assert lib.pi0b_time_embedding(s, dim, fs, a.ctypes.data_as(dp)) == 0
            ref.ref_time_embedding(s, dim, fs, b.ctypes.data_as(dp))
            assert np.array_equal(a, b), (dim, fs, s)
    assert lib.pi0b_time_embedding(0, 7, 10, np.zeros(7).ctypes.data_as(dp)) < 0  # odd dim: ShapeError


def test_premultiply_rows():
    from paper_2510_26742_b200 import engine as E
    lib = E.lib()
    dp = ctypes.POINTER(ctypes.c_double)
    lib.pi0b_premultiply_rows.argtypes = [dp, ctypes.c_int64, ctypes.c_int64, dp]
    rng = np.random.default_rng(3)
    w = rng.uniform(-1, 1, (5, 7))
    g = 1.0 + rng.uniform(-0.25, 0.25, 5)
    want = w * g[:, None]
    assert lib.pi0b_premultiply_rows(w.ctypes.data_as(dp), 5, 7, g.ctypes.data_as(dp)) == 0
    assert np.array_equal(w, want)
