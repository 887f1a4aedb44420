"""Host side of the C++ drop-in (include/pi0b_rtvla.hpp) without a GPU: pi0b::fuse turns the
reference's naive graph + WeightStore into the fused graph + weights with the reference's own
passes and weight rules; the result is isomorphic to rtvla::build_pi0_graph and evaluates to the
naive graph's fp64 output within the reference's 1e-9 (oracle/naive_fuse_check.cpp)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECK = os.path.join(ROOT, "oracle", "_ref", "naive_fuse_check")


@pytest.mark.skipif(not os.path.exists(CHECK), reason="reference not built here")
@pytest.mark.parametrize("views,prompt", [(1, 0), (2, 0), (3, 32)])
def test_naive_graph_fuse(views, prompt):
    r = subprocess.run([CHECK, str(views), str(prompt)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
