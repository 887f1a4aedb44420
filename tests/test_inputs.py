"""Host gen_inputs / seed_hash of the package are bit-identical to the reference's."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2510_26742_b200.config import default_config, mid_config, tiny_config
from paper_2510_26742_b200.inputs import gen_inputs, seed_hash


@pytest.mark.parametrize("cfg", [tiny_config(), mid_config(3, 32), default_config(2)], ids=["tiny", "mid", "full2v"])
def test_gen_inputs_bitwise(cfg):
    a = gen_inputs(cfg, 1)
    b = O.gen_inputs(cfg, 1, use_reference=O.ref_available())
    assert set(a) == {k for k in b if k != "prompt" or cfg.prompt_tokens > 0}
    for k in a:
        assert np.array_equal(a[k], b[k]), k


def test_seed_hash():
    if not O.ref_available():
        pytest.skip("reference not built")
    for args in [(1, "ve.qkv", 3, 1), (0, "", 0, 0), (2**64 - 1, "ae.action_proj", 9, 4)]:
        assert seed_hash(*args) == O.ref_lib().ref_seed_hash(args[0], args[1].encode(), args[2], args[3])
