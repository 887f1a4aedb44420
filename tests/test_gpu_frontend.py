"""the GPU image front-end (camera frames -> resize -> img2col -> ve.embed patches).

* pi0b_image_patches (device op) is bit-identical to the reference's rtvla::bilinear_resize
  (proj/src/tensor.cpp:180-212, compiled unmodified in oracle/_ref) followed by this engine's
  documented patch flattening, for down-, up- and same-size resizes;
* Engine.run_images(frames) equals Engine.run(patches of those frames).
"""
import ctypes

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2510_26742_b200 import engine as E
from paper_2510_26742_b200.config import mid_config

pytestmark = pytest.mark.gpu

SIDE, P, C = 224, 14, 3


def _ref_patches(frames):
    """reference resize per view + img2col: row view*256 + (y/14)*16 + x/14, col ((y%14)*14 + x%14)*3 + c"""
    lib = O.ref_lib()
    views, h, w, _ = frames.shape
    out = []
    for v in range(views):
        img = np.ascontiguousarray(frames[v].reshape(h, w * C))
        r = np.zeros((SIDE, SIDE * C))
        assert lib.ref_bilinear_resize(img.ctypes.data_as(O._dp), h, w, C, SIDE, SIDE, r.ctypes.data_as(O._dp)) == 0
        g = SIDE // P
        r = r.reshape(g, P, g, P, C).transpose(0, 2, 1, 3, 4).reshape(g * g, P * P * C)
        out.append(r)
    return np.concatenate(out, 0)


@pytest.mark.parametrize("views,h,w", [(2, 300, 400), (1, 224, 224), (3, 100, 150), (1, 2, 2), (2, 480, 640)])
def test_image_patches_bitexact(views, h, w):
    if not O.ref_available():
        pytest.skip("compiled reference not available")
    rng = np.random.default_rng(h * 1000 + w)
    frames = rng.uniform(-1, 1, size=(views, h, w, C))
    d_img = torch.from_numpy(frames).cuda()
    d_out = torch.zeros(views * (SIDE // P) ** 2, P * P * C, dtype=torch.float64, device="cuda")
    rc = E.lib().pi0b_image_patches(ctypes.c_void_p(d_img.data_ptr()), views, h, w, C, SIDE, P,
                                    ctypes.c_void_p(d_out.data_ptr()), None)
    assert rc == 0
    torch.cuda.synchronize()
    got = d_out.cpu().numpy()
    ref = _ref_patches(frames)
    assert np.array_equal(got, ref), float(np.abs(got - ref).max())


def test_engine_run_images():
    cfg = mid_config(views=2)
    x = O.gen_inputs(cfg, 1)
    rng = np.random.default_rng(5)
    frames = rng.uniform(-1, 1, size=(2, 360, 480, C))
    eng = E.Engine(cfg)
    eng.gen_weights(1)
    a = eng.run_images(frames, x["state"], x["noise"])
    if O.ref_available():
        patches = _ref_patches(frames)
    else:  # the device op itself
        d_img = torch.from_numpy(frames).cuda()
        d_out = torch.zeros(512, P * P * C, dtype=torch.float64, device="cuda")
        E.lib().pi0b_image_patches(ctypes.c_void_p(d_img.data_ptr()), 2, 360, 480, C, SIDE, P,
                                   ctypes.c_void_p(d_out.data_ptr()), None)
        patches = d_out.cpu().numpy()
    b = eng.run(patches, x["state"], x["noise"])
    assert np.isfinite(a).all()
    assert np.abs(a - b).max() < 0.02  # run-to-run (fp32 atomics ordering), same patches
