"""Pins of the oracle's a5 (gather + bilinear resize, reading R15/R16) against
closed forms, torch's bilinear interpolate at dyadic ratios (where torch's
float source coordinate is exact), and hand-derived taps."""
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as Fn

import oracle as O


def _gold():
    here = os.path.dirname(os.path.abspath(__file__))
    return json.load(open(os.path.join(here, "golden", "resize_remap_nms_golden.json")))


@pytest.mark.parametrize("case", _gold()["taps"], ids=lambda c: c["name"])
def test_taps_golden(case):
    got = [O.taps(case["in"], case["out"], d) for d in range(case["out"])]
    for (i0, i1, lam), (e0, e1, el) in zip(got, case["expect"]):
        assert (i0, i1) == (e0, e1)
        assert lam == pytest.approx(el, abs=1e-15)


def _frame_from_image(img):
    """img uint8 [h][w][3] -> frame [h][pitch] with pitch = 3w rounded to 16."""
    h, w, _ = img.shape
    pitch = (3 * w + 15) // 16 * 16
    fr = np.zeros((h, pitch), np.uint8)
    fr[:, : 3 * w] = img.reshape(h, 3 * w)
    return fr, pitch


def _resize_one(img, ow, oh, fmt=O.F64_NCHW, x=0, y=0, cw=None, chh=None):
    """Resize the crop (x, y, cw, chh) of img (uint8 HWC) to (ow, oh) with the oracle."""
    H, W, _ = img.shape
    cw = W if cw is None else cw
    chh = H if chh is None else chh
    fr, pitch = _frame_from_image(img)
    win = np.array([[0, x, y, cw, chh, 0, 0]], np.int32)
    st, outs = O.gather_resize([fr], pitch, W, H, win, [(cw, chh)], [(ow, oh)], [1], fmt)
    assert st == 0
    return outs[0][0]


def test_resize_ramp_and_2x2_means_golden():
    g = {c["name"]: c for c in _gold()["resize"]}
    row = np.array(g["G5c_ramp_in4_out3"]["row"], np.uint8)
    img = np.repeat(np.repeat(row[None, :, None], 3, axis=2), 2, axis=0)     # 2 x 4 x 3
    out = _resize_one(img, 3, 2)
    assert np.allclose(out[0, 0], g["G5c_ramp_in4_out3"]["expect"], atol=1e-12)
    n = g["G5d_2x2_means"]["image_10y_plus_x"]
    yy, xx = np.mgrid[0:n, 0:n]
    img = np.repeat((10 * yy + xx).astype(np.uint8)[:, :, None], 3, axis=2)
    out = _resize_one(img, 2, 2)
    assert np.allclose(out[1], g["G5d_2x2_means"]["expect"], atol=1e-12)


def test_scale_one_is_exact_copy():
    rng = np.random.default_rng(0)
    img = rng.integers(0, 256, (50, 70, 3), dtype=np.uint8)
    out = _resize_one(img, 30, 20, O.F32_NCHW, x=16, y=7, cw=30, chh=20)
    assert np.array_equal(out.transpose(1, 2, 0), img[7:27, 16:46].astype(np.float32))
    out8 = _resize_one(img, 30, 20, O.U8_NHWC, x=16, y=7, cw=30, chh=20)
    assert np.array_equal(out8, img[7:27, 16:46])


def test_exact_2x_downscale_is_block_mean():
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, (64, 96, 3), dtype=np.uint8)
    out = _resize_one(img, 48, 32)
    ref = img.astype(np.float64).reshape(32, 2, 48, 2, 3).mean(axis=(1, 3)).transpose(2, 0, 1)
    assert np.allclose(out, ref, atol=1e-12)


@pytest.mark.parametrize("src,dst", [((256, 256), (128, 128)), ((256, 256), (512, 512)),
                                     ((96, 64), (48, 32)), ((40, 24), (160, 96)), ((64, 64), (128, 32))])
def test_dyadic_ratios_match_torch_bilinear(src, dst):
    """At power-of-two ratios torch's float source coordinate (d+.5)*in/out-.5
    is exact, so F.interpolate(bilinear, align_corners=False) must agree."""
    rng = np.random.default_rng(2)
    w, h = src
    ow, oh = dst
    img = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    out = _resize_one(img, ow, oh)
    t = torch.from_numpy(img.astype(np.float64)).permute(2, 0, 1)[None]
    ref = Fn.interpolate(t, size=(oh, ow), mode="bilinear", align_corners=False)[0].numpy()
    assert np.abs(out - ref).max() < 1e-9


def test_non_dyadic_close_to_torch():
    """Sanity only: torch's float scale differs by a few 1e-3 at non-dyadic ratios."""
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (256, 256, 3), dtype=np.uint8)
    out = _resize_one(img, 192, 192)
    t = torch.from_numpy(img.astype(np.float64)).permute(2, 0, 1)[None]
    ref = Fn.interpolate(t, size=(192, 192), mode="bilinear", align_corners=False)[0].numpy()
    assert np.abs(out - ref).max() < 0.05


def test_constant_image_constant_output():
    img = np.full((45, 37, 3), (17, 200, 93), np.uint8)
    out = _resize_one(img, 29, 61)
    for c, v in enumerate((17, 200, 93)):
        assert np.abs(out[c] - v).max() < 1e-12


def test_affine_ramp_reproduced_at_interior_taps():
    """p(x,y) = 2x + 3y + 5 (channel 0); for taps not clamped the result is
    p at the source coordinate ((d+1/2) in/out - 1/2)."""
    h, w, oh, ow = 40, 60, 25, 45
    yy, xx = np.mgrid[0:h, 0:w]
    img = np.zeros((h, w, 3), np.uint8)
    img[..., 0] = (2 * xx + 3 * yy + 5) % 256
    assert img[..., 0].max() == 2 * 59 + 3 * 39 + 5
    out = _resize_one(img, ow, oh)
    for oy in range(oh):
        sy = (oy + 0.5) * h / oh - 0.5
        for ox in range(ow):
            sx = (ox + 0.5) * w / ow - 0.5
            if 0 <= sx <= w - 1 and 0 <= sy <= h - 1:
                assert out[0, oy, ox] == pytest.approx(2 * sx + 3 * sy + 5, abs=1e-9)


def test_u8_round_half_up_and_window_offset():
    """u8 output = floor(v + 0.5) of the f64 value (R16), and the crop origin
    is the window's (x, y)."""
    rng = np.random.default_rng(4)
    img = rng.integers(0, 256, (80, 120, 3), dtype=np.uint8)
    f64 = _resize_one(img, 33, 21, O.F64_NCHW, x=48, y=10, cw=50, chh=40)
    u8 = _resize_one(img, 33, 21, O.U8_NHWC, x=48, y=10, cw=50, chh=40)
    assert np.array_equal(u8, np.floor(f64 + 0.5).astype(np.uint8).transpose(1, 2, 0))
    crop = np.ascontiguousarray(img[10:50, 48:98])
    f64b = _resize_one(crop, 33, 21)
    assert np.array_equal(f64, f64b)


def test_gather_validation_and_capacity():
    rng = np.random.default_rng(5)
    img = rng.integers(0, 256, (64, 64, 3), dtype=np.uint8)
    fr, pitch = _frame_from_image(img)
    bad = np.array([[0, 40, 0, 32, 32, 0, 0]], np.int32)        # outside the frame
    st, _ = O.gather_resize([fr], pitch, 64, 64, bad, [(32, 32)], [(16, 16)], [1])
    assert st == O.ERR_INVALID
    over = np.array([[0, 0, 0, 32, 32, 0, 1]], np.int32)        # slot 1 >= cap 1
    st, _ = O.gather_resize([fr], pitch, 64, 64, over, [(32, 32)], [(16, 16)], [1])
    assert st == O.ERR_CAPACITY
