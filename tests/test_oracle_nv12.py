"""Pins of the oracle's NEXT-3 path (NV12 input, reading R23): the colour
conversion against published colour-bar codes, the chroma siting against
direct indexing at identity scale, and the NV12 resampler against the
(independently pinned) RGB resampler of test_oracle_resize.py applied to the
same image upsampled to 4:4:4."""
import json
import os

import numpy as np
import pytest

import oracle as O
from workloads import synth as S

MATRICES = {"bt709_limited": O.BT709_LIMITED, "bt601_limited": O.BT601_LIMITED}


def _bars():
    here = os.path.dirname(os.path.abspath(__file__))
    return json.load(open(os.path.join(here, "golden", "colour_bars.json")))


@pytest.mark.parametrize("std", sorted(MATRICES))
def test_colour_bars(std):
    # each published code is an integer: |dY|,|dCb|,|dCr| <= 0.5 moves R'G'B'
    # by at most 0.5*255/219 + 0.5*255/224*(2(1-Kr) or 2(1-Kb)) < 1.7 (8-bit);
    # a swapped U/V, a wrong Kr/Kb pair or a wrong offset is off by >= 15.
    for name, (yuv, rgb) in _bars()[std].items():
        got = O.yuv_to_rgb(*yuv, MATRICES[std])
        assert np.abs(got - np.asarray(rgb, float)).max() <= 2.0, (std, name, got)


def test_conversion_special_values():
    # grey axis: U = V = 128 -> R = G = B = 255 (Y - yo) / ys (no chroma term)
    for Y in (16, 17, 100, 128, 235):
        assert np.allclose(O.yuv_to_rgb(Y, 128, 128, O.BT709_LIMITED), (Y - 16) * 255 / 219, atol=1e-12)
        assert np.allclose(O.yuv_to_rgb(Y, 128, 128, O.BT601_FULL), Y, atol=1e-12)
    # clamping: below black / above white saturate
    assert np.all(O.yuv_to_rgb(0, 128, 128, O.BT709_LIMITED) == 0)
    assert np.all(O.yuv_to_rgb(255, 128, 128, O.BT709_LIMITED) == 255)
    # JFIF (BT.601 full range) primary red: Y = 76.245, Cb = 84.972, Cr = 255.5 -> (255, 0, 0)
    r = O.yuv_to_rgb(0.299 * 255, 128 - 0.168736 * 255, 128 + 0.5 * 255, O.BT601_FULL)
    assert np.allclose(r, (255, 0, 0), atol=1e-3)
    with pytest.raises(ValueError):
        O.yuv_to_rgb(1, 2, 3, 7)


def _nv12(seed, W, H, pitch):
    return S.frame_nv12_np(seed, H, pitch)


def _planes(fr, W, H):
    Y = fr[:H, :W].astype(np.float64)
    UV = fr[H:H + H // 2, :W]
    U = UV[:, 0::2].astype(np.float64)
    V = UV[:, 1::2].astype(np.float64)
    return Y, U, V


@pytest.mark.parametrize("matrix", [O.BT709_LIMITED, O.BT601_LIMITED, O.BT709_FULL])
def test_identity_scale_chroma_siting(matrix):
    """Scale 1 -> every output pixel is convert(Y[r][c], U[r>>1][c>>1], V[r>>1][c>>1])
    of the window's own pixels (windows at odd and even offsets)."""
    W, H = 64, 46
    pitch = 80
    fr = _nv12(7, W, H, pitch)
    Y, U, V = _planes(fr, W, H)
    win = [(0, 0, 0, 17, 9, 0, 0), (0, 3, 5, 17, 9, 0, 1), (0, 47, 37, 17, 9, 0, 2), (0, 0, 0, W, H, 1, 0)]
    st, out = O.gather_resize_nv12([fr], pitch, W, H, win, [(17, 9), (W, H)], [(17, 9), (W, H)], [3, 1],
                                   O.F64_NCHW, matrix)
    assert st == 0
    for (f, x, y, w, h, q, slot) in win:
        for r in range(h):
            for c in range(w):
                R, Cc = y + r, x + c
                e = O.yuv_to_rgb(Y[R, Cc], U[R >> 1, Cc >> 1], V[R >> 1, Cc >> 1], matrix)
                assert np.array_equal(out[q][slot, :, r, c], e), (x, y, r, c)


def test_resample_equals_rgb_resampler_on_444_upsampled_planes():
    """NV12 resize == R23 conversion of the RGB-path resize (pinned in
    test_oracle_resize.py) of the image packed as (Y, U444, V444) channels,
    U444 = nearest 2x upsampling of U; across up/down scales and odd offsets."""
    W, H = 96, 70
    pitch = 96
    fr = _nv12(11, W, H, pitch)
    Y, U, V = _planes(fr, W, H)
    up = lambda P: np.repeat(np.repeat(P, 2, 0), 2, 1)[:H, :W]
    img = np.stack([Y, up(U), up(V)], -1).astype(np.uint8)
    rgb_pitch = (3 * W + 15) // 16 * 16
    rgb_fr = np.zeros((H, rgb_pitch), np.uint8)
    rgb_fr[:, :3 * W] = img.reshape(H, 3 * W)
    sizes = [(33, 21), (50, 40), (W, H)]
    out_dims = [(47, 13), (19, 29), (40, 31)]
    win = [(0, 1, 3, 33, 21, 0, 0), (0, 62, 48, 33, 21, 0, 1), (0, 7, 0, 50, 40, 1, 0), (0, 0, 0, W, H, 2, 0)]
    st, yuv = O.gather_resize(np.stack([rgb_fr]), rgb_pitch, W, H, win, sizes, out_dims, [2, 1, 1], O.F64_NCHW)
    assert st == 0
    for matrix in (O.BT709_LIMITED, O.BT601_FULL):
        st, got = O.gather_resize_nv12([fr], pitch, W, H, win, sizes, out_dims, [2, 1, 1], O.F64_NCHW, matrix)
        assert st == 0
        for q in range(3):
            for s in range(got[q].shape[0]):
                _, oh, ow = got[q][s].shape
                for r in range(oh):
                    for c in range(ow):
                        e = O.yuv_to_rgb(*yuv[q][s, :, r, c], matrix)
                        assert np.allclose(got[q][s, :, r, c], e, rtol=0, atol=1e-9)


def test_grey_frame_matches_rgb_resampler():
    """U = V = 128: out = clamp(255 (Yresized - 16) / 219) with Yresized the RGB
    path's resize of the Y plane (BT.709 limited)."""
    W, H, pitch = 64, 48, 64
    fr = _nv12(3, W, H, pitch).copy()
    fr[H:] = 128
    Y = fr[:H, :W]
    rgb_pitch = 3 * W
    rgb_fr = np.repeat(Y[:, :, None], 3, 2).reshape(H, 3 * W)
    win = [(0, 5, 9, 40, 30, 0, 0)]
    st, a = O.gather_resize(np.stack([rgb_fr]), rgb_pitch, W, H, win, [(40, 30)], [(23, 41)], [1], O.F64_NCHW)
    st2, b = O.gather_resize_nv12([fr], pitch, W, H, win, [(40, 30)], [(23, 41)], [1], O.F64_NCHW)
    assert st == st2 == 0
    e = np.clip((a[0] - 16.0) * 255.0 / 219.0, 0, 255)
    assert np.allclose(b[0], e, atol=1e-9)


def test_u8_and_f32_outputs_follow_f64():
    W, H, pitch = 64, 48, 64
    fr = _nv12(5, W, H, pitch)
    win = [(0, 3, 1, 40, 30, 0, 0), (0, 24, 18, 40, 30, 0, 1)]
    args = ([fr], pitch, W, H, win, [(40, 30)], [(57, 21)], [2])
    _, d = O.gather_resize_nv12(*args, O.F64_NCHW)
    _, f = O.gather_resize_nv12(*args, O.F32_NCHW)
    _, u = O.gather_resize_nv12(*args, O.U8_NHWC)
    assert np.array_equal(f[0], d[0].astype(np.float32))
    assert np.array_equal(u[0], np.floor(d[0] + 0.5).astype(np.uint8).transpose(0, 2, 3, 1))
    assert d[0].min() >= 0 and d[0].max() <= 255


def test_invalid_inputs():
    W, H, pitch = 64, 48, 64
    fr = _nv12(5, W, H, pitch)
    good = [(0, 0, 0, 40, 30, 0, 0)]
    assert O.gather_resize_nv12([fr], pitch, W, H, [(0, 30, 0, 40, 30, 0, 0)], [(40, 30)], [(8, 8)], [1])[0] == 1
    assert O.gather_resize_nv12([fr], pitch, W, H, [(0, 0, 0, 40, 30, 0, 1)], [(40, 30)], [(8, 8)], [1])[0] == 3
    assert O.gather_resize_nv12([fr], pitch, W, H, good, [(40, 30)], [(8, 8)], [1], matrix=9)[0] == 1
    odd = S.frame_nv12_np(1, 47, 64)   # H odd: 4:2:0 needs even dims (R23)
    assert O.gather_resize_nv12([odd], 64, 64, 47, good, [(40, 30)], [(8, 8)], [1])[0] == 1
    with pytest.raises(ValueError):   # frame shape must be [H*3/2][pitch]
        O.gather_resize_nv12([fr[:H]], pitch, W, H, good, [(40, 30)], [(8, 8)], [1])
