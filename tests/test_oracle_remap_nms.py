"""Pins of the oracle's a6/a7 (remap + per-frame class-aware NMS, readings
R17-R20) against hand-derived golden values, torchvision.ops.nms (called per
class), closed forms and invariants."""
import json
import os

import numpy as np
import pytest
import torch
import torchvision

import oracle as O


def _gold():
    here = os.path.dirname(os.path.abspath(__file__))
    return json.load(open(os.path.join(here, "golden", "resize_remap_nms_golden.json")))


def _box(x1, y1, x2, y2, score=1.0, cls=0):
    b = np.zeros(1, O.BOX_DTYPE)[0]
    b["x1"], b["y1"], b["x2"], b["y2"], b["score"], b["cls"] = x1, y1, x2, y2, score, cls
    return b


def _boxes(rows):
    a = np.zeros(len(rows), O.BOX_DTYPE)
    for i, r in enumerate(rows):
        a[i] = tuple(r[:5]) + (int(r[5]),)
    return a


@pytest.mark.parametrize("case", _gold()["iou"], ids=lambda c: c["name"])
def test_iou_golden(case):
    assert O.iou(_box(*case["a"]), _box(*case["b"])) == pytest.approx(case["expect"], rel=1e-6)


@pytest.mark.parametrize("case", _gold()["remap"], ids=lambda c: c["name"])
def test_remap_golden(case):
    r = O.remap_box(_box(*case["box"][:4], case["box"][4], case["box"][5]), case["window"],
                    case["out_dim"], 0.25)
    assert [float(r[n]) for n in ("x1", "y1", "x2", "y2")] == case["expect"]


def test_remap_filters():
    w, od = (0, 0, 64, 64), (48, 48)
    assert O.remap_box(_box(1, 1, 5, 5, 0.25), w, od, 0.25) is None           # score == thr
    assert O.remap_box(_box(1, 1, 5, 5, np.nan), w, od, 0.25) is None         # NaN score
    assert O.remap_box(_box(5, 1, 5, 5, 0.9), w, od, 0.25) is None            # x2 == x1
    assert O.remap_box(_box(50, 1, 60, 5, 0.9), w, od, 0.25) is None          # clipped to empty
    assert O.remap_box(_box(1, 1, 5, 5, 0.26), w, od, 0.25) is not None


def test_remap_scale_one_integer_exact_and_inside_window():
    rng = np.random.default_rng(0)
    for _ in range(500):
        x, y = int(rng.integers(0, 1500)), int(rng.integers(0, 800))
        w, h = int(rng.integers(16, 400)), int(rng.integers(16, 300))
        a, b = sorted(rng.integers(0, w + 1, 2)); c, d = sorted(rng.integers(0, h + 1, 2))
        if a == b or c == d:
            continue
        r = O.remap_box(_box(a, c, b, d, 0.9), (x, y, w, h), (w, h), 0.25)
        assert [float(r[n]) for n in ("x1", "y1", "x2", "y2")] == [a + x, c + y, b + x, d + y]
    # containment for random scales and jittered boxes
    for _ in range(2000):
        x, y = int(rng.integers(0, 3000)), int(rng.integers(0, 1800))
        w, h = int(rng.integers(16, 800)), int(rng.integers(16, 800))
        ow, oh = int(rng.integers(8, 600)), int(rng.integers(8, 600))
        bx = rng.uniform(-20, ow + 20, 2); by = rng.uniform(-20, oh + 20, 2)
        r = O.remap_box(_box(bx.min(), by.min(), bx.max(), by.max(), 0.9), (x, y, w, h), (ow, oh), 0.25)
        if r is not None:
            assert x <= r["x1"] < r["x2"] <= x + w and y <= r["y1"] < r["y2"] <= y + h


def test_remap_dyadic_closed_form():
    # scale 1/2 in detector space (ow = w/2): X = 2 * x_l + x exactly
    rng = np.random.default_rng(1)
    for _ in range(300):
        x1, x2 = sorted(rng.uniform(0, 100, 2).astype(np.float32))
        if x1 == x2:
            continue
        r = O.remap_box(_box(x1, 1, x2, 2, 0.9), (1000, 500, 200, 200), (100, 100), 0.25)
        assert float(r["x1"]) == np.float32(np.float64(x1) * 2 + 1000)
        assert float(r["x2"]) == np.float32(np.float64(x2) * 2 + 1000)


def _one_frame_nms(rows, iou_thr, score_thr=-1.0):
    """Identity remap (window = out_dim at origin) so NMS sees the boxes as given."""
    bx = _boxes(rows)
    win = np.array([[0, 0, 0, 1 << 14, 1 << 14, 0, 0]], np.int32)
    res = O.remap_nms(bx, [0, len(bx)], win, [0, 1], [(1 << 14, 1 << 14)], 1 << 14, 1 << 14,
                      score_thr, iou_thr)
    return res


@pytest.mark.parametrize("case", _gold()["nms"], ids=lambda c: c["name"])
def test_nms_golden(case):
    res = _one_frame_nms(case["boxes"], case["iou_thr"])
    assert res["src"].tolist() == case["keep"]


def _tv_per_class(rows, thr):
    """torchvision.ops.nms called per class, merged by (score desc, index asc)."""
    a = np.asarray(rows, np.float64)
    keep = []
    for c in np.unique(a[:, 5]):
        idx = np.nonzero(a[:, 5] == c)[0]
        b = torch.tensor(a[idx, :4], dtype=torch.float32)
        s = torch.tensor(a[idx, 4], dtype=torch.float32)
        keep += idx[torchvision.ops.nms(b, s, thr).numpy()].tolist()
    sc = a[:, 4].astype(np.float32)
    return sorted(keep, key=lambda i: (-sc[i], i))


@pytest.mark.parametrize("seed", range(60))
def test_nms_matches_torchvision_per_class(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 120))
    rows = []
    for _ in range(n):
        x, y = rng.integers(0, 60, 2).astype(np.float64)       # integer-ish grid -> many exact ties
        w, h = rng.integers(1, 25, 2).astype(np.float64)
        if rng.random() < 0.5:
            x += rng.random(); w += rng.random()
        s = float(rng.choice([0.5, 0.75, 0.9])) if rng.random() < 0.4 else float(rng.random())
        rows.append((x, y, x + w, y + h, s, int(rng.integers(0, 3))))
    for thr in (0.5, 0.375, 0.625):
        res = _one_frame_nms(rows, thr)
        assert res["src"].tolist() == _tv_per_class(rows, thr)


def test_nms_invariants_and_certificate():
    rng = np.random.default_rng(7)
    for _ in range(50):
        n = int(rng.integers(1, 200))
        xy = rng.uniform(0, 200, (n, 2)); wh = rng.uniform(5, 60, (n, 2))
        rows = [(xy[i, 0], xy[i, 1], xy[i, 0] + wh[i, 0], xy[i, 1] + wh[i, 1], rng.random(),
                 int(rng.integers(0, 2))) for i in range(n)]
        res = _one_frame_nms(rows, 0.5)
        keep = res["src"].tolist()
        bx = _boxes(rows)
        assert len(set(keep)) == len(keep) and set(keep) <= set(range(n))
        for i in range(len(keep)):
            for j in range(i + 1, len(keep)):
                a, b = bx[keep[i]], bx[keep[j]]
                if a["cls"] == b["cls"]:
                    assert O.iou(a, b) <= 0.5
        # greedy certificate: every suppressed box has a higher-ranked kept same-class box with IoU > thr
        rank = {q: (-np.float32(bx[q]["score"]), q) for q in range(n)}
        for q in set(range(n)) - set(keep):
            assert any(bx[k]["cls"] == bx[q]["cls"] and rank[k] < rank[q] and O.iou(bx[k], bx[q]) > 0.5
                       for k in keep)
        # one class -> class-agnostic NMS (torchvision directly)
        one = [r[:5] + (0,) for r in rows]
        res1 = _one_frame_nms(one, 0.5)
        b = torch.tensor([r[:4] for r in one], dtype=torch.float32)
        s = torch.tensor([r[4] for r in one], dtype=torch.float32)
        assert res1["src"].tolist() == torchvision.ops.nms(b, s, 0.5).tolist()


def test_remap_nms_multi_frame_csr_and_negative_zero():
    # frame 0: two windows; frame 1: none; frame 2: one window with a -0.0 vs +0.0 score tie
    win = np.array([[0, 0, 0, 64, 64, 0, 0], [0, 32, 0, 64, 64, 0, 1], [2, 0, 0, 64, 64, 0, 2]], np.int32)
    rows = [(0, 0, 16, 16, 0.9, 0), (8, 0, 24, 16, 0.8, 0),          # window 0 (scale 64/32 = 2)
            (0, 0, 16, 16, 0.95, 0),                                   # window 1 -> frame (32..64)
            (0, 0, 10, 10, 0.0, 1), (20, 20, 30, 30, -0.0, 1)]         # window 2
    bx = _boxes(rows)
    res = O.remap_nms(bx, [0, 2, 3, 5], win, [0, 2, 2, 3], [(32, 32)], 640, 480, -1.0, 0.5)
    assert res["frame_off"].tolist() == [0, 3, 3, 5]
    # frame 0: candidates q0 (0,0,32,32) .9, q1 (16,0,48,32) .8, q2 (32,0,64,32) .95
    # order q2, q0, q1: IoU(q2,q0)=0 -> keep q0; IoU(q0,q1)=16*32/(1024+1024-512)=1/3 keep; IoU(q2,q1)=1/3 keep
    # frame 2: -0.0 == +0.0 -> tie broken by index: q3 before q4
    assert res["src"].tolist() == [2, 0, 1, 3, 4]


def test_remap_nms_capacity():
    rows = [(i * 20, 0, i * 20 + 10, 10, 0.9, 0) for i in range(5)]
    bx = _boxes(rows)
    win = np.array([[0, 0, 0, 256, 256, 0, 0]], np.int32)
    res = O.remap_nms(bx, [0, 5], win, [0, 1], [(256, 256)], 256, 256, 0.25, 0.5, max_out=3)
    assert res["status"] == O.ERR_CAPACITY and res["frame_off"].tolist() == [0, 5]
    assert len(res["boxes"]) == 3
