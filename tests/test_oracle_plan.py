"""Pins of the oracle's a1-a4 (threshold, components, merge, placement) against
things other than itself: SPEC/paper examples, hand-derived golden cases
(tests/golden/plan_golden.json), scipy.ndimage.label, brute-force optimal
covers on tiny grids, and the invariants the paper fixes."""
import itertools
import json
import os

import numpy as np
import pytest
import scipy.ndimage as ndi

import oracle as O


# --------------------------------------------------------------------------- a1
def test_threshold_spec_examples():
    # grid [0.2, 0.7, 0.9], b = 0.5 -> cells 2 and 3 (1-based)
    s = np.array([[0.2, 0.7, 0.9]], np.float32)
    assert O.threshold(s, 0.5).tolist() == [[0, 1, 1]]
    assert O.threshold(s, 1.0).sum() == 0             # b >= max score -> empty
    assert O.threshold(s, 0.1).sum() == 3             # b < min score -> full
    # strict '>' (R2): a score equal to B is not positive
    assert O.threshold(np.array([[0.5]], np.float32), 0.5).sum() == 0
    # NaN is never positive
    assert O.threshold(np.array([[np.nan, 1.0]], np.float32), 0.0).tolist() == [[0, 1]]


def test_threshold_matches_numpy_compare():
    rng = np.random.default_rng(1)
    for b in (0.1, 0.5, 0.77, 0.9):
        s = rng.random((34, 60), dtype=np.float32)
        s[0, :5] = np.float32(b)                        # exact ties
        assert np.array_equal(O.threshold(s, b), (s > np.float32(b)).astype(np.uint8))


def test_pack_mask_layout():
    rng = np.random.default_rng(2)
    pos = (rng.random((5, 70)) < 0.4).astype(np.uint8)
    m = O.pack_mask(pos)
    assert m.shape == (5, 3)
    for r in range(5):
        for c in range(96):
            bit = (int(m[r, c // 32]) >> (c % 32)) & 1
            assert bit == (pos[r, c] if c < 70 else 0)


# --------------------------------------------------------------------------- a2
def test_components_spec_examples():
    # empty -> []; diagonal-only neighbours -> 2 components
    assert O.components(np.zeros((3, 3), np.uint8))[1].shape == (0, 4)
    lab, bb = O.components(np.array([[1, 0], [0, 1]], np.uint8))
    assert len(bb) == 2 and bb.tolist() == [[0, 0, 0, 0], [1, 1, 1, 1]]


@pytest.mark.parametrize("seed", range(40))
def test_components_match_scipy_label(seed):
    """scipy.ndimage.label: default structure = 4-connectivity cross, labels in
    raster first-occurrence order -> labels and bboxes must be identical."""
    rng = np.random.default_rng(seed)
    R, C = rng.integers(1, 25), rng.integers(1, 40)
    pos = (rng.random((R, C)) < rng.uniform(0.05, 0.7)).astype(np.uint8)
    lab, bb = O.components(pos)
    ref, n = ndi.label(pos)
    assert len(bb) == n
    assert np.array_equal(lab + 1, ref)
    for i, sl in enumerate(ndi.find_objects(ref)):
        assert bb[i].tolist() == [sl[1].start, sl[0].start, sl[1].stop - 1, sl[0].stop - 1]


# --------------------------------------------------------------------------- golden
def _golden():
    here = os.path.dirname(os.path.abspath(__file__))
    return json.load(open(os.path.join(here, "golden", "plan_golden.json")))["cases"]


@pytest.mark.parametrize("case", _golden(), ids=lambda c: c["name"])
def test_plan_golden(case):
    cw = case.get("cell_w", case.get("cell", 32))
    ch = case.get("cell_h", case.get("cell", 32))
    W, H = case["W"], case["H"]
    R, C = -(-H // ch), -(-W // cw)
    s = np.zeros((1, R, C), np.float32)
    for r, c in case["cells"]:
        s[0, r, c] = 0.9
    res = O.plan_windows(W, H, cw, ch, 0.5, case["sizes"], case["cost"], s)
    assert res["status"] == 0
    assert res["windows"].tolist() == case["windows"]
    est = sum(case["cost"][w[5]] for w in res["windows"])
    assert est == case["est"]
    assert int(res["passes"][0]) == case["passes"]


def test_smallest_window_spec():
    # SPEC.md:225-229
    sizes = [(64, 32), (32, 64), (200, 100)]
    assert O.smallest_window(sizes, 60, 30) == 0
    assert O.smallest_window([(32, 32), (200, 100)], 32, 32) == 0
    assert O.smallest_window([(64, 64), (200, 100)], 65, 10) == 1


def test_smallest_window_tie_rule():
    # R6: equal area -> smaller w first.  32x64 (w=32) beats 64x32 for a bbox both contain.
    sizes = [(64, 32), (32, 64), (200, 100)]
    assert O.smallest_window(sizes, 20, 20) == 1


def test_invalid_params_rejected():
    s = np.zeros((1, 6, 8), np.float32)
    assert O.plan_windows(256, 192, 32, 32, .5, [(64, 64)], [20], s)["status"] == O.ERR_INVALID   # no full frame
    assert O.plan_windows(256, 192, 32, 32, .5, [(64, 64), (256, 192)], [70, 64], s)["status"] == O.ERR_INVALID
    assert O.plan_windows(256, 192, 32, 32, .5, [(300, 64), (256, 192)], [1, 64], s)["status"] == O.ERR_INVALID


# --------------------------------------------------------------------------- brute force
def _pix(cb, W, H, cw, ch):
    c0, r0, c1, r1 = cb
    x0, y0 = c0 * cw, r0 * ch
    return x0, y0, min((c1 + 1) * cw, W) - x0, min((r1 + 1) * ch, H) - y0


def _sw(sizes, bw, bh):
    fit = [i for i, (w, h) in enumerate(sizes) if w >= bw and h >= bh]
    return min(fit, key=lambda i: (sizes[i][0] * sizes[i][1], sizes[i][0], sizes[i][1]))


def _partitions(items):
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for p in _partitions(rest):
        yield [[first]] + p
        for i in range(len(p)):
            yield p[:i] + [[first] + p[i]] + p[i + 1:]


def _random_case(rng):
    W, H = 32 * int(rng.integers(3, 9)), 32 * int(rng.integers(2, 7))
    cand = sorted({(32 * int(rng.integers(1, W // 32 + 1)), 32 * int(rng.integers(1, H // 32 + 1)))
                   for _ in range(3)} - {(W, H)}, key=lambda s: s[0] * s[1])
    sizes = cand + [(W, H)]
    # strictly increasing in area: cells + per-window overhead (like the bench table)
    ov = int(rng.integers(0, 20))
    cost = [(w // 32) * (h // 32) * 4 + ov + 1 for (w, h) in sizes]
    # equal-area sizes must not violate "area_i < area_j -> T_i < T_j": fine by construction
    R, C = H // 32, W // 32
    pos = (rng.random((R, C)) < rng.uniform(0.1, 0.45)).astype(np.uint8)
    return W, H, sizes, cost, pos


def _check_invariants(W, H, sizes, cost, pos, res, cw=32, ch=32):
    lab, bb = O.components(pos)
    win = res["windows"]
    full = sizes.index((W, H))
    # sizes in S, inside the frame
    for f, x, y, w, h, k, slot in win:
        assert (w, h) == tuple(sizes[k])
        assert 0 <= x and 0 <= y and x + w <= W and y + h <= H
    # every component wholly inside one window => every positive cell covered
    for cb in bb:
        x0, y0, bw, bh = _pix(cb, W, H, cw, ch)
        assert any(x <= x0 and y <= y0 and x0 + bw <= x + w and y0 + bh <= y + h
                   for f, x, y, w, h, k, s in win), (cb, win)
    assert len(win) <= len(bb)
    est = sum(cost[w[5]] for w in win)
    assert est <= cost[full]
    # termination: each pass but the last merges, each merge shrinks the list
    assert int(res["passes"][0]) <= len(bb)
    return est, bb


def test_plan_bruteforce_and_invariants():
    """Greedy est >= brute-force optimum always; == optimum with <= 2
    components (the greedy then compares exactly the two partitions)."""
    rng = np.random.default_rng(20210314)
    n_checked = n_eq = 0
    for _ in range(1500):
        W, H, sizes, cost, pos = _random_case(rng)
        s = pos[None].astype(np.float32)
        res = O.plan_windows(W, H, 32, 32, 0.5, sizes, cost, s)
        assert res["status"] == 0
        est, bb = _check_invariants(W, H, sizes, cost, pos, res)
        if len(bb) == 0:
            assert len(res["windows"]) == 0
            continue
        if len(bb) > 7:
            continue
        best = None
        for part in _partitions(list(range(len(bb)))):
            tot = 0
            for block in part:
                c0 = min(bb[i][0] for i in block); r0 = min(bb[i][1] for i in block)
                c1 = max(bb[i][2] for i in block); r1 = max(bb[i][3] for i in block)
                _, _, bw, bh = _pix((c0, r0, c1, r1), W, H, 32, 32)
                tot += cost[_sw(sizes, bw, bh)]
            best = tot if best is None else min(best, tot)
        n_checked += 1
        assert est >= best
        if len(bb) <= 2:
            assert est == best
            n_eq += 1
    assert n_checked > 500 and n_eq > 50


def test_plan_batched_frames_independent_and_slots():
    """Frames are independent: the batched call equals per-frame calls;
    slots are ranks within size class in (frame, list) order; CSR is exact."""
    rng = np.random.default_rng(5)
    W, H = 320, 224
    sizes = [(64, 64), (128, 96), (320, 224)]
    cost = [20, 30, 90]
    F = 25
    s = rng.random((F, 7, 10), dtype=np.float32)
    res = O.plan_windows(W, H, 32, 32, 0.7, sizes, cost, s)
    allw = []
    for f in range(F):
        r1 = O.plan_windows(W, H, 32, 32, 0.7, sizes, cost, s[f:f + 1])
        w = r1["windows"].copy()
        w[:, 0] = f
        assert res["frame_off"][f + 1] - res["frame_off"][f] == len(w)
        allw.append(w)
    allw = np.concatenate(allw)
    assert np.array_equal(res["windows"][:, :6], allw[:, :6])
    for k in range(3):
        sel = res["windows"][res["windows"][:, 5] == k]
        assert sel[:, 6].tolist() == list(range(len(sel)))
        assert res["class_count"][k] == len(sel)


def test_plan_capacity_reports_true_total():
    rng = np.random.default_rng(6)
    s = rng.random((10, 6, 8), dtype=np.float32)
    full = O.plan_windows(256, 192, 32, 32, 0.8, [(32, 32), (256, 192)], [5, 100], s)
    n = int(full["frame_off"][-1])
    assert n > 3
    cut = O.plan_windows(256, 192, 32, 32, 0.8, [(32, 32), (256, 192)], [5, 100], s, max_windows=3)
    assert cut["status"] == O.ERR_CAPACITY
    assert np.array_equal(cut["frame_off"], full["frame_off"])
    assert np.array_equal(cut["windows"], full["windows"][:3])


def test_plan_checkerboard_worst_case():
    """Checkerboard: R*C/2 isolated components; merge terminates, invariants hold."""
    W, H = 640, 384
    R, C = 12, 20
    pos = ((np.add.outer(np.arange(R), np.arange(C)) % 2) == 0).astype(np.uint8)
    sizes = [(64, 64), (128, 128), (W, H)]
    cost = [4 + 16, 16 + 16, 240 + 16]
    res = O.plan_windows(W, H, 32, 32, 0.5, sizes, cost, pos[None].astype(np.float32))
    _check_invariants(W, H, sizes, cost, pos, res)
