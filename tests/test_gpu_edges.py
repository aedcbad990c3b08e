"""GPU parity on the edge cases SURVEY.md §7 (hard part 4) and the round-1
review single out, against the CPU oracle (bit-exact keep lists and
coordinates, R18-R20):

* remap/NMS at score thresholds <= 0 (-inf, -1, 0): +-0.0 (equal in fp32
  value order), negative, denormal, tied, NaN and +-inf scores reach the
  GPU sort;
* NaN and +-inf box coordinates (R18 clips with fmin/fmax: NaN -> the bound);
* frames with more raw boxes than the shared-memory tiers hold (> 1024):
  the global-memory path, alone and mixed with small frames in one call;
* Hungarian (R24): the GPU matching of tie-heavy problems is optimal —
  its total equals scipy's linear_sum_assignment optimum, computed
  independently of the shared tie rule — and uses only allowed pairs.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import gpu_util
    return gpu_util


def _nms_compare(G, boxes, wbo, windows, frame_off, out_dims, W, H, score_thr, iou_thr):
    ref = O.remap_nms(boxes, wbo, windows, frame_off, out_dims, W, H, score_thr, iou_thr)
    got = G.gpu_remap_nms(boxes, wbo, windows, frame_off, out_dims, W, H, score_thr, iou_thr)
    assert got["status"] == ref["status"] == 0
    assert np.array_equal(got["frame_off"], ref["frame_off"])
    assert np.array_equal(got["src"], ref["src"])
    assert np.array_equal(got["boxes"].view(np.uint32), ref["boxes"].view(np.float32).reshape(-1, 6).view(np.uint32))
    return ref, got


DENORM = np.float32(1e-45)      # smallest positive fp32 denormal (bit pattern 0x00000001)
EDGE_SCORES = np.array([0.0, -0.0, DENORM, -DENORM, np.float32(1.2e-38), -np.float32(1.2e-38), -0.5, -0.5, 0.5,
                        0.5, -1.0, -1.0000001, -3e38, 3e38, np.inf, -np.inf, np.nan, -np.nan, 1.0, 0.9999999],
                       np.float32)


def _edge_frame(rng, n, score_pool, coords=None):
    """n boxes in a 256x256 window's 192x192 detector input: heavy overlap so
    suppression order matters; scores drawn from `score_pool` (ties)."""
    rows = np.zeros(n, O.BOX_DTYPE)
    xy = rng.integers(0, 120, (n, 2)).astype(np.float32)
    wh = rng.integers(20, 70, (n, 2)).astype(np.float32)
    rows["x1"], rows["y1"] = xy[:, 0], xy[:, 1]
    rows["x2"], rows["y2"] = xy[:, 0] + wh[:, 0], xy[:, 1] + wh[:, 1]
    rows["score"] = rng.choice(score_pool, n)
    rows["cls"] = rng.integers(0, 2, n)
    if coords is not None:
        for i, (name, v) in enumerate(coords):
            rows[name][i] = v
    return rows


@pytest.mark.parametrize("thr", [-np.inf, -1.0, 0.0, -0.0, float(DENORM)])
@pytest.mark.parametrize("n", [20, 64, 300, 1500])
def test_nms_scores_le_zero_and_specials(G, thr, n):
    """Every special score value reaches the sort for thresholds <= 0 (one
    frame per tier: warp <= 64, CTA <= 512, large <= 1024)."""
    rng = np.random.default_rng(n + 7)
    rows = _edge_frame(rng, n, EDGE_SCORES)
    rows["score"][:len(EDGE_SCORES)] = EDGE_SCORES[:min(n, len(EDGE_SCORES))]
    win = np.array([[0, 32, 16, 256, 256, 0, 0]], np.int32)
    ref, got = _nms_compare(G, rows, [0, n], win, [0, 1], [(192, 192)], 512, 512, np.float32(thr), 0.5)
    # independent check of the sort key: kept boxes of one class never
    # increase in score (fp32 value order, -0 == +0), NaN never kept
    kept = got["boxes"].view(np.float32).reshape(-1, 6)
    assert not np.isnan(kept[:, 4]).any()
    assert (kept[:, 4] > np.float32(thr)).all()


@pytest.mark.parametrize("n", [40, 400, 1800])
def test_nms_nonfinite_coordinates(G, n):
    """NaN / +-inf / huge coordinates: clipped to the detector input with
    fmin/fmax (NaN -> the bound), then degenerate boxes dropped (R18)."""
    rng = np.random.default_rng(n)
    specials = [("x1", np.nan), ("y1", np.nan), ("x2", np.nan), ("y2", np.nan), ("x1", -np.inf), ("x2", np.inf),
                ("y1", -np.inf), ("y2", np.inf), ("x2", 3e38), ("x1", -3e38), ("x1", np.inf), ("x2", -np.inf),
                ("y2", np.nan), ("x1", 1e-45), ("x2", 191.99998), ("y2", 192.00002)]
    rows = _edge_frame(rng, n, np.array([0.3, 0.6, 0.6, 0.9], np.float32), specials)
    win = np.array([[0, 1700, 900, 220, 180, 0, 0]], np.int32)
    for thr in (0.25, -1.0):
        _nms_compare(G, rows, [0, n], win, [0, 1], [(192, 160)], 1920, 1080, thr, 0.5)


@pytest.mark.parametrize("n", [300, 1024, 1025, 2049, 3000, 6100])
def test_nms_beyond_shared_memory_tiers(G, n):
    """One frame around / beyond the 1024 raw boxes the shared-memory tiers
    hold (the large tier's 256-candidate bitmask, its tiled path, then the
    global-memory path), tie-heavy, two IoU thresholds."""
    rng = np.random.default_rng(n)
    rows = np.zeros(n, O.BOX_DTYPE)
    xy = rng.integers(0, 1800, (n, 2)).astype(np.float32)
    wh = rng.integers(8, 80, (n, 2)).astype(np.float32)
    rows["x1"], rows["y1"] = xy[:, 0], xy[:, 1]
    rows["x2"], rows["y2"] = xy[:, 0] + wh[:, 0], xy[:, 1] + wh[:, 1]
    rows["score"] = rng.choice(np.array([0.3, 0.5, 0.9, -0.0, 0.0], np.float32), n)
    rows["cls"] = rng.integers(0, 3, n)
    win = np.array([[0, 0, 0, 2048, 2048, 0, 0]], np.int32)
    for thr in (0.5, 0.375):
        _nms_compare(G, rows, [0, n], win, [0, 1], [(1920, 1920)], 2048, 2048, -0.5, thr)


def test_nms_mixed_tiers_in_one_call(G):
    """Frames of 0, 10, 64, 65, 600, 1024, 1025, 2049, 4500 and 30 raw boxes (spread
    over several windows each) in one call: every tier including the
    global-memory one runs in the same launch sequence, and each frame's
    keep list equals the oracle's."""
    rng = np.random.default_rng(77)
    sizes = [0, 10, 64, 65, 600, 1024, 1025, 2049, 4500, 30]
    windows, wbo, frame_off, chunks = [], [0], [0], []
    for f, n in enumerate(sizes):
        nw = 1 if n < 100 else 3
        cuts = np.sort(rng.integers(0, n + 1, nw - 1)) if nw > 1 else np.zeros(0, int)
        parts = np.diff(np.concatenate([[0], cuts, [n]]))
        for j, c in enumerate(parts):
            windows.append([f, 64 * j, 32 * j, 512, 512, 0, len(windows)])
            chunks.append(_edge_frame(rng, int(c), np.array([0.3, 0.5, 0.5, 0.9, 0.0, -0.0], np.float32)))
            wbo.append(wbo[-1] + int(c))
        frame_off.append(len(windows))
    boxes = np.concatenate(chunks)
    _nms_compare(G, boxes, wbo, np.array(windows, np.int32), frame_off, [(384, 384)], 1024, 1024, 0.1, 0.5)


# --------------------------------------------------------------------------- Hungarian optimality (R24)
def _allowed_weights(a, floor):
    w = np.where(np.isnan(a) | (a < np.float32(floor)), 0.0, a.astype(np.float64))
    return w


@pytest.mark.parametrize("floor", [0.25, 0.5])
def test_hungarian_tie_heavy_is_optimal(G, floor):
    """The GPU and the oracle share one arg-min tie rule (R24), so their
    pair-identity test checks a shared convention; this test checks what is
    unique: the total of the GPU's matching equals the optimum of the
    maximum-weight assignment computed by scipy (an independent solver), and
    every matched pair is allowed (score >= floor, not NaN), one-to-one."""
    from scipy.optimize import linear_sum_assignment
    rng = np.random.default_rng(int(floor * 1000))
    mats = []
    for i in range(160):
        m, n = (int(x) for x in rng.integers(1, 100, 2))
        a = rng.random((m, n)).astype(np.float32)
        a = (np.round(a * (2 + i % 5)) / (2 + i % 5)).astype(np.float32)     # heavy exact ties
        if i % 4 == 0:
            a[rng.random((m, n)) < 0.1] = np.nan
        if i % 9 == 0:
            a[:] = np.float32(floor)                                         # all ties at the floor
        mats.append(a)
    mats.append(np.full((200, 90), 0.75, np.float32))                        # CTA tier, one big plateau
    st, rows, cols, tot = G.gpu_hungarian(mats, floor)
    assert st == 0
    for b, a in enumerate(mats):
        w = _allowed_weights(a, floor)
        r, c = linear_sum_assignment(w, maximize=True)
        best = float(w[r, c].sum())
        rm = rows[b]
        matched = np.nonzero(rm >= 0)[0]
        assert len(set(rm[matched].tolist())) == len(matched)                 # one-to-one
        assert all(cols[b][rm[i]] == i for i in matched)
        vals = a[matched, rm[matched]]
        assert not np.isnan(vals).any() and (vals >= np.float32(floor)).all()  # allowed pairs only
        got = float(vals.astype(np.float64).sum())
        assert abs(got - best) <= 1e-9 * max(1.0, best), (b, got, best)
        assert abs(tot[b] - got) <= 1e-9 * max(1.0, got)


# --------------------------------------------------------------------------- spatial-grid NMS path
@pytest.mark.parametrize("iou", [0.0, 0.5, 0.9, 1.0, -0.25])
@pytest.mark.parametrize("n,layout", [(97, "spread"), (500, "spread"), (1000, "spread"), (900, "giant"),
                                      (1000, "stacked"), (480, "grid_edges")])
def test_nms_grid_path(G, n, layout, iou):
    """Frames above 96 candidates with iou_thr >= 0 take the spatial-grid
    path (sparse adjacency of intersecting same-class pairs, greedy over it);
    iou_thr < 0 keeps the dense paths.  Layouts: drone-like boxes spread over
    a 4K frame; the same plus one frame-sized box (cells become the whole
    frame); 1000 near-identical stacked boxes (the adjacency overflows its
    scratch -> dense fallback); boxes on exact cell-size multiples."""
    rng = np.random.default_rng(n * 7 + len(layout))
    rows = np.zeros(n, O.BOX_DTYPE)
    if layout == "stacked":
        xy = 100 + rng.integers(0, 3, (n, 2)).astype(np.float32)
        wh = np.full((n, 2), 40, np.float32)
    elif layout == "grid_edges":
        xy = (rng.integers(0, 40, (n, 2)) * 64).astype(np.float32)
        wh = np.full((n, 2), 64, np.float32)
    else:
        xy = np.stack([rng.uniform(0, 2800, n), rng.uniform(0, 1580, n)], 1).astype(np.float32)
        wh = rng.uniform(8, 60, (n, 2)).astype(np.float32)
        dup = rng.random(n) < 0.5                     # jittered duplicates of the previous box
        xy[1:][dup[1:]] = xy[:-1][dup[1:]] + rng.uniform(-4, 4, (int(dup[1:].sum()), 2)).astype(np.float32)
    rows["x1"], rows["y1"] = xy[:, 0], xy[:, 1]
    rows["x2"], rows["y2"] = xy[:, 0] + wh[:, 0], xy[:, 1] + wh[:, 1]
    if layout == "giant":
        rows[n // 2] = (0, 0, 2880, 1620, 0.7, 1)
    rows["score"] = rng.choice(np.array([0.3, 0.5, 0.5, 0.9, 0.7], np.float32), n)
    rows["cls"] = rng.integers(0, 2, n)
    win = np.array([[0, 0, 0, 3840, 2160, 0, 0]], np.int32)
    _nms_compare(G, rows, [0, n], win, [0, 1], [(2880, 1620)], 3840, 2160, 0.25, iou)
