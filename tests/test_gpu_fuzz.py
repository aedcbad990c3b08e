"""Randomised end-to-end parity: 48 seeded random problems — frame sizes that
are not multiples of the cell, non-square cells, 1-6 window sizes with random
monotone costs, blob-structured proxy scores at random thresholds — through
plan (exact), gather + resize of every window to random output sizes (f32
within 1e-3, u8 within 1 LSB, both staging paths) and remap + NMS of random
boxes (exact), all against the oracle."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from workloads import synth as S  # noqa: E402


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import gpu_util
    return gpu_util


def _problem(seed):
    rng = np.random.default_rng(9000 + seed)
    W, H = int(rng.integers(40, 900)), int(rng.integers(40, 600))
    W += W & 1
    H += H & 1
    cw = int(rng.choice([16, 24, 32, 48]))
    ch = cw if rng.random() < 0.6 else int(rng.choice([16, 32, 40]))
    R, C = -(-H // ch), -(-W // cw)
    k = int(rng.integers(0, 6))
    sizes = set()
    while len(sizes) < k:
        sizes.add((int(rng.integers(8, W + 1)), int(rng.integers(8, H + 1))))
    sizes.discard((W, H))
    sizes = sorted(sizes, key=lambda s: (s[0] * s[1], s)) + [(W, H)]
    # strictly area-monotone costs (equal areas get any order)
    areas = sorted({w * h for w, h in sizes})
    base = {a: 10 + 7 * i + int(rng.integers(0, 5)) for i, a in enumerate(areas)}
    cost = [base[w * h] for w, h in sizes]
    F = int(rng.integers(1, 6))
    scores = np.full((F, R, C), 0.0, np.float32)
    for f in range(F):
        z = rng.normal(-2.0, 1.0, (R, C))
        for _ in range(int(rng.integers(0, 8))):
            r0, c0 = rng.integers(0, R), rng.integers(0, C)
            rr, cc = int(rng.integers(1, 4)), int(rng.integers(1, 4))
            z[r0:r0 + rr, c0:c0 + cc] += rng.normal(4.0, 1.0)
        scores[f] = 1.0 / (1.0 + np.exp(-z))
    b = float(rng.choice([0.3, 0.5, 0.7]))
    return rng, W, H, cw, ch, sizes, cost, scores, b


@pytest.mark.parametrize("seed", range(48))
def test_random_end_to_end(G, seed):
    rng, W, H, cw, ch, sizes, cost, scores, b = _problem(seed)
    F = scores.shape[0]
    ref = O.plan_windows(W, H, cw, ch, b, sizes, cost, scores)
    got = G.gpu_plan(W, H, cw, ch, b, sizes, cost, scores)
    assert got["status"] == ref["status"] == 0
    assert np.array_equal(got["frame_off"], ref["frame_off"])
    assert np.array_equal(got["windows"], ref["windows"])
    assert np.array_equal(got["mask"], ref["mask"])
    win = ref["windows"]
    if len(win) == 0:
        return
    # gather + resize to random output dims (down- and up-scales)
    out_dims = [(max(1, int(w * s)), max(1, int(h * s))) for (w, h), s in
                zip(sizes, rng.uniform(0.2, 1.6, len(sizes)))]
    caps = [int((win[:, 5] == q).sum()) for q in range(len(sizes))]
    pitch = (3 * W + 15) // 16 * 16
    frames = [S.frame_pixels_np(S.frame_seed(seed, f), H, pitch) for f in range(F)]
    fmt = seed % 2
    strided = (seed // 2) % 2 == 0
    try:
        st_r, o_ref = O.gather_resize(frames, pitch, W, H, win, sizes, out_dims, caps,
                                      O.F32_NCHW if fmt == 0 else O.U8_NHWC)
        st_g, o_got = G.gpu_gather(frames, pitch, W, H, win, sizes, out_dims, caps, fmt, strided)
    except Exception as e:   # an unsupported (too strong) downscale of a very wide window is allowed
        import paper_2103_14695_b200 as mp
        assert isinstance(e, mp.MPError), e
        return
    assert st_g == st_r == 0
    for q in range(len(sizes)):
        if caps[q]:
            d = np.abs(o_got[q].astype(np.float64) - o_ref[q].astype(np.float64)).max()
            assert d <= (1e-3 if fmt == 0 else 1.0), (q, d)
    # remap + NMS of random boxes in each window's detector-input space
    rows, wbo = [], [0]
    for w in win:
        ow, oh = out_dims[int(w[5])]
        for _ in range(int(rng.integers(0, 12))):
            x1, y1 = rng.uniform(-5, ow), rng.uniform(-5, oh)
            rows.append((x1, y1, x1 + rng.uniform(-2, ow / 2), y1 + rng.uniform(-2, oh / 2),
                         float(rng.choice([rng.uniform(0, 1), 0.25, 0.5])), int(rng.integers(0, 3))))
        wbo.append(len(rows))
    boxes = np.zeros(len(rows), O.BOX_DTYPE)
    if rows:
        a = np.asarray(rows, np.float64)
        for i, name in enumerate(("x1", "y1", "x2", "y2", "score")):
            boxes[name] = a[:, i].astype(np.float32)
        boxes["cls"] = a[:, 5].astype(np.int32)
    wbo = np.asarray(wbo, np.int32)
    iou = float(rng.choice([0.3, 0.5, 0.7]))
    r = O.remap_nms(boxes, wbo, win, ref["frame_off"], out_dims, W, H, 0.25, iou)
    g = G.gpu_remap_nms(boxes, wbo, win, ref["frame_off"], out_dims, W, H, 0.25, iou)
    assert g["status"] == r["status"] == 0
    assert np.array_equal(g["frame_off"], r["frame_off"])
    assert np.array_equal(g["src"], r["src"])
    assert np.array_equal(g["boxes"].view(np.uint32), r["boxes"].view(np.float32).reshape(-1, 6).view(np.uint32))


def _merge_heavy_problem(seed):
    """Grids with many components (hundreds to thousands): every plan tier
    (fast + its cooperative merge above 96 components, full <= 960 runs,
    huge beyond) and cost tables from merge-averse to merge-happy."""
    rng = np.random.default_rng(77000 + seed)
    W, H = [(1920, 1080), (3840, 2160), (2560, 1440), (7680, 4320), (1280, 720)][seed % 5]
    cw = ch = 32
    R, C = -(-H // ch), -(-W // cw)
    k = int(rng.integers(1, 5))
    sizes = set()
    while len(sizes) < k:
        s = int(rng.choice([64, 96, 128, 192, 256, 384, 512, 768, 1024]))
        sizes.add((min(s, W), min(int(s * rng.choice([0.5, 1.0, 1.5])), H)))
    sizes.discard((W, H))
    sizes = sorted(sizes, key=lambda s: (s[0] * s[1], s)) + [(W, H)]
    areas = sorted({w * h for w, h in sizes})
    style = seed % 3   # 0: cost ~ area (merges pay), 1: big fixed overhead (merges pay a lot), 2: steep (rarely pay)
    base = {}
    for i, a in enumerate(areas):
        cells = a / (cw * ch)
        base[a] = int(cells + (64 if style == 1 else 4) + (cells * cells / 50 if style == 2 else 0)) + i
    cost = [base[w * h] for w, h in sizes]
    if seed % 4 != 3:   # full frame never pays: the greedy's clusters are the output (no R11 fallback)
        cost[-1] = 10 ** 9
    F = 2
    dens = float(rng.choice([0.03, 0.08, 0.2, 0.45]))
    scores = np.zeros((F, R, C), np.float32)
    for f in range(F):
        z = (rng.random((R, C)) < dens).astype(np.float32) * 0.9
        for _ in range(int(rng.integers(0, 40))):
            r0, c0 = rng.integers(0, R), rng.integers(0, C)
            z[r0:r0 + int(rng.integers(1, 6)), c0:c0 + int(rng.integers(1, 6))] = 0.9
        scores[f] = z
    return W, H, cw, ch, sizes, cost, scores


@pytest.mark.parametrize("seed", range(30))
def test_plan_merge_heavy(G, seed):
    W, H, cw, ch, sizes, cost, scores = _merge_heavy_problem(seed)
    ref = O.plan_windows(W, H, cw, ch, 0.5, sizes, cost, scores)
    got = G.gpu_plan(W, H, cw, ch, 0.5, sizes, cost, scores)
    assert got["status"] == ref["status"]
    assert np.array_equal(got["frame_off"], ref["frame_off"])
    assert np.array_equal(got["class_count"], ref["class_count"])
    assert np.array_equal(got["windows"], ref["windows"])
