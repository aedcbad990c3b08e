"""GPU parity of NEXT-3 (mp_gather_resize_nv12, reading R23) against the
oracle's mpo_gather_resize_nv12 on the same seeded NV12 frames: f32 pixels
within 1e-3 absolute, u8 within 1 LSB (the a5 tolerances), plus the full-frame
proxy-input downscale, odd window offsets (chroma parity), all four matrices,
frame edges and the error paths."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from workloads import synth as S  # noqa: E402

F32_TOL = 1e-3


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import gpu_util
    return gpu_util


def _frames(cfg, clip, F):
    return [S.frame_nv12_np(S.frame_seed(clip, f), cfg.H, cfg.pitch_nv12) for f in range(F)]


def _compare(G, frames, pitch, W, H, windows, sizes, out_dims, fmt, matrix=O.BT709_LIMITED):
    win = np.asarray(windows, np.int32).reshape(-1, 7)
    caps = [int((win[:, 5] == q).sum()) for q in range(len(sizes))]
    st_r, ref = O.gather_resize_nv12(frames, pitch, W, H, win, sizes, out_dims, caps,
                                     O.F32_NCHW if fmt == 0 else O.U8_NHWC, matrix)
    st_g, got = G.gpu_gather_nv12(frames, W, H, win, sizes, out_dims, caps, fmt, matrix)
    assert st_g == st_r == 0
    for q in range(len(sizes)):
        if caps[q] == 0:
            continue
        if fmt == 0:
            err = np.abs(got[q].astype(np.float64) - ref[q]).max()
            assert err <= F32_TOL, (q, err)
        else:
            d = np.abs(got[q].astype(np.int32) - ref[q].astype(np.int32))
            assert d.max() <= 1, (q, d.max())
    return ref, got


@pytest.mark.parametrize("fmt", [0, 1])
@pytest.mark.parametrize("name,frames", [("c1_540p", 30), ("c2_1080p_sparse", 24), ("c4_4k_drone", 2)])
def test_nv12_parity_configs(G, name, frames, fmt):
    cfg = S.CONFIGS[name]
    scene = S.make_scene(cfg, 4, frames)
    scores = S.score_grids(cfg, 4, scene)
    plan = O.plan_windows(cfg.W, cfg.H, 32, 32, cfg.b_proxy, cfg.sizes, cfg.cost, scores)
    _compare(G, _frames(cfg, 4, frames), cfg.pitch_nv12, cfg.W, cfg.H, plan["windows"], cfg.sizes,
             cfg.out_dims, fmt)


@pytest.mark.parametrize("matrix", [0, 1, 2, 3])
@pytest.mark.parametrize("fmt", [0, 1])
@pytest.mark.parametrize("scale", [1.0, 0.5, 0.7, 1.37, 0.26])
def test_nv12_scales_offsets_matrices(G, scale, fmt, matrix):
    """Every window offset parity (odd/even x and y), frame edges, up/down scales."""
    W, H = 640, 360
    pitch = 640
    sizes = [(96, 64), (250, 130), (640, 360)]
    out_dims = [(max(1, int(np.floor(scale * w + 0.5))), max(1, int(np.floor(scale * h + 0.5)))) for w, h in sizes]
    frames = [S.frame_nv12_np(S.frame_seed(77, f), H, pitch) for f in range(2)]
    rng = np.random.default_rng(int(scale * 1000) + matrix)
    win = []
    for f in range(2):
        for q, (w, h) in enumerate(sizes):
            xs = sorted({0, min(1, W - w), W - w, max(0, W - w - 1), int(rng.integers(0, W - w + 1))})
            ys = sorted({0, min(1, H - h), H - h, max(0, H - h - 1), int(rng.integers(0, H - h + 1))})
            for x in xs:
                for y in ys:
                    win.append([f, x, y, w, h, q, 0])
    win = np.array(win, np.int32)
    for q in range(3):
        sel = np.nonzero(win[:, 5] == q)[0]
        win[sel, 6] = np.arange(len(sel))
    _compare(G, frames, pitch, W, H, win, sizes, out_dims, fmt, matrix)


@pytest.mark.parametrize("name,proxy", [("c2_1080p_sparse", (384, 216)), ("c1_540p", (240, 135)),
                                        ("c4_4k_drone", (480, 270))])
def test_nv12_full_frame_proxy_input(G, name, proxy):
    """The proxy's low-resolution input: one full-frame window
    per frame in a class whose out_dims is the proxy resolution."""
    cfg = S.CONFIGS[name]
    F = 6 if cfg.W <= 1920 else 2
    win = np.array([[f, 0, 0, cfg.W, cfg.H, 0, f] for f in range(F)], np.int32)
    _compare(G, _frames(cfg, 9, F), cfg.pitch_nv12, cfg.W, cfg.H, win, [(cfg.W, cfg.H)], [proxy], 0)


def test_nv12_grey_equals_rgb_path(G):
    """U = V = 128 and R = G = B = Y: the NV12 kernel's output equals the RGB
    kernel's output mapped by 255 (v - 16) / 219 (within fp32 rounding)."""
    import paper_2103_14695_b200 as mp
    W, H, pitch = 512, 288, 512
    nv = S.frame_nv12_np(5, H, pitch).copy()
    nv[H:] = 128
    rgb = np.zeros((H, 3 * W), np.uint8)
    rgb[:, :] = np.repeat(nv[:H, :W], 3, 1)
    win = np.array([[0, 3, 7, 200, 150, 0, 0], [0, 311, 137, 200, 150, 0, 1]], np.int32)
    st, a = G.gpu_gather([rgb], 3 * W, W, H, win, [(200, 150)], [(131, 97)], [2])
    st2, b = G.gpu_gather_nv12([nv], W, H, win, [(200, 150)], [(131, 97)], [2])
    assert st == st2 == 0
    e = np.clip((a[0].astype(np.float64) - 16) * 255 / 219, 0, 255)
    assert np.abs(b[0] - e).max() <= 1e-3
    assert mp.MP_BT709_LIMITED == 0


def test_nv12_invalid(G):
    import paper_2103_14695_b200 as mp
    W, H, pitch = 256, 128, 256
    fr = [S.frame_nv12_np(5, H, pitch)]
    win = np.array([[0, 0, 0, 64, 64, 0, 0], [0, 64, 0, 64, 64, 0, 1]], np.int32)
    st, got = G.gpu_gather_nv12(fr, W, H, win, [(64, 64)], [(32, 32)], [1])
    assert st == O.ERR_CAPACITY
    st_r, ref = O.gather_resize_nv12(fr, pitch, W, H, win[:1], [(64, 64)], [(32, 32)], [1])
    assert np.abs(got[0] - ref[0]).max() <= F32_TOL
    bad = np.array([[0, 200, 0, 64, 64, 0, 0]], np.int32)
    st, _ = G.gpu_gather_nv12(fr, W, H, bad, [(64, 64)], [(32, 32)], [1])
    assert st == O.ERR_INVALID
    with pytest.raises(mp.MPError):
        G.gpu_gather_nv12(fr, W, H, win[:1], [(64, 64)], [(32, 32)], [1], matrix=4)
    odd = [S.frame_nv12_np(5, 127, pitch)]   # H odd
    with pytest.raises(mp.MPError):
        G.gpu_gather_nv12(odd, W, 127, win[:1], [(64, 64)], [(32, 32)], [1])


def test_pipeline_nv12_runner_matches_oracle(G):
    """WindowPipeline(src='nv12', proxy_dims) through the 4-stream runner:
    proxy input, windows and crops equal the oracle's (c1, 12 frames)."""
    import paper_2103_14695_b200 as mp
    cfg = S.CONFIGS["c1_540p"]
    F = 12
    scene = S.make_scene(cfg, 2, F)
    scores = S.score_grids(cfg, 2, scene)
    frames_np = _frames(cfg, 2, F)
    ref_plan = O.plan_windows(cfg.W, cfg.H, 32, 32, cfg.b_proxy, cfg.sizes, cfg.cost, scores)
    caps = [int(c) for c in ref_plan["class_count"]]
    dev = torch.device("cuda:0")
    pipes = []
    for _ in range(2):
        p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                              cfg.iou_thr, device=dev, src="nv12", proxy_dims=cfg.proxy_dims)
        p.reserve(F, len(ref_plan["windows"]), caps=caps, max_boxes=1)
        pipes.append(p)
    runner = mp.PipelinedRunner(pipes, device=dev)
    fr = torch.from_numpy(np.stack(frames_np)).to(dev)
    sc = torch.from_numpy(scores).to(dev)
    for _ in range(3):
        runner.step(sc, fr)
    runner.wait_all()
    torch.cuda.synchronize()
    for p in pipes:
        p.check_status()
        assert np.array_equal(p.windows[:len(ref_plan["windows"])].cpu().numpy(), ref_plan["windows"])
        st, ref = O.gather_resize_nv12(frames_np, cfg.pitch_nv12, cfg.W, cfg.H, ref_plan["windows"], cfg.sizes,
                                       cfg.out_dims, caps)
        for q in range(len(caps)):
            if caps[q]:
                assert np.abs(p.outs[q].cpu().numpy() - ref[q]).max() <= F32_TOL
        pw = [[f, 0, 0, cfg.W, cfg.H, 0, f] for f in range(F)]
        st, pref = O.gather_resize_nv12(frames_np, cfg.pitch_nv12, cfg.W, cfg.H, pw, [(cfg.W, cfg.H)],
                                        [cfg.proxy_dims], [F])
        assert np.abs(p.proxy_out.cpu().numpy() - pref[0]).max() <= F32_TOL


def test_full_size_nv12_bench_config_parity(G):
    """configs[1] at full size (1800 NV12 1080p frames) through the 4-stream
    PipelinedRunner as `bench.py --src nv12` runs it: windows exact; crop and
    proxy-input pixels on seeded samples, each recomputed by the oracle."""
    import paper_2103_14695_b200 as mp
    cfg = S.CONFIGS["c2_1080p_sparse"]
    F = cfg.frames
    scene = S.make_scene(cfg, 0, F)
    scores = S.score_grids(cfg, 0, scene)
    ref = O.plan_windows(cfg.W, cfg.H, 32, 32, cfg.b_proxy, cfg.sizes, cfg.cost, scores)
    caps = [int(c) for c in ref["class_count"]]
    n = len(ref["windows"])
    pipes = []
    for _ in range(2):
        p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                              cfg.iou_thr, device=G.DEV, src="nv12", proxy_dims=cfg.proxy_dims)
        p.reserve(F, n + 64, caps=caps, max_boxes=1)
        pipes.append(p)
    runner = mp.PipelinedRunner(pipes, device=G.DEV)
    frames = S.frame_pixels_torch([S.frame_seed(0, f) for f in range(F)], cfg.H + cfg.H // 2, cfg.pitch_nv12,
                                  device=G.DEV)
    sc = torch.from_numpy(scores).to(G.DEV)
    runner.capture_graphs(sc)
    for _ in range(3):
        runner.step(sc, frames)
    runner.wait_all()
    torch.cuda.synchronize()
    rng = np.random.default_rng(77)
    for p in pipes:
        p.check_status()
        assert np.array_equal(p.windows[:n].cpu().numpy(), ref["windows"])
        for wi in rng.choice(n, size=25, replace=False):
            w = ref["windows"][wi].copy()
            f, q, slot = int(w[0]), int(w[5]), int(w[6])
            fr = S.frame_nv12_np(S.frame_seed(0, f), cfg.H, cfg.pitch_nv12)
            one = w.copy(); one[0] = 0; one[6] = 0
            caps1 = [1 if qq == q else 0 for qq in range(len(cfg.sizes))]
            st, o = O.gather_resize_nv12([fr], cfg.pitch_nv12, cfg.W, cfg.H, one[None], cfg.sizes, cfg.out_dims,
                                         caps1)
            assert np.abs(p.outs[q][slot].cpu().numpy() - o[q][0]).max() <= F32_TOL
        for f in rng.choice(F, size=6, replace=False):
            fr = S.frame_nv12_np(S.frame_seed(0, int(f)), cfg.H, cfg.pitch_nv12)
            st, o = O.gather_resize_nv12([fr], cfg.pitch_nv12, cfg.W, cfg.H, [[0, 0, 0, cfg.W, cfg.H, 0, 0]],
                                         [(cfg.W, cfg.H)], [cfg.proxy_dims], [1])
            assert np.abs(p.proxy_out[int(f)].cpu().numpy() - o[0][0]).max() <= F32_TOL


@pytest.mark.parametrize("matrix", [0, 3])
def test_nv12_fixed_tap_4_3_classes(G, matrix):
    """The NV12 fixed-tap consumer (consume_tile_r43nv, f32 out): 4:3 classes
    tiled with every column-group width (ncg 16 / 8 / 4), windows on the
    16-px grid (fixed-tap path) and off it (per-column fallback in the same
    launch), odd and even window y (the chroma-row parity of the task rows),
    a full-frame class and ragged row tiles — within 1e-3 of the oracle."""
    W, H = 960, 540
    pitch = W
    sizes = [(64, 64), (128, 128), (256, 256), (512, 384), (960, 540)]
    out_dims = [(48, 48), (96, 96), (192, 192), (384, 288), (720, 405)]
    frames = [S.frame_nv12_np(S.frame_seed(71, f), H, pitch) for f in range(2)]
    rng = np.random.default_rng(434)
    win = []
    for f in range(2):
        for q, (w, h) in enumerate(sizes):
            xs = {0, W - w, 16 * int(rng.integers(0, (W - w) // 16 + 1)), int(rng.integers(0, W - w + 1))}
            ys = {0, H - h, 2 * int(rng.integers(0, (H - h) // 2 + 1))}
            if H - h >= 2:
                ys.add(2 * int(rng.integers(0, (H - h) // 2)) + 1)   # odd y: chroma rows at the other parity
            for x in sorted(xs):
                for y in sorted(y for y in ys if 0 <= y <= H - h):
                    win.append([f, x, y, w, h, q, 0])
    win = np.array(win, np.int32)
    for q in range(len(sizes)):
        sel = np.nonzero(win[:, 5] == q)[0]
        win[sel, 6] = np.arange(len(sel))
    _compare(G, frames, pitch, W, H, win, sizes, out_dims, 0, matrix)
