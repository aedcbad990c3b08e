"""GPU parity of the zero-copy input path: frames left in page-locked host
memory and read by the gather kernels over PCIe (only the window footprints
cross the bus).  Results must equal the oracle within the a5 tolerances and be
bit-identical to the same call on frames resident in HBM (the kernel is the
same; only the source address space differs)."""
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


def _check(got, ref, caps, fmt):
    for q in range(len(caps)):
        if caps[q] == 0:
            continue
        if fmt == 0:
            err = np.abs(got[q].astype(np.float64) - ref[q]).max()
            assert err <= F32_TOL, (q, err)
        else:
            d = np.abs(got[q].astype(np.int32) - ref[q].astype(np.int32))
            assert d.max() <= 1, (q, d.max())


@pytest.mark.parametrize("strided", [True, False], ids=["tma_tensor", "ptr_array"])
@pytest.mark.parametrize("fmt", [0, 1])
@pytest.mark.parametrize("name,frames", [("c1_540p", 30), ("c2_1080p_sparse", 24), ("c4_4k_drone", 2)])
def test_zero_copy_gather_parity(G, name, frames, fmt, strided):
    cfg = S.CONFIGS[name]
    scene = S.make_scene(cfg, 6, frames)
    scores = S.score_grids(cfg, 6, scene)
    plan = O.plan_windows(cfg.W, cfg.H, 32, 32, cfg.b_proxy, cfg.sizes, cfg.cost, scores)
    win = plan["windows"]
    caps = [int(c) for c in plan["class_count"]]
    fr = [S.frame_pixels_np(S.frame_seed(6, f), cfg.H, cfg.pitch) for f in range(frames)]
    st_r, ref = O.gather_resize(fr, cfg.pitch, cfg.W, cfg.H, win, cfg.sizes, cfg.out_dims, caps,
                                O.F32_NCHW if fmt == 0 else O.U8_NHWC)
    st_h, host = G.gpu_gather(fr, cfg.pitch, cfg.W, cfg.H, win, cfg.sizes, cfg.out_dims, caps, fmt, strided,
                              host=True)
    st_d, dev = G.gpu_gather(fr, cfg.pitch, cfg.W, cfg.H, win, cfg.sizes, cfg.out_dims, caps, fmt, strided)
    assert st_h == st_d == st_r == 0
    _check(host, ref, caps, fmt)
    for q in range(len(caps)):
        assert np.array_equal(host[q], dev[q])


@pytest.mark.parametrize("fmt", [0, 1])
@pytest.mark.parametrize("scale", [1.0, 0.37, 1.5])
def test_zero_copy_gather_edges(G, scale, fmt):
    """Windows touching every frame edge, odd output widths, strong downscale
    (row-sparse staging) and upscale, frames in pinned host memory."""
    W, H = 640, 360
    pitch = (3 * W + 15) // 16 * 16
    sizes = [(96, 64), (250, 130), (640, 360)]
    out_dims = [(max(1, int(np.floor(scale * w + 0.5))), max(1, int(np.floor(scale * h + 0.5)))) for w, h in sizes]
    frames = [S.frame_pixels_np(S.frame_seed(77, f), H, pitch) for f in range(3)]
    win = []
    for f in range(3):
        for q, (w, h) in enumerate(sizes):
            for x in sorted({0, W - w, (W - w) // 3}):
                for y in sorted({0, H - h, (H - h) // 2}):
                    win.append([f, x, y, w, h, q, 0])
    win = np.array(win, np.int32)
    for q in range(3):
        sel = np.nonzero(win[:, 5] == q)[0]
        win[sel, 6] = np.arange(len(sel))
    caps = [int((win[:, 5] == q).sum()) for q in range(3)]
    st_r, ref = O.gather_resize(frames, pitch, W, H, win, sizes, out_dims, caps,
                                O.F32_NCHW if fmt == 0 else O.U8_NHWC)
    for strided in (True, False):
        st, got = G.gpu_gather(frames, pitch, W, H, win, sizes, out_dims, caps, fmt, strided, host=True)
        assert st == st_r == 0
        _check(got, ref, caps, fmt)


@pytest.mark.parametrize("fmt", [0, 1])
def test_zero_copy_nv12_parity(G, fmt):
    cfg = S.CONFIGS["c2_1080p_sparse"]
    F = 12
    scene = S.make_scene(cfg, 8, F)
    scores = S.score_grids(cfg, 8, scene)
    plan = O.plan_windows(cfg.W, cfg.H, 32, 32, cfg.b_proxy, cfg.sizes, cfg.cost, scores)
    win = plan["windows"]
    caps = [int(c) for c in plan["class_count"]]
    fr = [S.frame_nv12_np(S.frame_seed(8, f), cfg.H, cfg.pitch_nv12) for f in range(F)]
    st_r, ref = O.gather_resize_nv12(fr, cfg.pitch_nv12, cfg.W, cfg.H, win, cfg.sizes, cfg.out_dims, caps,
                                     O.F32_NCHW if fmt == 0 else O.U8_NHWC, O.BT709_LIMITED)
    st_h, host = G.gpu_gather_nv12(fr, cfg.W, cfg.H, win, cfg.sizes, cfg.out_dims, caps, fmt, host=True)
    st_d, dev = G.gpu_gather_nv12(fr, cfg.W, cfg.H, win, cfg.sizes, cfg.out_dims, caps, fmt)
    assert st_h == st_d == st_r == 0
    _check(host, ref, caps, fmt)
    for q in range(len(caps)):
        assert np.array_equal(host[q], dev[q])


def test_zero_copy_pipeline_end_to_end(G):
    """The e2e leg of bench.py: scores and detector boxes copied H2D, frames
    read zero-copy from a pinned host pool through WindowPipeline's pointer
    path, kept boxes read back — windows and kept boxes bit-exact, sampled
    pixels within 1e-3 of the oracle."""
    import paper_2103_14695_b200 as mp
    cfg = S.CONFIGS["c2_1080p_sparse"]
    F, pool = 96, 32
    scene = S.make_scene(cfg, 2, F)
    scores = S.score_grids(cfg, 2, scene)
    ref = O.plan_windows(cfg.W, cfg.H, 32, 32, cfg.b_proxy, cfg.sizes, cfg.cost, scores)
    boxes, wbo = S.standin_boxes(cfg, 2, scene, ref["windows"])
    r = O.remap_nms(boxes, wbo, ref["windows"], ref["frame_off"], cfg.out_dims, cfg.W, cfg.H, cfg.score_thr,
                    cfg.iou_thr)
    host = torch.from_numpy(np.stack([S.frame_pixels_np(S.frame_seed(2, i), cfg.H, cfg.pitch)
                                      for i in range(pool)])).pin_memory()
    base = mp.WindowPipeline.frame_ptrs(host)          # host addresses, on the host
    assert not base.is_cuda
    ptrs = base[torch.arange(F) % pool].to(G.DEV)
    pipe = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                             cfg.iou_thr, device=G.DEV)
    n = len(ref["windows"])
    pipe.reserve(F, n, caps=[int(c) for c in ref["class_count"]], max_boxes=max(len(boxes), 1))
    pipe.plan(torch.from_numpy(scores).pin_memory().to(G.DEV, non_blocking=True))
    pipe.gather(ptrs)
    pipe.merge(G.boxes_to_t(boxes), torch.from_numpy(wbo).to(G.DEV))
    torch.cuda.synchronize()
    pipe.check_status()
    assert np.array_equal(pipe.windows[:n].cpu().numpy(), ref["windows"])
    nk = int(pipe.nms_frame_off[F].item())
    assert np.array_equal(pipe.nms_src[:nk].cpu().numpy(), r["src"])
    assert np.array_equal(pipe.nms_out[:nk].cpu().numpy().view(np.uint32),
                          r["boxes"].view(np.float32).reshape(-1, 6).view(np.uint32))
    rng = np.random.default_rng(9)
    for wi in rng.choice(n, size=min(24, n), replace=False):
        w = ref["windows"][wi].copy()
        f, q, slot = int(w[0]), int(w[5]), int(w[6])
        fr = S.frame_pixels_np(S.frame_seed(2, f % pool), cfg.H, cfg.pitch)
        one = w.copy(); one[0] = 0; one[6] = 0
        caps1 = [1 if qq == q else 0 for qq in range(len(cfg.sizes))]
        st, o = O.gather_resize([fr], cfg.pitch, cfg.W, cfg.H, one[None], cfg.sizes, cfg.out_dims, caps1)
        assert np.abs(pipe.outs[q][slot].cpu().numpy() - o[q][0]).max() <= F32_TOL


def test_pageable_host_frames_rejected(G):
    import paper_2103_14695_b200 as mp
    fr = torch.zeros((2, 8, 32), dtype=torch.uint8)      # pageable: the GPU cannot address it
    with pytest.raises(ValueError):
        mp.WindowPipeline.frame_ptrs(fr)
    pipe = mp.WindowPipeline(8, 8, [(8, 8)], [1], [(8, 8)], device=G.DEV)
    pipe.reserve(2, 2, caps=[2])
    with pytest.raises(ValueError):
        pipe.gather(fr)


@pytest.mark.parametrize("src", ["nv12", "rgb24"])
def test_zero_copy_proxy_input(G, src):
    """NEXT-3's full-frame proxy-input downscale (row-sparse TMA row gathers)
    reading the frames from pinned host memory: bit-identical to the same
    call on frames in HBM, and within 1e-3 of the oracle."""
    import paper_2103_14695_b200 as mp
    cfg = S.CONFIGS["c2_1080p_sparse"]
    F = 8
    if src == "nv12":
        fr = [S.frame_nv12_np(S.frame_seed(12, f), cfg.H, cfg.pitch_nv12) for f in range(F)]
    else:
        fr = [S.frame_pixels_np(S.frame_seed(12, f), cfg.H, cfg.pitch) for f in range(F)]
    host = torch.from_numpy(np.stack(fr)).pin_memory()
    dev = host.to(G.DEV)
    outs = []
    for frames in (host, dev):
        p = mp.WindowPipeline(cfg.W, cfg.H, cfg.sizes, cfg.cost, cfg.out_dims, cfg.b_proxy, cfg.score_thr,
                              cfg.iou_thr, device=G.DEV, src=src, proxy_dims=cfg.proxy_dims)
        p.reserve(F, 1)
        p.proxy_input(frames)
        torch.cuda.synchronize()
        p.check_status()
        outs.append(p.proxy_out.cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    win = np.array([[f, 0, 0, cfg.W, cfg.H, 0, f] for f in range(F)], np.int32)
    if src == "nv12":
        st, ref = O.gather_resize_nv12(fr, cfg.pitch_nv12, cfg.W, cfg.H, win, [(cfg.W, cfg.H)], [cfg.proxy_dims], [F],
                                       O.F32_NCHW, O.BT709_LIMITED)
    else:
        st, ref = O.gather_resize(fr, cfg.pitch, cfg.W, cfg.H, win, [(cfg.W, cfg.H)], [cfg.proxy_dims], [F])
    assert st == 0
    assert np.abs(outs[0].astype(np.float64) - ref[0]).max() <= F32_TOL
