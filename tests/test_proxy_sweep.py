"""NEXT-1 — proxy-module caching sweep: per-threshold
runtime estimate (sum of T over the planned windows) and recall (fraction of
theta_best detections covered by the windows).  CPU tests pin the oracle's
sweep to per-threshold plans + an independent numpy coverage count and to
hand-derived cases; GPU tests compare the CUDA sweep with the oracle exactly."""
import numpy as np
import pytest

import oracle as O
from workloads import synth as S


def _numpy_sweep(W, H, cw, ch, sizes, cost, scores, thresholds, dets, det_off):
    out = np.zeros((len(thresholds), 5), np.int64)
    full = [i for i, s in enumerate(sizes) if tuple(s) == (W, H)][0]
    for j, b in enumerate(thresholds):
        r = O.plan_windows(W, H, cw, ch, b, sizes, cost, scores)
        w, fo = r["windows"], r["frame_off"]
        out[j, 0] = sum(cost[x[5]] for x in w)
        out[j, 1] = len(w)
        for f in range(scores.shape[0]):
            ww = w[fo[f]:fo[f + 1]]
            if len(ww) == 1 and ww[0, 5] == full:
                out[j, 2] += 1
            d = dets[det_off[f]:det_off[f + 1]]
            if len(d) == 0:
                continue
            x0, y0 = ww[:, 1][None, :], ww[:, 2][None, :]
            x1, y1 = (ww[:, 1] + ww[:, 3])[None, :], (ww[:, 2] + ww[:, 4])[None, :]
            inside = (d[:, :1] >= x0) & (d[:, 2:3] <= x1) & (d[:, 1:2] >= y0) & (d[:, 3:4] <= y1)
            touch = (d[:, :1] < x1) & (d[:, 2:3] > x0) & (d[:, 1:2] < y1) & (d[:, 3:4] > y0)
            out[j, 3] += int(inside.any(axis=1).sum()) if len(ww) else 0
            out[j, 4] += int(touch.any(axis=1).sum()) if len(ww) else 0
    return out


def _workload(name, clip, frames):
    cfg = S.CONFIGS[name]
    scene = S.make_scene(cfg, clip, frames)
    scores = S.score_grids(cfg, clip, scene)
    dets = np.concatenate([b for b in scene.boxes]).astype(np.float32) if frames else np.zeros((0, 4), np.float32)
    det_off = np.concatenate([[0], np.cumsum([len(b) for b in scene.boxes])]).astype(np.int32)
    return cfg, scores, dets, det_off


def test_oracle_sweep_matches_per_threshold_plans():
    cfg, scores, dets, det_off = _workload("c5_1080p_clips", 7, 30)
    th = list(S.B_SWEEP)
    st, got = O.proxy_sweep(cfg.W, cfg.H, 32, 32, cfg.sizes, cfg.cost, scores, th, dets, det_off)
    assert st == 0
    ref = _numpy_sweep(cfg.W, cfg.H, 32, 32, cfg.sizes, cfg.cost, scores, th, dets, det_off)
    assert np.array_equal(got, ref)
    # noise-free proxy at B well below the positive scores covers (touches) every detection
    assert got[0, 4] <= len(dets)


def test_oracle_sweep_hand_cases():
    # 256x192 frame, 32-px cells, S = {64x64, 256x192}, T = {20, 64}
    W, H, sizes, cost = 256, 192, [(64, 64), (256, 192)], [20, 64]
    s = np.zeros((1, 6, 8), np.float32)
    s[0, 0, 0] = 0.9          # cell (0,0): window (0,0,64,64) (clamped, centred)
    s[0, 5, 7] = 0.6          # cell (5,7): window (192,128,64,64)
    dets = np.array([[2, 2, 30, 30],        # inside window 1
                     [40, 40, 70, 70],      # crosses window 1's edge: touched, not covered
                     [200, 140, 250, 190],  # inside window 2 (only when B < 0.6)
                     [100, 100, 120, 120]], np.float32)   # in no window
    st, out = O.proxy_sweep(W, H, 32, 32, sizes, cost, s, [0.5, 0.7, 0.95], dets, [0, 4])
    assert st == 0
    # B=0.5: two 64x64 windows (20+20 < 64), covered {d0, d2}, touched {d0, d1, d2}
    assert out[0].tolist() == [40, 2, 0, 2, 3]
    # B=0.7: one window (cell (0,0))
    assert out[1].tolist() == [20, 1, 0, 1, 2]
    # B=0.95: nothing positive, no windows, recall 0
    assert out[2].tolist() == [0, 0, 0, 0, 0]


@pytest.mark.gpu
@pytest.mark.parametrize("name,frames", [("c5_1080p_clips", 200), ("c4_4k_drone", 16), ("c1_540p", 30)])
def test_gpu_sweep_parity(name, frames):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2103_14695_b200 as mp
    cfg, scores, dets, det_off = _workload(name, 3, frames)
    th = list(S.B_SWEEP) + [0.0, 0.999, 0.5]
    st, ref = O.proxy_sweep(cfg.W, cfg.H, 32, 32, cfg.sizes, cfg.cost, scores, th, dets, det_off)
    dev = torch.device("cuda:0")
    p = mp.PlanParams(cfg.W, cfg.H, cfg.sizes, cfg.cost)
    out = torch.full((len(th), 5), -1, dtype=torch.int64, device=dev)
    ws = torch.empty(mp.mp_proxy_sweep_workspace_size(p, frames), dtype=torch.uint8, device=dev)
    d = torch.from_numpy(dets if len(dets) else np.zeros((1, 4), np.float32)).to(dev)
    mp.mp_proxy_sweep(p, torch.from_numpy(scores).to(dev), frames, th, d, torch.from_numpy(det_off).to(dev),
                      out, ws)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)


@pytest.mark.gpu
def test_gpu_sweep_single_pass_edges():
    """The single-pass sweep ranks each cell once against the SORTED
    thresholds and re-uses a plan when a threshold leaves the mask unchanged:
    unsorted / duplicated / +-inf thresholds, scores exactly equal to a
    threshold, NaN and +-inf scores, and a quantised score grid where most
    thresholds select identical masks."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2103_14695_b200 as mp
    cfg, scores, dets, det_off = _workload("c5_1080p_clips", 5, 60)
    rng = np.random.default_rng(11)
    q = np.round(scores * 4) / 4                      # values in {0, .25, .5, .75, 1}: few distinct masks
    q = q.astype(np.float32)
    q[rng.random(q.shape) < 0.01] = np.nan
    q[rng.random(q.shape) < 0.005] = np.inf
    q[rng.random(q.shape) < 0.005] = -np.inf
    th = [0.5, 0.25, 0.5, 0.3, 0.75, -np.inf, np.inf, 0.74999994, 0.25, 1.0, 0.0, 0.6, 0.7, 0.5]
    st, ref = O.proxy_sweep(cfg.W, cfg.H, 32, 32, cfg.sizes, cfg.cost, q, th, dets, det_off)
    assert st == 0
    dev = torch.device("cuda:0")
    p = mp.PlanParams(cfg.W, cfg.H, cfg.sizes, cfg.cost)
    F = q.shape[0]
    out = torch.full((len(th), 5), -1, dtype=torch.int64, device=dev)
    ws = torch.empty(mp.mp_proxy_sweep_workspace_size(p, F), dtype=torch.uint8, device=dev)
    mp.mp_proxy_sweep(p, torch.from_numpy(q).to(dev), F, th, torch.from_numpy(dets).to(dev),
                      torch.from_numpy(det_off).to(dev), out, ws)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.array_equal(got, ref)
    # duplicated thresholds give identical rows; thresholds between two grid values too
    assert np.array_equal(got[0], got[2]) and np.array_equal(got[1], got[8])
    assert np.array_equal(got[11], got[12]) and np.array_equal(got[11], got[0]) and np.array_equal(got[7], got[0])
