"""NEXT-2 — window-size set selection: greedy over all
multiple-of-32 candidates minimising tot_time(S + {(w,h)}) with a perfect
proxy.  CPU tests pin the oracle to SPEC.md:239-247's examples, to the
objective recomputed from independent per-candidate plans, and to the
monotonicity the greedy guarantees; GPU tests compare objectives and the
selected sets exactly."""
import numpy as np
import pytest

import oracle as O
from workloads import synth as S


def cost_fn(w, h):
    return -(-w // 32) * -(-h // 32) + 16


def _labels(name, clip, frames):
    cfg = S.CONFIGS[name]
    scene = S.make_scene(cfg, clip, frames)
    return cfg, np.stack([S.cell_labels(cfg, b) for b in scene.boxes]).astype(np.float32)


def test_spec_all_frames_empty_tie_break():
    # all frames empty -> every addition ties at tot 0 -> smallest area, then smaller w
    s = np.zeros((5, 3, 4), np.float32)
    sizes, hist = O.select_window_sizes(128, 96, 32, 32, s, 3, cost_fn)
    assert sizes == [(128, 96), (32, 32), (32, 64)] and hist == [0, 0]


def test_spec_one_cell_object_picks_one_cell_window():
    # every frame has one 32x32 object -> second size = the smallest size covering one cell
    s = np.zeros((4, 3, 4), np.float32)
    for f, (r, c) in enumerate([(0, 0), (1, 2), (2, 3), (1, 1)]):
        s[f, r, c] = 1.0
    sizes, hist = O.select_window_sizes(128, 96, 32, 32, s, 2, cost_fn)
    assert sizes == [(128, 96), (32, 32)] and hist == [4 * cost_fn(32, 32)]


def test_objective_equals_sum_of_independent_plans():
    cfg, lab = _labels("c1_540p", 2, 8)
    S0 = [(cfg.W, cfg.H)]
    cand = [(256, 256), (96, 64), (32, 32), (512, 288), (960, 32)]
    st, tot = O.window_set_cost(cfg.W, cfg.H, 32, 32, 0.5, S0, [cost_fn(*s) for s in S0], lab, cand,
                                [cost_fn(*c) for c in cand])
    assert st == 0
    for c, t in zip(cand, tot):
        sz = S0 + [c]
        cs = [cost_fn(*x) for x in sz]
        r = O.plan_windows(cfg.W, cfg.H, 32, 32, 0.5, sz, cs, lab)
        assert t == sum(cs[w[5]] for w in r["windows"])


def test_greedy_objective_is_monotone():
    cfg, lab = _labels("c1_540p", 3, 6)
    sizes, hist = O.select_window_sizes(cfg.W, cfg.H, 32, 32, lab, 4, cost_fn, step=64)
    full_only = sum(cost_fn(cfg.W, cfg.H) for f in range(lab.shape[0]) if lab[f].any())
    assert len(sizes) == 4 and len(set(sizes)) == 4 and sizes[0] == (cfg.W, cfg.H)
    assert hist[0] <= full_only and all(b <= a for a, b in zip(hist, hist[1:]))


@pytest.mark.gpu
@pytest.mark.parametrize("name,frames,k,step", [("c1_540p", 30, 3, 32), ("c2_1080p_sparse", 40, 3, 32)])
def test_gpu_window_selection_parity(name, frames, k, step):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2103_14695_b200 import window_sets
    cfg, lab = _labels(name, 5, frames)
    ref_sizes, ref_hist = O.select_window_sizes(cfg.W, cfg.H, 32, 32, lab, k, cost_fn, step=step)
    got_sizes, got_hist = window_sets.select_window_sizes(torch.from_numpy(lab).cuda(), cfg.W, cfg.H, k, cost_fn,
                                                          step=step)
    assert got_sizes == ref_sizes and got_hist == ref_hist
