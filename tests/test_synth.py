"""The shared input generator: numpy and torch produce identical frame bytes
(so the GPU bench can synthesise frames in HBM and the oracle can regenerate
any sampled frame on the host), and every draw is seed-deterministic."""
import numpy as np
import torch

from workloads import synth as S


def test_splitmix64_reference_values():
    # splitmix64 stream from state 0: first output 0xE220A8397B1DCDAF (Vigna's reference generator)
    assert S.splitmix64(0) == 0xE220A8397B1DCDAF
    z = np.asarray(S.frame_pixels_np(0, 1, 8)).view(np.uint64).ravel()[0]
    assert int(z) == 0xE220A8397B1DCDAF


def test_pixels_numpy_equals_torch():
    seeds = [S.frame_seed(3, f) for f in range(4)] + [2**64 - 5, 0]
    t = S.frame_pixels_torch(seeds, 37, 112)
    for i, sd in enumerate(seeds):
        assert np.array_equal(t[i].numpy(), S.frame_pixels_np(sd, 37, 112))


def test_scene_and_scores_deterministic():
    cfg = S.CONFIGS["c2_1080p_sparse"]
    a = S.make_scene(cfg, 7, 40)
    b = S.make_scene(cfg, 7, 40)
    assert all(np.array_equal(x, y) for x, y in zip(a.boxes, b.boxes))
    g1, g2 = S.score_grids(cfg, 7, a), S.score_grids(cfg, 7, b)
    assert np.array_equal(g1, g2) and g1.shape == (40, 34, 60) and g1.dtype == np.float32
    # a sub-range of frames regenerates the same objects (per-shard generation)
    c = S.make_scene(cfg, 7, 10, frame0=30)
    assert all(np.array_equal(x, y) for x, y in zip(a.boxes[30:], c.boxes))


def test_cell_labels_positive_area_rule():
    cfg = S.CONFIGS["c1_540p"]
    lab = S.cell_labels(cfg, np.array([[32.0, 32.0, 64.0, 64.0]]))     # exactly one cell
    assert lab.sum() == 1 and lab[1, 1] == 1
    lab = S.cell_labels(cfg, np.array([[31.5, 32.0, 64.5, 64.0]]))
    assert lab.sum() == 3
