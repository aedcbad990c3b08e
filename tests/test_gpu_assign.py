"""GPU parity of NEXT-4a (mp_hungarian, reading R24) against the oracle's
mpo_hungarian: the kernel runs the same shortest-augmenting-path steps in the
same fp64 order, so row/column matches and totals must be bit-identical —
across both tiers (warp per problem S <= 64, CTA per problem S <= 1024),
tie-heavy quantised scores, NaN, empty and rectangular problems, and the
capacity / invalid paths."""
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


def _check(G, mats, floor=0.5):
    st, rows, cols, tot = G.gpu_hungarian(mats, floor)
    assert st == 0
    for b, a in enumerate(mats):
        sr, rm, cm, t = O.hungarian(a, floor)
        assert sr == 0
        assert np.array_equal(rows[b], rm), b
        assert np.array_equal(cols[b], cm), b
        assert tot[b] == t, (b, tot[b], t)


@pytest.mark.parametrize("mr,nr", [((3, 40), (3, 40)), ((1, 64), (1, 64)), ((50, 130), (40, 150))])
def test_hungarian_parity_synth(G, mr, nr):
    mats = S.assign_batch(7 + mr[1], 300 if mr[1] <= 64 else 60, mr, nr)
    _check(G, mats)


@pytest.mark.parametrize("floor", [0.05, 0.5, 0.95])
def test_hungarian_parity_random_and_ties(G, floor):
    rng = np.random.default_rng(int(floor * 100))
    mats = []
    for i in range(200):
        m, n = (int(x) for x in rng.integers(1, 90, 2))
        a = rng.random((m, n)).astype(np.float32)
        if i % 3 == 0:
            a = (np.round(a * 4) / 4).astype(np.float32)   # many exact ties
        if i % 7 == 0:
            a[rng.random((m, n)) < 0.05] = np.nan
        mats.append(a)
    _check(G, mats, floor)


def test_hungarian_large_and_degenerate(G):
    rng = np.random.default_rng(5)
    mats = [rng.random((300, 280)).astype(np.float32), rng.random((1, 700)).astype(np.float32),
            rng.random((1024, 3)).astype(np.float32), np.zeros((0, 5), np.float32), np.zeros((4, 0), np.float32),
            np.full((6, 6), 0.2, np.float32), np.ones((65, 65), np.float32)]
    _check(G, mats)


def test_hungarian_capacity_and_invalid(G):
    import paper_2103_14695_b200 as mp
    rng = np.random.default_rng(9)
    mats = [rng.random((10, 10)).astype(np.float32), rng.random((80, 20)).astype(np.float32)]
    st, rows, cols, tot = G.gpu_hungarian(mats, 0.5, max_dim=64)
    assert st == O.ERR_CAPACITY
    assert (rows[1] == -1).all() and (cols[1] == -1).all()
    sr, rm, cm, t = O.hungarian(mats[0], 0.5)
    assert np.array_equal(rows[0], rm) and tot[0] == t
    with pytest.raises(mp.MPError):
        G.gpu_hungarian(mats, 0.0)
    with pytest.raises(mp.MPError):
        G.gpu_hungarian(mats, 0.5, max_dim=2000)
