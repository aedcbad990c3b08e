"""GPU parity of NEXT-4b (mp_track_resample, mp_dbscan, mp_cluster_centers,
mp_refine_tracks; readings R25-R27) against the oracle.  Every step runs the
oracle's fp64 operations in the oracle's order, so paths, labels, core flags,
centres, counts, refined endpoints and taken counts are compared
bit-for-bit."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
from workloads import synth as S  # noqa: E402

N = O.TRACK_N


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import gpu_util
    return gpu_util


def _oracle(train, query, eps, min_pts, cell=32.0, k=10):
    tp = np.stack([O.track_resample(O.box_centers(b), N) for b in train])
    qc = [O.box_centers(b) for b in query]
    qp = np.stack([O.track_resample(c, N) for c in qc])
    lab, core, nd, C = O.dbscan(tp, eps, min_pts)
    ctr, cnt = O.cluster_centers(tp, lab, C)
    outs, taken = [], []
    for p, c in zip(qp, qc):
        n, o = O.refine_track(p, c[0], c[-1], ctr, cnt, cell, k)
        outs.append(o)
        taken.append(n)
    return dict(train_paths=tp, query_paths=qp, labels=lab, is_core=core, nd=nd, C=C, centers=ctr, counts=cnt,
                out=np.asarray(outs), taken=np.asarray(taken))


@pytest.mark.parametrize("seed,n_train,n_query,lanes,eps_frac,min_pts",
                         [(1, 300, 200, 8, 0.05, 2), (2, 500, 300, 12, 0.03, 3), (3, 120, 80, 4, 0.08, 5),
                          (4, 200, 100, 16, 0.01, 2)])
def test_refine_pipeline_parity(G, seed, n_train, n_query, lanes, eps_frac, min_pts):
    _, train, query, _ = S.track_sets(seed, n_train, n_query, lanes, gap=16)
    eps = eps_frac * math.hypot(1920, 1080)
    ref = _oracle(train, query, eps, min_pts)
    got = G.gpu_refine_pipeline(train, query, eps, min_pts)
    assert got["status"] == 0
    assert np.array_equal(got["train_paths"], ref["train_paths"])
    assert np.array_equal(got["query_paths"], ref["query_paths"])
    assert np.array_equal(got["labels"], ref["labels"])
    assert np.array_equal(got["is_core"], ref["is_core"])
    assert got["nclust"].tolist() == [ref["nd"], ref["C"]]
    assert np.array_equal(got["counts"], ref["counts"])
    assert np.array_equal(got["centers"], ref["centers"])
    assert np.array_equal(got["taken"], ref["taken"])
    assert np.array_equal(got["out"], ref["out"])


def test_refine_degenerate_tracks(G):
    """Single-detection tracks, zero-length tracks, duplicates, tracks leaving
    the frame, and a query far from every cluster (unchanged)."""
    rng = np.random.default_rng(3)
    train = [np.array([[100, 100, 110, 110]], np.float32),
             np.array([[500, 500, 520, 520]] * 4, np.float32),
             np.array([[-50, 300, -10, 340], [300, 300, 340, 340], [2000, 320, 2040, 360]], np.float32)]
    for _ in range(40):
        y = rng.uniform(200, 900)
        pts = np.stack([np.linspace(0, 1920, 30), np.full(30, y) + rng.normal(0, 2, 30)], 1)
        train.append(np.concatenate([pts - 15, pts + 15], 1).astype(np.float32))
    query = [t[len(t) // 3: 2 * len(t) // 3: 3] if len(t) > 6 else t for t in train[3:20]]
    query += [np.array([[900, 20, 930, 50], [1000, 22, 1030, 52]], np.float32), train[0], train[1]]
    eps = 40.0
    ref = _oracle(train, query, eps, 2)
    got = G.gpu_refine_pipeline(train, query, eps, 2)
    assert got["status"] == 0
    for key in ("train_paths", "query_paths", "labels", "is_core", "counts", "centers", "taken", "out"):
        assert np.array_equal(got[key], ref[key]), key


def test_refine_invalid_and_capacity(G):
    import paper_2103_14695_b200 as mp
    _, train, query, _ = S.track_sets(5, 100, 20, 6, gap=16)
    with pytest.raises(mp.MPError):
        G.gpu_refine_pipeline(train, query, -1.0, 2)              # eps <= 0
    with pytest.raises(mp.MPError):
        G.gpu_refine_pipeline(train, query, 50.0, 2, N=1)         # N < 2
    got = G.gpu_refine_pipeline(train, query, 50.0, 2, C_max=2)   # more clusters than C_max
    assert got["status"] == O.ERR_CAPACITY
