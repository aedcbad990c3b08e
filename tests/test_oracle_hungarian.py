"""Pins of the oracle's NEXT-4a Hungarian matching (reading
R24): SPEC S:313-317's worked examples, brute force over every partial
matching on small matrices, scipy's linear_sum_assignment on larger ones, and
the optimality invariants of a maximum-weight matching."""
import itertools

import numpy as np
import pytest
from scipy.optimize import linear_sum_assignment

import oracle as O


def _brute(s, floor):
    """Best total over all matchings that use only pairs with score >= floor
    (exhaustive over injective partial maps rows -> columns)."""
    m, n = s.shape
    best, best_pairs = 0.0, []
    for k in range(0, min(m, n) + 1):
        for rows in itertools.combinations(range(m), k):
            for cols in itertools.permutations(range(n), k):
                if any(not (s[r, c] >= floor) for r, c in zip(rows, cols)):
                    continue
                t = sum(float(s[r, c]) for r, c in zip(rows, cols))
                if t > best + 1e-12:
                    best, best_pairs = t, list(zip(rows, cols))
    return best, sorted(best_pairs)


def _pairs(rm):
    return sorted((i, int(j)) for i, j in enumerate(rm) if j >= 0)


def test_spec_examples():
    st, rm, cm, t = O.hungarian([[0.9]], 0.5)
    assert st == 0 and rm.tolist() == [0] and cm.tolist() == [0]
    st, rm, cm, t = O.hungarian([[0.3]], 0.5)
    assert st == 0 and rm.tolist() == [-1] and cm.tolist() == [-1] and t == 0.0
    # all below floor -> nothing matched (SPEC step example)
    st, rm, cm, t = O.hungarian(np.full((3, 4), 0.2, np.float32), 0.5)
    assert (rm == -1).all() and (cm == -1).all()
    # greedy would take 0.9 (0,0) then nothing; the optimum is 0.8 + 0.85
    st, rm, cm, t = O.hungarian([[0.9, 0.8], [0.85, 0.1]], 0.5)
    assert _pairs(rm) == [(0, 1), (1, 0)]
    assert t == pytest.approx(float(np.float32(0.8)) + float(np.float32(0.85)), abs=1e-12)


def test_floor_boundary_nan_and_empty():
    f = np.float32(0.5)
    st, rm, cm, t = O.hungarian(np.array([[f]], np.float32), 0.5)
    assert rm.tolist() == [0]                         # score == floor is allowed
    st, rm, cm, t = O.hungarian(np.array([[np.nan, 0.7]], np.float32), 0.5)
    assert rm.tolist() == [1]                         # NaN never matched
    for shape in ((0, 0), (0, 4), (3, 0)):
        st, rm, cm, t = O.hungarian(np.zeros(shape, np.float32), 0.5)
        assert st == 0 and len(rm) == shape[0] and len(cm) == shape[1] and t == 0.0
    assert O.hungarian([[0.9]], 0.0)[0] == O.ERR_INVALID   # floor must be > 0


def test_brute_force_small():
    rng = np.random.default_rng(207)
    for it in range(250):
        m, n = int(rng.integers(1, 7)), int(rng.integers(1, 7))
        s = rng.random((m, n)).astype(np.float32)
        if it % 5 == 0:
            s = np.round(s * 4) / 4          # many exact ties
        floor = float(rng.choice([0.05, 0.3, 0.5, 0.8]))
        best, pairs = _brute(s, floor)
        st, rm, cm, t = O.hungarian(s, floor)
        assert st == 0
        assert t == pytest.approx(best, abs=1e-9)
        got = _pairs(rm)
        assert all(s[i, j] >= floor for i, j in got)
        assert sum(float(s[i, j]) for i, j in got) == pytest.approx(best, abs=1e-9)
        if it % 5:                               # continuous scores: the optimum is unique
            assert got == pairs


@pytest.mark.parametrize("m,n", [(10, 10), (37, 20), (20, 55), (120, 80), (1, 90)])
def test_scipy_linear_sum_assignment(m, n):
    rng = np.random.default_rng(m * 1000 + n)
    for floor in (0.1, 0.5, 0.9):
        s = rng.random((m, n)).astype(np.float32)
        w = np.where(s >= floor, s.astype(np.float64), 0.0)
        r, c = linear_sum_assignment(w, maximize=True)
        ref = float(w[r, c].sum())
        ref_pairs = sorted((int(i), int(j)) for i, j in zip(r, c) if w[i, j] > 0)
        st, rm, cm, t = O.hungarian(s, floor)
        assert st == 0 and t == pytest.approx(ref, abs=1e-9)
        assert _pairs(rm) == ref_pairs
        # consistency and optimality invariants
        for i, j in enumerate(rm):
            if j >= 0:
                assert cm[j] == i and s[i, j] >= floor
        free_r = [i for i in range(m) if rm[i] < 0]
        free_c = [j for j in range(n) if cm[j] < 0]
        if free_r and free_c:                     # no allowed pair between two unmatched vertices
            assert not (s[np.ix_(free_r, free_c)] >= floor).any()
