"""GPU seeding / Lloyd / cost vs the numpy oracle (pinned to the reference).

Seeding picks and Lloyd iteration counts must be identical; centers and
costs agree to 1e-9 relative (fp64, different summation order)."""

import numpy as np
import pytest

from oracle import piecy_oracle as O

pytestmark = pytest.mark.gpu


def _ev():
    from paper_1502_04265_b200 import evaluation
    return evaluation


def _blobs(seed, n, d, c, scale=10.0):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(-scale, scale, size=(c, d))
    X = cen[rng.integers(0, c, size=n)] + rng.normal(size=(n, d))
    w = rng.integers(1, 50, size=n).astype(np.float64)
    return X, w


@pytest.mark.parametrize("seed,n,d,k", [(0, 500, 5, 7), (1, 3000, 54, 50), (2, 2000, 128, 20), (3, 40, 3, 10)])
def test_repetitions_match_oracle(seed, n, d, k):
    X, w = _blobs(seed, n, d, max(2, k // 2))
    got = _ev().kmeans_repetitions(X, w, k, reps=5, seed=seed, max_iters=100, tol=1e-4)
    want = O.kmeans_reps(X, w, k, reps=5, seed=seed, max_iters=100, tol=1e-4)
    for (cg, vg), (cw, vw) in zip(got, want):
        np.testing.assert_allclose(cg, cw, rtol=1e-9, atol=1e-9)
        assert abs(vg - vw) <= 1e-9 * max(1.0, abs(vw))


def test_seeding_picks_identical():
    X, w = _blobs(5, 4000, 20, 30)
    for s in range(3):
        a = _ev().kmeanspp_seed(X, w, 25, np.random.default_rng(s))
        b = O.seed_dsquared(X, w, 25, np.random.default_rng(s))
        assert np.array_equal(a, b)


def test_lloyd_cost_log_and_iterations():
    X, w = _blobs(6, 2000, 10, 8)
    C0 = X[:8].copy()
    la, lb = [], []
    a = _ev().lloyd_iterate(X, w, C0, max_iters=50, tol=1e-6, cost_log=la)
    b = O.lloyd(X, w, C0, max_iters=50, tol=1e-6, cost_log=lb)
    assert len(la) == len(lb)
    np.testing.assert_allclose(la, lb, rtol=1e-10)
    np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-10)


def test_reference_known_answers():
    ev = _ev()
    pts = np.array([[0.0], [2.0], [10.0], [12.0]])
    log = []
    out = ev.lloyd_iterate(pts, None, np.array([[1.0], [11.0]]), cost_log=log)
    assert np.allclose(out, [[1.0], [11.0]]) and len(log) == 2
    out = ev.lloyd_iterate(np.array([[0.0], [2.0]]), None, np.array([[5.0]]))
    assert out[0, 0] == pytest.approx(1.0)
    pts = np.array([[0.0, 0.0], [0.1, 0.0], [10.0, 0.0], [10.1, 0.0]])
    out = ev.lloyd_iterate(pts, None, np.array([[0.05, 0.0], [0.05, 0.1], [50.0, 50.0]]), max_iters=20)
    assert ev.weighted_cost(pts, None, out) <= 0.011
    assert len(np.unique(np.round(out, 3), axis=0)) == 3
    pts = np.array([[0.0, 0.0], [5.0, 0.0], [0.0, 5.0], [5.0, 5.0]])
    c = ev.kmeanspp_seed(pts, None, 4, np.random.default_rng(1))
    assert ev.weighted_cost(pts, None, c) == pytest.approx(0.0, abs=1e-12)


def test_empty_cluster_repair_matches_oracle():
    pts = np.array([[0.0, 0.0], [0.1, 0.0], [10.0, 0.0], [10.1, 0.0], [20.0, 1.0]])
    C0 = np.array([[0.05, 0.0], [0.05, 0.1], [50.0, 50.0], [60.0, 60.0]])
    la, lb = [], []
    a = _ev().lloyd_iterate(pts, None, C0, max_iters=20, cost_log=la)
    b = O.lloyd(pts, np.ones(5), C0, max_iters=20, cost_log=lb)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(la, lb, rtol=1e-12, atol=1e-12)


def test_weighted_equals_repeated_and_determinism():
    ev = _ev()
    rng = np.random.default_rng(5)
    pts = rng.normal(size=(12, 3))
    w = rng.integers(1, 5, size=12)
    a = ev.lloyd_iterate(pts, w.astype(float), pts[:3].copy(), max_iters=30)
    b = ev.lloyd_iterate(np.repeat(pts, w, axis=0), None, pts[:3].copy(), max_iters=30)
    assert np.allclose(a, b, atol=1e-9)
    X = rng.normal(size=(60, 3))
    r1 = ev.kmeans_repetitions(X, None, 4, reps=3, seed=13)
    r2 = ev.kmeans_repetitions(X, None, 4, reps=3, seed=13)
    assert [c for _, c in r1] == [c for _, c in r2]
    for (c1, _), (c2, _) in zip(r1, r2):
        assert np.array_equal(c1, c2)
