"""GPU BICO engine vs the CPU oracle (oracle/bico_oracle.c) on seeded streams.

Membership, levels, weights, references and linear sums must be bit-exact;
square sums and T within 1e-12 relative (their dot products are summed in a
different order than the oracle's)."""

import numpy as np
import pytest

from oracle.piecy_oracle import OracleEngine

pytestmark = pytest.mark.gpu


def _engine(d, m, **kw):
    from paper_1502_04265_b200 import BicoEngine
    return BicoEngine(d, m, **kw)


def assert_same(gpu, ora, rtol=1e-12):
    assert gpu.total_weight == ora.total_weight
    assert gpu.num_features == ora.num_features
    tg, to = gpu.threshold, ora.threshold
    assert abs(tg - to) <= rtol * abs(to), (tg, to)
    lv, w, s, q, r = ora.features()
    feats = gpu.features()
    assert len(feats) == len(w)
    for i, (L, cf) in enumerate(feats):
        assert L == lv[i], f"level mismatch at feature {i}"
        assert cf.weight == w[i], f"weight mismatch at feature {i}: {cf.weight} vs {w[i]}"
        assert np.array_equal(cf.reference, r[i]), f"reference mismatch at feature {i}"
        assert np.array_equal(cf.linear_sum, s[i]), f"linear sum mismatch at feature {i}"
        assert abs(cf.square_sum - q[i]) <= rtol * max(1.0, abs(q[i]))
    cs = gpu.extract_coreset()
    pts, wts = ora.extract()
    assert np.array_equal(cs.weights, wts)
    assert np.array_equal(cs.points, pts)


def run_pair(X, W, d, m, block=None, **kw):
    g = _engine(d, m, **kw)
    o = OracleEngine(d, m, kw.get("bootstrap_cap", 1001))
    if block is None:
        g.insert_block(X, W)
    else:
        for a in range(0, len(X), block):
            g.insert_block(X[a:a + block], None if W is None else W[a:a + block])
    o.insert_block(X, W)
    return g, o


@pytest.mark.parametrize("seed,n,d,m", [(0, 3000, 5, 50), (1, 20000, 57, 2000), (2, 5000, 20, 100),
                                        (3, 4000, 128, 300), (4, 500, 2, 1), (5, 800, 3, 7)])
def test_unit_streams(seed, n, d, m):
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-20, 20, size=(30, d))
    X = centers[rng.integers(0, 30, size=n)] + rng.normal(size=(n, d))
    g, o = run_pair(X, None, d, m, block=1777)
    assert_same(g, o)


@pytest.mark.parametrize("seed", range(3))
def test_weighted_streams(seed):
    rng = np.random.default_rng(40 + seed)
    X = rng.normal(scale=4.0, size=(2000, 5))
    W = rng.integers(1, 9, size=2000)
    g, o = run_pair(X, W, 5, 25)
    assert_same(g, o)


def test_duplicates_and_bootstrap_features():
    rng = np.random.default_rng(7)
    base = rng.normal(size=(40, 4))
    X = np.repeat(base, 3, axis=0)
    g, o = run_pair(X, None, 4, 60)          # never builds: 40 distinct < 61
    assert_same(g, o)
    X2 = base[rng.integers(0, 40, size=500)]  # non-consecutive repeats
    g, o = run_pair(X2, None, 4, 60)
    assert_same(g, o)
    g, o = run_pair(np.repeat(rng.normal(size=(300, 4)), 2, axis=0), None, 4, 40)
    assert_same(g, o)


def test_single_point_inserts_match_block():
    rng = np.random.default_rng(11)
    X = rng.normal(scale=3.0, size=(700, 6))
    g = _engine(6, 30, host_buffer=64)
    for x in X:
        g.insert(x)
    o = OracleEngine(6, 30)
    o.insert_block(X)
    assert_same(g, o)


def test_invalid_point_stops_block():
    rng = np.random.default_rng(12)
    X = rng.normal(size=(300, 3))
    X[200, 1] = np.nan
    g = _engine(3, 20)
    with pytest.raises(ValueError, match="non-finite"):
        g.insert_block(X)
    o = OracleEngine(3, 20)
    o.insert_block(X[:200])
    assert_same(g, o)
    X[200, 1] = 1e200
    X[200, 2] = 1e200
    g2 = _engine(3, 20)
    with pytest.raises(ValueError, match="overflow"):
        g2.insert_block(X)


def test_fp32_input_upcast():
    rng = np.random.default_rng(13)
    X = (rng.normal(size=(3000, 54)) * np.geomspace(1, 3000, 54)).astype(np.float32)
    g, o = run_pair(X, None, 54, 500)
    assert_same(g, o)


@pytest.mark.parametrize("name,rows,m", [("cfg2", 120_000, 10_000), ("cfg4", 150_000, 20_000), ("cfg2", 60_000, 1_000),
                                         ("cfg1", 20_000, 1_000)])
def test_workload_streams(name, rows, m):
    """Long streams of the bench families: these run mostly through the
    subtree-parallel resolve (k_plan windows), with rebuilds in between."""
    from paper_1502_04265_b200 import workloads
    X = workloads.generate_rows(name, 0, rows)
    d = X.shape[1]
    g, o = run_pair(X, None, d, m, block=40_000)
    assert_same(g, o)


def test_bootstrap_runs_weights_and_invalid_row():
    """Bootstrap block semantics (coreset.py:283-295) on the parallel scan:
    runs of equal rows fold into one pending entry with summed weights,
    non-consecutive repeats grow the pending buffer, and an invalid row inside
    the bootstrap leaves exactly the earlier rows."""
    rng = np.random.default_rng(21)
    base = rng.normal(size=(90, 6))
    idx = np.repeat(rng.integers(0, 90, size=700), rng.integers(1, 4, size=700))
    X = base[idx]
    W = rng.integers(1, 5, size=len(X))
    for m in (50, 200):   # builds mid-block / stays in bootstrap
        g, o = run_pair(X, W, 6, m, block=333)
        assert_same(g, o)
    Xb = X.copy()
    Xb[400, 2] = np.inf
    g = _engine(6, 200)
    with pytest.raises(ValueError, match="non-finite"):
        g.insert_block(Xb, W)
    o = OracleEngine(6, 200)
    o.insert_block(X[:400], W[:400])
    assert_same(g, o)


def test_parallel_resolve_deterministic_and_equal_to_sequential(monkeypatch):
    """The subtree-parallel resolve allocates slots and groups through atomic
    tickets; the features (order, levels, weights, sums) must not depend on
    that, and must equal the one-CTA sequential resolve (PCY_K3PAR=0)."""
    from paper_1502_04265_b200 import workloads
    X = workloads.generate_rows("cfg2", 0, 60_000)
    d = X.shape[1]

    def feats():
        g = _engine(d, 2_000)
        g.insert_block(X)
        f = g.features()
        return ([L for L, _ in f], [cf.weight for _, cf in f],
                np.stack([cf.linear_sum for _, cf in f]), np.stack([cf.reference for _, cf in f]))

    a, b = feats(), feats()
    monkeypatch.setenv("PCY_K3PAR", "0")
    c = feats()
    for u, v, w in zip(a, b, c):
        assert np.array_equal(np.asarray(u), np.asarray(v))
        assert np.array_equal(np.asarray(u), np.asarray(w))


def test_weighted_long_stream():
    """Weighted items keep k_plan's windows at root keys with root opens as
    stoppers (K1 does not follow partial takes)."""
    rng = np.random.default_rng(77)
    centers = rng.uniform(-30, 30, size=(40, 12))
    X = centers[rng.integers(0, 40, size=30_000)] + rng.normal(size=(30_000, 12))
    W = rng.integers(1, 6, size=30_000)
    W[rng.random(30_000) < 0.7] = 1
    g, o = run_pair(X, W, 12, 800, block=7_000)
    assert_same(g, o)
