"""Host-side logic of the drop-in package (no GPU): configs, piece assembly,
closed forms, summaries, synthetic workloads.  Mirrors the reference's own
known-answer tests (pkg/tests/test_coreset.py:10-61, test_pipeline.py:38-70)."""

import numpy as np
import pytest

from paper_1502_04265_b200 import insertion_error_increment, max_insertable_copies
from paper_1502_04265_b200.coreset import ClusteringFeature
from paper_1502_04265_b200.evaluation import CostSummary
from paper_1502_04265_b200.pipeline import PiecyConfig, default_svd_dim, iter_pieces


def simulate_copy_insertions(group_points, new_point, copies, threshold):
    pts = [float(v) for v in group_points]
    n = 0
    for _ in range(copies):
        trial = np.array(pts + [float(new_point)])
        if float(((trial - trial.mean()) ** 2).sum()) > threshold:
            break
        pts.append(float(new_point))
        n += 1
    return n


def test_closed_forms_known_answers():
    assert insertion_error_increment(1, 1, 2.0) == pytest.approx(1.0)
    assert insertion_error_increment(2, 2, 3.0) == pytest.approx(3.0)
    assert max_insertable_copies(4, 10, 1.0, 5.0, 2.0) == 4
    assert max_insertable_copies(3, 1000, 4.0, 4.0, 0.0) == 1000
    assert max_insertable_copies(1, 10, 5.0, 5.0, 1.0) == 0


@pytest.mark.parametrize("seed", range(4))
def test_capacity_agrees_with_simulation(seed):
    rng = np.random.default_rng(seed)
    for _ in range(50):
        size = int(rng.integers(1, 30))
        spread = float(rng.uniform(0.0, 2.0))
        group = [spread] * (size // 2) + [-spread] * (size // 2) + [0.0] * (size % 2)
        arr = np.array(group)
        err = float(((arr - arr.mean()) ** 2).sum())
        new = float(rng.uniform(-4.0, 4.0))
        thr = err + float(rng.uniform(0.0, 20.0))
        copies = int(rng.integers(1, 100))
        got = max_insertable_copies(size, copies, err, thr, float((new - arr.mean()) ** 2))
        assert got == simulate_copy_insertions(group, new, copies, thr)


def test_clustering_feature_algebra():
    cf = ClusteringFeature(2, np.array([2.0, 0.0]), 4.0, np.array([0.0, 0.0]))
    assert cf.cost_to(np.array([1.0, 0.0])) == pytest.approx(2.0)
    assert cf.internal_error() == pytest.approx(2.0)
    m = ClusteringFeature.from_point([1.0, 0.0], 2).merged_with(ClusteringFeature.from_point([0.0, 2.0], 3))
    assert m.weight == 5 and np.allclose(m.linear_sum, [2.0, 6.0])


def test_configs_and_pieces():
    cfg = PiecyConfig(k=10, piece_size=2000)
    assert cfg.svd_dim == 15 and cfg.coreset_size == 2000 and default_svd_dim(1) == 2
    with pytest.raises(ValueError):
        PiecyConfig(k=10, piece_size=5)
    with pytest.raises(ValueError):
        PiecyConfig(k=0, piece_size=10)
    with pytest.raises(ValueError):
        PiecyConfig(k=10, piece_size=100, coreset_size=5)
    sizes = [p.shape[0] for p in iter_pieces(iter([np.full(3, float(i)) for i in range(10)]), 4, 3)]
    assert sizes == [4, 4, 2]


def test_cost_summary():
    s = CostSummary.of([5.0, 1.0, 3.0, 2.0, 4.0])
    assert (s.minimum, s.maximum, s.median) == (1.0, 5.0, 3.0)
    with pytest.raises(ValueError):
        CostSummary.of([])


def test_workloads_deterministic_and_shaped():
    from paper_1502_04265_b200 import workloads as W
    a = W.generate("cfg2", 5000)
    b = W.generate("cfg2", 5000)
    assert a.shape == (5000, 54) and a.dtype == np.float32 and np.array_equal(a, b)
    assert np.all(a[:, 10:14].sum(1) == 1) and np.all(a[:, 14:].sum(1) == 1)
    c = W.generate("cfg1")
    assert c.shape == (20000, 128) and c.dtype == np.float64
    e = W.generate("cfg5", 64)
    assert e.shape == (64, 4096)
    np.testing.assert_allclose(np.linalg.norm(e.astype(np.float64), axis=1), 1.0, rtol=1e-6)
