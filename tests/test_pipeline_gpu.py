"""run_bico / run_piecy on the device vs the oracle pipelines."""

import numpy as np
import pytest

from oracle import piecy_oracle as O

pytestmark = pytest.mark.gpu


def _mix(seed, n, d, c, spread=10.0):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(-spread, spread, size=(c, d))
    return cen[rng.integers(0, c, size=n)] + rng.normal(size=(n, d))


def test_run_bico_exact():
    from paper_1502_04265_b200.pipeline import run_bico
    X = _mix(0, 20000, 57, 40)
    cs = run_bico(X, 57, 1500)
    p, w = O.bico(X, 1500)
    assert np.array_equal(cs.weights, w) and np.array_equal(cs.points, p)


def test_run_piecy_skip_projection_exact():
    from paper_1502_04265_b200.pipeline import PiecyConfig, run_piecy
    X = _mix(1, 12000, 20, 30).astype(np.float32)
    cfg = PiecyConfig(k=10, piece_size=3000, svd_dim=20, coreset_size=800, seed=1)
    cs = run_piecy(X, 20, cfg)
    p, w = O.piecy(X, 10, 3000, 20, 800, seed=1)
    assert np.array_equal(cs.weights, w) and np.array_equal(cs.points, p)


@pytest.mark.parametrize("n,d,k,ps,ell,m", [(6000, 64, 5, 500, 8, 300), (20000, 128, 20, 1000, 30, 1000),
                                            (2043, 40, 4, 400, 6, 150)])
def test_run_piecy_projection_parity(n, d, k, ps, ell, m):
    from paper_1502_04265_b200.pipeline import PiecyConfig, PipelineStats, run_piecy
    X = _mix(n, n, d, k)
    st = PipelineStats()
    cs = run_piecy(X, d, PiecyConfig(k=k, piece_size=ps, svd_dim=ell, coreset_size=m, seed=3), st)
    stats = {}
    p, w = O.piecy(X, k, ps, ell, m, seed=3, stats=stats)
    assert st.svd_calls == stats["svd_calls"]
    assert np.array_equal(cs.weights, w)
    np.testing.assert_allclose(cs.points, p, rtol=1e-9, atol=1e-9 * np.abs(p).max())


def test_pipeline_structure_like_reference():
    from paper_1502_04265_b200.pipeline import PiecyConfig, PipelineStats, run_piecy
    rng = np.random.default_rng(1)
    st = PipelineStats()
    run_piecy(iter(rng.normal(size=(140, 8))), 8, PiecyConfig(k=2, piece_size=40, svd_dim=5, coreset_size=40, seed=1), st)
    assert st.pieces == 4 and st.svd_calls == 4
    st = PipelineStats()
    cs = run_piecy(iter(rng.normal(size=(43, 8))), 8, PiecyConfig(k=2, piece_size=40, svd_dim=5, coreset_size=40, seed=1), st)
    assert st.pieces == 2 and st.svd_calls == 1 and cs.total_weight == 43
    cs = run_piecy(iter([]), 5, PiecyConfig(k=2, piece_size=10, svd_dim=2, coreset_size=10))
    assert len(cs) == 0
