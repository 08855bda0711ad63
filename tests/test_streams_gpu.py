"""Device paths of SURVEY.md §8f rows 1-2: the streaming full-data evaluation
(evaluate_cost_multi, evaluation.py:157-180) and stream-file ingest (SCPT
files read block-wise, pinned double-buffered H2D) feeding run_piecy."""
import numpy as np
import pytest

from oracle import piecy_oracle as O
from paper_1502_04265_b200 import PiecyConfig, evaluate_cost, evaluate_cost_multi, run_piecy
from paper_1502_04265_b200 import streams as S

pytestmark = pytest.mark.gpu


def _data(n=3000, d=20, seed=0):
    rng = np.random.default_rng(seed)
    C = rng.uniform(-10, 10, size=(8, d))
    return C[rng.integers(0, 8, size=n)] + rng.normal(size=(n, d))


@pytest.mark.parametrize("chunk", [1, 777, 8192])
def test_evaluate_cost_multi_matches_oracle(chunk):
    import torch
    X = _data(2500 if chunk == 1 else 20000)
    rng = np.random.default_rng(1)
    sets = [X[rng.integers(0, X.shape[0], size=k)] + rng.normal(size=(k, X.shape[1])) for k in (1, 7, 70)]
    want = O.evaluate_cost_multi(sets, X, chunk)
    for src in (X, torch.from_numpy(X).cuda(), list(X)):
        got = evaluate_cost_multi(sets, src, chunk=chunk)
        assert np.allclose(got, want, rtol=1e-12, atol=0), (got, want)
    X32 = X.astype(np.float32)   # fp32 streams are upcast exactly (as np.asarray(float64) does)
    want32 = O.evaluate_cost_multi(sets, X32.astype(np.float64), chunk)
    assert np.allclose(evaluate_cost_multi(sets, torch.from_numpy(X32).cuda(), chunk=chunk), want32, rtol=1e-12, atol=0)
    assert np.isclose(evaluate_cost(sets[1], X, chunk=chunk), want[1], rtol=1e-12)


def test_stream_file_feeds_pipeline(tmp_path):
    import torch
    X = _data()
    path = str(tmp_path / "x.bin")
    S.write_bin(path, list(X), X.shape[1])
    src = S.PointSource(path, "bin")
    blocks = [b[0].cpu().numpy() for b in S.device_blocks(src, 700)]
    assert np.array_equal(np.concatenate(blocks), X)
    cfg = PiecyConfig(k=8, piece_size=500, svd_dim=8, coreset_size=200, seed=3)
    a = run_piecy(X, X.shape[1], cfg)
    b = run_piecy(src, X.shape[1], cfg)
    assert np.array_equal(a.points, b.points) and np.array_equal(a.weights, b.weights)
    # the full-data evaluation reads the file block-wise, same totals as the array
    C = a.points[:8]
    assert evaluate_cost_multi([C], src)[0] == evaluate_cost_multi([C], X)[0]
    torch.cuda.synchronize()
