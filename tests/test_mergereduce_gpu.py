"""piecy-mr on the device: single-process tree and the sharded driver vs
golden reference outputs / the oracle tree; reference structure tests
(pkg/tests/test_mergereduce.py)."""

import os

import numpy as np
import pytest

from oracle import piecy_oracle as O

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def _cfg(**kw):
    from paper_1502_04265_b200.mergereduce import MrConfig
    return MrConfig(**kw)


@pytest.mark.parametrize("name", ["run_piecy_mr", "run_piecy_mr_noproj"])
def test_golden(name):
    from paper_1502_04265_b200.mergereduce import run_piecy_mr
    g = dict(np.load(os.path.join(G, f"{name}.npz")))
    cfg = _cfg(k=int(g["k"]), piece_size=int(g["piece_size"]), num_pieces=int(g["num_pieces"]),
               svd_dim=int(g["svd_dim"]), coreset_size=int(g["m"]), seed=int(g["seed"]))
    trees = []
    cs = run_piecy_mr(g["X"], g["X"].shape[1], cfg, tree_out=trees)
    assert np.array_equal(cs.weights, g["wts"])
    np.testing.assert_allclose(cs.points, g["pts"], rtol=1e-9, atol=1e-9 * np.abs(g["pts"]).max())
    if "flush_sources" in g:
        assert trees[0].stats.flush_sources == list(g["flush_sources"])


def _data(n, d, seed=0):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(-8, 8, size=(6, d))
    return cen[rng.integers(0, 6, size=n)] + rng.normal(size=(n, d))


@pytest.mark.parametrize("n,d,ps,npc,ell,m", [(1170, 20, 90, 4, 5, 60), (2000, 12, 50, 3, 4, 40),
                                              (6000, 57, 500, 3, 57, 300), (150, 8, 40, 5, 3, 30)])
def test_sharded_one_gpu_equals_oracle_tree(n, d, ps, npc, ell, m):
    from paper_1502_04265_b200.distributed import run_piecy_mr_multi
    from paper_1502_04265_b200.mergereduce import run_piecy_mr
    X = _data(n, d)
    cfg = _cfg(k=3, piece_size=ps, num_pieces=npc, svd_dim=ell, coreset_size=m, seed=9)
    want_p, want_w = O.piecy_mr(X, 3, ps, npc, ell, m, seed=9)
    a = run_piecy_mr_multi(X, d, cfg, rank=0, world=1, concurrent=True)
    b = run_piecy_mr(X, d, cfg)
    for cs in (a, b):
        assert np.array_equal(cs.weights, want_w)
        np.testing.assert_allclose(cs.points, want_p, rtol=1e-9, atol=1e-9 * np.abs(want_p).max())


def test_flush_schedule_and_structure():
    from paper_1502_04265_b200.mergereduce import MergeReduceTree, run_piecy_mr
    rng = np.random.default_rng(0)
    rows = rng.normal(size=(45, 6))
    tree = MergeReduceTree(6, _cfg(k=2, piece_size=5, num_pieces=3, svd_dim=2, coreset_size=5, seed=1))
    for a in range(0, 45, 5):
        tree.push_piece(rows[a:a + 5])
    assert tree.stats.pieces == 9 and tree.stats.flush_sources == [0, 0, 0, 1]
    assert tree.stats.peak_live_engines == 2
    assert tree.finalize().total_weight == 45
    # Exactly repeated rows: the reference's LAPACK projection maps every piece
    # to bit-identical rows and BICO collapses them into one feature.  The
    # device projection reproduces them only to ~1 ulp, so the summary may keep
    # ulp-separated features (documented deviation); the
    # represented multiset is the same.
    cs = run_piecy_mr(np.tile([[2.0, -1.0, 3.0]], (24, 1)), 3,
                      _cfg(k=1, piece_size=4, num_pieces=2, svd_dim=1, coreset_size=4, seed=2))
    assert cs.total_weight == 24
    np.testing.assert_allclose(cs.points, np.tile([[2.0, -1.0, 3.0]], (len(cs), 1)), rtol=1e-13)
    empty = MergeReduceTree(3, _cfg(k=2, piece_size=5, num_pieces=2, svd_dim=2, coreset_size=5)).finalize()
    assert len(empty) == 0
    with pytest.raises(ValueError):
        MergeReduceTree(4, _cfg(k=2, piece_size=5, num_pieces=2, svd_dim=2, coreset_size=5)).push_piece(np.zeros((3, 7)))
