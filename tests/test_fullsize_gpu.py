"""GPU path vs the unmodified reference at the full BASELINE configs.

Every config end to end -- the public pipeline (run_piecy for cfg1-3; the
sharded run_piecy_mr, all eight level-0 groups on this GPU, for cfg4/cfg5)
then kmeans_repetitions(reps=5) on the coreset -- against the reference's
own outputs on the same bytes (tests/golden/full_<cfg>.npz, written by
tests/golden/make_fullsize.py from /root/reference; the stream is
regenerated here and its sha256 checked first).

Bar (SURVEY.md §8a parity contract): coreset weights/order exact; points
bit-exact where no projection runs (cfg2, cfg4), else within 1e-9 of the row
scale; k-means costs and centres within 1e-9 relative.
"""

import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
import fullsize as F  # noqa: E402

pytestmark = pytest.mark.gpu


def _run(name):
    import torch
    from paper_1502_04265_b200 import workloads as W
    from paper_1502_04265_b200.evaluation import kmeans_repetitions
    cfg = W.CONFIGS[name]
    fx = F.load(name)
    if fx is None:
        pytest.skip(f"no fixture for {name}")
    dev = torch.device("cuda", 0)
    if cfg.entry == "piecy":
        from paper_1502_04265_b200.pipeline import PiecyConfig, run_piecy
        X = W.generate(name)
        assert F.sha256(X) == str(fx["input_sha256"]), "stream bytes differ from the reference run's"
        cs = run_piecy(X, cfg.d, PiecyConfig(k=cfg.k, piece_size=cfg.piece_size, svd_dim=cfg.svd_dim,
                                             coreset_size=cfg.m, seed=cfg.seed))
    else:
        from paper_1502_04265_b200.distributed import DeviceOps, run_piecy_mr_sharded
        from paper_1502_04265_b200.mergereduce import MrConfig
        X = W.generate(name)
        assert F.sha256(X) == str(fx["input_sha256"]), "stream bytes differ from the reference run's"
        mcfg = MrConfig(k=cfg.k, piece_size=cfg.piece_size, num_pieces=cfg.num_pieces, svd_dim=cfg.svd_dim,
                        coreset_size=cfg.m, seed=cfg.seed)

        def source(a, b):
            return torch.from_numpy(X[a:b]).to(dev)
        trees = []
        cs = run_piecy_mr_sharded(source, X.shape[0], cfg.d, mcfg, ops=DeviceOps(mcfg, dev), tree_out=trees)
        if "flush_sources" in fx and trees:
            assert list(trees[0].stats.flush_sources) == list(fx["flush_sources"])
        del X
    runs = kmeans_repetitions(cs.points, cs.weights.astype(np.float64), cfg.k, reps=cfg.reps, seed=cfg.seed,
                              max_iters=cfg.max_iters, tol=1e-4)
    C = np.stack([c for c, _ in runs])
    costs = np.array([v for _, v in runs])
    return F.compare(fx, cs.points, cs.weights, C, costs, exact_points=cfg.svd_dim >= cfg.d)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_full_config_matches_reference(name):
    rep = _run(name)
    print(name, rep)
    assert rep["ok"], rep
