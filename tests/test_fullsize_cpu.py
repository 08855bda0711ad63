"""Full-size pins of the CPU oracle against the unmodified reference.

tests/golden/full_<cfg>.npz were written by tests/golden/make_fullsize.py,
which runs /root/reference's own run_piecy / run_piecy_mr and
kmeans_repetitions on the exact BASELINE streams (sha256 recorded).  Here:

* the frozen generators still produce those bytes (cfg1-3; cfg4/cfg5 are
  checked on the GPU box where their 2.6 / 16 GB streams are made anyway);
* the oracle reproduces the reference's coreset and k-means result on the
  whole cfg1 and cfg2 streams (cfg3 takes ~11 min in the C oracle at d=1024;
  its pin is recorded in profiles/r2_oracle_fullsize_pin.txt).
"""

import sys
import os

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
import fullsize as F  # noqa: E402

from paper_1502_04265_b200 import workloads as W  # noqa: E402


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_generator_bytes_match_fixture(name):
    fx = F.load(name)
    assert fx is not None, f"missing fixture {F.path(name)}"
    X = W.generate(name)
    assert X.shape == (int(fx["n"]), int(fx["d"]))
    assert F.sha256(X) == str(fx["input_sha256"])


def test_fixture_manifest_records_reference_run():
    import json
    for name in ("cfg1", "cfg2", "cfg3"):
        man = json.loads(str(F.load(name)["manifest"]))
        assert man["config"] == name and man["reference"].endswith("pkg/src")
        assert "numpy" in man and "OPENBLAS_NUM_THREADS" in man and "cpu" in man


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_oracle_matches_reference_full_size(name):
    from oracle import piecy_oracle as O
    cfg = W.CONFIGS[name]
    fx = F.load(name)
    X = W.generate(name)
    P, w = O.piecy(X, cfg.k, cfg.piece_size, cfg.svd_dim, cfg.m, seed=cfg.seed)
    runs = O.kmeans_reps(P, w.astype(np.float64), cfg.k, reps=cfg.reps, seed=cfg.seed, max_iters=cfg.max_iters)
    C = np.stack([c for c, _ in runs])
    costs = np.array([v for _, v in runs])
    rep = F.compare(fx, P, w, C, costs, exact_points=cfg.svd_dim >= cfg.d)
    assert rep["ok"], rep
