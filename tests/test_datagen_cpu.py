"""Paper generators: the oracle's draw-index restatement (the same bookkeeping
the device kernels use) against the reference's own streams
(tests/golden/datagen.npz from tests/golden/make_golden_datagen.py), plus the
drop-in configs' validation."""

import os
import sys

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(__file__), "golden")
sys.path.insert(0, HERE)
from make_golden_datagen import CUBE, LB, SWN  # noqa: E402

from oracle import piecy_oracle as O  # noqa: E402

G = np.load(os.path.join(HERE, "datagen.npz"))


@pytest.mark.parametrize("i", range(len(SWN)))
def test_swn_oracle_bit_exact(i):
    cl, ppc, dim, a, sp, no, seed = SWN[i]
    assert np.array_equal(O.gen_swn(cl, ppc, dim, a, spread=sp, noise=no, seed=seed), G[f"swn{i}"])


@pytest.mark.parametrize("i", range(len(CUBE)))
def test_cube_oracle_bit_exact(i):
    n, sp, seed = CUBE[i]
    assert np.array_equal(O.gen_cube(n, spread=sp, seed=seed), G[f"cube{i}"])


@pytest.mark.parametrize("i", range(len(LB)))
def test_lower_bound_oracle_bit_exact(i):
    k, n, sp, no = LB[i]
    assert np.array_equal(O.gen_lower_bound(k, n, spread=sp, noise=no), G[f"lb{i}"])


def test_philox_restatement_matches_numpy():
    t = np.array([0, 1, 2, 3, 4, 5, 17, 1000, 2**40 + 3], dtype=np.uint64)
    g = np.random.Philox(key=123)
    raw = g.random_raw(1001)
    want = (raw >> np.uint64(11)).astype(np.float64) / 9007199254740992.0
    got = O.philox_uniforms(123, t[:-1])
    assert np.array_equal(got, want[t[:-1].astype(np.int64)])
    tmp = np.random.Philox(key=123, counter=(2**40 + 3) // 4)
    tmp.random_raw(3)
    x = tmp.random_raw(1)[0]
    assert O.philox_uniforms(123, t[-1:])[0] == float(x >> np.uint64(11)) / 9007199254740992.0


def test_config_validation_like_reference():
    from paper_1502_04265_b200.datagen import LowerBoundConfig, RandomConfig, SwnConfig
    with pytest.raises(ValueError):
        SwnConfig(clusters=2, points_per_cluster=3, dim=4, active_dims=5)
    with pytest.raises(ValueError):
        SwnConfig(clusters=2, points_per_cluster=3, dim=4, active_dims=2, spread=1.0, noise=2.0)
    with pytest.raises(ValueError):
        LowerBoundConfig(k=1, n=10)
    with pytest.raises(ValueError):
        LowerBoundConfig(k=3, n=10)
    with pytest.raises(ValueError):
        RandomConfig(n=0)
    assert LowerBoundConfig(k=5, n=50).dim == 55 and RandomConfig(n=7).dim == 7
    assert SwnConfig(3, 4, 5, 2).n_points == 12
