"""Shared-memory-row K3/rebuild kernels (k_resolve3 / k_reattach3): every
dimension, including d > 256 where the new-node rows live in HBM, and the
forced shared-memory variant for small d (PCY_SMEM_RESOLVE)."""

import os

import numpy as np
import pytest

from oracle.piecy_oracle import OracleEngine
from tests.test_engine_gpu import assert_same

pytestmark = pytest.mark.gpu


def _pair(X, W, d, m):
    from paper_1502_04265_b200 import BicoEngine
    g = BicoEngine(d, m)
    g.insert_block(X, W)
    o = OracleEngine(d, m)
    o.insert_block(X, W)
    return g, o


@pytest.mark.parametrize("seed,n,d,m", [(0, 3000, 300, 200), (1, 2500, 1024, 300), (2, 1200, 4096, 150),
                                        (3, 3000, 257, 40)])
def test_high_dim_streams(seed, n, d, m):
    rng = np.random.default_rng(seed)
    cen = rng.uniform(-5, 5, size=(12, d))
    X = cen[rng.integers(0, 12, size=n)] + rng.normal(size=(n, d))
    g, o = _pair(X, None, d, m)
    assert_same(g, o)


def test_high_dim_weighted():
    rng = np.random.default_rng(9)
    X = rng.normal(scale=3.0, size=(900, 600))
    W = rng.integers(1, 6, size=900)
    g, o = _pair(X, W, 600, 40)
    assert_same(g, o)


@pytest.mark.parametrize("seed,n,d,m,weighted", [(4, 6000, 12, 150, False), (5, 2000, 5, 25, True),
                                                 (6, 8000, 54, 500, False)])
def test_forced_smem_variant_small_dim(seed, n, d, m, weighted, monkeypatch):
    monkeypatch.setenv("PCY_SMEM_RESOLVE", "1")
    rng = np.random.default_rng(seed)
    cen = rng.uniform(-20, 20, size=(30, d))
    X = cen[rng.integers(0, 30, size=n)] + rng.normal(size=(n, d))
    W = rng.integers(1, 9, size=n) if weighted else None
    g, o = _pair(X, W, d, m)
    assert_same(g, o)


@pytest.mark.parametrize("name,rows,m", [("cfg3", 40_000, 3_000), ("cfg5", 6_000, 1_500)])
def test_high_dim_workload_streams(name, rows, m):
    """Bench-family streams at d = 1024 / 4096: long enough for the
    subtree-parallel resolve and reattach windows (k_plan) between rebuilds."""
    from paper_1502_04265_b200 import workloads
    X = workloads.generate_rows(name, 0, rows)
    g, o = _pair(X, None, X.shape[1], m)
    assert_same(g, o)
