"""Seeded synthetic streams for the five BASELINE.json configurations.

The reference's paper benchmarks use real datasets that are not available
here; BASELINE.json names synthetic stand-ins with their shapes and value
distributions, and these generators restate them.  Details
the spec leaves open (mixture weights, scale assignment, draw order) are
fixed below once and for all.  Every generator is deterministic in its seed
and chunked so large configs never materialise fp64 copies.

Also holds the config -> reference-parameter mapping.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    entry: str          # "piecy" | "piecy-mr"
    n: int
    d: int
    dtype: str
    k: int
    m: int              # coreset size (per shard and merged for piecy-mr)
    svd_dim: int
    piece_size: int
    num_pieces: int | None
    seed: int
    max_iters: int = 100
    reps: int = 5


CONFIGS = {
    "cfg1": Workload("cfg1", "piecy", 20_000, 128, "float64", 20, 1_000, 30, 1_000, None, 0, max_iters=20),
    "cfg2": Workload("cfg2", "piecy", 581_012, 54, "float32", 50, 10_000, 54, 10_000, None, 1),
    "cfg3": Workload("cfg3", "piecy", 200_000, 1_024, "float32", 100, 20_000, 150, 20_000, None, 2),
    "cfg4": Workload("cfg4", "piecy-mr", 11_620_300, 57, "float32", 50, 20_000, 57, 20_000, 73, 3),
    "cfg5": Workload("cfg5", "piecy-mr", 1_000_000, 4_096, "float32", 250, 25_000, 375, 12_500, 10, 4),
}


def _zipf_sizes(n: int, count: int, a: float) -> np.ndarray:
    p = 1.0 / np.arange(1, count + 1) ** a
    p /= p.sum()
    raw = p * n
    sizes = np.floor(raw).astype(np.int64)
    rest = n - int(sizes.sum())
    order = np.argsort(-(raw - sizes), kind="stable")
    sizes[order[:rest]] += 1
    return sizes


def gen_cfg1(seed: int = 0) -> np.ndarray:
    """20 centers U[-10,10]^128, isotropic sigma 1, 1,000 points each, shuffled (fp64)."""
    rng = np.random.default_rng(seed)
    centers = rng.uniform(-10.0, 10.0, size=(20, 128))
    lab = np.repeat(np.arange(20), 1_000)
    rng.shuffle(lab)
    return centers[lab] + rng.standard_normal((20_000, 128))


def gen_cfg2(seed: int = 1, n: int = 581_012) -> np.ndarray:
    """Covertype-shaped mixed stream (fp32): 10 continuous columns from a
    7-component Gaussian mixture with column scales geometric in [1, 3000];
    one-hot groups of 4 and 40 with category p_i ~ i^-1.2."""
    rng = np.random.default_rng(seed)
    wts = rng.uniform(0.5, 1.5, size=7)
    comp = rng.choice(7, size=n, p=wts / wts.sum())
    scales = np.geomspace(1.0, 3000.0, 10)
    means = rng.uniform(-1.0, 1.0, size=(7, 10)) * scales
    stds = rng.uniform(0.05, 0.3, size=(7, 10)) * scales
    X = np.zeros((n, 54), dtype=np.float32)
    X[:, :10] = means[comp] + rng.standard_normal((n, 10)) * stds[comp]
    rows = np.arange(n)
    for off, size in ((10, 4), (14, 40)):
        p = 1.0 / np.arange(1, size + 1) ** 1.2
        cat = rng.choice(size, size=n, p=p / p.sum())
        X[rows, off + cat] = 1.0
    return X


def gen_cfg3(seed: int = 2, n: int = 200_000, d: int = 1_024, clusters: int = 100) -> np.ndarray:
    """100 anisotropic clusters: centers N(0, 25 I), per-cluster diagonal std
    log-uniform in [0.1, 2], Zipf(1.0) sizes, random order (fp32)."""
    rng = np.random.default_rng(seed)
    centers = rng.normal(0.0, 5.0, size=(clusters, d))
    stds = np.exp(rng.uniform(np.log(0.1), np.log(2.0), size=(clusters, d)))
    lab = np.repeat(np.arange(clusters), _zipf_sizes(n, clusters, 1.0))
    rng.shuffle(lab)
    X = np.empty((n, d), dtype=np.float32)
    for a in range(0, n, 16_384):
        b = min(n, a + 16_384)
        L = lab[a:b]
        X[a:b] = centers[L] + rng.standard_normal((b - a, d)) * stds[L]
    return X


_CH4 = 262_144
_CH5 = 8_192


def _cfg4_params(seed: int, d: int):
    rng = np.random.default_rng(seed)
    return rng.uniform(0.0, 100.0, size=(500, d)), rng.uniform(0.5, 5.0, size=500)


def gen_cfg4(seed: int = 3, n: int = 11_620_300, d: int = 57, rows: tuple | None = None) -> np.ndarray:
    """BigCross-shaped: 500 components, centers U[0,100]^57, sigma U[0.5,5]
    per component, 1% uniform outliers in [0,100]^57 (fp32).  Chunk c of
    262,144 rows draws from PCG64([seed, c]), so any row range can be made
    on its own (``rows=(a, b)``) -- each rank generates only its groups."""
    centers, sig = _cfg4_params(seed, d)
    a0, b0 = rows if rows is not None else (0, n)
    X = np.empty((b0 - a0, d), dtype=np.float32)
    for c in range(a0 // _CH4, (b0 + _CH4 - 1) // _CH4):
        ca, cb = c * _CH4, min(n, (c + 1) * _CH4)
        rng = np.random.default_rng([seed, c])
        m = cb - ca
        lab = rng.integers(0, 500, size=m)
        blk = centers[lab] + rng.standard_normal((m, d)) * sig[lab, None]
        out = rng.random(m) < 0.01
        blk[out] = rng.uniform(0.0, 100.0, size=(int(out.sum()), d))
        lo, hi = max(ca, a0), min(cb, b0)
        X[lo - a0:hi - a0] = blk[lo - ca:hi - ca]
    return X


def gen_cfg5(seed: int = 4, n: int = 1_000_000, d: int = 4_096, topics: int = 250,
             active: int = 400, nnz: int = 205, rows: tuple | None = None) -> np.ndarray:
    """Sparse-valued dense rows: topic t (uniform of 250) active on 400 dims;
    ~5% of coordinates (205) nonzero at random positions among them with
    values lognormal(0,1) times the topic profile; rows L2-normalised (fp32).
    Chunk c of 8,192 rows draws from PCG64([seed, c]) (row ranges as cfg4)."""
    rng0 = np.random.default_rng(seed)
    dims = np.stack([rng0.choice(d, size=active, replace=False) for _ in range(topics)])
    prof = rng0.uniform(0.5, 1.5, size=(topics, active))
    a0, b0 = rows if rows is not None else (0, n)
    X = np.zeros((b0 - a0, d), dtype=np.float32)
    for c in range(a0 // _CH5, (b0 + _CH5 - 1) // _CH5):
        ca, cb = c * _CH5, min(n, (c + 1) * _CH5)
        rng = np.random.default_rng([seed, c])
        m = cb - ca
        t = rng.integers(0, topics, size=m)
        pick = np.argsort(rng.random((m, active)), axis=1)[:, :nnz]
        cols = dims[t[:, None], pick]
        vals = rng.lognormal(0.0, 1.0, size=(m, nnz)) * prof[t[:, None], pick]
        vals /= np.sqrt((vals * vals).sum(axis=1, keepdims=True))
        blk = np.zeros((m, d), dtype=np.float32)
        np.put_along_axis(blk, cols, vals.astype(np.float32), axis=1)
        lo, hi = max(ca, a0), min(cb, b0)
        X[lo - a0:hi - a0] = blk[lo - ca:hi - ca]
    return X


GENERATORS = {"cfg1": gen_cfg1, "cfg2": gen_cfg2, "cfg3": gen_cfg3, "cfg4": gen_cfg4, "cfg5": gen_cfg5}


def generate_rows(name: str, a: int, b: int, n: int | None = None) -> np.ndarray:
    """Rows [a, b) of a config's stream (cfg4/cfg5 without generating the rest)."""
    cfg = CONFIGS[name]
    total = cfg.n if n is None else n
    if name == "cfg4":
        return gen_cfg4(cfg.seed, n=total, rows=(a, b))
    if name == "cfg5":
        return gen_cfg5(cfg.seed, n=total, rows=(a, b))
    return generate(name, n)[a:b]


def generate(name: str, n: int | None = None) -> np.ndarray:
    """The stream of a config (or a smaller stream of the same family with n rows)."""
    cfg = CONFIGS[name]
    if name == "cfg1":
        X = gen_cfg1(cfg.seed)
        return X if n is None else X[:n]
    if n is None:
        return GENERATORS[name](cfg.seed)
    return GENERATORS[name](cfg.seed, n=n)
