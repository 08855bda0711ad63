"""Checker for the full-size reference fixtures (tests/golden/full_<cfg>.npz).

Test infrastructure, shared by tests/golden/make_fullsize.py (which writes the
fixtures from the unmodified reference), the parity tests and bench.py's
``parity`` field.  No reference code is needed to read or check a fixture.

Contract (SURVEY.md §8a "Parity contract", BASELINE.json north_star):
* coreset weights and order: exact;
* coreset points: bit-exact (sha256 of the fp64 bytes) when the config has no
  projection (cfg2, cfg4); otherwise the sketch (row sums, squared norms, four
  fixed random directions) within 1e-9 relative to the row scale;
* k-means: per-repetition costs within 1e-9 relative and the centre sketch
  within 1e-9 of the centre scale (full centres too when the fixture has them).
"""

from __future__ import annotations

import hashlib
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SKETCH_SEED = 20260101
SKETCH_DIRS = 4
RTOL = 1e-9


def sha256(a: np.ndarray) -> str:
    h = hashlib.sha256()
    a = np.ascontiguousarray(a)
    flat = a.reshape(-1).view(np.uint8)
    step = 1 << 28
    for i in range(0, flat.size, step):
        h.update(memoryview(flat[i:i + step]))
    return h.hexdigest()


def sketch(P: np.ndarray) -> np.ndarray:
    """(rows, 2 + SKETCH_DIRS): row sum, squared norm, projections on fixed directions."""
    P = np.asarray(P, dtype=np.float64)
    d = P.shape[1]
    R = np.random.default_rng([SKETCH_SEED, d]).standard_normal((d, SKETCH_DIRS))
    return np.concatenate([P.sum(axis=1, keepdims=True), (P * P).sum(axis=1, keepdims=True), P @ R], axis=1)


def path(name: str) -> str:
    return os.path.join(HERE, f"full_{name}.npz")


def load(name: str):
    p = path(name)
    if not os.path.exists(p):
        return None
    return dict(np.load(p, allow_pickle=False))


def _sketch_close(got: np.ndarray, want: np.ndarray, d: int) -> float:
    """Largest deviation of two sketches relative to the rows' scale."""
    if got.shape != want.shape:
        return float("inf")
    nrm = np.sqrt(np.maximum(want[:, 1], 0.0))                      # |row|
    scale = np.stack([nrm * np.sqrt(d), np.maximum(want[:, 1], 1e-300)] +
                     [nrm * np.sqrt(d)] * (want.shape[1] - 2), axis=1)  # |sum| <= sqrt(d)|row|, |P r| ~ sqrt(d)|row|
    scale = np.maximum(scale, 1e-300)
    return float(np.max(np.abs(got - want) / scale)) if got.size else 0.0


def compare(fx: dict, points: np.ndarray, weights: np.ndarray, centers: np.ndarray | None = None,
            costs: np.ndarray | None = None, exact_points: bool | None = None) -> dict:
    """Compare one run against a fixture; returns a report with ``ok``."""
    d = int(fx["d"])
    rep = {"rows": int(len(weights)), "rows_ref": int(len(fx["weights"]))}
    rep["weights_exact"] = bool(np.array_equal(np.asarray(weights, dtype=np.int64), fx["weights"]))
    P = np.ascontiguousarray(points, dtype=np.float64)
    rep["points_sha256_equal"] = sha256(P) == str(fx["points_sha256"])
    rep["points_rel_err"] = _sketch_close(sketch(P), fx["points_sketch"], d) if len(P) else 0.0
    if "points" in fx and fx["points"].shape == P.shape:
        den = np.maximum(np.abs(fx["points"]), np.abs(fx["points"]).max() * 1e-300 + 1e-300)
        rep["points_max_rel"] = float(np.max(np.abs(P - fx["points"]) / np.maximum(den, np.abs(fx["points"]).max())))
    if exact_points is None:
        exact_points = False
    ok = rep["weights_exact"] and (rep["points_sha256_equal"] if exact_points else rep["points_rel_err"] <= RTOL)
    if costs is not None:
        c = np.asarray(costs, dtype=np.float64)
        want = fx["costs"]
        rep["costs_max_rel"] = float(np.max(np.abs(c - want) / np.abs(want))) if c.shape == want.shape else float("inf")
        ok = ok and rep["costs_max_rel"] <= RTOL
    if centers is not None:
        C = np.asarray(centers, dtype=np.float64)
        cs = fx["centers_sketch"]
        if C.shape[0] != cs.shape[0]:
            rep["centers_rel_err"] = float("inf")
        else:
            rep["centers_rel_err"] = max(_sketch_close(sketch(C[r]), cs[r], d) for r in range(C.shape[0]))
        ok = ok and rep["centers_rel_err"] <= RTOL
        if "centers" in fx and fx["centers"].shape == C.shape:
            ref = fx["centers"]
            rep["centers_max_abs_over_scale"] = float(np.max(np.abs(C - ref)) / max(np.abs(ref).max(), 1e-300))
            ok = ok and rep["centers_max_abs_over_scale"] <= RTOL
    rep["ok"] = bool(ok)
    return rep
