"""GPU path vs golden outputs of the unmodified reference (tests/golden/).

Membership, levels, weights, references and linear sums bit-exact; square
sums / T within 1e-12 relative; projected coresets, centers and costs within
1e-9 relative (fp64, different summation order)."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
G = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    return dict(np.load(os.path.join(G, f"{name}.npz")))


@pytest.mark.parametrize("name", ["engine_unit", "engine_weighted", "engine_dups", "engine_budget1",
                                  "engine_bootstrap", "engine_scales"])
def test_engine(name):
    from paper_1502_04265_b200 import BicoEngine
    g = load(name)
    e = BicoEngine(int(g["d"]), int(g["m"]))
    e.insert_block(g["X"], g["W"] if g["W"].size else None)
    assert e.total_weight == int(g["total_weight"])
    assert abs(e.threshold - float(g["T"])) <= 1e-12 * max(1.0, abs(float(g["T"])))
    lv, w, s, q, r = (t.cpu().numpy() for t in e.features_device())
    assert np.array_equal(lv, g["lv"]) and np.array_equal(w, g["w"])
    assert np.array_equal(r, g["r"]) and np.array_equal(s, g["s"])
    np.testing.assert_allclose(q, g["q"], rtol=1e-12)
    cs = e.extract_coreset()
    assert np.array_equal(cs.weights, g["wts"]) and np.array_equal(cs.points, g["pts"])


def test_run_bico():
    from paper_1502_04265_b200.pipeline import run_bico
    g = load("run_bico")
    cs = run_bico(iter(g["X"]), g["X"].shape[1], int(g["m"]))
    assert np.array_equal(cs.weights, g["wts"]) and np.array_equal(cs.points, g["pts"])


def test_run_piecy():
    from paper_1502_04265_b200.pipeline import PiecyConfig, run_piecy
    g = load("run_piecy")
    cfg = PiecyConfig(k=int(g["k"]), piece_size=int(g["piece_size"]), svd_dim=int(g["svd_dim"]),
                      coreset_size=int(g["m"]), seed=int(g["seed"]))
    cs = run_piecy(g["X"], g["X"].shape[1], cfg)
    assert np.array_equal(cs.weights, g["wts"])
    np.testing.assert_allclose(cs.points, g["pts"], rtol=1e-9, atol=1e-9 * np.abs(g["pts"]).max())


@pytest.mark.parametrize("name", ["rsvd_two_sided", "rsvd_one_sided", "weighted_fit"])
def test_projection(name):
    from paper_1502_04265_b200 import linalg
    g = load(name)
    tr = linalg.SvdTruncation(int(g["rank"]), int(g["ov"]), int(g["power"]), int(g["seed"]))
    pr = (linalg.weighted_best_fit(g["A"], g["w"], tr) if "w" in g else linalg.randomized_truncated_svd(g["A"], tr))
    np.testing.assert_allclose(pr.singular_values, g["sigma"], rtol=1e-10)
    np.testing.assert_allclose(pr.vectors, g["V"], atol=1e-9)
    if "proj" in g:
        np.testing.assert_allclose(linalg.project(g["A"], pr), g["proj"], atol=1e-9 * np.abs(g["proj"]).max())


def test_clustering():
    from paper_1502_04265_b200 import evaluation as ev
    g = load("kmeans_reps")
    runs = ev.kmeans_repetitions(g["P"], g["w"], int(g["k"]), reps=int(g["reps"]), seed=int(g["seed"]))
    np.testing.assert_allclose(np.stack([c for c, _ in runs]), g["centers"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose([c for _, c in runs], g["costs"], rtol=1e-9)
    g = load("lloyd")
    log = []
    C = ev.lloyd_iterate(g["P"], g["w"], g["C0"], max_iters=50, tol=1e-6, cost_log=log)
    assert len(log) == len(g["log"])
    np.testing.assert_allclose(C, g["C"], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(log, g["log"], rtol=1e-10)
    g = load("seed")
    assert np.array_equal(ev.kmeanspp_seed(g["P"], g["w"], int(g["k"]), np.random.default_rng(5)), g["C"])
