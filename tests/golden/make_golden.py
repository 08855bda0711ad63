"""Generate golden fixtures by running the UNMODIFIED reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports ``piecy`` from /root/reference/pkg/src (read-only, never copied) and
records its outputs on small seeded inputs into tests/golden/*.npz.  The
fixtures pin the CPU oracle (tests/test_oracle_golden.py) and the GPU path
(tests/test_golden_gpu.py); /root/reference does not exist on the GPU box,
only these files travel.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _features(engine):
    feats = engine.features()
    n = len(feats)
    d = engine.dim
    lv = np.array([L for L, _ in feats], dtype=np.int32)
    w = np.array([cf.weight for _, cf in feats], dtype=np.int64)
    s = np.stack([cf.linear_sum for _, cf in feats]) if n else np.zeros((0, d))
    q = np.array([cf.square_sum for _, cf in feats], dtype=np.float64)
    r = np.stack([cf.reference for _, cf in feats]) if n else np.zeros((0, d))
    return lv, w, s, q, r


def engine_case(name, X, W, d, m, out):
    from piecy.coreset import BicoEngine
    e = BicoEngine(d, m)
    for i in range(X.shape[0]):
        e.insert(X[i], 1 if W is None else int(W[i]))
    lv, w, s, q, r = _features(e)
    cs = e.extract_coreset()
    out[name] = dict(X=X, W=np.zeros(0, np.int64) if W is None else W, d=d, m=m, T=e.threshold,
                     total_weight=e.total_weight, lv=lv, w=w, s=s, q=q, r=r, pts=cs.points, wts=cs.weights)


def main():
    sys.path.insert(0, REF)
    import piecy
    from piecy import evaluation as ev
    from piecy import linalg as la
    from piecy.mergereduce import MergeReduceTree, MrConfig, run_piecy_mr
    from piecy.pipeline import PiecyConfig, run_bico, run_piecy
    from piecy.util import mix_seed

    cases = {}
    rng = np.random.default_rng(2024)
    # --- BICO engine: unit, weighted, duplicates, budget 1, bootstrap-only, fp32 mixed scales
    cen = rng.uniform(-20, 20, size=(25, 12))
    X = cen[rng.integers(0, 25, size=3000)] + rng.normal(size=(3000, 12))
    engine_case("engine_unit", X, None, 12, 120, cases)
    X = rng.normal(scale=4.0, size=(1500, 5))
    W = rng.integers(1, 9, size=1500)
    engine_case("engine_weighted", X, W, 5, 25, cases)
    base = rng.normal(size=(60, 4))
    X = np.repeat(base, 3, axis=0)[rng.permutation(180)]
    engine_case("engine_dups", X, None, 4, 30, cases)
    engine_case("engine_budget1", rng.normal(size=(200, 2)), None, 2, 1, cases)
    engine_case("engine_bootstrap", np.repeat(rng.normal(size=(20, 3)), 2, axis=0), None, 3, 50, cases)
    X = (rng.normal(size=(4000, 54)) * np.geomspace(1, 3000, 54)).astype(np.float32).astype(np.float64)
    engine_case("engine_scales", X, None, 54, 400, cases)

    # --- pipelines
    X = cen[rng.integers(0, 25, size=2400)] + rng.normal(size=(2400, 12))
    cs = run_bico(iter(X), 12, 200)
    cases["run_bico"] = dict(X=X, m=200, pts=cs.points, wts=cs.weights)
    Xp = rng.uniform(-10, 10, size=(8, 64))[rng.integers(0, 8, size=3000)] + rng.normal(size=(3000, 64))
    cfg = PiecyConfig(k=5, piece_size=500, svd_dim=8, coreset_size=250, seed=3)
    cs = run_piecy(iter(Xp), 64, cfg)
    cases["run_piecy"] = dict(X=Xp, k=5, piece_size=500, svd_dim=8, m=250, seed=3, pts=cs.points, wts=cs.weights)
    mcfg = MrConfig(k=4, piece_size=300, num_pieces=3, svd_dim=6, coreset_size=150, seed=5)
    trees = []
    cs = run_piecy_mr(iter(Xp), 64, mcfg, tree_out=trees)
    cases["run_piecy_mr"] = dict(X=Xp, k=4, piece_size=300, num_pieces=3, svd_dim=6, m=150, seed=5,
                                 pts=cs.points, wts=cs.weights,
                                 flush_sources=np.array(trees[0].stats.flush_sources, dtype=np.int64))
    mcfg2 = MrConfig(k=4, piece_size=300, num_pieces=3, svd_dim=64, coreset_size=150, seed=5)
    cs = run_piecy_mr(iter(Xp), 64, mcfg2)
    cases["run_piecy_mr_noproj"] = dict(X=Xp, k=4, piece_size=300, num_pieces=3, svd_dim=64, m=150, seed=5,
                                        pts=cs.points, wts=cs.weights)

    # --- linalg
    U = rng.normal(size=(900, 40)) * np.geomspace(50, 1, 40)
    A = U @ rng.normal(size=(40, 100)) + 1e-3 * rng.normal(size=(900, 100))
    pr = la.randomized_truncated_svd(A, la.SvdTruncation(20, 10, 2, 77))
    cases["rsvd_two_sided"] = dict(A=A, rank=20, ov=10, power=2, seed=77, V=pr.vectors, sigma=pr.singular_values,
                                   proj=la.project(A, pr))
    A2 = A[:100]
    pr = la.randomized_truncated_svd(A2, la.SvdTruncation(15, 10, 2, 78))
    cases["rsvd_one_sided"] = dict(A=A2, rank=15, ov=10, power=2, seed=78, V=pr.vectors, sigma=pr.singular_values)
    wts = rng.integers(1, 30, size=900)
    pr = la.weighted_best_fit(A, wts, la.SvdTruncation(12, 10, 2, 79))
    cases["weighted_fit"] = dict(A=A, w=wts, rank=12, ov=10, power=2, seed=79, V=pr.vectors, sigma=pr.singular_values)

    # --- clustering
    P = cen[rng.integers(0, 25, size=800)] + rng.normal(size=(800, 12))
    pw = rng.integers(1, 40, size=800).astype(np.float64)
    runs = ev.kmeans_repetitions(P, pw, 10, reps=5, seed=11, max_iters=100, tol=1e-4)
    cases["kmeans_reps"] = dict(P=P, w=pw, k=10, reps=5, seed=11, centers=np.stack([c for c, _ in runs]),
                                costs=np.array([c for _, c in runs]))
    log = []
    C0 = P[:10].copy()
    C = ev.lloyd_iterate(P, pw, C0, max_iters=50, tol=1e-6, cost_log=log)
    cases["lloyd"] = dict(P=P, w=pw, C0=C0, C=C, log=np.array(log))
    cases["seed"] = dict(P=P, w=pw, k=15, C=ev.kmeanspp_seed(P, pw, 15, np.random.default_rng(5)))
    cases["mix_seed"] = dict(args=np.array([[0, 0], [1, 2], [3, 1], [2**63, 7], [123456789, 987654321]], dtype=np.uint64),
                             vals=np.array([mix_seed(0, 0), mix_seed(1, 2), mix_seed(3, 1), mix_seed(2**63, 7),
                                            mix_seed(123456789, 987654321)], dtype=np.uint64))

    for name, dct in cases.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **{k: np.asarray(v) for k, v in dct.items()})
    with open(os.path.join(HERE, "MANIFEST.txt"), "w") as f:
        f.write(f"generated by tests/golden/make_golden.py from piecy {piecy.__version__} at {REF}\n")
        f.write(f"numpy {np.__version__}\n")
        for name in sorted(cases):
            f.write(name + "\n")
    print("wrote", len(cases), "fixtures")


if __name__ == "__main__":
    main()
