"""Full-size reference fixtures for the five BASELINE configs (build container only).

    python tests/golden/make_fullsize.py cfg1 cfg2 cfg3      # minutes
    python tests/golden/make_fullsize.py cfg4                # ~25 min, one core
    python tests/golden/make_fullsize.py cfg5                # ~1.5 h

Runs the UNMODIFIED reference (``piecy`` imported from /root/reference/pkg/src,
read-only, never copied) through its own public entry points on the exact
streams ``paper_1502_04265_b200.workloads`` generates:

* cfg1-3: ``run_piecy(iter(X), d, PiecyConfig(...))``   (pipeline.py:102-139)
* cfg4-5: ``run_piecy_mr(iter(X), d, MrConfig(...))``   (mergereduce.py:190-202)
* then ``kmeans_repetitions(P, w, k, reps=5, seed, max_iters, tol=1e-4)``
  (evaluation.py:199-210) on the coreset, exactly as ``coreset_cost_report``
  (pipeline.py:142-149) and the CLI (cli.py:263-265) call it.

Nothing of size travels: each ``full_<cfg>.npz`` holds the input's sha256
(the GPU box regenerates the stream and checks it), the coreset weights in
order (int64, exact), the sha256 of the coreset point bytes, a sketch of the
points (row sums, squared norms, four fixed random directions) for the
tolerance checks of projected configs, and the k-means costs plus a sketch of
the centres (full centres when small).  The run manifest (numpy version,
OPENBLAS_NUM_THREADS, CPU, wall times) goes into the same file.
"""

from __future__ import annotations

import json
import os
import platform
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

sys.path.insert(0, HERE)
from fullsize import sha256, sketch  # noqa: E402  (the checker's own digests)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def run(name: str) -> None:
    sys.path.insert(0, REF)
    import piecy
    from piecy.evaluation import kmeans_repetitions
    from piecy.mergereduce import MrConfig, run_piecy_mr
    from piecy.pipeline import PiecyConfig, run_piecy

    from paper_1502_04265_b200 import workloads as W

    cfg = W.CONFIGS[name]
    t0 = time.perf_counter()
    X = W.generate(name)
    t_gen = time.perf_counter() - t0
    in_sha = sha256(X)
    print(f"{name}: generated {X.shape} {X.dtype} in {t_gen:.1f}s sha256 {in_sha[:16]}", flush=True)

    t0 = time.perf_counter()
    extra = {}
    if cfg.entry == "piecy":
        pc = PiecyConfig(k=cfg.k, piece_size=cfg.piece_size, svd_dim=cfg.svd_dim, coreset_size=cfg.m,
                         seed=cfg.seed)
        cs = run_piecy(iter(X), cfg.d, pc)
    else:
        mc = MrConfig(k=cfg.k, piece_size=cfg.piece_size, num_pieces=cfg.num_pieces, svd_dim=cfg.svd_dim,
                      coreset_size=cfg.m, seed=cfg.seed)
        trees = []
        cs = run_piecy_mr(iter(X), cfg.d, mc, tree_out=trees)
        extra["flush_sources"] = np.array(trees[0].stats.flush_sources, dtype=np.int64)
    t_build = time.perf_counter() - t0
    P, w = cs.points, cs.weights
    print(f"{name}: coreset {P.shape} mass {int(w.sum())} in {t_build:.1f}s", flush=True)

    t0 = time.perf_counter()
    runs = kmeans_repetitions(P, w.astype(np.float64), cfg.k, reps=cfg.reps, seed=cfg.seed,
                              max_iters=cfg.max_iters, tol=1e-4)
    t_cluster = time.perf_counter() - t0
    C = np.stack([c for c, _ in runs])
    costs = np.array([c for _, c in runs], dtype=np.float64)
    print(f"{name}: kmeans costs {costs} in {t_cluster:.1f}s", flush=True)

    manifest = {
        "config": name, "entry": cfg.entry, "piecy_version": piecy.__version__, "reference": REF,
        "numpy": np.__version__, "python": platform.python_version(),
        "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS"), "cpu": cpu_model(),
        "nproc": os.cpu_count(), "seconds": {"generate": t_gen, "build": t_build, "cluster": t_cluster},
        "points_per_s": cfg.n / t_build,
    }
    out = dict(
        input_sha256=np.array(in_sha), n=np.int64(X.shape[0]), d=np.int64(X.shape[1]),
        weights=w.astype(np.int64), points_sha256=np.array(sha256(P)), points_sketch=sketch(P),
        costs=costs, centers_sketch=np.stack([sketch(c) for c in C]),
        manifest=np.array(json.dumps(manifest)), **extra,
    )
    if C.size <= 40_000:
        out["centers"] = C
    if P.size <= 200_000:
        out["points"] = P
    path = os.path.join(HERE, f"full_{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["cfg1", "cfg2", "cfg3"]:
        run(nm)
