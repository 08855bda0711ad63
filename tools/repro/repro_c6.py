"""Reproduce the reference acceptance criterion 6 streams (SWN 20x500x200,
seed 7) through the drop-in and compare with the oracle."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_1502_04265_b200 import datagen as D
from paper_1502_04265_b200.mergereduce import MrConfig, run_piecy_mr
from paper_1502_04265_b200.pipeline import PiecyConfig, run_bico, run_piecy
from oracle import piecy_oracle as O

X = D.structured_with_noise_device(D.SwnConfig(20, 500, 200, 20, seed=7)).cpu().numpy()
k, budget = 20, 4000
for name, fn, ofn in [
        ("bico", lambda: run_bico(X, 200, budget), lambda: O.bico(X, budget)),
        ("piecy", lambda: run_piecy(X, 200, PiecyConfig(k=k, piece_size=2000, svd_dim=30, coreset_size=budget, seed=3)),
         lambda: O.piecy(X, k, 2000, 30, budget, seed=3)),
        ("mr", lambda: run_piecy_mr(X, 200, MrConfig(k=k, piece_size=2000, num_pieces=3, svd_dim=30, coreset_size=budget, seed=3)),
         lambda: O.piecy_mr(X, k, 2000, 3, 30, budget, seed=3))]:
    try:
        cs = fn()
        p, w = ofn()
        print(name, len(cs), len(w), np.array_equal(cs.weights, w), float(np.abs(cs.points - p).max()) if len(w) == len(cs) else None, flush=True)
    except Exception as e:
        print(name, "ERROR", e, flush=True)
