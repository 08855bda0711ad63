"""Identical input rows must project to bit-identical rows (the reference's
LAPACK/BLAS path does; BICO then collapses them)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1502_04265_b200 import linalg as L
from paper_1502_04265_b200.mergereduce import MrConfig, run_piecy_mr

rows = np.tile([[2.0, -1.0, 3.0]], (24, 1))
cs = run_piecy_mr(iter(rows), 3, MrConfig(k=1, piece_size=4, num_pieces=2, svd_dim=1, coreset_size=4, seed=2))
print("all-equal:", len(cs), cs.weights, cs.points.tolist())
A = torch.from_numpy(np.tile([[2.0, -1.0, 3.0]], (4, 1))).cuda()
for seed in range(3):
    P = L.project_piece_device(A, L.SvdTruncation(1, 2, 2, seed)).cpu().numpy()
    print("piece", seed, P.tolist(), [np.array_equal(P[0], P[i]) for i in range(4)])
w = torch.tensor([3, 5, 7, 9], dtype=torch.int64).cuda()
P = L.weighted_project_device(A, w, L.SvdTruncation(1, 2, 2, 5)).cpu().numpy()
print("weighted", P.tolist(), [np.array_equal(P[0], P[i]) for i in range(4)])
