"""Trace run_piecy_mr on 24 identical rows (reference test_all_equal_points_collapse)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1502_04265_b200 import linalg as L
from paper_1502_04265_b200.coreset import BicoEngine
from paper_1502_04265_b200.util import mix_seed

x = np.array([2.0, -1.0, 3.0])
hexs = lambda a: [v.hex() for v in np.asarray(a).ravel()]
A = torch.from_numpy(np.tile(x, (4, 1))).cuda()
for pi in range(6):
    P = L.project_piece_device(A, L.SvdTruncation(1, 2, 2, 2 ^ pi)).cpu().numpy()
    print("piece", pi, hexs(P[0]), all(np.array_equal(P[0], P[i]) for i in range(4)))
for f in (1, 2, 3):
    e = BicoEngine(3, 4)
    e.insert_block(np.tile(x, (8, 1)))
    cs = e.extract_coreset()
    print("L0 flush", f, len(cs), cs.weights, hexs(cs.points[0]))
    Pd = torch.from_numpy(cs.points).cuda()
    wd = torch.from_numpy(cs.weights).cuda()
    q = L.weighted_project_device(Pd, wd, L.SvdTruncation(1, 0, 2, mix_seed(2, 1, f))).cpu().numpy()
    print("   weighted proj", hexs(q[0]))
