"""One piece projection (rsvd + project) at a config's piece shape, timed
with CUDA events; with --ncu a single call for the launch list."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1502_04265_b200 import linalg as L
from paper_1502_04265_b200 import workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
cfg = W.CONFIGS[name]
X = W.generate_rows(name, 0, cfg.piece_size) if cfg.entry != "piecy" else W.generate(name)[:cfg.piece_size]
A = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float64)).cuda()
r = cfg.svd_dim + min(10, min(A.shape) - cfg.svd_dim)
tr = L.SvdTruncation(cfg.svd_dim, r - cfg.svd_dim, 2, 7)
reps = 1 if "--ncu" in sys.argv else 20
for _ in range(2 if reps > 1 else 0):
    L.project_piece_device(A, tr)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    P = L.project_piece_device(A, tr)
torch.cuda.synchronize()
print(f"{name} piece {tuple(A.shape)} r={r}: {(time.perf_counter() - t0) / reps * 1e3:.3f} ms per projection")
