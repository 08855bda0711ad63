"""Debug probe: per-phase device time of run_piecy on the first rows of a config."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_04265_b200 import workloads as W  # noqa: E402
from paper_1502_04265_b200 import linalg  # noqa: E402
from paper_1502_04265_b200 import _native as nat  # noqa: E402
from paper_1502_04265_b200.coreset import BicoEngine  # noqa: E402
from paper_1502_04265_b200.util import MASK64  # noqa: E402

name = sys.argv[1]
rows = int(sys.argv[2])
cfg = W.CONFIGS[name]
X = W.generate_rows(name, 0, rows) if cfg.entry != "piecy" else W.generate(name, rows)
Xd = torch.from_numpy(X).cuda()
ell = cfg.svd_dim
eng = BicoEngine(cfg.d, cfg.m)
tm = {"rng": 0.0, "rsvd": 0.0, "project": 0.0, "insert": 0.0, "cast": 0.0}


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


nat.prof_reset(); nat.prof_enable(True)
t_all = tick()
for index in range(0, (rows + cfg.piece_size - 1) // cfg.piece_size):
    piece = Xd[index * cfg.piece_size:(index + 1) * cfg.piece_size]
    block = piece
    if ell < cfg.d and piece.shape[0] >= ell:
        over = min(10, min(piece.shape[0], cfg.d) - ell)
        t0 = tick()
        A = linalg.to_f64_device(piece)
        t1 = tick(); tm["cast"] += t1 - t0
        r = ell + over
        rng = np.random.default_rng((cfg.seed ^ index) & MASK64)
        rng.standard_normal((cfg.d, r)); rng.standard_normal((r, r))
        t2 = tick(); tm["rng"] += t2 - t1
        V, _ = linalg.rsvd_device(A, ell, over, 2, (cfg.seed ^ index) & MASK64)
        t3 = tick(); tm["rsvd"] += t3 - t2
        block = linalg.project_device(A, V)
        t4 = tick(); tm["project"] += t4 - t3
    t5 = tick()
    eng.insert_device(block)
    tm["insert"] += tick() - t5
t_end = tick()
print(name, rows, "total", round(t_end - t_all, 3), {k: round(v, 3) for k, v in tm.items()})
print({k: nat.prof_read(k) for k in nat.PROF_SLOTS})
