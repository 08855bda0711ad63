"""Debug probe: one engine over the first rows of a config, with K3 counters."""
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1502_04265_b200 import workloads as W  # noqa: E402
from paper_1502_04265_b200 import _native as nat  # noqa: E402
from paper_1502_04265_b200.pipeline import PiecyConfig, run_piecy_device  # noqa: E402

name = sys.argv[1]
rows = int(sys.argv[2])
cfg = W.CONFIGS[name]
X = W.generate_rows(name, 0, rows) if cfg.entry != "piecy" else W.generate(name, rows)
Xd = torch.from_numpy(X).cuda()
pc = PiecyConfig(k=cfg.k, piece_size=cfg.piece_size, svd_dim=cfg.svd_dim, coreset_size=cfg.m, seed=cfg.seed)
nat.prof_reset(); nat.prof_enable(True)
torch.cuda.synchronize(); t0 = time.time()
eng = run_piecy_device(Xd, cfg.d, pc)
torch.cuda.synchronize(); t1 = time.time()
print(name, rows, "secs", round(t1 - t0, 3), "F", eng.num_features, "T", eng.threshold)
print("counters", eng.counters())
print({k: nat.prof_read(k) for k in ("resolve", "chain", "reattach")})
