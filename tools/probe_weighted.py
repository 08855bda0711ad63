"""Debug probe: one engine over a weighted point set shaped like the piecy-mr merge
(8 group summaries of a cfg4 stream), with K3 counters and kernel times."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_04265_b200 import workloads as W  # noqa: E402
from paper_1502_04265_b200 import _native as nat  # noqa: E402
from paper_1502_04265_b200.coreset import BicoEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 160000
X = W.generate_rows("cfg4", 0, n)
rng = np.random.default_rng(0)
w = rng.integers(1, 400, size=n).astype(np.int64)
Xd = torch.from_numpy(X).cuda()
wd = torch.from_numpy(w).cuda()
nat.prof_reset(); nat.prof_enable(True)
torch.cuda.synchronize(); t0 = time.time()
eng = BicoEngine(57, 20000)
eng.insert_device(Xd, wd)
torch.cuda.synchronize(); t1 = time.time()
print("weighted", n, "secs", round(t1 - t0, 3), "F", eng.num_features)
print("counters", eng.counters())
print({k: nat.prof_read(k) for k in ("resolve", "chain", "reattach")})
