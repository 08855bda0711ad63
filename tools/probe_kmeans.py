"""Debug probe: seeding / Lloyd / cost device time on a coreset-shaped point set."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1502_04265_b200 import evaluation as ev  # noqa: E402

n, d, k, reps, iters = (int(a) for a in sys.argv[1:6])
rng = np.random.default_rng(0)
cent = rng.normal(0, 5, size=(k, d))
P = cent[rng.integers(0, k, size=n)] + rng.normal(0, 1, size=(n, d))
w = rng.integers(1, 50, size=n).astype(np.float64)
Pd, wd = torch.from_numpy(P).cuda(), torch.from_numpy(w).cuda()


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(2):
    t0 = tick()
    U = ev._uniforms(1, reps, k)
    C = ev.seed_device(Pd, wd, k, U)
    t1 = tick()
    logs = ev.lloyd_device(Pd, wd, C, iters, 1e-4)
    t2 = tick()
    costs = ev.cost_device(Pd, wd, C)
    t3 = tick()
    print(f"n={n} d={d} k={k} reps={reps}: seed {1e3*(t1-t0):.1f} ms, lloyd {1e3*(t2-t1):.1f} ms "
          f"({[len(l) for l in logs]} iters), cost {1e3*(t3-t2):.1f} ms")
