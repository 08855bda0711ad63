import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_1502_04265_b200 import linalg, _native as nat
A = torch.randn(12500, 4096, dtype=torch.float64, device="cuda")
def t():
    torch.cuda.synchronize(); return time.perf_counter()
for it in range(4):
    t0 = t()
    rng = np.random.default_rng(it); om = rng.standard_normal((4096, 385)); om2 = rng.standard_normal((385, 385))
    t1 = t()
    omd = torch.from_numpy(om).to("cuda"); om2d = torch.from_numpy(om2).to("cuda")
    t2 = t()
    V = torch.empty((4096, 375), dtype=torch.float64, device="cuda"); sig = np.zeros(375)
    nat.check(nat.lib().pcy_rsvd(nat.ptr(A), 12500, 4096, 375, 385, 2, nat.ptr(omd), nat.ptr(om2d), nat.ptr(V), sig.ctypes.data, nat.stream_ptr()), "x")
    t3 = t()
    out = linalg.project_device(A, V)
    t4 = t()
    print(f"rng {1e3*(t1-t0):.1f} h2d {1e3*(t2-t1):.1f} rsvd {1e3*(t3-t2):.1f} project {1e3*(t4-t3):.1f} ms")
