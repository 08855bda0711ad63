import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1502_04265_b200 import workloads as W
from paper_1502_04265_b200.pipeline import PiecyConfig, run_piecy, run_piecy_device
cfg = W.CONFIGS["cfg2"]
X = W.generate("cfg2")
pc = PiecyConfig(k=cfg.k, piece_size=cfg.piece_size, svd_dim=cfg.svd_dim, coreset_size=cfg.m, seed=cfg.seed)
Xd = torch.from_numpy(X).cuda()
def bench(name, fn):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(name, [round(t * 1e3, 1) for t in ts], "ms", flush=True)
bench("device", lambda: run_piecy_device(Xd, cfg.d, pc).extract_coreset())
bench("host   ", lambda: run_piecy(X, cfg.d, pc))
sys.setswitchinterval(5e-5)
bench("host si=50us", lambda: run_piecy(X, cfg.d, pc))
bench("device si=50us", lambda: run_piecy_device(Xd, cfg.d, pc).extract_coreset())
