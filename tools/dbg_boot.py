import numpy as np, sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from oracle.piecy_oracle import OracleEngine
from paper_1502_04265_b200 import BicoEngine
rng = np.random.default_rng(1)
d, m, n = 57, 2000, 20000
centers = rng.uniform(-20, 20, size=(30, d))
X = centers[rng.integers(0, 30, size=n)] + rng.normal(size=(n, d))
for seqboot in (0, 1):
    if seqboot: os.environ["PCY_SEQ_BOOT"] = "1"
    g = BicoEngine(d, m); o = OracleEngine(d, m)
    for a in range(0, 6000, 1777):
        g.insert_block(X[a:a+1777]); o.insert_block(X[a:a+1777])
        print(seqboot, a, g.total_weight, o.total_weight, g.num_features, o.num_features, flush=True)
