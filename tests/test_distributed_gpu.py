"""The sharded piecy-mr driver with the CUDA engine on both ranks and the
exchange over gloo (world size 2; both ranks use this box's one GPU -- their
kernels never wait on each other, only the host-side gloo exchange connects
them).  The result must equal the oracle's merge-and-reduce tree, with the
merge on rank 0 streamed in group order while shards are still running."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CASES = [  # (n, d, piece, num_pieces, svd_dim, m)
    (6000, 57, 250, 3, 57, 300),    # 8 groups, projection skipped (cfg4-like)
    (3000, 40, 200, 2, 8, 150),     # 8 groups, projection active (cfg5-like)
    (2100, 20, 100, 4, 20, 120),    # 6 groups incl. a partial tail
]


def _data(n, d):
    rng = np.random.default_rng(n + d)
    cen = rng.uniform(-8, 8, size=(9, d))
    return cen[rng.integers(0, 9, size=n)] + rng.normal(size=(n, d))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    from paper_1502_04265_b200 import distributed as D
    from paper_1502_04265_b200.mergereduce import MrConfig
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for (n, d, ps, npc, ell, m) in CASES:
        X = _data(n, d)
        cfg = MrConfig(k=4, piece_size=ps, num_pieces=npc, svd_dim=ell, coreset_size=m, seed=7)
        ph = {}
        res = D.run_piecy_mr_sharded(lambda a, b: torch.from_numpy(X[a:b]).to(dev), n, d, cfg, rank=rank,
                                     world=world, ops=D.DeviceOps(cfg, dev), phases=ph)
        if rank == 0:
            out.append((res.points, res.weights, ph))
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        q.put(out)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_ranks_gloo_exchange_equals_oracle_tree():
    from oracle import piecy_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for (n, d, ps, npc, ell, m), (pts, wts, ph) in zip(CASES, results):
        X = _data(n, d)
        want_p, want_w = O.piecy_mr(X, 4, ps, npc, ell, m, seed=7)
        assert np.array_equal(wts, want_w)
        np.testing.assert_allclose(pts, want_p, rtol=1e-9, atol=1e-9 * np.abs(want_p).max())
        assert ph["world"] == 2 and ph["groups_local"] >= 1 and ph["merge_s"] >= 0.0
