"""The sharded piecy-mr driver (distributed.py) on CPU with world_size 2 over
gloo, the per-group work done by the CPU oracle.  Its result must equal the
single-process merge-and-reduce tree for any group count (no GPU)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import piecy_oracle as O
from paper_1502_04265_b200 import distributed as D
from paper_1502_04265_b200.mergereduce import MrConfig


class OracleTreeAdapter:
    """Upper levels of the oracle tree with the insert_reduced entry point."""

    def __init__(self, dim, cfg):
        self.t = O.OracleTree(dim, cfg.k, cfg.piece_size, cfg.num_pieces, cfg.svd_dim, cfg.coreset_size,
                              cfg.oversample, cfg.power_iterations, cfg.seed)

        class _S:
            flush_sources = []
            pieces = 0
            points_read = 0
        self.stats = _S()
        self.stats.flush_sources = self.t.flush_sources

    def insert_reduced(self, level, pts, wts):
        up = self.t._slot(level)
        if pts.shape[0]:
            up[0].insert_block(pts, wts)
        up[1] += 1
        if up[1] == self.t.np_:
            self.t._flush(level)


class OracleOps:
    def __init__(self, cfg, dim):
        self.cfg, self.dim = cfg, dim
        self.red = O.OracleTree(dim, cfg.k, cfg.piece_size, cfg.num_pieces, cfg.svd_dim, cfg.coreset_size,
                                cfg.oversample, cfg.power_iterations, cfg.seed)

    def stream_scope(self):
        import contextlib
        return contextlib.nullcontext()

    def engine(self, dim, m):
        return O.OracleEngine(dim, m)

    def reduce(self, pts, wts, seed):
        return self.red._reduce(np.asarray(pts, dtype=np.float64), wts, seed)

    def insert(self, eng, block, wts):
        eng.insert_block(block, wts)

    def extract(self, eng):
        return eng.extract()

    def sync(self):
        pass

    def tree(self, dim, cfg):
        return OracleTreeAdapter(dim, cfg)

    def coreset(self, pts, wts):
        return pts, wts

    def finish(self, tree, _):
        return tree.t.finalize()

    def ready(self, item):
        pass

    def send(self, item, dst):
        pts, wts, flushed = item
        dist.send(torch.tensor([pts.shape[0], int(flushed)], dtype=torch.int64), dst)
        if pts.shape[0]:
            dist.send(torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float64)), dst)
            dist.send(torch.from_numpy(np.ascontiguousarray(wts, dtype=np.int64)), dst)

    def recv(self, src, dim):
        hdr = torch.zeros(2, dtype=torch.int64)
        dist.recv(hdr, src)
        n = int(hdr[0])
        pts = torch.empty((n, dim), dtype=torch.float64)
        wts = torch.empty(n, dtype=torch.int64)
        if n:
            dist.recv(pts, src)
            dist.recv(wts, src)
        return pts.numpy(), wts.numpy(), bool(hdr[1])


CASES = [  # (n, d, piece, num_pieces, svd_dim, m)
    (1170, 20, 90, 4, 5, 60),     # 4 groups, partial tail, projection active
    (1170, 20, 90, 4, 20, 60),    # projection skipped
    (2000, 12, 50, 3, 4, 40),     # 14 groups: level-1 cascades
    (150, 8, 40, 5, 3, 30),       # one partial group
    (200, 8, 40, 5, 3, 30),       # exactly one full group
]


def _data(n, d):
    rng = np.random.default_rng(n + d)
    cen = rng.uniform(-8, 8, size=(6, d))
    return cen[rng.integers(0, 6, size=n)] + rng.normal(size=(n, d))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    for (n, d, ps, npc, ell, m) in CASES:
        X = _data(n, d)
        cfg = MrConfig(k=3, piece_size=ps, num_pieces=npc, svd_dim=ell, coreset_size=m, seed=9)
        res = D.run_piecy_mr_sharded(lambda a, b: X[a:b], n, d, cfg, rank=rank, world=world,
                                     ops=OracleOps(cfg, d), concurrent=False)
        if rank == 0:
            out.append(res)
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


def test_groups_cover_the_stream():
    gs = D.level0_groups(1170, 90, 4)
    assert [g.pieces for g in gs] == [4, 4, 4, 1]
    assert gs[-1].row_end == 1170 and not gs[-1].full and gs[0].full
    assert [D.owner(g.index, 2) for g in gs] == [0, 1, 0, 1]
    assert D.level0_groups(0, 10, 3) == []


@pytest.mark.parametrize("world", [1, 2])
def test_sharded_equals_sequential_tree(world):
    if world == 1:
        results = []
        for (n, d, ps, npc, ell, m) in CASES:
            X = _data(n, d)
            cfg = MrConfig(k=3, piece_size=ps, num_pieces=npc, svd_dim=ell, coreset_size=m, seed=9)
            results.append(D.run_piecy_mr_sharded(lambda a, b: X[a:b], n, d, cfg, ops=OracleOps(cfg, d),
                                                  concurrent=False))
    else:
        ctx = mp.get_context("spawn")
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
        for p in procs:
            p.start()
        results = q.get(timeout=300)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    for (n, d, ps, npc, ell, m), (pts, wts) in zip(CASES, results):
        want_p, want_w = O.piecy_mr(_data(n, d), 3, ps, npc, ell, m, seed=9)
        assert np.array_equal(wts, want_w)
        assert np.array_equal(pts, want_p)
