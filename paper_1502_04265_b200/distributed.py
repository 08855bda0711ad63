"""Sharded piecy-mr: level-0 groups of the merge-and-reduce tree on N GPUs.

In the reference tree (mergereduce.py:128-171) every run of ``num_pieces``
consecutive pieces feeds one level-0 engine that is flushed (extracted,
weight-projected with seed mix_seed(seed, 1, g+1), inserted into level 1)
before the next run starts.  The level-0 groups are therefore independent:
group g only needs its own pieces and the global piece index of each (piece
seed = seed ^ index, :140).  Only levels >= 1 are sequential.

Here group g runs on rank g mod N (several groups per GPU run concurrently on
separate CUDA streams).  The reduced level-0 summaries are gathered to rank 0
in group order -- the one exchange step, NCCL point-to-point over NVLink --
and rank 0 replays them into the upper levels with
``MergeReduceTree.insert_reduced``.  The result is identical to
``run_piecy_mr`` for any number of groups and any N.

The per-group work goes through an ``ops`` object so the same driver runs
with the CUDA engine (DeviceOps, NCCL) or, in the CPU tests, with the oracle
(gloo); see tests/test_distributed_cpu.py.
"""

from __future__ import annotations

import math
import os
import threading
import time
from dataclasses import dataclass

import numpy as np

from .util import MASK64, mix_seed


@dataclass(frozen=True)
class Group:
    index: int
    row_start: int
    row_end: int
    piece_start: int     # global index of the group's first piece
    pieces: int
    full: bool


def level0_groups(n_rows: int, piece_size: int, num_pieces: int) -> list[Group]:
    """Level-0 groups of the tree for a stream of n_rows (pieces of piece_size)."""
    n_pieces = math.ceil(n_rows / piece_size) if n_rows else 0
    out = []
    for g in range(math.ceil(n_pieces / num_pieces) if n_pieces else 0):
        p0 = g * num_pieces
        p1 = min(n_pieces, p0 + num_pieces)
        out.append(Group(g, p0 * piece_size, min(n_rows, p1 * piece_size), p0, p1 - p0, p1 - p0 == num_pieces))
    return out


def owner(g: int, world: int) -> int:
    return g % world


def group_summary(ops, source, grp: Group, dim: int, cfg, n_groups: int):
    """Run one level-0 group: projected pieces -> engine -> coreset, then the
    group's flush reduction.  Returns (points, weights, flushed)."""
    eng = ops.engine(dim, cfg.coreset_size)
    for p in range(grp.pieces):
        a = grp.row_start + p * cfg.piece_size
        b = min(grp.row_end, a + cfg.piece_size)
        block = source(a, b)
        red = ops.reduce(block, None, (cfg.seed ^ (grp.piece_start + p)) & MASK64)
        ops.insert(eng, red, None)
    pts, wts = ops.extract(eng)
    del eng
    # full groups flush when their last piece arrives; the trailing partial
    # group flushes in finalize() only if an earlier flush made level 1 live
    flushed = grp.full or n_groups > 1
    if flushed:
        pts = ops.reduce(pts, wts, mix_seed(cfg.seed, 1, grp.index + 1))
    return pts, wts, flushed


def run_piecy_mr_sharded(source, n_rows: int, dim: int, cfg, *, rank: int = 0, world: int = 1,
                         ops=None, concurrent: bool = True, tree_out: list | None = None):
    """Sharded run_piecy_mr.  ``source(a, b)`` returns rows [a, b) of the stream
    (any rank may read any range; each reads only its own groups).  Returns the
    Coreset on rank 0 and None elsewhere."""
    if ops is None:
        ops = DeviceOps(cfg)
    if cfg.svd_dim > dim:
        raise ValueError(f"svd_dim {cfg.svd_dim} exceeds point dimension {dim}")
    groups = level0_groups(n_rows, cfg.piece_size, cfg.num_pieces)
    mine = [g for g in groups if owner(g.index, world) == rank]
    results = {}

    def work(grp):
        with ops.stream_scope():
            results[grp.index] = group_summary(ops, source, grp, dim, cfg, len(groups))

    _dbg = os.environ.get("PCY_DEBUG_MR")
    _t0 = time.perf_counter()
    if concurrent and len(mine) > 1:
        errs = []

        def guard(fn, g):
            try:
                fn(g)
            except BaseException as exc:   # surface worker failures on the caller
                errs.append(exc)
        threads = [threading.Thread(target=guard, args=(work, g)) for g in mine]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        if errs:
            raise errs[0]
    else:
        for g in mine:
            work(g)
    ops.sync()
    if _dbg:
        print(f"[mr] rank {rank}: {len(mine)} level-0 groups in {time.perf_counter() - _t0:.3f} s", flush=True)
        _t0 = time.perf_counter()

    # gather to rank 0 in group order (the exchange step)
    if world > 1:
        if rank == 0:
            for g in groups:
                if owner(g.index, world) != 0:
                    results[g.index] = ops.recv(owner(g.index, world), dim)
        else:
            for g in mine:
                ops.send(results[g.index], 0)
            return None

    tree = ops.tree(dim, cfg)
    if tree_out is not None:
        tree_out.append(tree)
    if not groups:
        return ops.finish(tree, None)
    if len(groups) == 1 and not groups[0].full:
        pts, wts, _ = results[0]
        tree.stats.pieces = groups[0].pieces
        return ops.coreset(pts, wts)
    for g in groups:
        pts, wts, flushed = results[g.index]
        tree.stats.flush_sources.append(0)
        tree.insert_reduced(1, pts, wts)
    tree.stats.pieces = sum(g.pieces for g in groups)
    tree.stats.points_read = n_rows
    if _dbg:
        ops.sync()
        print(f"[mr] rank {rank}: merge of {len(groups)} summaries in {time.perf_counter() - _t0:.3f} s", flush=True)
        _t0 = time.perf_counter()
    out = ops.finish(tree, None)
    if _dbg:
        ops.sync()
        print(f"[mr] rank {rank}: finalize in {time.perf_counter() - _t0:.3f} s", flush=True)
    return out


class DeviceOps:
    """Group work on the CUDA engine; exchange over torch.distributed (NCCL)."""

    def __init__(self, cfg, device=None):
        import torch
        self.torch = torch
        self.cfg = cfg
        self.device = device or torch.device("cuda", torch.cuda.current_device())

    def stream_scope(self):
        torch = self.torch
        s = torch.cuda.Stream(device=self.device)
        return _StreamCtx(torch, s, self.device)

    def engine(self, dim, m):
        from .coreset import BicoEngine
        return BicoEngine(dim, m, device=self.device)

    def reduce(self, pts, wts, seed):
        from .mergereduce import reduce_device
        return reduce_device(pts, wts, pts.shape[1], self.cfg, seed)

    def insert(self, eng, block, wts):
        eng.insert_device(block, wts)

    def extract(self, eng):
        return eng.extract_device()

    def sync(self):
        self.torch.cuda.synchronize(self.device)

    def tree(self, dim, cfg):
        from .mergereduce import MergeReduceTree
        return MergeReduceTree(dim, cfg, device=self.device)

    def coreset(self, pts, wts):
        from .coreset import Coreset
        return Coreset(pts.cpu().numpy(), wts.cpu().numpy())

    def finish(self, tree, _):
        return tree.finalize()

    def send(self, item, dst):
        import torch.distributed as dist
        pts, wts, flushed = item
        torch = self.torch
        pts = pts.to(torch.float64).contiguous()
        hdr = torch.tensor([pts.shape[0], 1 if flushed else 0], dtype=torch.int64, device=self.device)
        dist.send(hdr, dst)
        if pts.shape[0]:
            dist.send(pts, dst)
            dist.send(wts.contiguous(), dst)

    def recv(self, src, dim):
        import torch.distributed as dist
        torch = self.torch
        hdr = torch.zeros(2, dtype=torch.int64, device=self.device)
        dist.recv(hdr, src)
        n = int(hdr[0])
        pts = torch.empty((n, dim), dtype=torch.float64, device=self.device)
        wts = torch.empty(n, dtype=torch.int64, device=self.device)
        if n:
            dist.recv(pts, src)
            dist.recv(wts, src)
        return pts, wts, bool(hdr[1])


class _StreamCtx:
    def __init__(self, torch, stream, device):
        self.torch, self.stream, self.device = torch, stream, device

    def __enter__(self):
        self.torch.cuda.set_device(self.device)
        self.ctx = self.torch.cuda.stream(self.stream)
        self.ctx.__enter__()
        return self

    def __exit__(self, *exc):
        self.stream.synchronize()
        return self.ctx.__exit__(*exc)


def run_piecy_mr_multi(X, dim: int, cfg, *, rank: int, world: int, device=None, concurrent: bool = True,
                       tree_out: list | None = None):
    """Convenience wrapper: X is the full stream (host ndarray or CUDA tensor
    visible to every rank); each rank uploads only its groups' rows."""
    import torch
    ops = DeviceOps(cfg, device)
    dev = ops.device

    def source(a, b):
        blk = X[a:b]
        if isinstance(blk, torch.Tensor):
            return blk.to(dev)
        return torch.from_numpy(np.ascontiguousarray(blk)).to(dev)

    return run_piecy_mr_sharded(source, X.shape[0], dim, cfg, rank=rank, world=world, ops=ops,
                                concurrent=concurrent, tree_out=tree_out)
