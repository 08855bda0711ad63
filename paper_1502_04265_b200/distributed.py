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
                         ops=None, concurrent: bool = True, tree_out: list | None = None,
                         phases: dict | None = None):
    """Sharded run_piecy_mr.  ``source(a, b)`` returns rows [a, b) of the stream
    (any rank may read any range; each reads only its own groups).  Returns the
    Coreset on rank 0 and None elsewhere.

    Rank 0 merges in group order *as the summaries become available*: its own
    groups run on worker threads (one CUDA stream each) and group g is
    replayed into level 1 as soon as it -- and every group before it -- is
    done, local or received, so the merge overlaps the remaining shard work.
    The other ranks post their summaries with non-blocking sends.  ``phases``
    (optional dict) receives the per-phase wall times of this rank: shard
    compute, gather wait (rank 0: time blocked on remote summaries), merge."""
    if ops is None:
        ops = DeviceOps(cfg)
    if cfg.svd_dim > dim:
        raise ValueError(f"svd_dim {cfg.svd_dim} exceeds point dimension {dim}")
    groups = level0_groups(n_rows, cfg.piece_size, cfg.num_pieces)
    mine = [g for g in groups if owner(g.index, world) == rank]
    results = {}
    done = {g.index: threading.Event() for g in mine}
    errs = []
    ph = {"shard_s": 0.0, "gather_wait_s": 0.0, "merge_s": 0.0, "groups_local": len(mine),
          "groups_total": len(groups), "world": world}
    t_start = time.perf_counter()

    def work(grp):
        try:
            with ops.stream_scope():
                results[grp.index] = group_summary(ops, source, grp, dim, cfg, len(groups))
        except BaseException as exc:   # surface worker failures on the caller
            errs.append(exc)
        finally:
            done[grp.index].set()

    threads = []
    if concurrent and len(mine) > 1:
        threads = [threading.Thread(target=work, args=(g,), daemon=True) for g in mine]
        for t in threads:
            t.start()
    else:
        for g in mine:
            work(g)

    def finish_local():
        for t in threads:
            t.join()
        if errs:
            raise errs[0]
        ops.sync()
        ph["shard_s"] = time.perf_counter() - t_start

    if rank != 0:   # post every summary to rank 0 as it completes, in group order
        pending = []
        for g in mine:
            done[g.index].wait()
            if errs:
                break
            pending.append(ops.send(results[g.index], 0))
        finish_local()
        for h in pending:
            if h is not None:
                h.wait()
        if phases is not None:
            phases.update(ph)
        return None

    tree = ops.tree(dim, cfg)
    if tree_out is not None:
        tree_out.append(tree)
    if not groups:
        finish_local()
        return ops.finish(tree, None)
    if len(groups) == 1 and not groups[0].full:
        finish_local()
        pts, wts, _ = results[0]
        tree.stats.pieces = groups[0].pieces
        return ops.coreset(pts, wts)
    for g in groups:
        if owner(g.index, world) == 0:
            done[g.index].wait()
            if errs:
                finish_local()
            item = results[g.index]
            ops.ready(item)
        else:
            t0 = time.perf_counter()
            item = ops.recv(owner(g.index, world), dim)
            ph["gather_wait_s"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        pts, wts, flushed = item
        tree.stats.flush_sources.append(0)
        tree.insert_reduced(1, pts, wts)
        ph["merge_s"] += time.perf_counter() - t0
    finish_local()
    tree.stats.pieces = sum(g.pieces for g in groups)
    tree.stats.points_read = n_rows
    t0 = time.perf_counter()
    out = ops.finish(tree, None)
    ops.sync()
    ph["merge_s"] += time.perf_counter() - t0
    ph["total_s"] = time.perf_counter() - t_start
    if os.environ.get("PCY_DEBUG_MR"):
        print(f"[mr] rank {rank}: {ph}", flush=True)
    if phases is not None:
        phases.update(ph)
    return out


class Exchange:
    """Point-to-point transport of the reduced summaries over the default
    process group: NCCL sends device tensors directly (NVLink); gloo stages
    them through host memory.  send() is non-blocking and returns a handle."""

    def __init__(self, device):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.device = torch, dist, device
        self.host = dist.is_initialized() and dist.get_backend() == "gloo"

    def _out(self, t):
        return t.cpu() if self.host else t

    def send(self, tensors, dst):
        dist = self.dist
        works = []
        keep = []
        for t in tensors:
            t = self._out(t.contiguous())
            keep.append(t)
            works.append(dist.isend(t, dst))
        return _Handles(works, keep)

    def recv(self, shape, dtype, src):
        torch = self.torch
        t = torch.empty(shape, dtype=dtype, device="cpu" if self.host else self.device)
        self.dist.recv(t, src)
        return t.to(self.device) if self.host else t


class _Handles:
    def __init__(self, works, keep):
        self.works, self.keep = works, keep

    def wait(self):
        for w in self.works:
            w.wait()


class DeviceOps:
    """Group work on the CUDA engine; exchange over the default process group
    (NCCL device-to-device, or gloo through host memory: ``Exchange``)."""

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

    def ready(self, item):
        """A locally produced summary is about to be merged: nothing to wait
        for -- the worker synchronised its stream before signalling."""

    def _xchg(self):
        if not hasattr(self, "_ex"):
            self._ex = Exchange(self.device)
        return self._ex

    def send(self, item, dst):
        pts, wts, flushed = item
        torch = self.torch
        pts = pts.to(torch.float64).contiguous()
        hdr = torch.tensor([pts.shape[0], 1 if flushed else 0], dtype=torch.int64, device=self.device)
        torch.cuda.current_stream(self.device).synchronize()
        return self._xchg().send([hdr, pts, wts.contiguous()] if pts.shape[0] else [hdr], dst)

    def recv(self, src, dim):
        torch = self.torch
        ex = self._xchg()
        hdr = ex.recv((2,), torch.int64, src)
        n = int(hdr[0])
        if n:
            pts = ex.recv((n, dim), torch.float64, src)
            wts = ex.recv((n,), torch.int64, src)
        else:
            pts = torch.empty((0, dim), dtype=torch.float64, device=self.device)
            wts = torch.empty(0, dtype=torch.int64, device=self.device)
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
