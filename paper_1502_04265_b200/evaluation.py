"""Weighted k-means++ seeding, weighted Lloyd and costs on the GPU.

Drop-in for ``piecy.evaluation`` (/root/reference/pkg/src/piecy/evaluation.py).
The random stream is the reference's: repetition ``rep`` draws exactly k
uniforms from ``numpy.random.default_rng(mix_seed(seed, rep))`` (one per
center, :49-53, :72-78); they are generated on the host and uploaded, and the
seeding / Lloyd / cost arithmetic runs in csrc/kmeans.cu.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat
from .util import mix_seed

DEFAULT_REPETITIONS = 5
DEFAULT_MAX_ITERS = 100
DEFAULT_TOL = 1e-4

c_i32, c_i64, c_f64, c_vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p
nat.register("pcy_kmeanspp", c_i32, [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp])
nat.register("pcy_lloyd", c_i32, [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_i32, c_f64, c_vp, c_vp, c_vp])
nat.register("pcy_cast_i64_f64", c_i32, [c_vp, c_i64, c_vp, c_vp])
nat.register("pcy_weighted_cost", c_i32, [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp])
nat.register("pcy_weighted_cost_dev", c_i32, [c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp])
nat.register("pcy_cost_chunks", c_i32, [c_vp, c_i64, c_i32, c_vp, c_i32, c_i64, c_vp, c_i64, c_vp])


def _as_points(points) -> np.ndarray:
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2:
        raise ValueError("points must be a 2-d array (one point per row)")
    return pts


def _as_weights(weights, count: int) -> np.ndarray:
    if weights is None:
        return np.ones(count)
    w = np.asarray(weights, dtype=np.float64)
    if w.shape != (count,):
        raise ValueError("weights must be one per point")
    if not np.all(w > 0):
        raise ValueError("weights must be positive")
    return w


def _dev_points(points, weights, device=None):
    """(P, w) as contiguous float64 CUDA tensors; accepts numpy or torch."""
    import torch
    if isinstance(points, torch.Tensor):
        P = points.to(device or points.device, dtype=torch.float64).contiguous()
        if P.dim() != 2:
            raise ValueError("points must be a 2-d array (one point per row)")
        if weights is None:
            w = torch.ones(P.shape[0], dtype=torch.float64, device=P.device)
        else:
            w = (weights if isinstance(weights, torch.Tensor) else torch.as_tensor(np.asarray(weights)))
            w = w.to(P.device).contiguous()
            if w.dtype == torch.int64:
                wf = torch.empty(w.shape, dtype=torch.float64, device=P.device)
                nat.check(nat.lib().pcy_cast_i64_f64(nat.ptr(w), w.numel(), nat.ptr(wf), nat.stream_ptr()), "cast")
                w = wf
            elif w.dtype != torch.float64:
                w = w.to(torch.float64)
            if w.shape != (P.shape[0],):
                raise ValueError("weights must be one per point")
        return P, w
    pts = _as_points(points)
    wts = _as_weights(weights, pts.shape[0])
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return (torch.from_numpy(np.ascontiguousarray(pts)).to(dev),
            torch.from_numpy(np.ascontiguousarray(wts)).to(dev))


REPS_PER_LAUNCH = 64   # csrc/kmeans.cu: repetitions per seeding / Lloyd launch


def _uniforms(seed: int, reps: int, k: int, start: int = 0) -> np.ndarray:
    return np.stack([np.random.default_rng(mix_seed(seed, r)).random(k) for r in range(start, reps)])


def seed_device(P, w, k: int, U: np.ndarray):
    """k-means++ for every row of U (reps x k uniforms) -> (reps, k, d) tensor."""
    import torch
    reps = U.shape[0]
    n, d = P.shape
    Ud = torch.from_numpy(np.ascontiguousarray(U, dtype=np.float64)).to(P.device)
    C = torch.empty((reps, k, d), dtype=torch.float64, device=P.device)
    nat.check(nat.lib().pcy_kmeanspp(nat.ptr(P), nat.ptr(w), n, d, k, reps, nat.ptr(Ud), nat.ptr(C), None,
                                     nat.stream_ptr()), "pcy_kmeanspp")
    return C


def _check_centers(P, C) -> None:
    """Centres (reps, k, d) must share the points' row length: the kernels take
    d from the centres (the reference fails in sq_distances, evaluation.py:41)."""
    if C.dim() != 3 or C.shape[2] != P.shape[1] or C.shape[1] < 1:
        raise ValueError("centers must match the point dimension")


def lloyd_device(P, w, C, max_iters: int, tol: float):
    """Lloyd in place on C (reps, k, d); returns per-rep cost logs."""
    _check_centers(P, C)
    reps, k, d = C.shape
    n = P.shape[0]
    logs = np.zeros((reps, max(1, max_iters)))
    iters = np.zeros(reps, dtype=np.int32)
    if max_iters > 0:
        nat.check(nat.lib().pcy_lloyd(nat.ptr(P), nat.ptr(w), n, d, k, reps, nat.ptr(C), int(max_iters),
                                      float(tol), logs.ctypes.data, iters.ctypes.data, nat.stream_ptr()),
                  "pcy_lloyd")
    return [list(logs[r, :iters[r]]) for r in range(reps)]


def cost_device(P, w, C) -> np.ndarray:
    _check_centers(P, C)
    reps, k, d = C.shape
    out = np.zeros(reps)
    nat.check(nat.lib().pcy_weighted_cost(nat.ptr(P), nat.ptr(w), P.shape[0], d, k, reps, nat.ptr(C),
                                          out.ctypes.data, nat.stream_ptr()), "pcy_weighted_cost")
    return out


def kmeanspp_seed(points, weights, k: int, rng: np.random.Generator) -> np.ndarray:
    """Draw ``k`` centers by the weighted D^2 rule (evaluation.py:56-82)."""
    pts = _as_points(points) if not _is_tensor(points) else points
    n = pts.shape[0]
    if n == 0:
        raise ValueError("cannot seed centers from an empty point set")
    if k < 1:
        raise ValueError("k must be >= 1")
    P, w = _dev_points(points, weights)
    U = rng.random(k)[None, :]
    return seed_device(P, w, k, U)[0].cpu().numpy()


def lloyd_iterate(points, weights, centers, max_iters: int = DEFAULT_MAX_ITERS,
                  tol: float = DEFAULT_TOL, cost_log: list | None = None) -> np.ndarray:
    """Weighted Lloyd with empty-cluster repair (evaluation.py:85-139)."""
    import torch
    P, w = _dev_points(points, weights)
    ctr = np.array(centers, dtype=np.float64, copy=True)
    if ctr.ndim != 2 or ctr.shape[1] != P.shape[1]:
        raise ValueError("centers must match the point dimension")
    if P.shape[0] == 0:
        return ctr
    C = torch.from_numpy(ctr).to(P.device)[None].contiguous()
    logs = lloyd_device(P, w, C, int(max_iters), float(tol))
    if cost_log is not None:
        cost_log.extend(float(c) for c in logs[0])
    return C[0].cpu().numpy()


def weighted_cost(points, weights, centers) -> float:
    """Weighted SSE of points against their nearest center (evaluation.py:142-149)."""
    import torch
    if not _is_tensor(points):
        pts = _as_points(points)
        _as_weights(weights, pts.shape[0])
        if pts.shape[0] == 0:
            return 0.0
    P, w = _dev_points(points, weights)
    ctr = np.asarray(centers, dtype=np.float64)
    if ctr.ndim != 2 or ctr.shape[1] != P.shape[1] or ctr.shape[0] < 1:
        raise ValueError("centers must match the point dimension")
    C = torch.from_numpy(np.ascontiguousarray(ctr)).to(P.device)[None].contiguous()
    return float(cost_device(P, w, C)[0])


def kmeans_repetitions(points, weights, k: int, reps: int = DEFAULT_REPETITIONS,
                       seed: int = 0, max_iters: int = DEFAULT_MAX_ITERS,
                       tol: float = DEFAULT_TOL):
    """Seeding + Lloyd ``reps`` times, repetition rng = PCG64(mix_seed(seed, rep))
    (evaluation.py:199-210).  All repetitions run concurrently on the device.
    Returns [(centers, cost), ...]."""
    if reps <= 0:
        return []
    C, costs = kmeans_repetitions_device(points, weights, k, reps, seed, max_iters, tol)
    Ch = C.cpu().numpy()
    return [(Ch[r], float(costs[r])) for r in range(reps)]


def kmeans_repetitions_device(points, weights, k: int, reps: int = DEFAULT_REPETITIONS,
                              seed: int = 0, max_iters: int = DEFAULT_MAX_ITERS,
                              tol: float = DEFAULT_TOL, cost_logs: list | None = None):
    """Device form: returns (centers (reps, k, d) CUDA tensor, costs ndarray)."""
    P, w = _dev_points(points, weights)
    if P.shape[0] == 0:
        raise ValueError("cannot seed centers from an empty point set")
    if k < 1:
        raise ValueError("k must be >= 1")
    import torch
    if reps <= 0:
        return torch.empty((0, k, int(P.shape[1])), dtype=torch.float64, device=P.device), np.zeros(0)
    # every repetition owns its PCG64(mix_seed(seed, rep)) stream, so running
    # them in chunks of REPS_PER_LAUNCH gives the same results as one launch
    Cs, costs = [], []
    for r0 in range(0, reps, REPS_PER_LAUNCH):
        U = _uniforms(seed, min(reps, r0 + REPS_PER_LAUNCH), k, start=r0)
        C = seed_device(P, w, k, U)
        logs = lloyd_device(P, w, C, int(max_iters), float(tol))
        if cost_logs is not None:
            cost_logs.extend(logs)
        Cs.append(C)
        costs.append(cost_device(P, w, C))
    if len(Cs) == 1:
        return Cs[0], costs[0]
    return torch.cat(Cs), np.concatenate(costs)


def _is_tensor(x) -> bool:
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except Exception:
        return False


@dataclass(frozen=True)
class CostSummary:
    minimum: float
    maximum: float
    average: float
    median: float

    @classmethod
    def of(cls, costs) -> "CostSummary":
        arr = np.asarray(list(costs), dtype=np.float64)
        if arr.size == 0:
            raise ValueError("no costs to summarize")
        return cls(float(arr.min()), float(arr.max()), float(arr.mean()), float(np.median(arr)))


def _stream_blocks(point_stream, chunk: int):
    """The reference's chunk framing (evaluation.py:172-179): consecutive blocks
    of ``chunk`` rows, the last one partial.  Arrays and tensors are sliced;
    a ``streams.PointSource`` is read block-wise; other iterables are gathered
    row by row."""
    if _is_tensor(point_stream) or isinstance(point_stream, np.ndarray):
        n = int(point_stream.shape[0])
        for a in range(0, n, chunk):
            yield point_stream[a:a + chunk]
        return
    blocks = getattr(point_stream, "blocks", None)
    if callable(blocks):
        for blk in blocks(chunk):
            yield blk[0] if isinstance(blk, tuple) else blk
        return
    buf = []
    for x in point_stream:
        buf.append(np.asarray(x, dtype=np.float64))
        if len(buf) == chunk:
            yield np.stack(buf)
            buf = []
    if buf:
        yield np.stack(buf)


def evaluate_cost_multi(center_sets, point_stream, chunk: int = 8192) -> list:
    """One streaming pass; unweighted SSE of the stream against each center
    set (evaluation.py:157-180).  The stream is taken in super-blocks of 64
    chunks; per block and set one device call computes the GEMM-form distances
    (fp64 tensor pipe), the first minimum and the per-chunk sums.  The chunk
    sums stay on the device until the end and are then added in chunk order,
    like the reference's running totals."""
    import torch
    from .linalg import to_f64_device
    if chunk < 1:
        raise ValueError("chunk must be >= 1")
    sets = [np.asarray(c, dtype=np.float64) for c in center_sets]
    if not sets:
        return []
    dev = torch.device("cuda", torch.cuda.current_device())
    Cs = [torch.from_numpy(np.ascontiguousarray(c)).to(dev) for c in sets]
    parts = []
    for blk in _stream_blocks(point_stream, chunk * 64):
        P = to_f64_device(blk)
        if P.dim() != 2 or any(P.shape[1] != c.shape[1] for c in sets):
            raise ValueError("points and centers must have the same dimension")
        nb = int(P.shape[0])
        out = torch.empty(((nb + chunk - 1) // chunk, len(sets)), dtype=torch.float64, device=dev)
        for i, C in enumerate(Cs):
            nat.check(nat.lib().pcy_cost_chunks(nat.ptr(P), nb, int(P.shape[1]), nat.ptr(C), int(C.shape[0]),
                                                chunk, nat.ptr(out[:, i:]), len(sets), nat.stream_ptr()),
                      "pcy_cost_chunks")
        parts.append(out)
    totals = [0.0] * len(sets)
    if parts:
        for row in torch.cat(parts).cpu().numpy():
            for i in range(len(sets)):
                totals[i] += float(row[i])
    return [float(t) for t in totals]


def evaluate_cost(centers, point_stream, chunk: int = 8192) -> float:
    """Unweighted SSE of a stream against its nearest center (evaluation.py:152-154)."""
    return evaluate_cost_multi([centers], point_stream, chunk=chunk)[0]
