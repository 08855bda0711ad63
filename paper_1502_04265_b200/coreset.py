"""Drop-in BICO engine backed by the device-resident CF tree.

Mirrors ``piecy.coreset`` (/root/reference/pkg/src/piecy/coreset.py): same
names, argument meaning and ValueError contracts.  The tree (references,
linear/square sums, groups) lives in HBM; ``insert`` buffers points on the
host and hands them to the GPU in blocks before any observer runs, so the
observable state is the same as one-at-a-time insertion.

The closed-form helpers and the ClusteringFeature snapshot type are scalar
API conveniences (reference :30-99) and are plain Python.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat

_BAD_MESSAGES = {
    1: "point has non-finite coordinates",
    2: "point coordinates overflow",
    3: "weight must be a positive integer",
}


def insertion_error_increment(group_weight: int, copies: int, dist_sq: float) -> float:
    """SSE increase s*w/(s+w)*dist_sq of adding ``copies`` copies at squared
    distance ``dist_sq`` from the centroid (coreset.py:30-34)."""
    return group_weight * copies / (group_weight + copies) * dist_sq


def max_insertable_copies(group_weight: int, copies: int, cur_error: float,
                          threshold: float, dist_sq: float) -> int:
    """Largest w' <= copies with cur_error + s*w'/(s+w')*dist_sq <= threshold
    (coreset.py:37-55); the same expression order the kernel uses."""
    slack = group_weight * dist_sq - threshold + cur_error
    if slack <= 0.0:
        return copies
    limit = (group_weight * threshold - group_weight * cur_error) / slack
    if limit >= copies:
        return copies
    if limit <= 0.0:
        return 0
    return int(limit)


@dataclass
class ClusteringFeature:
    """Feature snapshot (weight n, linear sum s, squared sum q, reference)."""

    weight: int
    linear_sum: np.ndarray
    square_sum: float
    reference: np.ndarray

    @classmethod
    def from_point(cls, point, weight: int = 1) -> "ClusteringFeature":
        x = np.asarray(point, dtype=np.float64)
        return cls(weight, weight * x, weight * float(x @ x), x.copy())

    @property
    def centroid(self) -> np.ndarray:
        return self.linear_sum / self.weight

    def internal_error(self) -> float:
        e = self.square_sum - float(self.linear_sum @ self.linear_sum) / self.weight
        return e if e > 0.0 else 0.0

    def cost_to(self, center) -> float:
        c = np.asarray(center, dtype=np.float64)
        if c.shape != self.linear_sum.shape:
            raise ValueError("center dimension does not match the feature")
        v = self.square_sum - 2.0 * float(c @ self.linear_sum) + self.weight * float(c @ c)
        return v if v > 0.0 else 0.0

    def merged_with(self, other: "ClusteringFeature") -> "ClusteringFeature":
        return ClusteringFeature(self.weight + other.weight,
                                 self.linear_sum + other.linear_sum,
                                 self.square_sum + other.square_sum,
                                 self.reference.copy())


@dataclass
class Coreset:
    """Weighted summary: one row per feature centroid (coreset.py:102-121)."""

    points: np.ndarray
    weights: np.ndarray

    def __len__(self) -> int:
        return self.points.shape[0]

    def __iter__(self):
        return zip(self.points, self.weights)

    @property
    def dim(self) -> int:
        return self.points.shape[1]

    @property
    def total_weight(self) -> int:
        return int(self.weights.sum())


def _device(device):
    import torch
    if device is None:
        if not torch.cuda.is_available():
            raise nat.NativeError("piecy_b200 needs a CUDA device (no CPU fallback)")
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise nat.NativeError("piecy_b200 engines live on CUDA devices only")
    return torch.device("cuda", d.index if d.index is not None else torch.cuda.current_device())


class BicoEngine:
    """Single-pass summarizer with a hard feature budget (coreset.py:213-451).

    Extra keyword arguments (not in the reference): ``device`` (CUDA device),
    ``block_rows`` (rows per device block) and ``host_buffer`` (rows the
    single-point ``insert`` buffers before a device flush).
    """

    def __init__(self, dim: int, budget: int, *, bootstrap_cap: int = 1001,
                 device=None, block_rows: int = 0, host_buffer: int = 8192):
        if dim < 1:
            raise ValueError("dim must be >= 1")
        if budget < 1:
            raise ValueError("budget must be >= 1")
        self._dim = int(dim)
        self._budget = int(budget)
        self._dev = _device(device)
        self._h = None
        L = nat.lib()
        h = ctypes.c_void_p()
        import torch
        with torch.cuda.device(self._dev):
            nat.check(L.pcy_engine_create(self._dev.index, self._dim, self._budget, int(bootstrap_cap),
                                          int(block_rows), ctypes.byref(h)), "pcy_engine_create")
        self._h = h
        self._hb = np.empty((max(1, int(host_buffer)), self._dim))
        self._hw = np.empty(self._hb.shape[0], dtype=np.int64)
        self._hn = 0
        self._hunit = True

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                nat.lib().pcy_engine_destroy(h)
            except Exception:
                pass
            self._h = None

    # -- properties ---------------------------------------------------------
    @property
    def dim(self) -> int:
        return self._dim

    @property
    def budget(self) -> int:
        return self._budget

    @property
    def device(self):
        return self._dev

    def _stats(self):
        self._flush()
        nf, T, tw, b = ctypes.c_longlong(), ctypes.c_double(), ctypes.c_longlong(), ctypes.c_int()
        nat.check(nat.lib().pcy_engine_stats(self._h, ctypes.byref(nf), ctypes.byref(T), ctypes.byref(tw),
                                             ctypes.byref(b), nat.stream_ptr()), "pcy_engine_stats")
        return nf.value, T.value, tw.value, bool(b.value)

    @property
    def total_weight(self) -> int:
        return self._stats()[2]

    @property
    def threshold(self) -> float:
        return self._stats()[1]

    @property
    def num_features(self) -> int:
        return self._stats()[0]

    # -- ingestion ----------------------------------------------------------
    def insert(self, point, weight: int = 1) -> None:
        """Absorb ``weight`` copies of ``point`` (coreset.py:264-281)."""
        x = np.asarray(point, dtype=np.float64)
        if x.ndim != 1 or x.shape[0] != self._dim:
            raise ValueError(f"expected a point of dimension {self._dim}")
        w = int(weight)
        if w < 1:
            raise ValueError("weight must be a positive integer")
        x_sq = float(x @ x)
        if not math.isfinite(x_sq):
            if not np.isfinite(x).all():
                raise ValueError("point has non-finite coordinates")
            raise ValueError("point coordinates overflow")
        self._hb[self._hn] = x
        self._hw[self._hn] = w
        self._hunit &= (w == 1)
        self._hn += 1
        if self._hn == self._hb.shape[0]:
            self._flush()

    def _flush(self) -> None:
        n = self._hn
        if n == 0:
            return
        import torch
        self._hn = 0
        x = torch.from_numpy(self._hb[:n]).to(self._dev, non_blocking=False)
        w = None if self._hunit else torch.from_numpy(self._hw[:n]).to(self._dev)
        self._hunit = True
        self._insert_dev(x, w)

    def insert_block(self, points, weights=None) -> None:
        """Insert the rows of ``points`` in order (host array or CUDA tensor,
        float32 or float64).  Raises ValueError at the first invalid row; the
        engine then holds exactly the rows before it."""
        import torch
        self._flush()
        if isinstance(points, torch.Tensor):
            x = points
        else:
            arr = np.asarray(points)
            if arr.dtype not in (np.float32, np.float64):
                arr = arr.astype(np.float64)
            x = torch.from_numpy(np.ascontiguousarray(arr))
        if x.dim() != 2 or x.shape[1] != self._dim:
            raise ValueError(f"expected a point of dimension {self._dim}")
        if x.device != self._dev:
            x = x.to(self._dev)
        w = None
        if weights is not None:
            w = weights if isinstance(weights, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(np.asarray(weights, dtype=np.int64)))
            w = w.to(self._dev, dtype=torch.int64)
        self._insert_dev(x, w)

    def insert_device(self, x, w=None, stream=None) -> int:
        """Insert rows of CUDA tensor ``x`` (n x dim, f32/f64, row stride may
        exceed dim) with optional int64 weights ``w``.  Returns rows consumed.
        Rows buffered by ``insert`` go first, so the stream order holds."""
        import torch
        if not isinstance(x, torch.Tensor) or x.dim() != 2 or x.shape[1] != self._dim:
            raise ValueError(f"expected a point of dimension {self._dim}")
        if x.device != self._dev:
            raise ValueError(f"points must be on the engine's device {self._dev}")
        if w is not None:
            if not isinstance(w, torch.Tensor) or w.shape != (x.shape[0],) or w.device != self._dev:
                raise ValueError("weights must be one per point, on the engine's device")
            if w.dtype != torch.int64:
                w = w.to(torch.int64)
        self._flush()
        return self._insert_dev(x, w, stream)

    def _insert_dev(self, x, w=None, stream=None) -> int:
        import torch
        n = int(x.shape[0])
        if n == 0:
            return 0
        if x.dtype == torch.float64:
            dt = 0
        elif x.dtype == torch.float32:
            dt = 1
        else:
            raise ValueError("points must be float32 or float64")
        if x.stride(1) != 1:
            x = x.contiguous()
        if w is not None:
            w = w.contiguous()
        consumed, bad = ctypes.c_longlong(), ctypes.c_int()
        nat.check(nat.lib().pcy_engine_insert(self._h, nat.ptr(x), dt, x.stride(0), nat.ptr(w), n,
                                              nat.stream_ptr(stream), ctypes.byref(consumed),
                                              ctypes.byref(bad)), "pcy_engine_insert")
        if bad.value:
            raise ValueError(_BAD_MESSAGES.get(bad.value, "invalid point"))
        return consumed.value

    def counters(self) -> dict:
        """K3 instrumentation: levels walked, direct scans, demand row loads,
        full capacity evaluations, items resolved, deepest level."""
        self._flush()
        out = np.zeros(6, dtype=np.int64)
        nat.check(nat.lib().pcy_engine_counters(self._h, out.ctypes.data), "pcy_engine_counters")
        keys = ("levels", "tc_rechecks", "demand_loads", "slow_capacity", "items", "max_depth")
        return {k: int(v) for k, v in zip(keys, out)}

    def work(self) -> dict:
        """K1 work counters (pcy_engine_work): member visits of the chain walks
        (the reference's own dgemv work), those served by direct fp64 scans,
        tensor-pipe flops of the big-group panel and its launches.  The
        useful fraction of SURVEY.md §8d is 2*d*visits / executed flops."""
        self._flush()
        out = np.zeros(4, dtype=np.float64)
        nat.check(nat.lib().pcy_engine_work(self._h, out.ctypes.data), "pcy_engine_work")
        d = float(self._dim)
        useful = 2.0 * d * out[0]
        executed = 2.0 * d * out[1] + out[2]
        return {"member_visits": int(out[0]), "direct_visits": int(out[1]), "tensor_flops": float(out[2]),
                "panel_launches": int(out[3]), "useful_flops": useful, "executed_flops": executed,
                "useful_fraction": useful / executed if executed > 0 else None}

    # -- extraction ---------------------------------------------------------
    def features_device(self):
        """(levels, weights, linear sums, square sums, references) as CUDA tensors, DFS order."""
        import torch
        nf = self.num_features
        lv = torch.empty(nf, dtype=torch.int32, device=self._dev)
        w = torch.empty(nf, dtype=torch.int64, device=self._dev)
        s = torch.empty((nf, self._dim), dtype=torch.float64, device=self._dev)
        q = torch.empty(nf, dtype=torch.float64, device=self._dev)
        r = torch.empty((nf, self._dim), dtype=torch.float64, device=self._dev)
        cnt = ctypes.c_longlong()
        nat.check(nat.lib().pcy_engine_features(self._h, nat.ptr(lv), nat.ptr(w), nat.ptr(s), nat.ptr(q),
                                                nat.ptr(r), nf, ctypes.byref(cnt), nat.stream_ptr()),
                  "pcy_engine_features")
        k = cnt.value
        return lv[:k], w[:k], s[:k], q[:k], r[:k]

    def features(self):
        """[(level, ClusteringFeature)] in deterministic traversal order (coreset.py:425-441)."""
        lv, w, s, q, r = (t.cpu().numpy() for t in self.features_device())
        return [(int(lv[i]), ClusteringFeature(int(w[i]), s[i].copy(), float(q[i]), r[i].copy()))
                for i in range(lv.shape[0])]

    def extract_device(self):
        """Coreset rows (s/n) and int64 weights as CUDA tensors."""
        import torch
        nf = self.num_features
        pts = torch.empty((nf, self._dim), dtype=torch.float64, device=self._dev)
        w = torch.empty(nf, dtype=torch.int64, device=self._dev)
        cnt = ctypes.c_longlong()
        nat.check(nat.lib().pcy_engine_extract(self._h, nat.ptr(pts), nat.ptr(w), nf, ctypes.byref(cnt),
                                               nat.stream_ptr()), "pcy_engine_extract")
        k = cnt.value
        return pts[:k], w[:k]

    def extract_coreset(self) -> Coreset:
        """One weighted point per feature (coreset.py:443-451)."""
        pts, w = self.extract_device()
        if pts.shape[0] == 0:
            return Coreset(np.zeros((0, self._dim)), np.zeros(0, dtype=np.int64))
        return Coreset(pts.cpu().numpy(), w.cpu().numpy())
