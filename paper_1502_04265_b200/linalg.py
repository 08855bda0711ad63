"""Randomized best-fit projection on the GPU.

Drop-in for the hot-path part of ``piecy.linalg``
(/root/reference/pkg/src/piecy/linalg.py): ``SvdTruncation``, ``Projector``,
``randomized_truncated_svd``, ``project``, ``weighted_best_fit``.  The
Gaussian sketches are the reference's exact numpy PCG64 draws (generated on
the host, uploaded); GEMMs, CholeskyQR2 and the Jacobi core SVD run in
csrc/linalg.cu.  Only the sketched span reaches the result, so the basis
conventions of the QR do not matter (SURVEY.md §7 hard part 5).
"""

from __future__ import annotations

import ctypes
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native as nat

DEFAULT_OVERSAMPLE = 10
DEFAULT_POWER_ITERATIONS = 2
EXACT_ENTRY_LIMIT = 4_000_000
_SIGMA_CLIP = 1e-12

c_i32, c_i64, c_f64, c_vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_double, ctypes.c_void_p
nat.register("pcy_dgemm", c_i32, [c_i32, c_i32, c_i32, c_f64, c_vp, c_i64, c_i32, c_vp, c_i64, c_i32, c_f64,
                                  c_vp, c_i64, c_vp])
nat.register("pcy_cast_f32_f64", c_i32, [c_vp, c_i64, c_vp, c_vp])
nat.register("pcy_scale_rows_sqrtw", c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp, c_vp])
nat.register("pcy_rsvd", c_i32, [c_vp, c_i64, c_i32, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp])
nat.register("pcy_project", c_i32, [c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_vp])
nat.register("pcy_all_finite", c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp])


def as_matrix(a) -> np.ndarray:
    """Dense, finite, float64, one point per row (linalg.py:26-35)."""
    mat = np.ascontiguousarray(a, dtype=np.float64)
    if mat.ndim != 2:
        raise ValueError(f"expected a 2-d matrix, got ndim={mat.ndim}")
    if mat.shape[1] < 1:
        raise ValueError("matrix must have at least one column")
    if not np.isfinite(mat).all():
        raise ValueError("matrix contains non-finite entries")
    return mat


@dataclass(frozen=True)
class SvdTruncation:
    """Configuration for the randomized truncated SVD (linalg.py:38-53)."""

    rank: int
    oversample: int = DEFAULT_OVERSAMPLE
    power_iterations: int = DEFAULT_POWER_ITERATIONS
    seed: int = 0

    def __post_init__(self):
        if self.rank < 1:
            raise ValueError("rank must be >= 1")
        if self.oversample < 0:
            raise ValueError("oversample must be >= 0")
        if self.power_iterations < 0:
            raise ValueError("power_iterations must be >= 0")


@dataclass(frozen=True)
class Projector:
    """Rank-l best-fit subspace: orthonormal right singular vectors plus the
    retained singular values (linalg.py:56-74)."""

    vectors: np.ndarray
    singular_values: np.ndarray

    def __post_init__(self):
        self.vectors.setflags(write=False)
        self.singular_values.setflags(write=False)

    @property
    def rank(self) -> int:
        return self.vectors.shape[1]

    @property
    def dim(self) -> int:
        return self.vectors.shape[0]


# ----------------------------------------------------------------- device
def to_f64_device(a, device=None):
    """float64 CUDA copy/view of a host array or tensor (fp32 upcast by kernel)."""
    import torch
    if isinstance(a, torch.Tensor):
        t = a if device is None else a.to(device)
        if not t.is_cuda:
            t = t.to(torch.device("cuda", torch.cuda.current_device()))
    else:
        arr = np.asarray(a)
        if arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        arr = np.ascontiguousarray(arr)
        with warnings.catch_warnings():
            # read-only inputs (memory-mapped stream files): the host view is
            # only read by the H2D copy below, so no host copy is made
            warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
            host = torch.from_numpy(arr)
        t = host.to(device or torch.device("cuda", torch.cuda.current_device()))
    t = t.contiguous()
    if t.dtype == torch.float64:
        return t
    if t.dtype != torch.float32:
        raise ValueError("expected float32 or float64 data")
    out = torch.empty(t.shape, dtype=torch.float64, device=t.device)
    nat.check(nat.lib().pcy_cast_f32_f64(nat.ptr(t), t.numel(), nat.ptr(out), nat.stream_ptr()), "cast")
    return out


def check_finite_device(t) -> None:
    """Raise ValueError if a CUDA tensor holds a non-finite entry.  The kernel
    scans numel() contiguous f32/f64 elements, so anything else (another dtype,
    a strided or sliced view) is first made a contiguous float64 copy."""
    import torch
    if t.dtype not in (torch.float32, torch.float64) or not t.is_contiguous():
        t = t.to(torch.float64).contiguous()
    flag = np.zeros(1, dtype=np.int32)
    dt = 0 if t.dtype == torch.float64 else 1
    nat.check(nat.lib().pcy_all_finite(nat.ptr(t), t.numel(), dt, flag.ctypes.data, nat.stream_ptr()),
              "all_finite")
    if not flag[0]:
        raise ValueError("matrix contains non-finite entries")


def rsvd_device(A, rank: int, oversample: int, power: int, seed: int):
    """Randomized truncated SVD of a float64 CUDA matrix -> (V (cols x rank) tensor, sigma ndarray)."""
    import torch
    rows, cols = int(A.shape[0]), int(A.shape[1])
    r = rank + oversample
    if r > min(rows, cols):
        raise ValueError(f"rank + oversample = {r} exceeds min(rows, cols) = {min(rows, cols)}")
    rng = np.random.default_rng(seed)
    om = rng.standard_normal((cols, r))
    om2 = rng.standard_normal((r, r)) if rows > 4 * r else None
    dev = A.device
    omd = torch.from_numpy(om).to(dev)
    om2d = torch.from_numpy(om2).to(dev) if om2 is not None else None
    V = torch.empty((cols, rank), dtype=torch.float64, device=dev)
    sig = np.zeros(rank)
    rc = nat.lib().pcy_rsvd(nat.ptr(A), rows, cols, rank, r, power, nat.ptr(omd), nat.ptr(om2d),
                            nat.ptr(V), sig.ctypes.data, nat.stream_ptr())
    if rc == nat.PCY_ENONFINITE:   # checked on the device, read back with sigma
        raise ValueError("matrix contains non-finite entries")
    nat.check(rc, "pcy_rsvd")
    return V, sig


def project_device(A, V):
    """(A V) V^T for float64 CUDA tensors."""
    import torch
    rows, cols = int(A.shape[0]), int(A.shape[1])
    out = torch.empty((rows, cols), dtype=torch.float64, device=A.device)
    nat.check(nat.lib().pcy_project(nat.ptr(A), rows, cols, nat.ptr(V.contiguous()), int(V.shape[1]),
                                    nat.ptr(out), nat.stream_ptr()), "pcy_project")
    return out


def project_piece_device(piece, trunc: SvdTruncation):
    """Piece projection of run_piecy (pipeline.py:120-126) on the device
    (a non-finite entry raises ValueError from rsvd_device before anything is
    inserted, as the reference's as_matrix check does)."""
    A = to_f64_device(piece)
    V, _ = rsvd_device(A, trunc.rank, trunc.oversample, trunc.power_iterations, trunc.seed)
    return project_device(A, V)


def weighted_project_device(P, w, trunc: SvdTruncation):
    """weighted_best_fit + project of a coreset (mergereduce.py:118-122):
    sqrt(w)-scaled rows decide the subspace, the unscaled rows are projected."""
    import torch
    A = to_f64_device(P)
    w = w.to(A.device, dtype=torch.int64).contiguous()
    S = torch.empty_like(A)
    nat.check(nat.lib().pcy_scale_rows_sqrtw(nat.ptr(A), nat.ptr(w), int(A.shape[0]), int(A.shape[1]),
                                             nat.ptr(S), nat.stream_ptr()), "scale_rows")
    V, _ = rsvd_device(S, trunc.rank, trunc.oversample, trunc.power_iterations, trunc.seed)
    return project_device(A, V)


# ------------------------------------------------------------- public API
def randomized_truncated_svd(a, trunc: SvdTruncation) -> Projector:
    """Approximate top-``rank`` Projector via Gaussian sketching (linalg.py:167-206)."""
    mat = as_matrix(a)
    rows, cols = mat.shape
    r = trunc.rank + trunc.oversample
    if r > min(rows, cols):
        raise ValueError(f"rank + oversample = {r} exceeds min(rows, cols) = {min(rows, cols)}")
    V, sig = rsvd_device(to_f64_device(mat), trunc.rank, trunc.oversample, trunc.power_iterations, trunc.seed)
    return Projector(V.cpu().numpy(), sig)


def project(a, projector: Projector) -> np.ndarray:
    """Project rows of ``a`` onto the subspace: A V V^T (linalg.py:209-221)."""
    import torch
    mat = as_matrix(a)
    v = projector.vectors
    if mat.shape[1] != v.shape[0]:
        raise ValueError(f"matrix has {mat.shape[1]} columns but the projector expects {v.shape[0]}")
    A = to_f64_device(mat)
    # Projector freezes its vectors; hand torch a writable f64 copy
    Vd = torch.as_tensor(np.array(v, dtype=np.float64, order="C", copy=True), device=A.device)
    return project_device(A, Vd).cpu().numpy()


def weighted_best_fit(points, weights, trunc: SvdTruncation, *, exact: bool = False,
                      max_entries: int = EXACT_ENTRY_LIMIT) -> Projector:
    """Best-fit subspace of the row multiset given by integer weights (linalg.py:231-250)."""
    import torch
    mat = as_matrix(points)
    w = np.asarray(weights)
    if w.ndim != 1 or w.shape[0] != mat.shape[0]:
        raise ValueError("weights must be one per row")
    if not np.all(w >= 1):
        raise ValueError("weights must be positive integers (>= 1)")
    rows, cols = mat.shape
    if exact:   # exact_truncated_svd's contract (linalg.py:120-164): rank range, entry limit
        if trunc.rank < 1 or trunc.rank > min(rows, cols):
            raise ValueError(f"rank {trunc.rank} out of range for a {rows}x{cols} matrix")
        if rows * cols > max_entries:
            raise ValueError(f"matrix with {rows * cols} entries exceeds the exact-backend "
                             f"limit of {max_entries}")
    A = to_f64_device(mat)
    wd = torch.from_numpy(np.ascontiguousarray(w.astype(np.int64))).to(A.device)
    S = torch.empty_like(A)
    nat.check(nat.lib().pcy_scale_rows_sqrtw(nat.ptr(A), nat.ptr(wd), mat.shape[0], mat.shape[1], nat.ptr(S),
                                             nat.stream_ptr()), "scale_rows")
    if exact:
        # the exact backend: a sketch as wide as min(rows, cols) spans the whole
        # row space, so the device range finder + Jacobi core SVD return the
        # exact decomposition (to rounding; no squared condition number)
        full = min(rows, cols)
        V, sig = rsvd_device(S, trunc.rank, full - trunc.rank, 2, 0)
        return Projector(V.cpu().numpy(), sig)
    r = trunc.rank + trunc.oversample
    if r > min(mat.shape):
        raise ValueError(f"rank + oversample = {r} exceeds min(rows, cols) = {min(mat.shape)}")
    V, sig = rsvd_device(S, trunc.rank, trunc.oversample, trunc.power_iterations, trunc.seed)
    return Projector(V.cpu().numpy(), sig)
