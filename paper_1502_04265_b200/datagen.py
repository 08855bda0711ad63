"""Paper instance families, generated on the device.

Drop-in for ``piecy.datagen`` (/root/reference/pkg/src/piecy/datagen.py):
the same configs, validation and bit-identical streams.  The coordinates come
from numpy's Philox4x64-10 generator exactly as the reference draws them
(``Generator(Philox(key=seed)).random``, datagen.py:15-16); csrc/datagen.cu
evaluates draw t of that stream directly on the GPU (word t % 4 of the
counter block t // 4 + 1), so an instance is written into HBM in one launch.
Only SWN's per-cluster ``permutation`` calls (a few ints per cluster) run on
the host, on numpy's own generator, which also yields each cluster's first
draw index.

``*_device(cfg)`` return the (n_points x dim) float64 CUDA tensor; the
reference-named generators yield the rows one by one like the reference.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Iterator

import numpy as np

from . import _native as nat

c_i32, c_i64, c_u64, c_f64, c_vp = ctypes.c_int, ctypes.c_longlong, ctypes.c_ulonglong, ctypes.c_double, ctypes.c_void_p
nat.register("pcy_gen_swn", c_i32, [c_vp, c_i64, c_i32, c_i64, c_i32, c_i32, c_u64, c_u64, c_vp, c_vp, c_f64, c_f64,
                                    c_vp])
nat.register("pcy_gen_cube", c_i32, [c_vp, c_i64, c_i64, c_i64, c_u64, c_u64, c_u64, c_f64, c_vp])
nat.register("pcy_gen_lower_bound", c_i32, [c_vp, c_i64, c_i32, c_i64, c_f64, c_f64, c_vp])

_MASK = (1 << 64) - 1


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=seed))


def _key(seed: int) -> tuple[int, int]:
    k = int(seed) & ((1 << 128) - 1)
    return k & _MASK, k >> 64


def _next_draw(bitgen: np.random.Philox) -> int:
    """Global index of the next 64-bit output numpy's Philox will hand out."""
    st = bitgen.state
    c = st["state"]["counter"]
    ctr = int(c[0]) | (int(c[1]) << 64)
    return ctr * 4 if st["buffer_pos"] >= 4 else (ctr - 1) * 4 + int(st["buffer_pos"])


def _seek(bitgen: np.random.Philox, seed: int, t: int) -> None:
    """Move numpy's Philox to global draw t (keeps its 32-bit half buffer)."""
    st = bitgen.state
    tmp = np.random.Philox(key=seed, counter=t // 4)
    if t % 4:
        tmp.random_raw(t % 4)
    nst = tmp.state
    nst["has_uint32"], nst["uinteger"] = st["has_uint32"], st["uinteger"]
    bitgen.state = nst


@dataclass(frozen=True)
class SwnConfig:
    """Hidden-cluster instance (datagen.py:19-45)."""

    clusters: int
    points_per_cluster: int
    dim: int
    active_dims: int
    spread: float = 10.0
    noise: float = 0.5
    seed: int = 0

    def __post_init__(self):
        if self.clusters < 1 or self.points_per_cluster < 1 or self.dim < 1:
            raise ValueError("clusters, points_per_cluster and dim must be >= 1")
        if not 1 <= self.active_dims <= self.dim:
            raise ValueError("active_dims must be in [1, dim]")
        if not self.spread > self.noise > 0:
            raise ValueError("need spread > noise > 0")

    @property
    def n_points(self) -> int:
        return self.clusters * self.points_per_cluster


@dataclass(frozen=True)
class LowerBoundConfig:
    """Nested-simplex instance (datagen.py:48-78); deterministic."""

    k: int
    n: int
    spread: float = 1000.0
    noise: float = 100.0
    seed: int = 0

    def __post_init__(self):
        if self.k < 2:
            raise ValueError("k must be >= 2")
        if self.n < self.k or self.n % self.k != 0:
            raise ValueError("n must be a positive multiple of k")
        if not self.spread > self.noise > 0:
            raise ValueError("need spread > noise > 0")

    @property
    def n_points(self) -> int:
        return self.n

    @property
    def dim(self) -> int:
        return self.k + self.n


@dataclass(frozen=True)
class RandomConfig:
    """n-by-n cube instance (datagen.py:81-101)."""

    n: int
    spread: float = 10.0
    seed: int = 0

    def __post_init__(self):
        if self.n < 1:
            raise ValueError("n must be >= 1")
        if self.spread <= 0:
            raise ValueError("spread must be positive")

    @property
    def n_points(self) -> int:
        return self.n

    @property
    def dim(self) -> int:
        return self.n


def _device(device):
    import torch
    return device or torch.device("cuda", torch.cuda.current_device())


def structured_with_noise_device(cfg: SwnConfig, device=None):
    """The SWN stream (cluster-major, datagen.py:104-112) as a CUDA tensor."""
    import torch
    dev = _device(device)
    rng = _rng(cfg.seed)
    bg = rng.bit_generator
    per_point = cfg.dim + cfg.active_dims
    base = np.zeros(cfg.clusters, dtype=np.uint64)
    inv = np.full((cfg.clusters, cfg.dim), -1, dtype=np.int32)
    for c in range(cfg.clusters):
        active = rng.permutation(cfg.dim)[: cfg.active_dims]
        inv[c, active] = np.arange(cfg.active_dims, dtype=np.int32)
        t = _next_draw(bg)
        base[c] = t
        _seek(bg, cfg.seed, t + cfg.points_per_cluster * per_point)   # the cluster's points
    out = torch.empty((cfg.n_points, cfg.dim), dtype=torch.float64, device=dev)
    bd = torch.from_numpy(base.view(np.int64)).to(dev)
    invd = torch.from_numpy(inv).to(dev)
    k0, k1 = _key(cfg.seed)
    nat.check(nat.lib().pcy_gen_swn(nat.ptr(out), cfg.dim, cfg.clusters, cfg.points_per_cluster, cfg.dim,
                                    cfg.active_dims, k0, k1, nat.ptr(bd), nat.ptr(invd), float(cfg.noise),
                                    float(cfg.spread), nat.stream_ptr()), "pcy_gen_swn")
    return out


def random_cube_device(cfg: RandomConfig, device=None):
    """The cube instance (datagen.py:131-135) as a CUDA tensor."""
    import torch
    dev = _device(device)
    out = torch.empty((cfg.n, cfg.n), dtype=torch.float64, device=dev)
    k0, k1 = _key(cfg.seed)
    nat.check(nat.lib().pcy_gen_cube(nat.ptr(out), cfg.n, cfg.n, cfg.n, k0, k1, 0, float(cfg.spread),
                                     nat.stream_ptr()), "pcy_gen_cube")
    return out


def lower_bound_device(cfg: LowerBoundConfig, device=None):
    """The nested-simplex instance (datagen.py:115-128) as a CUDA tensor."""
    import torch
    dev = _device(device)
    out = torch.empty((cfg.n, cfg.dim), dtype=torch.float64, device=dev)
    nat.check(nat.lib().pcy_gen_lower_bound(nat.ptr(out), cfg.dim, cfg.k, cfg.n, float(cfg.spread),
                                            float(cfg.noise), nat.stream_ptr()), "pcy_gen_lower_bound")
    return out


def generate_device(cfg, device=None):
    if isinstance(cfg, SwnConfig):
        return structured_with_noise_device(cfg, device)
    if isinstance(cfg, LowerBoundConfig):
        return lower_bound_device(cfg, device)
    if isinstance(cfg, RandomConfig):
        return random_cube_device(cfg, device)
    raise TypeError("unknown generator config")


def _rows(t, block: int = 4096) -> Iterator[np.ndarray]:
    n = int(t.shape[0])
    for a in range(0, n, block):
        host = t[a:a + block].cpu().numpy()
        for row in host:
            yield row.copy()


def structured_with_noise(cfg: SwnConfig) -> Iterator[np.ndarray]:
    """Yield the hidden-cluster points in cluster-major order."""
    return _rows(structured_with_noise_device(cfg))


def lower_bound(cfg: LowerBoundConfig) -> Iterator[np.ndarray]:
    """Yield the nested-simplex points in vertex-major order."""
    return _rows(lower_bound_device(cfg))


def random_cube(cfg: RandomConfig) -> Iterator[np.ndarray]:
    """Yield n points with n iid uniform coordinates each."""
    return _rows(random_cube_device(cfg))
