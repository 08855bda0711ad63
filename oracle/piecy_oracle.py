"""CPU oracle for the piecy / piecy-mr hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module.  It is the checker, never
the product: ``paper_1502_04265_b200`` does not import it.

It restates the reference algorithm (``/root/reference/pkg/src/piecy``):

* the BICO engine -> plain C in ``bico_oracle.c`` (loaded through ctypes);
* seeding / Lloyd / cost (evaluation.py:39-149, :199-210) -> numpy below;
* randomized truncated SVD, projection, weighted fit (linalg.py:77-94,
  :167-250) -> numpy below;
* piece pipeline (pipeline.py:66-139) and merge-and-reduce tree
  (mergereduce.py:73-202) -> plain Python drivers below;
* splitmix64 seed folding (util.py:8-21).

Pinning: ``tests/golden/`` holds outputs of the unmodified reference run in
the build container (script: ``tests/golden/make_golden.py``); the
``-m "not gpu"`` tests check this oracle against them.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libbico_oracle.so")
_MASK64 = (1 << 64) - 1
_PHI64 = 0x9E3779B97F4A7C15


def build() -> str:
    """Compile the C restatement (gcc, no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        lib.bico_create.restype = vp
        lib.bico_create.argtypes = [i32, i64, i64]
        lib.bico_destroy.argtypes = [vp]
        lib.bico_insert.restype = i32
        lib.bico_insert.argtypes = [vp, vp, i64]
        lib.bico_insert_block.restype = i64
        lib.bico_insert_block.argtypes = [vp, vp, vp, i64, ctypes.POINTER(i32)]
        lib.bico_num_features.restype = i64
        lib.bico_num_features.argtypes = [vp]
        lib.bico_threshold.restype = dp
        lib.bico_threshold.argtypes = [vp]
        lib.bico_total_weight.restype = i64
        lib.bico_total_weight.argtypes = [vp]
        lib.bico_features.restype = i64
        lib.bico_features.argtypes = [vp, i64, vp, vp, vp, vp, vp]
        lib.bico_extract.restype = i64
        lib.bico_extract.argtypes = [vp, i64, vp, vp]
        _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


# --------------------------------------------------------------------- util
def mix_seed(*parts: int) -> int:
    """splitmix64 finaliser folded over the parts (util.py:8-21)."""
    state = _PHI64
    for p in parts:
        z = ((state ^ (int(p) & _MASK64)) + _PHI64) & _MASK64
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
        state = z ^ (z >> 31)
    return state


# ------------------------------------------------------------------- engine
class OracleEngine:
    """ctypes handle on the C restatement of BicoEngine (coreset.py:213-451)."""

    def __init__(self, dim: int, budget: int, bootstrap_cap: int = 1001):
        self._lib = _load()
        self.dim = int(dim)
        self.budget = int(budget)
        self._h = self._lib.bico_create(self.dim, self.budget, int(bootstrap_cap))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.bico_destroy(h)
            self._h = None

    def insert(self, x, weight: int = 1) -> None:
        x = np.ascontiguousarray(x, dtype=np.float64)
        rc = self._lib.bico_insert(self._h, _ptr(x), int(weight))
        if rc:
            raise ValueError({-1: "non-finite", -2: "overflow", -3: "bad weight"}[rc])

    def insert_block(self, X, W=None) -> int:
        X = np.ascontiguousarray(X, dtype=np.float64).reshape(-1, self.dim)
        Wa = None if W is None else np.ascontiguousarray(W, dtype=np.int64)
        st = ctypes.c_int(0)
        n = self._lib.bico_insert_block(self._h, _ptr(X), _ptr(Wa), X.shape[0], ctypes.byref(st))
        if st.value:
            raise ValueError(f"row {n} rejected ({st.value})")
        return n

    @property
    def num_features(self) -> int:
        return int(self._lib.bico_num_features(self._h))

    @property
    def threshold(self) -> float:
        return float(self._lib.bico_threshold(self._h))

    @property
    def total_weight(self) -> int:
        return int(self._lib.bico_total_weight(self._h))

    def features(self):
        """(levels, weights, linear sums, square sums, references) in DFS pre-order."""
        n = int(self._lib.bico_features(self._h, 0, None, None, None, None, None))
        lv = np.zeros(n, np.int32)
        w = np.zeros(n, np.int64)
        s = np.zeros((n, self.dim))
        q = np.zeros(n)
        r = np.zeros((n, self.dim))
        self._lib.bico_features(self._h, n, _ptr(lv), _ptr(w), _ptr(s), _ptr(q), _ptr(r))
        return lv, w, s, q, r

    def extract(self):
        n = self.num_features
        pts = np.zeros((n, self.dim))
        wts = np.zeros(n, np.int64)
        got = int(self._lib.bico_extract(self._h, n, _ptr(pts), _ptr(wts)))
        return pts[:got], wts[:got]


# ---------------------------------------------------------------- clustering
def pairwise_sq(P: np.ndarray, C: np.ndarray) -> np.ndarray:
    """GEMM-form squared distances with clamp (evaluation.py:39-46)."""
    out = P @ C.T
    out *= -2.0
    out += np.einsum("ij,ij->i", P, P)[:, None]
    out += np.einsum("ij,ij->i", C, C)[None, :]
    np.maximum(out, 0.0, out=out)
    return out


def weighted_draw(rng, mass: np.ndarray) -> int:
    """Inverse-CDF draw: first index with cumsum > u*total (evaluation.py:49-53)."""
    c = np.cumsum(mass)
    target = rng.random() * c[-1]
    return min(int(np.searchsorted(c, target, side="right")), c.shape[0] - 1)


def seed_dsquared(P: np.ndarray, w: np.ndarray, k: int, rng) -> np.ndarray:
    """Weighted D^2 seeding (evaluation.py:56-82); diff-based distances."""
    centers = np.empty((k, P.shape[1]))
    pick = weighted_draw(rng, w)
    centers[0] = P[pick]
    delta = P - centers[0]
    nearest = np.einsum("ij,ij->i", delta, delta)
    for c in range(1, k):
        mass = w * nearest
        pick = weighted_draw(rng, mass) if mass.sum() > 0.0 else weighted_draw(rng, w)
        centers[c] = P[pick]
        delta = P - centers[c]
        np.minimum(nearest, np.einsum("ij,ij->i", delta, delta), out=nearest)
    return centers


def lloyd(P: np.ndarray, w: np.ndarray, C0: np.ndarray, max_iters: int = 100,
          tol: float = 1e-4, cost_log: list | None = None) -> np.ndarray:
    """Weighted Lloyd with empty-cluster repair (evaluation.py:85-139)."""
    n = P.shape[0]
    C = np.array(C0, dtype=np.float64, copy=True)
    k = C.shape[0]
    rows = np.arange(n)
    last = math.inf
    for _ in range(max_iters):
        d2 = pairwise_sq(P, C)
        lab = d2.argmin(axis=1)
        dist = d2[rows, lab]
        used = np.bincount(lab, minlength=k) > 0
        while not used.all():
            gain = w * dist
            if gain.max() <= 0.0:
                break
            hole = int(np.flatnonzero(~used)[0])
            far = int(np.argmax(gain))
            C[hole] = P[far]
            delta = P - C[hole]
            cand = np.einsum("ij,ij->i", delta, delta)
            better = cand < dist
            lab[better] = hole
            dist[better] = cand[better]
            lab[far] = hole
            dist[far] = 0.0
            used = np.bincount(lab, minlength=k) > 0
        total = float(w @ dist)
        if cost_log is not None:
            cost_log.append(total)
        if math.isfinite(last) and last - total <= tol * last:
            break
        last = total
        member = np.zeros((n, k))
        member[rows, lab] = w
        mass = member.sum(axis=0)
        has = mass > 0
        moved = (member.T @ P) / np.where(has, mass, 1.0)[:, None]
        C = np.where(has[:, None], moved, C)
    return C


def cost(P: np.ndarray, w: np.ndarray, C: np.ndarray) -> float:
    """Weighted SSE to the nearest center (evaluation.py:142-149)."""
    if P.shape[0] == 0:
        return 0.0
    return float(w @ pairwise_sq(P, np.asarray(C, dtype=np.float64)).min(axis=1))


def kmeans_reps(P, w, k: int, reps: int = 5, seed: int = 0, max_iters: int = 100,
                tol: float = 1e-4):
    """[(centers, cost)] per repetition, rng = PCG64(mix_seed(seed, rep))
    (evaluation.py:199-210)."""
    P = np.asarray(P, dtype=np.float64)
    w = np.ones(P.shape[0]) if w is None else np.asarray(w, dtype=np.float64)
    out = []
    for rep in range(reps):
        rng = np.random.default_rng(mix_seed(seed, rep))
        C = seed_dsquared(P, w, k, rng)
        C = lloyd(P, w, C, max_iters, tol)
        out.append((C, cost(P, w, C)))
    return out


# ------------------------------------------------------------------ linalg
def _signs(V: np.ndarray) -> np.ndarray:
    """First non-negligible entry of each column made >= 0 (linalg.py:77-88)."""
    V = np.array(V, copy=True)
    for j in range(V.shape[1]):
        a = np.abs(V[:, j])
        top = a.max()
        if top == 0.0:
            continue
        lead = np.nonzero(a > 1e-12 * top)[0]
        if lead.size and V[lead[0], j] < 0.0:
            V[:, j] = -V[:, j]
    return V


def rsvd(A: np.ndarray, rank: int, oversample: int, power: int, seed: int):
    """HMT randomized truncated SVD (linalg.py:167-206) -> (V d x rank, sigma)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    rows, cols = A.shape
    r = rank + oversample
    if r > min(rows, cols):
        raise ValueError("rank + oversample exceeds min(rows, cols)")
    gen = np.random.default_rng(seed)
    Om = gen.standard_normal((cols, r))
    Q = np.linalg.qr(A @ Om)[0]
    for _ in range(power):
        Z = np.linalg.qr(A.T @ Q)[0]
        Q = np.linalg.qr(A @ Z)[0]
    B = Q.T @ A
    if rows > 4 * r:
        Om2 = gen.standard_normal((r, r))
        W = np.linalg.qr(B.T @ Om2)[0]
        _, sig, vt = np.linalg.svd(B @ W)
        V = W @ vt.T
    else:
        _, sig, vt = np.linalg.svd(B, full_matrices=False)
        V = vt.T
    sig = np.array(sig[:rank])
    if sig.size and sig[0] > 0.0:
        sig[sig < 1e-12 * sig[0]] = 0.0
    return _signs(V[:, :rank]), sig


def project(A: np.ndarray, V: np.ndarray) -> np.ndarray:
    """A V V^T (linalg.py:209-221)."""
    return (np.asarray(A, dtype=np.float64) @ V) @ V.T


def weighted_fit(P, w, rank, oversample, power, seed):
    """sqrt(w)-scaled rows through rsvd (linalg.py:231-250)."""
    P = np.asarray(P, dtype=np.float64)
    scaled = P * np.sqrt(np.asarray(w).astype(np.float64))[:, None]
    return rsvd(scaled, rank, oversample, power, seed)


# --------------------------------------------------------------- pipelines
def _pieces(X: np.ndarray, size: int):
    for a in range(0, X.shape[0], size):
        yield X[a:a + size]


def piecy(X, k: int, piece_size: int, svd_dim: int | None = None,
          coreset_size: int | None = None, oversample: int = 10, power: int = 2,
          seed: int = 0, stats: dict | None = None):
    """run_piecy restated (pipeline.py:102-139) -> (points, weights)."""
    X = np.asarray(X, dtype=np.float64)
    d = X.shape[1]
    ell = svd_dim if svd_dim is not None else (3 * k + 1) // 2
    m = coreset_size if coreset_size is not None else 200 * k
    if ell > d:
        raise ValueError("svd_dim exceeds point dimension")
    eng = OracleEngine(d, m)
    for idx, piece in enumerate(_pieces(X, piece_size)):
        blk = piece
        if ell < d and piece.shape[0] >= ell:
            ov = min(oversample, min(piece.shape[0], d) - ell)
            V, _ = rsvd(piece, ell, ov, power, (seed ^ idx) & _MASK64)
            blk = project(piece, V)
            if stats is not None:
                stats["svd_calls"] = stats.get("svd_calls", 0) + 1
        eng.insert_block(blk)
    return eng.extract()


def bico(X, coreset_size: int):
    """run_bico restated (pipeline.py:87-99)."""
    X = np.asarray(X, dtype=np.float64)
    eng = OracleEngine(X.shape[1], coreset_size)
    eng.insert_block(X)
    return eng.extract()


class OracleTree:
    """MergeReduceTree restated (mergereduce.py:73-187)."""

    def __init__(self, dim, k, piece_size, num_pieces, svd_dim=None, coreset_size=None,
                 oversample=10, power=2, seed=0):
        self.dim = dim
        self.ell = svd_dim if svd_dim is not None else (3 * k + 1) // 2
        self.m = coreset_size if coreset_size is not None else 200 * k
        self.np_ = num_pieces
        self.piece_size = piece_size
        self.ov, self.power, self.seed = oversample, power, seed
        self.levels = []     # [engine|None, batches, flushes]
        self.piece_index = 0
        self.flush_sources = []

    def _reduce(self, P, w, seed):
        rows = P.shape[0]
        if self.ell >= self.dim or rows < self.ell:
            return P
        ov = min(self.ov, min(rows, self.dim) - self.ell)
        if w is None:
            w = np.ones(rows, dtype=np.int64)
        V, _ = weighted_fit(P, w, self.ell, ov, self.power, seed)
        return project(P, V)

    def _slot(self, lvl):
        while len(self.levels) <= lvl:
            self.levels.append([None, 0, 0])
        s = self.levels[lvl]
        if s[0] is None:
            s[0] = OracleEngine(self.dim, self.m)
        return s

    def push_piece(self, piece):
        blk = np.asarray(piece, dtype=np.float64)
        red = self._reduce(blk, None, (self.seed ^ self.piece_index) & _MASK64)
        self.piece_index += 1
        s = self._slot(0)
        s[0].insert_block(red)
        s[1] += 1
        if s[1] == self.np_:
            self._flush(0)

    def _flush(self, lvl):
        s = self.levels[lvl]
        pts, wts = s[0].extract()
        s[0] = None
        s[1] = 0
        s[2] += 1
        self.flush_sources.append(lvl)
        red = self._reduce(pts, wts, mix_seed(self.seed, lvl + 1, s[2]))
        up = self._slot(lvl + 1)
        up[0].insert_block(red, wts)
        up[1] += 1
        if up[1] == self.np_:
            self._flush(lvl + 1)

    def finalize(self):
        while True:
            live = [i for i, s in enumerate(self.levels) if s[0] is not None]
            if len(live) <= 1:
                break
            self._flush(live[0])
        live = [i for i, s in enumerate(self.levels) if s[0] is not None]
        if not live:
            return np.zeros((0, self.dim)), np.zeros(0, np.int64)
        return self.levels[live[0]][0].extract()


def piecy_mr(X, k, piece_size, num_pieces, svd_dim=None, coreset_size=None,
             oversample=10, power=2, seed=0):
    """run_piecy_mr restated (mergereduce.py:190-202)."""
    X = np.asarray(X, dtype=np.float64)
    t = OracleTree(X.shape[1], k, piece_size, num_pieces, svd_dim, coreset_size,
                   oversample, power, seed)
    for piece in _pieces(X, piece_size):
        t.push_piece(piece)
    return t.finalize()


def evaluate_cost_multi(center_sets, X: np.ndarray, chunk: int = 8192) -> list:
    """Streaming unweighted SSE against several center sets (evaluation.py:157-180):
    chunks of ``chunk`` rows, GEMM-form distances to the stacked centers, per-set
    minimum, chunk sums accumulated in chunk order."""
    sets = [np.asarray(c, dtype=np.float64) for c in center_sets]
    stacked = np.vstack(sets)
    bounds = np.cumsum([0] + [c.shape[0] for c in sets])
    totals = np.zeros(len(sets))
    X = np.asarray(X, dtype=np.float64)
    for a in range(0, X.shape[0], chunk):
        d2 = pairwise_sq(X[a:a + chunk], stacked)
        for i in range(len(sets)):
            totals[i] += d2[:, bounds[i]:bounds[i + 1]].min(axis=1).sum()
    return [float(t) for t in totals]


# ------------------------------------------------------------ paper generators
# datagen.py:15-16 draws every coordinate from numpy's Philox4x64-10 as
# Generator.random(): output t of the stream is word t % 4 of the counter
# block t // 4 + 1 (numpy bumps the counter before each block), u = (x >> 11)
# * 2^-53.  Restated here in vectorised uint64 arithmetic (the third-party
# algorithm, numpy 2.x philox.h), with the reference's own draw order.
_PM0, _PM1 = np.uint64(0xD2E7470EE14C6C93), np.uint64(0xCA5A826395121157)
_PW0, _PW1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
_M32 = np.uint64(0xFFFFFFFF)


def _mulhilo(a: np.uint64, b: np.ndarray):
    a_lo, a_hi = a & _M32, a >> np.uint64(32)
    b_lo, b_hi = b & _M32, b >> np.uint64(32)
    ll = a_lo * b_lo
    lh = a_lo * b_hi
    hl = a_hi * b_lo
    hh = a_hi * b_hi
    mid = (ll >> np.uint64(32)) + (lh & _M32) + (hl & _M32)
    hi = hh + (lh >> np.uint64(32)) + (hl >> np.uint64(32)) + (mid >> np.uint64(32))
    return hi, a * b


def philox_uniforms(seed: int, t: np.ndarray) -> np.ndarray:
    """Generator(Philox(key=seed)).random() values at global draw indices t."""
    t = np.asarray(t, dtype=np.uint64)
    key = int(seed) & ((1 << 128) - 1)
    k0, k1 = key & ((1 << 64) - 1), key >> 64
    with np.errstate(over="ignore"):
        x0 = (t >> np.uint64(2)) + np.uint64(1)
        x1 = np.zeros_like(x0)
        x2 = np.zeros_like(x0)
        x3 = np.zeros_like(x0)
        for r in range(10):
            if r:
                k0 = (k0 + _PW0) & ((1 << 64) - 1)
                k1 = (k1 + _PW1) & ((1 << 64) - 1)
            hi0, lo0 = _mulhilo(_PM0, x0)
            hi1, lo1 = _mulhilo(_PM1, x2)
            x0, x1, x2, x3 = hi1 ^ x1 ^ np.uint64(k0), lo1, hi0 ^ x3 ^ np.uint64(k1), lo0
    w = np.stack([x0, x1, x2, x3])[(t & np.uint64(3)).astype(np.int64), np.arange(t.size)]
    return (w >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _centred(u, scale):
    return (2.0 * u - 1.0) * scale


def gen_swn(clusters, ppc, dim, active_dims, spread=10.0, noise=0.5, seed=0) -> np.ndarray:
    """structured_with_noise (datagen.py:104-112) by global draw index: the
    per-cluster permutation on numpy's generator, every coordinate from
    philox_uniforms."""
    rng = np.random.Generator(np.random.Philox(key=seed))
    bg = rng.bit_generator
    out = np.empty((clusters * ppc, dim))
    per = dim + active_dims
    for c in range(clusters):
        active = rng.permutation(dim)[:active_dims]
        st = bg.state
        ctr = int(st["state"]["counter"][0]) | (int(st["state"]["counter"][1]) << 64)
        t0 = ctr * 4 if st["buffer_pos"] >= 4 else (ctr - 1) * 4 + int(st["buffer_pos"])
        j = np.arange(ppc, dtype=np.uint64)[:, None] * np.uint64(per)
        noise_u = philox_uniforms(seed, (np.uint64(t0) + j + np.arange(dim, dtype=np.uint64)).ravel())
        sig_u = philox_uniforms(seed, (np.uint64(t0 + dim) + j + np.arange(active_dims, dtype=np.uint64)).ravel())
        blk = _centred(noise_u.reshape(ppc, dim), noise)
        blk[:, active] = _centred(sig_u.reshape(ppc, active_dims), spread)
        out[c * ppc:(c + 1) * ppc] = blk
        t1 = t0 + ppc * per
        tmp = np.random.Philox(key=seed, counter=t1 // 4)
        if t1 % 4:
            tmp.random_raw(t1 % 4)
        nst = tmp.state
        nst["has_uint32"], nst["uinteger"] = st["has_uint32"], st["uinteger"]
        bg.state = nst
    return out


def gen_cube(n, spread=10.0, seed=0) -> np.ndarray:
    """random_cube (datagen.py:131-135)."""
    return _centred(philox_uniforms(seed, np.arange(n * n, dtype=np.uint64)).reshape(n, n), spread)


def gen_lower_bound(k, n, spread=1000.0, noise=100.0) -> np.ndarray:
    """lower_bound (datagen.py:115-128)."""
    per = n // k
    out = np.zeros((n, k + n))
    for v in range(k):
        for j in range(per):
            out[v * per + j, v] = spread
            out[v * per + j, k + v * per + j] = noise
    return out
