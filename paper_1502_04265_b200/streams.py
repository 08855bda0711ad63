"""Point-stream files: the reference's two formats, plus block readers that feed
the device path.

Formats (reference streams.py:1-14):
* ``csv`` -- one point per line, comma-separated decimals; the weighted form
  has an integer weight in the first column.
* ``bin`` -- ``SCPT``, little-endian u32 version 1, u32 dimension, then per
  point d little-endian float64 values; the weighted form prefixes each record
  with a little-endian u64 weight.

``PointSource`` keeps the reference's row iteration and error positions
(1-based line for csv, byte offset for bin).  What is new is ``blocks(rows)``,
which returns whole ``(coords, weights)`` arrays per block (binary files are
sliced from the read buffer without a per-row Python loop), and
``device_blocks``, which moves blocks through pinned host buffers on a
separate copy stream so the next block's H2D overlaps the current block's
kernels.
"""
from __future__ import annotations

import struct
from typing import Iterable, Iterator

import numpy as np

MAGIC = b"SCPT"
VERSION = 1
FORMATS = ("csv", "bin")
_HDR = struct.Struct("<4sII")
_READ_BYTES = 1 << 20   # the reference's read framing (streams.py:176); see _bin_frames


class StreamFormatError(ValueError):
    """Malformed stream file; the message names the offending position."""


# ------------------------------------------------------------------ writers
def write_csv(path, rows: Iterable, *, weighted: bool = False) -> int:
    """Points (or ``(point, weight)`` pairs) as csv lines; returns the count.
    Floats are written with ``repr`` so a csv round trip is exact."""
    n = 0
    with open(path, "w", encoding="ascii") as out:
        for item in rows:
            point, weight = item if weighted else (item, None)
            fields = [repr(float(v)) for v in point]
            if weighted:
                fields.insert(0, str(int(weight)))
            out.write(",".join(fields) + "\n")
            n += 1
    return n


def write_bin(path, rows: Iterable, dim: int, *, weighted: bool = False) -> int:
    """Points (or ``(point, weight)`` pairs) in the binary format."""
    n = 0
    with open(path, "wb") as out:
        out.write(_HDR.pack(MAGIC, VERSION, dim))
        for item in rows:
            point, weight = item if weighted else (item, None)
            coords = np.ascontiguousarray(point, dtype="<f8")
            if coords.shape != (dim,):
                raise ValueError(f"point of dimension {coords.shape} does not match d={dim}")
            if weighted:
                out.write(struct.pack("<Q", int(weight)))
            out.write(coords.tobytes())
            n += 1
    return n


def write_stream(path, rows: Iterable, dim: int, fmt: str, *, weighted: bool = False) -> int:
    if fmt == "csv":
        return write_csv(path, rows, weighted=weighted)
    if fmt == "bin":
        return write_bin(path, rows, dim, weighted=weighted)
    raise ValueError(f"unknown format {fmt!r}")


# ------------------------------------------------------------------ readers
def _bin_header(path, fh):
    """(dim) from an open binary stream, or None for an empty file."""
    head = fh.read(_HDR.size)
    if not head:
        return None
    if len(head) < _HDR.size:
        raise StreamFormatError(f"{path}: truncated header at byte {len(head)}")
    magic, version, dim = _HDR.unpack(head)
    if magic != MAGIC:
        raise StreamFormatError(f"{path}: bad magic at byte 0")
    if version != VERSION:
        raise StreamFormatError(f"{path}: unsupported version {version}")
    return dim


def _bin_frames(path, weighted: bool):
    """Yield (coords [r x d] float64, weights [r] int64 | None) per read frame.
    A frame is max(1, 1 MiB // record) records, as in the reference: a file
    whose tail record is truncated yields every complete frame before the
    error and nothing of the frame that holds the truncation."""
    with open(path, "rb") as fh:
        dim = _bin_header(path, fh)
        if dim is None:
            return
        rec = 8 * dim + (8 if weighted else 0)
        per = max(1, _READ_BYTES // rec)
        offset = _HDR.size
        while True:
            raw = fh.read(rec * per)
            if not raw:
                return
            whole = len(raw) - len(raw) % rec
            if whole != len(raw):
                raise StreamFormatError(f"{path}: truncated record at byte {offset + whole}")
            if weighted:
                arr = np.frombuffer(raw, dtype=np.dtype([("w", "<u8"), ("x", "<f8", (dim,))]))
                yield arr["x"], arr["w"].astype(np.int64)
            else:
                yield np.frombuffer(raw, dtype="<f8").reshape(-1, dim), None
            offset += len(raw)


def _csv_rows(path, weighted: bool):
    """Yield (line number, coords, weight | None) with the reference's checks."""
    dim = None
    with open(path, "r", encoding="ascii") as fh:
        for lineno, line in enumerate(fh, start=1):
            if not line.strip():
                continue
            fields = line.rstrip("\n").split(",")
            try:
                weight = int(fields[0]) if weighted else None
                coords = np.array([float(f) for f in (fields[1:] if weighted else fields)])
            except (ValueError, IndexError) as exc:
                raise StreamFormatError(f"{path}: line {lineno}: {exc}") from exc
            if dim is None:
                dim = coords.shape[0]
            elif coords.shape[0] != dim:
                raise StreamFormatError(f"{path}: line {lineno}: expected {dim} coordinates, got {coords.shape[0]}")
            if weighted and weight < 1:
                raise StreamFormatError(f"{path}: line {lineno}: weight must be >= 1")
            yield lineno, coords, weight


def _probe_dim(path, fmt: str, weighted: bool):
    if fmt == "bin":
        with open(path, "rb") as fh:
            dim = _bin_header(path, fh)
        if dim is not None and dim < 1:
            raise StreamFormatError(f"{path}: dimension {dim} in header")
        return dim
    with open(path, "r", encoding="ascii") as fh:
        for line in fh:
            if line.strip():
                dim = len(line.rstrip("\n").split(",")) - (1 if weighted else 0)
                if dim < 1:
                    raise StreamFormatError(f"{path}: line 1: no coordinates")
                return dim
    return None


class PointSource:
    """Re-iterable reader (reference streams.py:91-114): ``dim`` is probed up
    front (None for an empty file); each iteration is a fresh one-pass scan."""

    def __init__(self, path: str, fmt: str, weighted: bool = False):
        if fmt not in FORMATS:
            raise StreamFormatError(f"unknown format {fmt!r}")
        self.path, self.fmt, self.weighted = path, fmt, weighted
        self.dim = _probe_dim(path, fmt, weighted)

    def __iter__(self) -> Iterator:
        if self.fmt == "csv":
            for _, coords, weight in _csv_rows(self.path, self.weighted):
                yield (coords, weight) if self.weighted else coords
        else:
            for coords, weights in _bin_frames(self.path, self.weighted):
                for i in range(coords.shape[0]):
                    yield (coords[i], int(weights[i])) if self.weighted else coords[i]

    def points(self) -> Iterator[np.ndarray]:
        """Coordinates only (weights dropped)."""
        if not self.weighted:
            return iter(self)
        return (p for p, _ in self)

    def blocks(self, rows: int):
        """Consecutive blocks of ``rows`` points: (coords [r x d] float64,
        weights [r] int64 | None); the last block may be shorter.  Errors are
        raised at the same stream position as row iteration raises them."""
        if rows < 1:
            raise ValueError("rows must be >= 1")
        pend_x, pend_w, have = [], [], 0
        if self.fmt == "bin":
            frames = _bin_frames(self.path, self.weighted)
        else:
            def frames():
                xs, ws = [], []
                for _, coords, weight in _csv_rows(self.path, self.weighted):
                    xs.append(coords)
                    ws.append(weight)
                    if len(xs) == rows:
                        yield np.stack(xs), (np.asarray(ws, dtype=np.int64) if self.weighted else None)
                        xs, ws = [], []
                if xs:
                    yield np.stack(xs), (np.asarray(ws, dtype=np.int64) if self.weighted else None)
            frames = frames()
        for coords, weights in frames:
            pos = 0
            while pos < coords.shape[0]:
                take = min(rows - have, coords.shape[0] - pos)
                pend_x.append(coords[pos:pos + take])
                if weights is not None:
                    pend_w.append(weights[pos:pos + take])
                have += take
                pos += take
                if have == rows:
                    yield _join(pend_x, pend_w, self.weighted)
                    pend_x, pend_w, have = [], [], 0
        if have:
            yield _join(pend_x, pend_w, self.weighted)


def _join(xs, ws, weighted):
    x = xs[0] if len(xs) == 1 else np.concatenate(xs)
    w = (ws[0] if len(ws) == 1 else np.concatenate(ws)) if weighted else None
    return x, w


def device_blocks(source: PointSource, rows: int, device=None):
    """``source.blocks(rows)`` moved to the device: yields (coords fp64 CUDA
    tensor, weights int64 CUDA tensor | None).  Two pinned host buffers and a
    copy stream: block b+1 is staged and copied while the caller's kernels
    run on block b; the caller's stream waits on an event before use."""
    import torch
    dev = device or torch.device("cuda", torch.cuda.current_device())
    dim = source.dim
    if dim is None:
        return
    copy = torch.cuda.Stream(device=dev)
    pins = [torch.empty((rows, dim), dtype=torch.float64, pin_memory=True) for _ in range(2)]
    wpins = [torch.empty(rows, dtype=torch.int64, pin_memory=True) for _ in range(2)] if source.weighted else None
    done = [None, None]
    slot = 0
    pending = None
    for coords, weights in source.blocks(rows):
        r = coords.shape[0]
        if done[slot] is not None:
            done[slot].synchronize()           # the pinned buffer's previous copy has finished
        pins[slot][:r].numpy()[...] = coords
        if weights is not None:
            wpins[slot][:r].numpy()[...] = weights
        with torch.cuda.stream(copy):
            xd = pins[slot][:r].to(dev, non_blocking=True)
            wd = wpins[slot][:r].to(dev, non_blocking=True) if weights is not None else None
            ev = torch.cuda.Event()
            ev.record(copy)
        done[slot] = ev
        if pending is not None:
            yield pending
        torch.cuda.current_stream(dev).wait_event(ev)
        xd.record_stream(torch.cuda.current_stream(dev))
        if wd is not None:
            wd.record_stream(torch.cuda.current_stream(dev))
        pending = (xd, wd)
        slot ^= 1
    if pending is not None:
        yield pending
