"""Stream files: the reference's csv / SCPT formats,
row iteration, block reads and error positions (reference streams.py)."""
import importlib.util
import os
import sys

import numpy as np
import pytest

from paper_1502_04265_b200 import streams as S

REF_SRC = "/root/reference/pkg/src"


def _rows(n=37, d=5, seed=0):
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(n, d)) * 10.0 ** rng.integers(-3, 4, size=(n, 1))
    w = rng.integers(1, 1000, size=n)
    return X, w


@pytest.mark.parametrize("fmt", ["bin", "csv"])
@pytest.mark.parametrize("weighted", [False, True])
def test_round_trip_exact(tmp_path, fmt, weighted):
    X, w = _rows()
    path = str(tmp_path / f"s.{fmt}")
    rows = list(zip(X, w)) if weighted else list(X)
    assert S.write_stream(path, rows, X.shape[1], fmt, weighted=weighted) == X.shape[0]
    src = S.PointSource(path, fmt, weighted=weighted)
    assert src.dim == X.shape[1]
    got = list(src)
    if weighted:
        assert np.array_equal(np.stack([p for p, _ in got]), X)      # bitwise (repr / raw bytes)
        assert [q for _, q in got] == [int(v) for v in w]
        assert np.array_equal(np.stack(list(src.points())), X)
    else:
        assert np.array_equal(np.stack(got), X)
    for rows_per in (1, 5, 36, 37, 100):
        blocks = list(src.blocks(rows_per))
        assert all(b[0].shape[0] == rows_per for b in blocks[:-1])
        assert np.array_equal(np.concatenate([b[0] for b in blocks]), X)
        if weighted:
            assert np.array_equal(np.concatenate([b[1] for b in blocks]), w)


def test_bin_errors(tmp_path):
    p = str(tmp_path / "e.bin")
    open(p, "wb").write(b"SCP")
    with pytest.raises(S.StreamFormatError, match="truncated header at byte 3"):
        S.PointSource(p, "bin")
    open(p, "wb").write(b"XXXX" + (1).to_bytes(4, "little") + (3).to_bytes(4, "little"))
    with pytest.raises(S.StreamFormatError, match="bad magic at byte 0"):
        S.PointSource(p, "bin")
    open(p, "wb").write(b"SCPT" + (2).to_bytes(4, "little") + (3).to_bytes(4, "little"))
    with pytest.raises(S.StreamFormatError, match="unsupported version 2"):
        S.PointSource(p, "bin")
    X, _ = _rows(4, 3)
    S.write_bin(p, list(X), 3)
    with open(p, "ab") as f:
        f.write(b"\0" * 10)                        # a partial fifth record
    src = S.PointSource(p, "bin")
    with pytest.raises(S.StreamFormatError, match=f"truncated record at byte {12 + 4 * 24}"):
        list(src)
    with pytest.raises(S.StreamFormatError, match=f"truncated record at byte {12 + 4 * 24}"):
        list(src.blocks(2))
    open(p, "wb").write(b"")
    assert S.PointSource(p, "bin").dim is None and list(S.PointSource(p, "bin")) == []


def test_csv_errors(tmp_path):
    p = str(tmp_path / "e.csv")
    open(p, "w").write("1,2,3\n4,5\n")
    with pytest.raises(S.StreamFormatError, match="line 2: expected 3 coordinates, got 2"):
        list(S.PointSource(p, "csv"))
    open(p, "w").write("1,2\n\n3,x\n")
    with pytest.raises(S.StreamFormatError, match="line 3: could not convert string to float"):
        list(S.PointSource(p, "csv"))
    open(p, "w").write("0,1.5,2\n")
    with pytest.raises(S.StreamFormatError, match="line 1: weight must be >= 1"):
        list(S.PointSource(p, "csv", weighted=True))
    with pytest.raises(S.StreamFormatError, match="unknown format"):
        S.PointSource(p, "parquet")


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference tree not present")
@pytest.mark.parametrize("fmt", ["bin", "csv"])
@pytest.mark.parametrize("weighted", [False, True])
def test_matches_reference_reader(tmp_path, fmt, weighted):
    """Pinned against the unmodified reference reader on the same files,
    including a truncated binary tail larger than one 1 MiB read frame."""
    spec = importlib.util.spec_from_file_location("ref_streams", os.path.join(REF_SRC, "piecy", "streams.py"))
    ref = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ref)
    X, w = _rows(3000 if fmt == "bin" else 50, 57)
    path = str(tmp_path / f"r.{fmt}")
    rows = list(zip(X, w)) if weighted else list(X)
    ref.write_stream(path, rows, X.shape[1], fmt, weighted=weighted)
    mine = S.PointSource(path, fmt, weighted=weighted)
    theirs = ref.PointSource(path, fmt, weighted=weighted)
    assert mine.dim == theirs.dim
    for a, b in zip(mine, theirs):
        if weighted:
            assert np.array_equal(a[0], b[0]) and a[1] == b[1]
        else:
            assert np.array_equal(a, b)
    if fmt == "bin":
        with open(path, "ab") as f:
            f.write(b"\1" * 17)
        got_m, got_r, err_m, err_r = 0, 0, None, None
        try:
            for _ in S.PointSource(path, fmt, weighted=weighted):
                got_m += 1
        except S.StreamFormatError as e:
            err_m = str(e)
        try:
            for _ in ref.PointSource(path, fmt, weighted=weighted):
                got_r += 1
        except ref.StreamFormatError as e:
            err_r = str(e)
        assert (got_m, err_m) == (got_r, err_r)
