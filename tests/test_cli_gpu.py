"""The CLI on the device vs the reference CLI's own reports
(tests/golden/cli_reports.json, from tests/golden/make_golden_cli.py):
every report v1 key in the same order with the same value (costs within 1e-9
relative; timings excluded), the GPU fields appended, and the --out coreset
(weights exact, points within 1e-9)."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(__file__), "golden")
CASES = json.load(open(os.path.join(HERE, "cli_reports.json")))


def _parse(text):
    out = {}
    for line in text.strip().splitlines():
        key, _, value = line.partition(" = ")
        out[key.strip()] = value.strip()
    return out


@pytest.mark.parametrize("name", sorted(CASES))
def test_report_matches_reference(name, tmp_path, capsys):
    from paper_1502_04265_b200.cli import main
    from paper_1502_04265_b200.streams import PointSource
    case = CASES[name]
    out = tmp_path / "cs.bin"
    rep_file = tmp_path / "rep.txt"
    assert main(case["argv"] + ["--out", str(out), "--report", str(rep_file)]) == 0
    got = _parse(capsys.readouterr().out)
    assert _parse(rep_file.read_text()) == got
    want = case["report"]
    keys = [k for k in got if not k.endswith("_seconds")]
    assert keys[:len(want)] == list(want), "v1 keys / order"
    for k, v in want.items():
        if "_cost_" in k:
            assert abs(float(got[k]) - float(v)) <= 1e-9 * abs(float(v)), (k, got[k], v)
        else:
            assert got[k] == v, (k, got[k], v)
    for extra in ("gpu_name", "gpus", "gpu_kernel_launches"):
        assert extra in got
    assert int(got["gpu_kernel_launches"]) > 0
    rows = list(PointSource(str(out), "bin", weighted=True))
    assert [w for _, w in rows] == case["coreset_weights"]
    P = np.array([p for p, _ in rows])
    W = np.array(case["coreset_points"])
    np.testing.assert_allclose(P, W, rtol=1e-9, atol=1e-9 * max(1.0, np.abs(W).max()))


def test_generator_mode_writes_reference_stream(tmp_path, capsys):
    """--gen without --algo: the device-generated file equals the reference generator's rows."""
    from oracle import piecy_oracle as O
    from paper_1502_04265_b200.cli import main
    from paper_1502_04265_b200.streams import PointSource
    out = tmp_path / "swn.bin"
    assert main(["--gen", "swn", "--clusters", "4", "--y", "6", "--d", "10", "--x", "2", "--seed", "1",
                 "--out", str(out)]) == 0
    assert "24 points" in capsys.readouterr().out
    X = np.array(list(PointSource(str(out), "bin")))
    assert np.array_equal(X, O.gen_swn(4, 6, 10, 2, seed=1))


def test_projected_lower_bound_keeps_invariants(capsys):
    """piecy on a LowerBound instance: the pieces' singular values are
    degenerate (a 49-dimensional eigenspace), so the rank-6 subspace -- and
    with it the coreset -- is not unique.  The mass, budget and
    report structure must still hold."""
    from paper_1502_04265_b200.cli import main
    assert main(["--algo", "piecy", "--gen", "lb", "--k", "4", "--n", "200", "--coreset-size", "60",
                 "--piece-size", "50", "--svd-dim", "6"]) == 0
    rep = _parse(capsys.readouterr().out)
    assert rep["coreset_total_weight"] == "200" and int(rep["coreset_size"]) <= 60 and rep["svd_calls"] == "4"
