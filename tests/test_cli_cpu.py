"""CLI host logic without a GPU: flag surface and the usage errors the
reference maps to exit status 2 (cli.py:126-156, :210-231, :307-317)."""

import json
import os

from paper_1502_04265_b200.cli import build_parser, main

HERE = os.path.join(os.path.dirname(__file__), "golden")


def test_flags_cover_reference_surface():
    p = build_parser()
    dests = {a.dest for a in p._actions}
    for want in ("algo", "gen", "input", "format", "weighted", "out", "report", "k", "coreset_size", "piece_size",
                 "svd_dim", "num_pieces", "seed", "reps", "eval_mode", "clusters", "points_per_cluster", "dim",
                 "active_dims", "n", "spread", "noise"):
        assert want in dests
    a = p.parse_args([])
    assert a.num_pieces == 10 and a.reps == 5 and a.seed == 0 and a.eval_mode == "coreset"


def test_golden_argv_parse():
    cases = json.load(open(os.path.join(HERE, "cli_reports.json")))
    p = build_parser()
    for case in cases.values():
        p.parse_args(case["argv"])


def test_usage_errors_exit_2(tmp_path, capsys):
    assert main([]) == 2
    assert "nothing to do" in capsys.readouterr().err
    assert main(["--gen", "swn", "--clusters", "4", "--out", str(tmp_path / "x.bin")]) == 2
    assert "--y" in capsys.readouterr().err
    assert main(["--algo", "piecy", "--gen", "swn", "--clusters", "2", "--y", "3", "--d", "4", "--x", "2"]) == 2
    assert "--k" in capsys.readouterr().err
    assert main(["--algo", "piecy", "--k", "2"]) == 2
    assert "--input or --gen" in capsys.readouterr().err
    assert main(["--algo", "piecy", "--k", "2", "--weighted", "--gen", "random", "--n", "4"]) == 2
    assert "weighted input" in capsys.readouterr().err
    assert main(["--algo", "bico", "--k", "0", "--gen", "random", "--n", "4"]) == 2
    assert main(["--algo", "bico", "--k", "2", "--input", str(tmp_path / "missing.bin")]) == 2
