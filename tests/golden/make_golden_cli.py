"""Golden CLI reports of the reference (build container only).

    python tests/golden/make_golden_cli.py

Runs the UNMODIFIED reference CLI (``piecy.cli.main``, cli.py:307-317,
imported from /root/reference/pkg/src, read-only) on small generated
instances for every pipeline and evaluation mode, and records the report
lines (cli.py:280-303) -> tests/golden/cli_reports.json.  The ``*_seconds``
timings are not reproducible and are dropped.  The coreset written by
``--out`` is recorded too (weights exact, points as floats).
"""

import contextlib
import io
import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    "bico_swn": ["--algo", "bico", "--gen", "swn", "--clusters", "5", "--y", "60", "--d", "20", "--x", "4",
                 "--k", "5", "--coreset-size", "80", "--seed", "3"],
    "piecy_swn": ["--algo", "piecy", "--gen", "swn", "--clusters", "6", "--y", "100", "--d", "40", "--x", "5",
                  "--k", "6", "--coreset-size", "150", "--piece-size", "200", "--seed", "1", "--eval", "both"],
    "piecy_mr_swn": ["--algo", "piecy-mr", "--gen", "swn", "--clusters", "4", "--y", "150", "--d", "30", "--x", "6",
                     "--k", "4", "--coreset-size", "100", "--piece-size", "100", "--np", "3", "--seed", "2",
                     "--eval", "full"],
    # LowerBound pieces have a 49-fold degenerate singular value: a rank-6
    # projection picks an arbitrary basis of that eigenspace (LAPACK's choice
    # is not reproducible by any other SVD), so LB runs without projection here
    "bico_lb": ["--algo", "bico", "--gen", "lb", "--k", "4", "--n", "200", "--coreset-size", "60"],
    "bico_random": ["--algo", "bico", "--gen", "random", "--n", "90", "--k", "3", "--coreset-size", "40",
                    "--seed", "5", "--reps", "2"],
}


def parse(text):
    out = {}
    for line in text.strip().splitlines():
        key, _, value = line.partition(" = ")
        out[key.strip()] = value.strip()
    return out


def main():
    sys.path.insert(0, REF)
    from piecy.cli import main as ref_main
    from piecy.streams import PointSource
    res = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, argv in CASES.items():
            out = os.path.join(tmp, name + ".bin")
            buf = io.StringIO()
            with contextlib.redirect_stdout(buf):
                code = ref_main(argv + ["--out", out])
            assert code == 0, name
            rep = {k: v for k, v in parse(buf.getvalue()).items() if not k.endswith("_seconds")}
            rows = list(PointSource(out, "bin", weighted=True))
            res[name] = {"argv": argv, "report": rep,
                         "coreset_weights": [int(w) for _, w in rows],
                         "coreset_points": [np.asarray(p, dtype=float).tolist() for p, _ in rows]}
    with open(os.path.join(HERE, "cli_reports.json"), "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", len(res), "reports")


if __name__ == "__main__":
    main()
