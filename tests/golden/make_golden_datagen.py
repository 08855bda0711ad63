"""Golden fixtures of the reference's paper generators (build container only).

    python tests/golden/make_golden_datagen.py

Runs the UNMODIFIED reference ``piecy.datagen`` (/root/reference/pkg/src,
read-only, never copied): structured_with_noise, lower_bound and random_cube
on small configs (datagen.py:104-135) -> tests/golden/datagen.npz.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

SWN = [(6, 15, 40, 8, 10.0, 0.5, 4), (3, 7, 13, 13, 10.0, 0.5, 1), (20, 50, 200, 20, 10.0, 0.5, 1),
       (2, 1, 1, 1, 3.0, 1.0, 9), (4, 33, 64, 5, 7.5, 0.25, 2**70 + 5)]
CUBE = [(5, 10.0, 0), (33, 2.5, 7), (128, 10.0, 3)]
LB = [(5, 50, 1000.0, 100.0), (2, 8, 10.0, 1.0), (10, 200, 1000.0, 100.0)]


def main():
    sys.path.insert(0, REF)
    from piecy import datagen as D
    out = {}
    for i, (cl, ppc, dim, a, sp, no, seed) in enumerate(SWN):
        X = np.array(list(D.structured_with_noise(D.SwnConfig(cl, ppc, dim, a, spread=sp, noise=no, seed=seed))))
        out[f"swn{i}"] = X
        out[f"swn{i}_cfg"] = np.array([cl, ppc, dim, a, sp, no, seed], dtype=object).astype(str)
    for i, (n, sp, seed) in enumerate(CUBE):
        out[f"cube{i}"] = np.array(list(D.random_cube(D.RandomConfig(n, spread=sp, seed=seed))))
    for i, (k, n, sp, no) in enumerate(LB):
        out[f"lb{i}"] = np.array(list(D.lower_bound(D.LowerBoundConfig(k, n, spread=sp, noise=no))))
    np.savez_compressed(os.path.join(HERE, "datagen.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
