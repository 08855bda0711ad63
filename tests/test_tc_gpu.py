"""Split-TF32 tensor-core distance contraction (csrc/tc_dots.cu) against fp64.

The contraction feeds the full-set nearest-reference search (coreset.py:318-330)
at d >= 256; its products are fp32-faithful, so the test checks the rigorous
error bound the engine's near-tie recheck relies on: |approx - exact| <=
tau |a - c| |b - c| (c = first row of A), for padded and unpadded shapes.
"""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,d", [(1, 1, 3), (300, 700, 57), (129, 257, 300), (1000, 333, 1024),
                                   (64, 200, 4096)])
def test_tc_dots_error_bound(m, n, d):
    import torch
    from paper_1502_04265_b200 import _native as nat
    rng = np.random.default_rng(m * 7 + n + d)
    A = rng.normal(50.0, 3.0, size=(m, d))          # offset data: centring matters
    B = rng.normal(50.0, 3.0, size=(n, d))
    B[: n // 3] = A[rng.integers(0, m, size=n // 3)]   # exact duplicates of A rows
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    out = torch.empty((m, n), dtype=torch.float32, device="cuda")
    tau = ctypes.c_double()
    nat.check(nat.lib().pcy_tc_dots_f64(nat.ptr(Ad), d, m, nat.ptr(Bd), d, n, d, nat.ptr(out),
                                        ctypes.byref(tau), nat.stream_ptr()), "tc_dots")
    torch.cuda.synchronize()
    c = A[0]
    Ac, Bc = A - c, B - c
    exact = Ac @ Bc.T
    bound = tau.value * np.linalg.norm(Ac, axis=1)[:, None] * np.linalg.norm(Bc, axis=1)[None, :]
    err = np.abs(out.cpu().numpy().astype(np.float64) - exact)
    assert np.all(err <= bound + 1e-300), float((err / np.maximum(bound, 1e-300)).max())
    # typical errors sit well inside the worst-case window the recheck uses
    assert np.median(err / np.maximum(bound, 1e-300)) < 0.25
