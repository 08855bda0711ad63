"""Device projection (GEMM / CholeskyQR2 / Jacobi) vs the numpy oracle."""

import numpy as np
import pytest

from oracle import piecy_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K,ta,tb", [(1, 1, 1, 0, 0), (70, 33, 129, 0, 0), (64, 64, 64, 1, 0),
                                         (130, 17, 300, 0, 1), (5, 200, 77, 1, 1)])
def test_dgemm(M, N, K, ta, tb):
    import torch
    from paper_1502_04265_b200 import _native as nat, linalg  # noqa: F401
    rng = np.random.default_rng(M * 7 + N)
    A = rng.normal(size=(K, M) if ta else (M, K))
    B = rng.normal(size=(N, K) if tb else (K, N))
    want = (A.T if ta else A) @ (B.T if tb else B)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    C = torch.zeros((M, N), dtype=torch.float64, device="cuda")
    nat.check(nat.lib().pcy_dgemm(M, N, K, 1.0, nat.ptr(Ad), A.shape[1], ta, nat.ptr(Bd), B.shape[1], tb, 0.0,
                                  nat.ptr(C), N, nat.stream_ptr()), "dgemm")
    np.testing.assert_allclose(C.cpu().numpy(), want, rtol=1e-12, atol=1e-12 * np.abs(want).max())


def _lowrank(seed, rows, cols, rank, noise=1e-3):
    rng = np.random.default_rng(seed)
    U = rng.normal(size=(rows, rank))
    V = rng.normal(size=(rank, cols))
    s = np.geomspace(100.0, 1.0, rank)
    return (U * s) @ V + noise * rng.normal(size=(rows, cols))


@pytest.mark.parametrize("rows,cols,ell,ov,seed", [(1000, 128, 30, 10, 0), (100, 64, 10, 10, 1),
                                                   (3000, 300, 40, 10, 2), (45, 50, 20, 5, 3)])
def test_rsvd_and_project_match_oracle(rows, cols, ell, ov, seed):
    from paper_1502_04265_b200 import linalg
    A = _lowrank(seed, rows, cols, min(60, cols))
    pr = linalg.randomized_truncated_svd(A, linalg.SvdTruncation(ell, ov, 2, seed))
    V, sig = O.rsvd(A, ell, ov, 2, seed)
    np.testing.assert_allclose(pr.singular_values, sig, rtol=1e-10)
    np.testing.assert_allclose(pr.vectors, V, atol=1e-9)
    got = linalg.project(A, pr)
    want = O.project(A, V)
    np.testing.assert_allclose(got, want, atol=1e-9 * np.abs(want).max())


def test_weighted_best_fit_matches_oracle():
    from paper_1502_04265_b200 import linalg
    A = _lowrank(5, 800, 90, 30)
    w = np.random.default_rng(5).integers(1, 40, size=800)
    pr = linalg.weighted_best_fit(A, w, linalg.SvdTruncation(12, 10, 2, 99))
    V, sig = O.weighted_fit(A, w, 12, 10, 2, 99)
    np.testing.assert_allclose(pr.singular_values, sig, rtol=1e-10)
    np.testing.assert_allclose(pr.vectors, V, atol=1e-9)


@pytest.mark.parametrize("rows,cols,rank_true,ell,ov", [(4, 3, 1, 1, 2), (60, 30, 3, 8, 10), (500, 80, 5, 12, 10)])
def test_rank_deficient_sketch_projects_like_reference(rows, cols, rank_true, ell, ov):
    """LAPACK QR stays orthonormal on rank-deficient sketches; the device
    CholeskyQR2 falls back to Gram-Schmidt with completion.  Only the span
    reaches the projection, which must match the oracle."""
    from paper_1502_04265_b200 import linalg
    rng = np.random.default_rng(rows)
    A = rng.normal(size=(rows, rank_true)) @ rng.normal(size=(rank_true, cols))
    pr = linalg.randomized_truncated_svd(A, linalg.SvdTruncation(ell, ov, 2, 5))
    V, sig = O.rsvd(A, ell, ov, 2, 5)
    np.testing.assert_allclose(pr.singular_values[:rank_true], sig[:rank_true], rtol=1e-9)
    np.testing.assert_allclose(linalg.project(A, pr), O.project(A, V), atol=1e-9 * np.abs(A).max())
    np.testing.assert_allclose(pr.vectors.T @ pr.vectors, np.eye(ell), atol=1e-9)
