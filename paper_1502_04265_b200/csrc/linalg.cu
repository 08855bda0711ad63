// Randomized best-fit projection on B200 (sm_100a), all fp64.
//
// Reference: /root/reference/pkg/src/piecy/linalg.py
//   randomized_truncated_svd :167-206   (sketch, q power iterations with QR,
//                                         two-sided core when rows > 4r)
//   _fix_signs / _clip_small :77-94
//   project                  :209-221   A V V^T
//   weighted_best_fit        :231-250   rows scaled by sqrt(w)
// Building blocks (all hand-written; no cuBLAS, no host round trip inside
// the decomposition -- a device status word picks the code path):
//   pcy_gemm_f64 (gemm.cu) -- strided split-K fp64 DMMA GEMM for the range
//                finder, the core products and the projection
//   CholeskyQR2 -- Gram by GEMM, k_chol (one CTA, shared memory up to r = 160)
//                with a rank-deficiency pivot test, k_trsm_rows (Y <- Y L^-T,
//                one thread per row, L broadcast from shared memory):
//                orthonormal basis of the same span as LAPACK's Householder Q
//                (only the span reaches the result; SURVEY.md §7 hard part 5);
//                k_cgs2 runs instead when the factorisation breaks down
//   k_jacobi_smem / k_jacobi -- one-sided (Hestenes) Jacobi SVD, tournament
//                ordering: one CTA with the matrix in shared memory when it
//                fits, else a persistent cooperative grid
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include "common.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace {

// ------------------------------------------------------------ Cholesky
// Blocked right-looking Cholesky of the r x r Gram (row-major; lower factor
// written in place) in CHB-wide column blocks, and the triangular solve
// Y <- Y L^-T applied block by block -- the GEMM parts on pcy_gemm_f64.
// status[0]: sticky failure flag of one orthonormalisation (0 = CholeskyQR
// holding so far); status[1]: CGS2 completion failure; status[4..5] (as a
// double): the Gram's largest diagonal, the scale of a rounding-level pivot.
constexpr int CHB = 64;

// Whole-Gram checks of a pass: largest diagonal; with expect_identity (second
// CholeskyQR pass) the Gram must be within 1e-3 of I, else the first pass
// lost orthogonality.  Skips when status[0] is set.
__global__ void k_gram_check(const double* __restrict__ G, int r, int expect_identity, int* __restrict__ status) {
  if (*(volatile int*)status) return;
  unsigned long long* gmax = reinterpret_cast<unsigned long long*>(status + 4);
  const long long n = (long long)r * r;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / r), j = (int)(e % r);
    const double v = G[e];
    if (expect_identity && !(fabs(v - (i == j ? 1.0 : 0.0)) <= 1e-3)) atomicOr(status, 1);
    if (i == j) atomicMax(gmax, (unsigned long long)__double_as_longlong(fabs(v)));
  }
}

// Diagonal block (k0, k0) of size kb <= CHB: Cholesky in shared memory (the
// trailing updates of earlier blocks are already applied), L11 written back
// (zeros above), and D = L11^-1 (kb x CHB, row-major) for the panel and the
// solve.  A pivot that is not positive, not finite or at rounding level of the
// Gram's scale (a rank-deficient sketch, where CholeskyQR amplifies noise)
// sets status[0].
__global__ void __launch_bounds__(4 * CHB) k_chol_blk(double* __restrict__ G, int r, int k0, int kb,
                                                      double* __restrict__ D, int* __restrict__ status) {
  // Four threads per row (factor) / per column (inverse), each taking every
  // fourth element: two barriers per pivot column, warp shuffles in the inverse.
  extern __shared__ double blk_sm[];   // a (L11) and x (its inverse), CHB x (CHB + 1) each
  double (*a)[CHB + 1] = reinterpret_cast<double (*)[CHB + 1]>(blk_sm);
  double (*x)[CHB + 1] = reinterpret_cast<double (*)[CHB + 1]>(blk_sm + CHB * (CHB + 1));
  __shared__ double colj[CHB];
  __shared__ double s_piv;
  __shared__ int bad;
  if (*(volatile int*)status) return;
  const int tid = threadIdx.x;
  const double gmax = __longlong_as_double(*reinterpret_cast<const long long*>(status + 4));
  const double thr = 16.0 * 2.220446049250313e-16 * gmax;
  if (tid == 0) bad = 0;
  for (int e = tid; e < kb * kb; e += 4 * CHB) {
    const int i = e / kb, c = e % kb;
    a[i][c] = G[(long long)(k0 + i) * r + k0 + c];
  }
  __syncthreads();
  {
    const int i = tid & (CHB - 1), part = tid >> 6;   // row i, columns c = part (mod 4)
    for (int j = 0; j < kb; ++j) {
      if (tid == j) {
        const double t = a[j][j];
        if (!(t > 0.0) || !isfinite(t) || t <= thr) bad = 1;
        else { const double piv = sqrt(t); a[j][j] = piv; s_piv = piv; }
      }
      __syncthreads();
      if (bad) break;
      if (part == 0 && i > j && i < kb) { const double l = a[i][j] / s_piv; a[i][j] = l; colj[i] = l; }
      __syncthreads();
      if (i > j && i < kb) {
        const double l = colj[i];
        double* __restrict__ row = a[i];
        for (int c = j + 1 + part; c <= i; c += 4) row[c] = fma(-l, colj[c], row[c]);
      }
    }
  }
  __syncthreads();
  if (bad) { if (tid == 0) atomicOr(status, 1); return; }
  // D = L11^-1: x[i][j] = -(sum_{k=j}^{i-1} L[i][k] x[k][j]) / L[i][i].  Column j
  // belongs to four adjacent lanes (k = j + q, j + q + 4, ...), their partial
  // sums added in lane order.
  {
    const int j = tid >> 2, q = tid & 3;
    const bool on = j < kb;
    if (on && q == 0) x[j][j] = 1.0 / a[j][j];
    __syncwarp();
    for (int i = 1; i < kb; ++i) {   // uniform trip count: the shuffles need the whole warp
      double acc = 0.0;
      if (on && i > j)
        for (int k = j + q; k < i; k += 4) acc = fma(a[i][k], x[k][j], acc);
      const double a1 = __shfl_down_sync(0xffffffffu, acc, 1);
      const double a2 = __shfl_down_sync(0xffffffffu, acc, 2);
      const double a3 = __shfl_down_sync(0xffffffffu, acc, 3);
      if (on && i > j && q == 0) x[i][j] = -(((acc + a1) + a2) + a3) / a[i][i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int e = tid; e < kb * kb; e += 4 * CHB) {
    const int i = e / kb, c = e % kb;
    G[(long long)(k0 + i) * r + k0 + c] = c <= i ? a[i][c] : 0.0;
    D[(long long)i * CHB + c] = c <= i ? x[i][c] : 0.0;
  }
}

// dst[i][c] = src[i][c] for a rows x cols block with leading dims (skip flag)
__global__ void k_copy_block(double* __restrict__ dst, long long ldd, const double* __restrict__ src, long long lds,
                             long long rows, int cols, const int* __restrict__ status) {
  if (*(volatile const int*)status) return;
  const long long n = rows * cols;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols;
    const int c = (int)(e % cols);
    dst[i * ldd + c] = src[i * lds + c];
  }
}

// zero the strictly upper triangle of the factor (the GEMM updates touch it)
__global__ void k_lower_only(double* __restrict__ G, int r, const int* __restrict__ status) {
  if (*(volatile const int*)status) return;
  const long long n = (long long)r * r;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    if (e % r > e / r) G[e] = 0.0;
}

// Rank-robust orthonormalisation (fallback when CholeskyQR breaks down on a
// rank-deficient sketch, where LAPACK's Householder QR still returns an
// orthonormal Q).  Classical Gram-Schmidt with re-orthogonalisation; a column
// that vanishes is replaced by the next standard basis vector orthogonalised
// against the accepted ones (the completion rule of linalg.py:97-117).  Only
// the span reaches the projection, so any orthonormal completion is valid.
__global__ void __launch_bounds__(1024) k_cgs2(double* __restrict__ Y, long long rows, int r,
                                              double* __restrict__ coef, int* __restrict__ status) {
  if (!*(volatile int*)status) return;   // CholeskyQR held: nothing to do
  __shared__ double red[32];
  __shared__ double s_val;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  auto block_sum = [&](double v) -> double {
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (warp == 0) { double t = lane < nw ? red[lane] : 0.0; t = warp_sum(t); if (lane == 0) s_val = t; }
    __syncthreads();
    return s_val;
  };
  auto orthogonalise = [&](int j) {
    for (int pass = 0; pass < 2; ++pass) {
      for (int k = warp; k < j; k += nw) {
        double acc = 0.0;
        for (long long i = lane; i < rows; i += 32) acc = fma(Y[i * r + k], Y[i * r + j], acc);
        acc = warp_sum(acc);
        if (lane == 0) coef[k] = acc;
      }
      __syncthreads();
      for (long long i = tid; i < rows; i += blockDim.x) {
        double v = Y[i * r + j];
        for (int k = 0; k < j; ++k) v = fma(-Y[i * r + k], coef[k], v);
        Y[i * r + j] = v;
      }
      __syncthreads();
    }
  };
  long long basis = 0;
  for (int j = 0; j < r; ++j) {
    double acc = 0.0;
    for (long long i = tid; i < rows; i += blockDim.x) acc = fma(Y[i * r + j], Y[i * r + j], acc);
    const double orig = sqrt(block_sum(acc));
    orthogonalise(j);
    acc = 0.0;
    for (long long i = tid; i < rows; i += blockDim.x) acc = fma(Y[i * r + j], Y[i * r + j], acc);
    double nrm = sqrt(block_sum(acc));
    if (!(nrm > 1e-10 * orig) || orig == 0.0) {
      for (;;) {
        if (basis >= rows) { if (tid == 0) status[1] = 2; return; }
        for (long long i = tid; i < rows; i += blockDim.x) Y[i * r + j] = (i == basis) ? 1.0 : 0.0;
        ++basis;
        __syncthreads();
        orthogonalise(j);
        acc = 0.0;
        for (long long i = tid; i < rows; i += blockDim.x) acc = fma(Y[i * r + j], Y[i * r + j], acc);
        nrm = sqrt(block_sum(acc));
        if (nrm > 0.5) break;
      }
    }
    // true division (not a reciprocal multiply): a column c * e normalises to
    // exactly +-e / |e| whatever c is, so degenerate (duplicated-row) sketches
    // give the same basis for every seed, as LAPACK's Householder QR does
    for (long long i = tid; i < rows; i += blockDim.x) Y[i * r + j] /= nrm;
    __syncthreads();
  }
}

// ---------------------------------------------------------- Jacobi SVD
// One-sided (Hestenes) Jacobi on G (m rows x n cols, column j at G + j*m),
// tournament ordering.  On exit sig[j] (descending) and U (m x n, row-major
// with leading dim ldu) hold the normalised columns of G*J; these are the
// right singular vectors of G^T.  perm scratch (n ints), rot scratch
// (max_sweeps ints, zeroed by the caller).
//
// Persistent cooperative kernel: one warp per pair of a round, the CTAs of
// the grid meet at a grid barrier between rounds (the pairs of one round are
// disjoint, so the result does not depend on how pairs map to warps).
__global__ void __launch_bounds__(256) k_jacobi(double* __restrict__ G, int m, int n, double tol, int max_sweeps,
                                               double* __restrict__ sig, double* __restrict__ U, int ldu,
                                               int* __restrict__ perm, int* __restrict__ sweeps_out,
                                               int* __restrict__ rot) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nw = (int)((gridDim.x * blockDim.x) >> 5);
  const long long gt = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nt = (long long)gridDim.x * blockDim.x;
  const int np = (n + 1) & ~1;   // even count (one dummy when n is odd)
  int sweep = 0;
  for (; sweep < max_sweeps; ++sweep) {
    for (int round = 0; round < np - 1; ++round) {
      // tournament pairing: position 0 fixed, others rotate
      for (int pr = gw; pr < np / 2; pr += nw) {
        int a = (pr == 0) ? 0 : 1 + (pr - 1 + round) % (np - 1);
        int b = 1 + (np - 2 - pr + round) % (np - 1);
        if (a >= n || b >= n) continue;
        if (a > b) { const int t = a; a = b; b = t; }
        double* gp = G + (long long)a * m;
        double* gq = G + (long long)b * m;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < m; i += 32) {
          const double x = gp[i], y = gq[i];
          al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        if (fabs(ga) > tol * sqrt(al * be) && ga != 0.0) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int i = lane; i < m; i += 32) {
            const double x = gp[i], y = gq[i];
            gp[i] = c * x - s * y;
            gq[i] = s * x + c * y;
          }
          if (lane == 0) atomicOr(rot + sweep, 1);
        }
      }
      grid.sync();
    }
    if (!*(volatile int*)(rot + sweep)) break;
  }
  // column norms
  for (int j = gw; j < n; j += nw) {
    const double* gj = G + (long long)j * m;
    double acc = 0.0;
    for (int i = lane; i < m; i += 32) acc = fma(gj[i], gj[i], acc);
    acc = warp_sum(acc);
    if (lane == 0) sig[j] = sqrt(acc);
  }
  grid.sync();
  // order by sigma descending (stable on ties), rank by counting
  for (long long j = gt; j < n; j += nt) {
    const double sj = sig[j];
    int rank = 0;
    for (int k = 0; k < n; ++k) rank += (sig[k] > sj) || (sig[k] == sj && k < j);
    perm[rank] = (int)j;
  }
  grid.sync();
  for (int jj = gw; jj < n; jj += nw) {
    const int j = perm[jj];
    const double* gj = G + (long long)j * m;
    const double sj = sig[j];
    for (int i = lane; i < m; i += 32) U[(long long)i * ldu + jj] = sj > 0.0 ? gj[i] / sj : 0.0;
  }
  if (gt == 0) *sweeps_out = sweep;
}

// The same one-sided Jacobi with G (m x n, column-major) resident in shared
// memory and one CTA: a __syncthreads per round instead of a grid barrier.
// The per-pair arithmetic is the cooperative kernel's (same rotations, same
// order), so both give identical results.
__global__ void __launch_bounds__(1024) k_jacobi_smem(double* __restrict__ Gg, int m, int n, double tol,
                                                      int max_sweeps, double* __restrict__ sig,
                                                      double* __restrict__ U, int ldu, int* __restrict__ perm,
                                                      int* __restrict__ sweeps_out) {
  extern __shared__ double jac_sm[];
  __shared__ int s_rot;
  double* G = jac_sm;
  const int lane = threadIdx.x & 31, gw = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (long long e = threadIdx.x; e < (long long)m * n; e += blockDim.x) G[e] = Gg[e];
  const int np = (n + 1) & ~1;
  int sweep = 0;
  __syncthreads();
  for (; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int round = 0; round < np - 1; ++round) {
      for (int pr = gw; pr < np / 2; pr += nw) {
        int a = (pr == 0) ? 0 : 1 + (pr - 1 + round) % (np - 1);
        int b = 1 + (np - 2 - pr + round) % (np - 1);
        if (a >= n || b >= n) continue;
        if (a > b) { const int t = a; a = b; b = t; }
        double* gp = G + (long long)a * m;
        double* gq = G + (long long)b * m;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < m; i += 32) {
          const double x = gp[i], y = gq[i];
          al = fma(x, x, al); be = fma(y, y, be); ga = fma(x, y, ga);
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        if (fabs(ga) > tol * sqrt(al * be) && ga != 0.0) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int i = lane; i < m; i += 32) {
            const double x = gp[i], y = gq[i];
            gp[i] = c * x - s * y;
            gq[i] = s * x + c * y;
          }
          if (lane == 0) s_rot = 1;
        }
      }
      __syncthreads();
    }
    if (!s_rot) break;
  }
  for (int j = gw; j < n; j += nw) {
    const double* gj = G + (long long)j * m;
    double acc = 0.0;
    for (int i = lane; i < m; i += 32) acc = fma(gj[i], gj[i], acc);
    acc = warp_sum(acc);
    if (lane == 0) sig[j] = sqrt(acc);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const double sj = sig[j];
    int rank = 0;
    for (int k = 0; k < n; ++k) rank += (sig[k] > sj) || (sig[k] == sj && k < j);
    perm[rank] = j;
  }
  __syncthreads();
  for (int jj = gw; jj < n; jj += nw) {
    const int j = perm[jj];
    const double* gj = G + (long long)j * m;
    const double sj = sig[j];
    for (int i = lane; i < m; i += 32) U[(long long)i * ldu + jj] = sj > 0.0 ? gj[i] / sj : 0.0;
  }
  if (threadIdx.x == 0) *sweeps_out = sweep;
}

// Sorted singular values: sorted[jj] = sig[perm[jj]] computed by rank again
// (same ranking rule as k_jacobi's column order).
// out[n] = completion failure (status[1]), out[n + 1] = A finite (status[2]).
__global__ void k_sorted_sigma(const double* __restrict__ sig, int n, double* __restrict__ out,
                               const int* __restrict__ status) {
  if (blockIdx.x == 0 && threadIdx.x == 0) { out[n] = (double)status[1]; out[n + 1] = (double)status[2]; }
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const double sj = sig[j];
    int rank = 0;
    for (int k = 0; k < n; ++k) rank += (sig[k] > sj) || (sig[k] == sj && k < j);
    out[rank] = sj;
  }
}

// _fix_signs: first entry with |v| > 1e-12 * max|v| made nonnegative, per
// column of V (rows x cols row-major, leading dim ldv).  One warp per column.
__global__ void k_fix_signs(double* __restrict__ V, int rows, int cols, int ldv) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= cols) return;
  double pk = 0.0;
  for (int i = lane; i < rows; i += 32) pk = fmax(pk, fabs(V[(long long)i * ldv + j]));
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) pk = fmax(pk, __shfl_xor_sync(PCY_FULL, pk, o));
  if (pk == 0.0) return;
  const double thr = 1e-12 * pk;
  int first = 0x7fffffff;
  for (int i = lane; i < rows; i += 32)
    if (fabs(V[(long long)i * ldv + j]) > thr) { first = i; break; }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) first = min(first, __shfl_xor_sync(PCY_FULL, first, o));
  if (first == 0x7fffffff) return;
  const bool neg = V[(long long)first * ldv + j] < 0.0;
  if (neg) for (int i = lane; i < rows; i += 32) V[(long long)i * ldv + j] = -V[(long long)i * ldv + j];
}

__global__ void k_cast_f32(const float* __restrict__ src, long long n, double* __restrict__ dst) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = (double)src[i];
}

// rows scaled by sqrt(w) (linalg.py:247)
__global__ void k_scale_rows(const double* __restrict__ A, const long long* __restrict__ w, long long rows, int cols,
                             double* __restrict__ out) {
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < rows * cols; e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / cols;
    out[e] = A[e] * sqrt((double)w[i]);
  }
}

__global__ void k_cast_i64(const long long* __restrict__ src, long long n, double* __restrict__ dst) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    dst[i] = (double)src[i];
}

__global__ void k_all_finite(const void* __restrict__ p, long long n, int dt, int* __restrict__ flag) {
  bool ok = true;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    ok &= dt ? isfinite(((const float*)p)[i]) : isfinite(((const double*)p)[i]);
  if (!__all_sync(PCY_FULL, ok) && (threadIdx.x & 31) == 0) *flag = 0;
}

}  // namespace

// ==================================================================== host
int pcy_gemm_f64(cudaStream_t st, int M, int N, int K, double alpha, const double* A, long long lda, int ta,
                 const double* B, long long ldb, int tb, double beta, double* C, long long ldc, const int* skip);

// C[M x N] = alpha * op(A) * op(B) + beta * C, row-major with leading dims.
// op(A) is M x K: A[m*lda + k] (ta=0) or A[k*lda + m] (ta=1).
// op(B) is K x N: B[k*ldb + n] (tb=0) or B[n*ldb + k] (tb=1).
static int gemm(cudaStream_t st, int M, int N, int K, double alpha, const double* A, long long lda, int ta,
                const double* B, long long ldb, int tb, double beta, double* C, long long ldc,
                const int* skip = nullptr) {
  return pcy_gemm_f64(st, M, N, K, alpha, A, lda, ta, B, ldb, tb, beta, C, ldc, skip);
}

static int jacobi(cudaStream_t st, double* G, int m, int n, double tol, int max_sweeps, double* sig, double* U,
                  int ldu, int* perm, int* sweeps, int* rot) {
  const size_t sm = sizeof(double) * (size_t)m * n;
  // one CTA with the matrix in shared memory for narrow problems (few pairs
  // per round: the grid barrier would dominate); the cooperative grid else
  if (n <= 64 && sm <= 200 * 1024) {
    static thread_local bool attr = false;
    if (!attr) {
      PCY_CUDA(cudaFuncSetAttribute(k_jacobi_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      attr = true;
    }
    const int threads = std::min(1024, std::max(64, ((n + 1) / 2) * 32));
    k_jacobi_smem<<<1, threads, sm, st>>>(G, m, n, tol, max_sweeps, sig, U, ldu, perm, sweeps);
    pcy_count_launch();
    PCY_LAUNCH_CHECK();
    return PCY_OK;
  }
  PCY_CUDA(cudaMemsetAsync(rot, 0, sizeof(int) * max_sweeps, st));
  // co-resident CTA limit of the cooperative launch, per device (threads of
  // distributed.py may drive different GPUs)
  thread_local int max_blocks_dev[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& max_blocks = max_blocks_dev[dev & 15];
  if (max_blocks <= 0) {
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_jacobi, 256, 0);
    max_blocks = sms * (per > 0 ? per : 1);
  }
  const int pairs = (n + 1) / 2;
  int blocks = (pairs + 7) / 8;
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  void* args[] = {&G, &m, &n, &tol, &max_sweeps, &sig, &U, &ldu, &perm, &sweeps, &rot};
  PCY_CUDA(cudaLaunchCooperativeKernel((const void*)k_jacobi, dim3(blocks), dim3(256), args, 0, st));
  pcy_count_launch();
  return PCY_OK;
}

// Orthonormalise Y (rows x r, row-major) in place: CholeskyQR2, or, when a
// factorisation breaks down, CGS2 with completion.  Each pass: Gram (GEMM),
// blocked Cholesky (k_chol_blk on the diagonal blocks, GEMM panel solves and
// trailing updates), then Y <- Y L^-T block column by block column (GEMMs with
// the diagonal blocks' inverses).  No host read: status[0] (device) skips the
// remaining launches once a factorisation fails and turns k_cgs2 on.
// Scratch: Gs (r x r), D (r x CHB), T (rows x CHB).
static int cholqr(cudaStream_t st, double* Y, long long rows, int r, double* Gs, double* D, double* T,
                  double* coef, int* status) {
  constexpr size_t blk_smem = sizeof(double) * 2 * CHB * (CHB + 1);
  static thread_local bool attr = false;
  if (!attr) {
    PCY_CUDA(cudaFuncSetAttribute(k_chol_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)blk_smem));
    attr = true;
  }
  PCY_CUDA(cudaMemsetAsync(status, 0, sizeof(int), st));
  const unsigned eb = (unsigned)std::min<long long>(((long long)r * r + 255) / 256, 148 * 4);
  int rc;
  for (int pass = 0; pass < 2; ++pass) {
    PCY_CUDA(cudaMemsetAsync(status + 4, 0, sizeof(double), st));
    if ((rc = gemm(st, r, r, (int)rows, 1.0, Y, r, 1, Y, r, 0, 0.0, Gs, r, status))) return rc;
    k_gram_check<<<eb, 256, 0, st>>>(Gs, r, pass, status); pcy_count_launch();
    for (int k0 = 0; k0 < r; k0 += CHB) {
      const int kb = std::min(CHB, r - k0), rest = r - k0 - kb;
      k_chol_blk<<<1, 4 * CHB, blk_smem, st>>>(Gs, r, k0, kb, D + (long long)k0 * CHB, status); pcy_count_launch();
      if (rest > 0) {
        // panel L21 = A21 L11^-T (through T), trailing A22 -= L21 L21^T
        double* A21 = Gs + (long long)(k0 + kb) * r + k0;
        if ((rc = gemm(st, rest, kb, kb, 1.0, A21, r, 0, D + (long long)k0 * CHB, CHB, 1, 0.0, T, CHB, status))) return rc;
        k_copy_block<<<(unsigned)std::min<long long>(((long long)rest * kb + 255) / 256, 148 * 4), 256, 0, st>>>(
            A21, r, T, CHB, rest, kb, status);
        pcy_count_launch();
        double* A22 = Gs + (long long)(k0 + kb) * r + k0 + kb;
        if ((rc = gemm(st, rest, rest, kb, -1.0, A21, r, 0, A21, r, 1, 1.0, A22, r, status))) return rc;
      }
    }
    k_lower_only<<<eb, 256, 0, st>>>(Gs, r, status); pcy_count_launch();
    // Y <- Y L^-T: block column b: Y_b <- (Y_b - Y_<b L_b,<b^T) D_b^T
    for (int k0 = 0; k0 < r; k0 += CHB) {
      const int kb = std::min(CHB, r - k0);
      double* Yb = Y + k0;
      if (k0 > 0 && (rc = gemm(st, (int)rows, kb, k0, -1.0, Y, r, 0, Gs + (long long)k0 * r, r, 1, 1.0, Yb, r, status)))
        return rc;
      if ((rc = gemm(st, (int)rows, kb, kb, 1.0, Yb, r, 0, D + (long long)k0 * CHB, CHB, 1, 0.0, T, CHB, status)))
        return rc;
      k_copy_block<<<(unsigned)std::min<long long>((rows * kb + 255) / 256, 148 * 8), 256, 0, st>>>(Yb, r, T, CHB, rows,
                                                                                                   kb, status);
      pcy_count_launch();
    }
  }
  // rank-deficient sketch or lost orthogonality: Gram-Schmidt with completion
  // (only when status[0] is set; Y spans the sketch's range either way)
  k_cgs2<<<1, 1024, 0, st>>>(Y, rows, r, coef, status); pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

extern "C" {

int pcy_all_finite(const void* p, long long n, int dtype, int* out_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int* flag;
  PCY_CUDA(pcy_malloc_async(&flag, sizeof(int), st));
  const int one = 1;
  PCY_CUDA(cudaMemcpyAsync(flag, &one, sizeof(int), cudaMemcpyHostToDevice, st));
  if (n > 0) { k_all_finite<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 8), 256, 0, st>>>(p, n, dtype, flag); pcy_count_launch(); }
  PCY_LAUNCH_CHECK();
  PCY_CUDA(pcy_d2h(out_host, flag, sizeof(int), st));
  cudaFreeAsync(flag, st);
  return PCY_OK;
}

int pcy_dgemm(int M, int N, int K, double alpha, const double* A, long long lda, int ta, const double* B,
              long long ldb, int tb, double beta, double* C, long long ldc, void* stream) {
  return gemm((cudaStream_t)stream, M, N, K, alpha, A, lda, ta, B, ldb, tb, beta, C, ldc);
}

int pcy_cast_f32_f64(const float* src, long long n, double* dst, void* stream) {
  if (n <= 0) return PCY_OK;
  k_cast_f32<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(src, n, dst); pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

int pcy_cast_i64_f64(const long long* src, long long n, double* dst, void* stream) {
  if (n <= 0) return PCY_OK;
  k_cast_i64<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(src, n, dst); pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

int pcy_scale_rows_sqrtw(const double* A, const long long* w, long long rows, int cols, double* out, void* stream) {
  if (rows <= 0) return PCY_OK;
  const long long n = rows * cols;
  k_scale_rows<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(A, w, rows, cols, out); pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

// Randomized truncated SVD (linalg.py:167-206) of A (rows x cols, fp64,
// row-major).  omega (cols x r) and omega2 (r x r, used when rows > 4r) are
// the host-drawn standard normals of the reference's rng.  Outputs V
// (cols x ell, row-major, signs fixed) and sigma (ell, host, clipped).
// Returns PCY_ENONFINITE (nothing written) when A has a non-finite entry --
// checked on the device and read back with sigma, the call's only host read.
int pcy_rsvd(const double* A, long long rows, int cols, int ell, int r, int power, const double* omega,
             const double* omega2, double* V, double* sigma_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (r > rows || r > cols || ell > r || ell < 1) { pcy_set_error("rsvd: bad rank"); return PCY_EINVAL; }
  const bool two = rows > 4LL * r;
  double *Q = nullptr, *Z = nullptr, *Bm = nullptr, *Gs = nullptr, *coef = nullptr, *Wm = nullptr, *core = nullptr,
         *Uj = nullptr, *sig = nullptr, *Vfull = nullptr, *Db = nullptr, *Tb = nullptr;
  int *status = nullptr, *perm = nullptr, *sweeps = nullptr, *rot = nullptr;
  int rc = PCY_OK;
  do {
    if ((rc = pcy_malloc_async(&Q, sizeof(double) * rows * r, st)) ||
        (rc = pcy_malloc_async(&Z, sizeof(double) * cols * r, st)) ||
        (rc = pcy_malloc_async(&Bm, sizeof(double) * (long long)r * cols, st)) ||
        (rc = pcy_malloc_async(&Gs, sizeof(double) * r * r, st)) ||
        (rc = pcy_malloc_async(&coef, sizeof(double) * r, st)) ||
        (rc = pcy_malloc_async(&Wm, sizeof(double) * cols * r, st)) ||
        (rc = pcy_malloc_async(&core, sizeof(double) * r * r, st)) ||
        (rc = pcy_malloc_async(&Uj, sizeof(double) * cols * r, st)) ||
        (rc = pcy_malloc_async(&sig, sizeof(double) * (2 * r + 2), st)) ||
        (rc = pcy_malloc_async(&Vfull, sizeof(double) * cols * r, st)) ||
        (rc = pcy_malloc_async(&status, sizeof(int) * 8, st)) ||
        (rc = pcy_malloc_async(&Db, sizeof(double) * ((long long)r + CHB) * CHB, st)) ||
        (rc = pcy_malloc_async(&Tb, sizeof(double) * std::max<long long>(rows, cols) * CHB, st)) ||
        (rc = pcy_malloc_async(&perm, sizeof(int) * r, st)) ||
        (rc = pcy_malloc_async(&sweeps, sizeof(int), st)) ||
        (rc = pcy_malloc_async(&rot, sizeof(int) * 64, st))) {
      pcy_set_error("rsvd: device allocation failed"); rc = PCY_ENOMEM; break;
    }
    PCY_CUDA(cudaMemsetAsync(status, 0, sizeof(int) * 8, st));
    // finiteness of A into status[2] (cleared on a non-finite entry)
    {
      const int one = 1;
      PCY_CUDA(cudaMemcpyAsync(status + 2, &one, sizeof(int), cudaMemcpyHostToDevice, st));
      const long long n = rows * (long long)cols;
      k_all_finite<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 8), 256, 0, st>>>(A, n, 0, status + 2);
      pcy_count_launch();
    }
    // Q = qr(A omega)
    if ((rc = gemm(st, (int)rows, r, cols, 1.0, A, cols, 0, omega, r, 0, 0.0, Q, r))) break;
    if ((rc = cholqr(st, Q, rows, r, Gs, Db, Tb, coef, status))) break;
    for (int it = 0; it < power; ++it) {
      // Z = qr(A^T Q); Q = qr(A Z)
      if ((rc = gemm(st, cols, r, (int)rows, 1.0, A, cols, 1, Q, r, 0, 0.0, Z, r))) break;
      if ((rc = cholqr(st, Z, cols, r, Gs, Db, Tb, coef, status))) break;
      if ((rc = gemm(st, (int)rows, r, cols, 1.0, A, cols, 0, Z, r, 0, 0.0, Q, r))) break;
      if ((rc = cholqr(st, Q, rows, r, Gs, Db, Tb, coef, status))) break;
    }
    if (rc) break;
    // small = Q^T A  (r x cols)
    if ((rc = gemm(st, r, cols, (int)rows, 1.0, Q, r, 1, A, cols, 0, 0.0, Bm, cols))) break;
    const double tol = 2.220446049250313e-16 * (double)std::max(r, 8);
    if (two) {
      // W = qr(small^T omega2) (cols x r); core = small W (r x r)
      if ((rc = gemm(st, cols, r, r, 1.0, Bm, cols, 1, omega2, r, 0, 0.0, Wm, r))) break;
      if ((rc = cholqr(st, Wm, cols, r, Gs, Db, Tb, coef, status))) break;
      if ((rc = gemm(st, r, r, cols, 1.0, Bm, cols, 0, Wm, r, 0, 0.0, core, r))) break;
      // Jacobi on core^T: column j of core^T = row j of core (contiguous)
      if ((rc = jacobi(st, core, r, r, tol, 60, sig, Uj, r, perm, sweeps, rot))) break;
      // Uj (r x r row-major) columns = right singular vectors of core: V = W Uj
      if ((rc = gemm(st, cols, r, r, 1.0, Wm, r, 0, Uj, r, 0, 0.0, Vfull, r))) break;
    } else {
      // Jacobi on small^T: column j of small^T = row j of small (contiguous)
      if ((rc = jacobi(st, Bm, cols, r, tol, 60, sig, Vfull, r, perm, sweeps, rot))) break;
    }
    k_sorted_sigma<<<1, 256, 0, st>>>(sig, r, sig + r, status); pcy_count_launch();
    // keep the first ell columns
    PCY_CUDA(cudaMemcpy2DAsync(V, sizeof(double) * ell, Vfull, sizeof(double) * r, sizeof(double) * ell, cols,
                               cudaMemcpyDeviceToDevice, st));
    k_fix_signs<<<(ell + 7) / 8, 256, 0, st>>>(V, cols, ell, ell); pcy_count_launch();
    PCY_LAUNCH_CHECK();
    // the one host read: sorted sigma + [completion failure, finiteness]
    std::vector<double> hs(r + 2);
    PCY_CUDA(pcy_d2h(hs.data(), sig + r, sizeof(double) * (r + 2), st));
    if (hs[r + 1] == 0.0) { pcy_set_error("matrix contains non-finite entries"); rc = PCY_ENONFINITE; break; }
    if (hs[r] != 0.0) { pcy_set_error("orthonormal completion failed"); rc = PCY_ESTATE; break; }
    for (int j = 0; j < ell; ++j) sigma_host[j] = hs[j];
    if (ell > 0 && sigma_host[0] > 0.0)
      for (int j = 0; j < ell; ++j) if (sigma_host[j] < 1e-12 * sigma_host[0]) sigma_host[j] = 0.0;
  } while (0);
  for (void* q : {(void*)Q, (void*)Z, (void*)Bm, (void*)Gs, (void*)coef, (void*)Wm, (void*)core, (void*)Uj,
                  (void*)sig, (void*)Vfull, (void*)status, (void*)perm, (void*)sweeps, (void*)rot, (void*)Db,
                  (void*)Tb})
    if (q) cudaFreeAsync(q, st);
  return rc;
}

// project (linalg.py:209-221): out = (A V) V^T, A rows x cols, V cols x ell.
int pcy_project(const double* A, long long rows, int cols, const double* V, int ell, double* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  double* P;
  PCY_CUDA(pcy_malloc_async(&P, sizeof(double) * rows * ell, st));
  int rc = gemm(st, (int)rows, ell, cols, 1.0, A, cols, 0, V, ell, 0, 0.0, P, ell);
  if (!rc) rc = gemm(st, (int)rows, cols, ell, 1.0, P, ell, 0, V, ell, 1, 0.0, out, cols);
  cudaFreeAsync(P, st);
  return rc;
}

}  // extern "C"
