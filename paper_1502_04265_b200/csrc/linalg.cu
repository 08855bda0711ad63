// Randomized best-fit projection on B200 (sm_100a), all fp64.
//
// Reference: /root/reference/pkg/src/piecy/linalg.py
//   randomized_truncated_svd :167-206   (sketch, q power iterations with QR,
//                                         two-sided core when rows > 4r)
//   _fix_signs / _clip_small :77-94
//   project                  :209-221   A V V^T
//   weighted_best_fit        :231-250   rows scaled by sqrt(w)
// Building blocks:
//   gemm      -- plain fp64 GEMMs of the range finder on cuBLAS (library GEMM)
//   CholeskyQR2 (k_gram_prep, k_chol_diag + cuBLAS trsm/syrk, blocked):
//                orthonormal basis of the same span as LAPACK's Householder Q
//                (only the span reaches the result; SURVEY.md §7 hard part 5),
//                k_cgs2 when the Gram factorisation breaks down
//   k_jacobi  -- one-sided (Hestenes) Jacobi SVD, tournament ordering,
//                persistent cooperative grid (grid barrier per round)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cublas_v2.h>
#include "common.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace {

// ------------------------------------------------------------ Cholesky
// Blocked Cholesky pieces (column-major lower, as LAPACK potrf 'L'; the
// Gram is symmetric so its row-major buffer is its column-major buffer).
// k_gram_prep: add the shift to the diagonal, and in the second CholeskyQR
// pass check that the Gram of the already orthonormalised basis is close to I
// (otherwise the first pass lost orthogonality).  Resets *status.
__global__ void k_gram_prep(double* __restrict__ G, int r, double shift, int expect_identity,
                            int* __restrict__ status) {
  const long long n = (long long)r * r;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const bool diag = (e / r) == (e % r);
    if (expect_identity && fabs(G[e] - (diag ? 1.0 : 0.0)) > 1e-3) atomicOr(status, 1);
    if (diag && shift != 0.0) G[e] += shift;
    if (diag)   // nonnegative doubles order like their bit patterns
      atomicMax(reinterpret_cast<unsigned long long*>(status + 2), (unsigned long long)__double_as_longlong(fabs(G[e])));
  }
}

// In-place Cholesky of the kb x kb diagonal block at A + k0*(lda+1) (kb <= 64),
// staged in shared memory.  A non-positive or non-finite pivot sets *status.
constexpr int CHB = 64;
__global__ void __launch_bounds__(256) k_chol_diag(double* __restrict__ A, int lda, int k0, int kb,
                                                   int* __restrict__ status) {
  __shared__ double a[CHB][CHB + 1];
  __shared__ int bad;
  __shared__ double gmax;
  const int tid = threadIdx.x;
  double* blk = A + (long long)k0 * lda + k0;
  if (tid == 0) {
    bad = 0;
    // largest diagonal of the original Gram (k_gram_prep): the scale of a rounding-level pivot
    gmax = __longlong_as_double(*reinterpret_cast<const long long*>(status + 2));
  }
  for (int e = tid; e < kb * kb; e += blockDim.x) {
    const int c = e / kb, rr = e % kb;      // column-major: element (rr, c) at blk[c*lda + rr]
    a[rr][c] = blk[(long long)c * lda + rr];
  }
  __syncthreads();
  for (int j = 0; j < kb; ++j) {
    if (tid == 0) {
      const double t = a[j][j];
      // a pivot at rounding level of the Gram's scale: the sketch is rank
      // deficient and CholeskyQR would amplify noise -- use the CGS2 path
      if (!(t > 0.0) || !isfinite(t) || t <= 16.0 * 2.220446049250313e-16 * gmax) bad = 1;
      a[j][j] = sqrt(fmax(t, 1e-300));
    }
    __syncthreads();
    const double piv = a[j][j];
    for (int i = j + 1 + tid; i < kb; i += blockDim.x) a[i][j] /= piv;
    __syncthreads();
    const int m = kb - j - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int i = j + 1 + e / m, c = j + 1 + e % m;
      if (c <= i) a[i][c] = fma(-a[i][j], a[c][j], a[i][c]);
    }
    __syncthreads();
  }
  for (int e = tid; e < kb * kb; e += blockDim.x) {
    const int c = e / kb, rr = e % kb;
    blk[(long long)c * lda + rr] = rr >= c ? a[rr][c] : 0.0;
  }
  if (tid == 0 && bad) atomicOr(status, 1);
}

// Rank-robust orthonormalisation (fallback when CholeskyQR breaks down on a
// rank-deficient sketch, where LAPACK's Householder QR still returns an
// orthonormal Q).  Classical Gram-Schmidt with re-orthogonalisation; a column
// that vanishes is replaced by the next standard basis vector orthogonalised
// against the accepted ones (the completion rule of linalg.py:97-117).  Only
// the span reaches the projection, so any orthonormal completion is valid.
__global__ void __launch_bounds__(1024) k_cgs2(double* __restrict__ Y, long long rows, int r,
                                              double* __restrict__ coef, int* __restrict__ status) {
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
        if (basis >= rows) { if (tid == 0) status[0] = 2; return; }
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
  if (tid == 0) status[0] = 0;
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

// Sorted singular values: sorted[jj] = sig[perm[jj]] computed by rank again
// (same ranking rule as k_jacobi's column order).
__global__ void k_sorted_sigma(const double* __restrict__ sig, int n, double* __restrict__ out) {
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
// C[M x N] = alpha * op(A) * op(B) + beta * C, row-major with leading dims.
// op(A) is M x K: A[m*lda + k] (ta=0) or A[k*lda + m] (ta=1).
// op(B) is K x N: B[k*ldb + n] (tb=0) or B[n*ldb + k] (tb=1).
// Plain fp64 GEMMs of the range finder go to cuBLAS (library GEMM; the
// distance contraction of the BICO path stays on our own kernels).  Row-major
// C = op(A) op(B) is column-major C^T = op(B)^T op(A)^T.
static cublasHandle_t blas_handle() {
  thread_local cublasHandle_t h[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!h[dev & 15]) cublasCreate(&h[dev & 15]);
  return h[dev & 15];
}

static int jacobi(cudaStream_t st, double* G, int m, int n, double tol, int max_sweeps, double* sig, double* U,
                  int ldu, int* perm, int* sweeps, int* rot) {
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

static int gemm(cudaStream_t st, int M, int N, int K, double alpha, const double* A, long long lda, int ta,
                const double* B, long long ldb, int tb, double beta, double* C, long long ldc) {
  if (M <= 0 || N <= 0) return PCY_OK;
  cublasHandle_t h = blas_handle();
  if (!h) { pcy_set_error("cublasCreate failed"); return PCY_ECUDA; }
  cublasSetStream(h, st);
  const cublasStatus_t rc = cublasDgemm(h, tb ? CUBLAS_OP_T : CUBLAS_OP_N, ta ? CUBLAS_OP_T : CUBLAS_OP_N,
                                        N, M, K, &alpha, B, (int)ldb, A, (int)lda, &beta, C, (int)ldc);
  if (rc != CUBLAS_STATUS_SUCCESS) { pcy_set_error("cublasDgemm failed (%d)", (int)rc); return PCY_ECUDA; }
  return PCY_OK;
}

// Orthonormalise Y (rows x r, row-major) in place: CholeskyQR2, falling back
// to shifted CholeskyQR3 when the Gram factorisation breaks down.
static int cholqr(cudaStream_t st, double* Y, long long rows, int r, double* Gs, double* Ls, double* Li,
                  double* T, int* status) {
  (void)Ls; (void)Li; (void)T;
  int hs = 0;
  auto pass = [&](double shift, int* ok, int check) -> int {
    int rc;
    if ((rc = gemm(st, r, r, (int)rows, 1.0, Y, r, 1, Y, r, 0, 0.0, Gs, r))) return rc;
    PCY_CUDA(cudaMemsetAsync(status, 0, sizeof(int) * 4, st));   // flag + the Gram's diagonal max (status + 2)
    k_gram_prep<<<(unsigned)std::min((r * r + 255) / 256, 148 * 4), 256, 0, st>>>(Gs, r, shift, check, status);
    pcy_count_launch();
    // blocked right-looking Cholesky, lower, column-major (Gs symmetric)
    cublasHandle_t h = blas_handle();
    cublasSetStream(h, st);
    const double one = 1.0, mone = -1.0;
    for (int k0 = 0; k0 < r; k0 += CHB) {
      const int kb = std::min(CHB, r - k0), rest = r - k0 - kb;
      k_chol_diag<<<1, 256, 0, st>>>(Gs, r, k0, kb, status); pcy_count_launch();
      if (rest > 0) {
        double* A11 = Gs + (long long)k0 * r + k0;
        double* A21 = A11 + kb;
        double* A22 = Gs + (long long)(k0 + kb) * r + k0 + kb;
        if (cublasDtrsm(h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, CUBLAS_DIAG_NON_UNIT, rest, kb,
                        &one, A11, r, A21, r) != CUBLAS_STATUS_SUCCESS) { pcy_set_error("trsm failed"); return PCY_ECUDA; }
        if (cublasDsyrk(h, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, rest, kb, &mone, A21, r, &one, A22, r)
            != CUBLAS_STATUS_SUCCESS) { pcy_set_error("syrk failed"); return PCY_ECUDA; }
      }
    }
    PCY_LAUNCH_CHECK();
    PCY_CUDA(pcy_d2h(&hs, status, sizeof(int), st));
    *ok = hs == 0;
    if (!*ok) return PCY_OK;
    // Y <- Y L^-T  (row-major Y is column-major Y^T: Y^T <- L^-1 Y^T)
    if (cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, r, (int)rows,
                    &one, Gs, r, Y, r) != CUBLAS_STATUS_SUCCESS) { pcy_set_error("trsm failed"); return PCY_ECUDA; }
    return PCY_OK;
  };
  int ok = 0, rc;
  if ((rc = pass(0.0, &ok, 0))) return rc;
  if (ok) {
    if ((rc = pass(0.0, &ok, 1))) return rc;
    if (ok) return PCY_OK;
  }
  // rank-deficient sketch: Gram-Schmidt with completion
  {
    double* coef = nullptr;
    PCY_CUDA(pcy_malloc_async(&coef, sizeof(double) * r, st));
    k_cgs2<<<1, 1024, 0, st>>>(Y, rows, r, coef, status); pcy_count_launch();
    PCY_LAUNCH_CHECK();
    PCY_CUDA(pcy_d2h(&hs, status, sizeof(int), st));
    cudaFreeAsync(coef, st);
    if (hs != 0) { pcy_set_error("orthonormal completion failed"); return PCY_ESTATE; }
  }
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
int pcy_rsvd(const double* A, long long rows, int cols, int ell, int r, int power, const double* omega,
             const double* omega2, double* V, double* sigma_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (r > rows || r > cols || ell > r || ell < 1) { pcy_set_error("rsvd: bad rank"); return PCY_EINVAL; }
  const bool two = rows > 4LL * r;
  double *Q, *Z, *Bm, *Gs, *Ls, *Li, *T, *Wm, *core, *Uj, *sig, *Vfull;
  int *status, *perm, *sweeps, *rot;
  const long long big = std::max<long long>(rows, cols);
  PCY_CUDA(pcy_malloc_async(&Q, sizeof(double) * rows * r, st));
  PCY_CUDA(pcy_malloc_async(&Z, sizeof(double) * cols * r, st));
  PCY_CUDA(pcy_malloc_async(&Bm, sizeof(double) * (long long)r * cols, st));
  PCY_CUDA(pcy_malloc_async(&Gs, sizeof(double) * r * r, st));
  PCY_CUDA(pcy_malloc_async(&Ls, sizeof(double) * r * r, st));
  PCY_CUDA(pcy_malloc_async(&Li, sizeof(double) * r * r, st));
  PCY_CUDA(pcy_malloc_async(&T, sizeof(double) * big * r, st));
  PCY_CUDA(pcy_malloc_async(&Wm, sizeof(double) * cols * r, st));
  PCY_CUDA(pcy_malloc_async(&core, sizeof(double) * r * r, st));
  PCY_CUDA(pcy_malloc_async(&Uj, sizeof(double) * cols * r, st));
  PCY_CUDA(pcy_malloc_async(&sig, sizeof(double) * 2 * r, st));
  PCY_CUDA(pcy_malloc_async(&Vfull, sizeof(double) * cols * r, st));
  PCY_CUDA(pcy_malloc_async(&status, sizeof(int) * 4, st));
  PCY_CUDA(pcy_malloc_async(&perm, sizeof(int) * r, st));
  PCY_CUDA(pcy_malloc_async(&sweeps, sizeof(int), st));
  PCY_CUDA(pcy_malloc_async(&rot, sizeof(int) * 64, st));
  int rc = PCY_OK;
  const bool dbg = getenv("PCY_DEBUG_RSVD") != nullptr;
  cudaEvent_t evs[4];
  if (dbg) for (auto& e : evs) { cudaEventCreate(&e); }
  if (dbg) cudaEventRecord(evs[0], st);
  do {
    // Q = qr(A omega)
    if ((rc = gemm(st, (int)rows, r, cols, 1.0, A, cols, 0, omega, r, 0, 0.0, Q, r))) break;
    if ((rc = cholqr(st, Q, rows, r, Gs, Ls, Li, T, status))) break;
    for (int it = 0; it < power; ++it) {
      // Z = qr(A^T Q); Q = qr(A Z)
      if ((rc = gemm(st, cols, r, (int)rows, 1.0, A, cols, 1, Q, r, 0, 0.0, Z, r))) break;
      if ((rc = cholqr(st, Z, cols, r, Gs, Ls, Li, T, status))) break;
      if ((rc = gemm(st, (int)rows, r, cols, 1.0, A, cols, 0, Z, r, 0, 0.0, Q, r))) break;
      if ((rc = cholqr(st, Q, rows, r, Gs, Ls, Li, T, status))) break;
    }
    if (rc) break;
    if (dbg) cudaEventRecord(evs[1], st);
    // small = Q^T A  (r x cols)
    if ((rc = gemm(st, r, cols, (int)rows, 1.0, Q, r, 1, A, cols, 0, 0.0, Bm, cols))) break;
    const double tol = 2.220446049250313e-16 * (double)std::max(r, 8);
    if (two) {
      // W = qr(small^T omega2) (cols x r); core = small W (r x r)
      if ((rc = gemm(st, cols, r, r, 1.0, Bm, cols, 1, omega2, r, 0, 0.0, Wm, r))) break;
      if ((rc = cholqr(st, Wm, cols, r, Gs, Ls, Li, T, status))) break;
      if ((rc = gemm(st, r, r, cols, 1.0, Bm, cols, 0, Wm, r, 0, 0.0, core, r))) break;
      // Jacobi on core^T: column j of core^T = row j of core (contiguous)
      if (dbg) cudaEventRecord(evs[2], st);
      if ((rc = jacobi(st, core, r, r, tol, 60, sig, Uj, r, perm, sweeps, rot))) break;
      if (dbg) {
        cudaEventRecord(evs[3], st); cudaEventSynchronize(evs[3]);
        float a = 0, b = 0, c = 0; int sw = 0;
        cudaEventElapsedTime(&a, evs[0], evs[1]); cudaEventElapsedTime(&b, evs[1], evs[2]);
        cudaEventElapsedTime(&c, evs[2], evs[3]);
        cudaMemcpy(&sw, sweeps, sizeof(int), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[pcy] rsvd %lldx%d r=%d: range %.2f ms, small+core %.2f ms, jacobi %.2f ms (%d sweeps)\n",
                rows, cols, r, a, b, c, sw);
      }
      // Uj (r x r row-major) columns = right singular vectors of core: V = W Uj
      if ((rc = gemm(st, cols, r, r, 1.0, Wm, r, 0, Uj, r, 0, 0.0, Vfull, r))) break;
    } else {
      // Jacobi on small^T: column j of small^T = row j of small (contiguous)
      if ((rc = jacobi(st, Bm, cols, r, tol, 60, sig, Vfull, r, perm, sweeps, rot))) break;
    }
    k_sorted_sigma<<<1, 256, 0, st>>>(sig, r, sig + r); pcy_count_launch();
    // keep the first ell columns
    PCY_CUDA(cudaMemcpy2DAsync(V, sizeof(double) * ell, Vfull, sizeof(double) * r, sizeof(double) * ell, cols,
                               cudaMemcpyDeviceToDevice, st));
    k_fix_signs<<<(ell + 7) / 8, 256, 0, st>>>(V, cols, ell, ell); pcy_count_launch();
    PCY_LAUNCH_CHECK();
    std::vector<double> hs(r);
    PCY_CUDA(pcy_d2h(hs.data(), sig + r, sizeof(double) * r, st));
    for (int j = 0; j < ell; ++j) sigma_host[j] = hs[j];
    if (ell > 0 && sigma_host[0] > 0.0)
      for (int j = 0; j < ell; ++j) if (sigma_host[j] < 1e-12 * sigma_host[0]) sigma_host[j] = 0.0;
  } while (0);
  cudaFreeAsync(Q, st); cudaFreeAsync(Z, st); cudaFreeAsync(Bm, st); cudaFreeAsync(Gs, st);
  cudaFreeAsync(Ls, st); cudaFreeAsync(Li, st); cudaFreeAsync(T, st); cudaFreeAsync(Wm, st);
  cudaFreeAsync(core, st); cudaFreeAsync(Uj, st); cudaFreeAsync(sig, st); cudaFreeAsync(Vfull, st);
  cudaFreeAsync(status, st); cudaFreeAsync(perm, st); cudaFreeAsync(sweeps, st);
  cudaFreeAsync(rot, st);
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
