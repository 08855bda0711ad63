// Distance contraction on the fp64 tensor pipe (sm_100a DMMA).
//
// The BICO decisions compare parts |r|^2 - 2 r.x in fp64 (coreset.py:172-176),
// so the contraction runs on DMMA (mma.sync m8n8k4 f64, exact fp64 products
// and sums) -- tcgen05 has no fp64 kind.  Two forms:
//   k_dist_tile<0>  C[m][n] = A[ia(m)] . B[ib(n)]          (block Gram for K3)
//   k_dist_tile<1>  per-(row, 64-column tile) argmin of rn[ib(n)] - 2 A.B,
//                   first column on ties; k_argmin_reduce folds the tiles.
// Rows of A and B may be gathered through index arrays (tree nodes live at
// arbitrary slots), so no operand is ever copied into a packed buffer.
#include <cstdlib>
#include "common.cuh"

namespace {

constexpr int DBM = 64, DBN = 64, DBK = 16;

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" :: "r"(sa), "l"(src), "r"(ok ? 8 : 0));
}

// CPA: operand tiles go global -> shared with cp.async (no register staging:
// fewer registers, five CTAs per SM instead of four), double-buffered as in
// the register-staged form; the k4 steps and the epilogue are unchanged, so
// the results are bitwise the same.
template <int MODE, bool CPA = false>
__global__ void __launch_bounds__(128, CPA ? 5 : 1) k_dist_tile(int M, int N, int K,
                                                  const double* __restrict__ A, const int* __restrict__ aidx, long long lda,
                                                  const double* __restrict__ B, const int* __restrict__ bidx, long long ldb,
                                                  const double* __restrict__ rn,
                                                  double* __restrict__ C, long long ldc,
                                                  double* __restrict__ ppart, int* __restrict__ ppos, int ntiles,
                                                  const int* __restrict__ n_dev = nullptr,
                                                  const double* __restrict__ rv = nullptr, int lower = 0,
                                                  int kslice = 0, long long cstride = 0,
                                                  const int* __restrict__ zactive = nullptr, long long zB = 0,
                                                  long long zrn = 0) {
  __shared__ double As[2][DBM][DBK + 4];
  __shared__ double Bs[2][DBK][DBN + 4];
  __shared__ long long arow[DBM], brow[DBN];
  __shared__ double s_rn[DBN];
  __shared__ double red_p[DBM][2];
  __shared__ int red_c[DBM][2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int m0 = blockIdx.y * DBM, n0 = blockIdx.x * DBN;
  if (lower && n0 > m0) return;   // tile strictly above the diagonal (DBM == DBN)
  if (kslice > 0) {   // split K: slice blockIdx.z of the contraction into partial z of C
    const int kb = blockIdx.z * kslice;
    A += kb; B += kb; K = min(kslice, K - kb); C += blockIdx.z * cstride;
  } else if (gridDim.z > 1 || zactive) {   // batch z (Lloyd: one centre set per repetition)
    const int z = blockIdx.z;
    if (zactive && !zactive[z]) return;
    B += z * zB; rn += z * zrn;
    ppart += (long long)z * M * ntiles; ppos += (long long)z * M * ntiles;
  }
  if (n_dev) { N = min(N, *n_dev); if (n0 >= N) return; }
  if (tid < DBM) {
    const int m = m0 + tid;
    arow[tid] = m < M ? (long long)(aidx ? aidx[m] : m) * lda : -1;
  } else {
    const int nn = tid - DBM, n = n0 + nn;
    brow[nn] = n < N ? (long long)(bidx ? bidx[n] : n) * ldb : -1;
    if (MODE != 0) s_rn[nn] = n < N ? rn[bidx ? bidx[n] : n] : INFINITY;
  }
  __syncthreads();
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }

  // register-staged double buffering of the 64x16 operand tiles
  double ra[8], rb[8];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int e = tid + r * 128;
      const int mm = e >> 4, kk = e & 15;
      const long long ar = arow[mm], br = brow[mm];
      ra[r] = (ar >= 0 && k0 + kk < K) ? A[ar + k0 + kk] : 0.0;
      rb[r] = (br >= 0 && k0 + kk < K) ? B[br + k0 + kk] : 0.0;
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int e = tid + r * 128;
      const int mm = e >> 4, kk = e & 15;
      As[buf][mm][kk] = ra[r];
      Bs[buf][kk][mm] = rb[r];
    }
  };
  auto issue = [&](int k0, int b) {   // CPA: the tile k0 straight into buffer b
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const int e = tid + r * 128;
      const int mm = e >> 4, kk = e & 15;
      const long long ar = arow[mm], br = brow[mm];
      const bool ka = k0 + kk < K;
      cp_async8(&As[b][mm][kk], ar >= 0 && ka ? A + ar + k0 + kk : A, ar >= 0 && ka);
      cp_async8(&Bs[b][kk][mm], br >= 0 && ka ? B + br + k0 + kk : B, br >= 0 && ka);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  int buf = 0;
  if constexpr (CPA) {
    issue(0, 0);
    asm volatile("cp.async.wait_group 0;\n" ::);
  } else {
    fetch(0);
    stash(0);
  }
  __syncthreads();
  for (int k0 = 0; k0 < K; k0 += DBK) {
    const bool more = k0 + DBK < K;
    if constexpr (CPA) { if (more) issue(k0 + DBK, buf ^ 1); }
    else if (more) fetch(k0 + DBK);
#pragma unroll
    for (int ks = 0; ks < DBK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][wm + i * 8 + g][ks + t4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][ks + t4][wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (more) {
      if constexpr (CPA) asm volatile("cp.async.wait_group 0;\n" ::);
      else stash(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

  if (MODE == 0 || MODE == 2) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int m = m0 + wm + i * 8 + g, cl = wn + j * 8 + 2 * t4 + h, n = n0 + cl;
          if (m < M && n < N)
            C[(long long)m * ldc + n] = MODE == 0 ? acc[i][j][h] : radd(s_rn[cl], rmul(acc[i][j][h], -2.0));
        }
    return;
  }
  // MODE 1: argmin of rn[n] - 2 g over this tile's 64 columns per row;
  // MODE 3: argmin of max(((-2 g) + rv[m]) + rn[n], 0) (evaluation.py:41-46);
  // lowest column on ties
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    double bp = INFINITY; int bc = 0x7fffffff;
    double rvm = 0.0;
    if (MODE == 3) { const int mm = m0 + wm + i * 8 + g; rvm = mm < M ? rv[mm] : 0.0; }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cl = wn + j * 8 + 2 * t4 + h;
        if (n0 + cl < N) {
          double p;
          if (MODE == 3) { p = radd(radd(rmul(-2.0, acc[i][j][h]), rvm), s_rn[cl]); if (p < 0.0) p = 0.0; }
          else p = radd(s_rn[cl], rmul(acc[i][j][h], -2.0));
          if (p < bp || (p == bp && cl < bc)) { bp = p; bc = cl; }
        }
      }
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const double op = __shfl_xor_sync(PCY_FULL, bp, o);
      const int oc = __shfl_xor_sync(PCY_FULL, bc, o);
      if (op < bp || (op == bp && oc < bc)) { bp = op; bc = oc; }
    }
    if (t4 == 0) { red_p[wm + i * 8 + g][warp & 1] = bp; red_c[wm + i * 8 + g][warp & 1] = bc; }
  }
  __syncthreads();
  if (tid < DBM) {
    const int m = m0 + tid;
    double p0 = red_p[tid][0], p1 = red_p[tid][1];
    int c0 = red_c[tid][0], c1 = red_c[tid][1];
    if (p1 < p0 || (p1 == p0 && c1 < c0)) { p0 = p1; c0 = c1; }
    if (m < M) {
      ppart[(long long)m * ntiles + blockIdx.x] = p0;
      ppos[(long long)m * ntiles + blockIdx.x] = c0 == 0x7fffffff ? 0x7fffffff : n0 + c0;
    }
  }
}

// per row: argmin over tiles (positions increase with the tile index)
// Sum of the split-K partials in slice order (fixed order: deterministic), on
// and below the diagonal.
__global__ void k_gram_sum(const double* __restrict__ part, int S, long long pstride, int M, double* __restrict__ C,
                           long long ldc) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (long long)M * M) return;
  const int m = (int)(e / M), n = (int)(e % M);
  if (n > m) return;
  const long long o = (long long)m * ldc + n;
  double v = part[o];
  for (int z = 1; z < S; ++z) v += part[z * pstride + o];
  C[o] = v;
}

__global__ void k_argmin_reduce(int M, int ntiles, const double* __restrict__ ppart, const int* __restrict__ ppos,
                                int* __restrict__ out_pos, double* __restrict__ out_part,
                                const int* __restrict__ zactive = nullptr) {
  const int lane = threadIdx.x & 31;
  const int m = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (m >= M) return;
  if (gridDim.y > 1 || zactive) {   // batch y (one repetition per y)
    const int z = blockIdx.y;
    if (zactive && !zactive[z]) return;
    ppart += (long long)z * M * ntiles; ppos += (long long)z * M * ntiles;
    out_pos += (long long)z * M; out_part += (long long)z * M;
  }
  double bp = INFINITY; int bc = 0x7fffffff;
  for (int t = lane; t < ntiles; t += 32) {
    const double p = ppart[(long long)m * ntiles + t];
    const int c = ppos[(long long)m * ntiles + t];
    if (p < bp || (p == bp && c < bc)) { bp = p; bc = c; }
  }
  warp_argmin(bp, bc);
  if (lane == 0) { out_pos[m] = bc; out_part[m] = bp; }
}

}  // namespace

int pcy_launch_gram(const double* A, const int* aidx, long long lda, int M, const double* B, const int* bidx,
                    long long ldb, int N, int K, double* C, long long ldc, cudaStream_t st) {
  if (M <= 0 || N <= 0) return PCY_OK;
  dim3 grid((unsigned)((N + DBN - 1) / DBN), (unsigned)((M + DBM - 1) / DBM));
  // only the tiles on or below the diagonal: the engine's batch Grams are
  // symmetric and read at (later item, earlier item) only
  k_dist_tile<0, true><<<grid, 128, 0, st>>>(M, N, K, A, aidx, lda, B, bidx, ldb, nullptr, C, ldc, nullptr, nullptr, 0,
                                       nullptr, nullptr, A == B && aidx == bidx && M == N ? 1 : 0);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

// Self-Gram of a block (lower triangle) with K split over S slices: a tile's
// K loop is latency-bound at large d (one stage of loads ahead), so S slices
// run S times more tiles at once; the partials (scratch, S x M x ldc) are
// summed in slice order.
int pcy_launch_gram_split(const double* A, const int* aidx, long long lda, int M, int K, double* C, long long ldc,
                          double* scratch, int S, cudaStream_t st) {
  if (M <= 0) return PCY_OK;
  int kslice = (K + S - 1) / S;
  kslice = (kslice + DBK - 1) / DBK * DBK;
  S = (K + kslice - 1) / kslice;
  if (S <= 1 || !scratch) return pcy_launch_gram(A, aidx, lda, M, A, aidx, lda, M, K, C, ldc, st);
  const long long pstride = (long long)M * ldc;
  dim3 grid((unsigned)((M + DBN - 1) / DBN), (unsigned)((M + DBM - 1) / DBM), (unsigned)S);
  k_dist_tile<0, true><<<grid, 128, 0, st>>>(M, M, K, A, aidx, lda, A, aidx, lda, nullptr, scratch, ldc, nullptr, nullptr, 0,
                                       nullptr, nullptr, 1, kslice, pstride);
  pcy_count_launch();
  k_gram_sum<<<(unsigned)(((long long)M * M + 255) / 256), 256, 0, st>>>(scratch, S, pstride, M, C, ldc);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

// Parts matrix: C[m][n] = rn[ib(n)] - 2 A[ia(m)].B[ib(n)] (the full-set form
// of K1: every block row against every live reference slot; n_dev, when set,
// caps N with a device-side count).
int pcy_launch_parts(const double* A, const int* aidx, long long lda, int M, const double* B, const int* bidx,
                     long long ldb, const double* rn, int N, const int* n_dev, int K, double* C, long long ldc,
                     cudaStream_t st) {
  if (M <= 0 || N <= 0) return PCY_OK;
  dim3 grid((unsigned)((N + DBN - 1) / DBN), (unsigned)((M + DBM - 1) / DBM));
  k_dist_tile<2, true><<<grid, 128, 0, st>>>(M, N, K, A, aidx, lda, B, bidx, ldb, rn, C, ldc, nullptr, nullptr, 0, n_dev);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

// Nearest reference per row: out_pos[m] = column (position) of the minimum
// part rn[ib(n)] - 2 A[ia(m)].B[ib(n)], lowest position on ties.  Scratch:
// ppart / ppos of M x ceil(N/64).
int pcy_launch_nearest(const double* A, const int* aidx, long long lda, int M, const double* B, const int* bidx,
                       long long ldb, const double* rn, int N, int K, double* ppart, int* ppos, int* out_pos,
                       double* out_part, cudaStream_t st) {
  if (M <= 0) return PCY_OK;
  const int ntiles = (N + DBN - 1) / DBN;
  dim3 grid((unsigned)ntiles, (unsigned)((M + DBM - 1) / DBM));
  k_dist_tile<1, true><<<grid, 128, 0, st>>>(M, N, K, A, aidx, lda, B, bidx, ldb, rn, nullptr, 0, ppart, ppos, ntiles);
  pcy_count_launch();
  k_argmin_reduce<<<(unsigned)((M + 7) / 8), 256, 0, st>>>(M, ntiles, ppart, ppos, out_pos, out_part);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

// Lloyd assignment (evaluation.py:104-107): assign[m] = first argmin over
// centres of max(((-2 P C^T) + pn) + cn, 0), best[m] = that value.  Scratch
// ppart / ppos of n x ceil(k/64).
int pcy_launch_assign_d2(const double* P, long long ldp, int n, const double* pn, const double* C, long long ldc,
                         const double* cn, int k, int d, double* ppart, int* ppos, int* assign, double* best,
                         cudaStream_t st) {
  if (n <= 0 || k <= 0) return PCY_OK;
  const int ntiles = (k + DBN - 1) / DBN;
  dim3 grid((unsigned)ntiles, (unsigned)((n + DBM - 1) / DBM));
  k_dist_tile<3, true><<<grid, 128, 0, st>>>(n, k, d, P, nullptr, ldp, C, nullptr, ldc, cn, nullptr, 0, ppart, ppos, ntiles,
                                      nullptr, pn);
  pcy_count_launch();
  k_argmin_reduce<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(n, ntiles, ppart, ppos, assign, best);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

// Batched Lloyd assignment: repetition z uses centres C + z*k*ldc and norms
// cn + z*k, writes assign/best + z*n; repetitions with active[z] == 0 skip.
// Scratch ppart / ppos of reps x n x ceil(k/64).
int pcy_launch_assign_d2_batch(const double* P, long long ldp, int n, const double* pn, const double* C, long long ldc,
                               const double* cn, int k, int d, int reps, const int* active, double* ppart, int* ppos,
                               int* assign, double* best, cudaStream_t st) {
  if (n <= 0 || k <= 0 || reps <= 0) return PCY_OK;
  const int ntiles = (k + DBN - 1) / DBN;
  dim3 grid((unsigned)ntiles, (unsigned)((n + DBM - 1) / DBM), (unsigned)reps);
  k_dist_tile<3, true><<<grid, 128, 0, st>>>(n, k, d, P, nullptr, ldp, C, nullptr, ldc, cn, nullptr, 0, ppart, ppos, ntiles,
                                      nullptr, pn, 0, 0, 0, active, (long long)k * ldc, (long long)k);
  pcy_count_launch();
  k_argmin_reduce<<<dim3((unsigned)((n + 7) / 8), (unsigned)reps), 256, 0, st>>>(n, ntiles, ppart, ppos, assign, best,
                                                                              active);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

extern "C" int pcy_nearest_refs(const double* X, long long ldx, int M, const double* R, const int* ridx,
                                long long ldr, const double* rn, int N, int K, int* out_pos, double* out_part,
                                void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int ntiles = (N + DBN - 1) / DBN;
  double* pp = nullptr; int* pc = nullptr;
  PCY_CUDA(pcy_malloc_async(&pp, sizeof(double) * (size_t)M * (ntiles > 0 ? ntiles : 1), st));
  PCY_CUDA(pcy_malloc_async(&pc, sizeof(int) * (size_t)M * (ntiles > 0 ? ntiles : 1), st));
  int rc = pcy_launch_nearest(X, nullptr, ldx, M, R, ridx, ldr, rn, N, K, pp, pc, out_pos, out_part, st);
  cudaFreeAsync(pp, st);
  cudaFreeAsync(pc, st);
  return rc;
}

extern "C" int pcy_gram(const double* A, long long lda, int M, const double* B, long long ldb, int N, int K,
                        double* C, long long ldc, void* stream) {
  return pcy_launch_gram(A, nullptr, lda, M, B, nullptr, ldb, N, K, C, ldc, (cudaStream_t)stream);
}
