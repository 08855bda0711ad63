// Dense fp64 GEMM on the fp64 tensor pipe (DMMA) for the projection path
// (linalg.py:186-201 range finder, :221 projection; replaces cuBLAS DGEMM).
//
//   C[m][n] = alpha * sum_k opA(m, k) * opB(k, n) + beta * C[m][n]
//
// Row-major operands with leading dimensions; opA(m, k) = A[m*lda + k]
// (ta = 0) or A[k*lda + m] (ta = 1); opB(k, n) = B[k*ldb + n] (tb = 0) or
// B[n*ldb + k] (tb = 1).  The range finder's products are tall and skinny
// (K up to the piece's row count with M x N a few tiles), so K is split into
// S slices whose partial tiles land in scratch and are summed in slice order
// (deterministic, no atomics).  64 x 64 x 16 tiles, 4 warps of 32 x 32
// m8n8k4 DMMA fragments, operand tiles global -> shared with cp.async (8-byte
// copies along whichever operand axis is contiguous, double-buffered).
// `skip` (device, nullable): the launch does nothing when *skip != 0 (lets a
// device-side status pick between two code paths without a host round trip).
#include <algorithm>
#include "common.cuh"

namespace {

constexpr int GBM = 64, GBN = 64, GBK = 16;

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" :: "r"(sa), "l"(src), "r"(ok ? 8 : 0));
}

// A tile (64 x 16 of opA) and B tile (16 x 64 of opB) into shared memory.
template <int TA, int TB>
__device__ __forceinline__ void load_tiles(double (*As)[GBK + 4], double (*Bs)[GBN + 4], const double* __restrict__ A,
                                           long long lda, const double* __restrict__ B, long long ldb, int M, int N,
                                           int K, int m0, int n0, int k0, int tid) {
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int e = tid + r * 128;
    int mm, kk;
    if (TA == 0) { mm = e >> 4; kk = e & 15; } else { mm = e & 63; kk = e >> 6; }
    const int m = m0 + mm, k = k0 + kk;
    const bool ok = m < M && k < K;
    const double* src = TA == 0 ? A + (long long)m * lda + k : A + (long long)k * lda + m;
    cp_async8(&As[mm][kk], ok ? src : A, ok);
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int e = tid + r * 128;
    int nn, kk;
    if (TB == 0) { nn = e & 63; kk = e >> 6; } else { nn = e >> 4; kk = e & 15; }
    const int n = n0 + nn, k = k0 + kk;
    const bool ok = n < N && k < K;
    const double* src = TB == 0 ? B + (long long)k * ldb + n : B + (long long)n * ldb + k;
    cp_async8(&Bs[kk][nn], ok ? src : B, ok);
  }
  asm volatile("cp.async.commit_group;\n" ::);
}

// grid (ceil(N/64), ceil(M/64), S); slice z covers k in [z*kslice, min(K, (z+1)*kslice))
// and writes its partial tile to P + z*pstride (ldp = N) -- or, with S == 1 and
// P == nullptr, the final alpha/beta result to C directly.
template <int TA, int TB>
__global__ void __launch_bounds__(128, 4) k_gemm(int M, int N, int K, const double* __restrict__ A, long long lda,
                                                 const double* __restrict__ B, long long ldb, int kslice,
                                                 double* __restrict__ P, long long pstride, double alpha, double beta,
                                                 double* __restrict__ C, long long ldc, const int* __restrict__ skip) {
  if (skip && *skip) return;
  __shared__ __align__(16) double As[2][GBM][GBK + 4];
  __shared__ __align__(16) double Bs[2][GBK][GBN + 4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int m0 = blockIdx.y * GBM, n0 = blockIdx.x * GBN;
  const int kb = blockIdx.z * kslice;
  const int ke = min(K, kb + kslice);
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }
  int buf = 0;
  if (kb < ke) {
    load_tiles<TA, TB>(As[0], Bs[0], A, lda, B, ldb, M, N, ke, m0, n0, kb, tid);
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  __syncthreads();
  for (int k0 = kb; k0 < ke; k0 += GBK) {
    const bool more = k0 + GBK < ke;
    if (more) load_tiles<TA, TB>(As[buf ^ 1], Bs[buf ^ 1], A, lda, B, ldb, M, N, ke, m0, n0, k0 + GBK, tid);
#pragma unroll
    for (int ks = 0; ks < GBK; ks += 4) {
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
      asm volatile("cp.async.wait_group 0;\n" ::);
      __syncthreads();
      buf ^= 1;
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int m = m0 + wm + i * 8 + g, n = n0 + wn + j * 8 + 2 * t4 + h;
        if (m < M && n < N) {
          if (P) P[blockIdx.z * pstride + (long long)m * N + n] = acc[i][j][h];
          else {
            const long long o = (long long)m * ldc + n;
            C[o] = beta == 0.0 ? alpha * acc[i][j][h] : alpha * acc[i][j][h] + beta * C[o];
          }
        }
      }
}

// C = alpha * (sum of the S partials, slice order) + beta * C
__global__ void k_gemm_reduce(int M, int N, int S, const double* __restrict__ P, long long pstride, double alpha,
                              double beta, double* __restrict__ C, long long ldc, const int* __restrict__ skip) {
  if (skip && *skip) return;
  const long long total = (long long)M * N;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    double v = P[e];
    for (int z = 1; z < S; ++z) v += P[z * pstride + e];
    const long long o = (e / N) * ldc + (e % N);
    C[o] = beta == 0.0 ? alpha * v : alpha * v + beta * C[o];
  }
}

}  // namespace

// Host entry used by linalg.cu (stream-ordered; scratch from the pool).
int pcy_gemm_f64(cudaStream_t st, int M, int N, int K, double alpha, const double* A, long long lda, int ta,
                 const double* B, long long ldb, int tb, double beta, double* C, long long ldc, const int* skip) {
  if (M <= 0 || N <= 0) return PCY_OK;
  const long long tiles = (long long)((M + GBM - 1) / GBM) * ((N + GBN - 1) / GBN);
  // slices: enough CTAs for the 148 SMs (about 4 resident each), >= 256 k per slice
  int S = 1;
  if (K > 512) {
    const long long want = (4LL * 148 + tiles - 1) / tiles;
    const long long maxs = std::max<long long>(1, K / 256);
    S = (int)std::min<long long>(std::min<long long>(want, maxs), 64);
    if (S < 1) S = 1;
  }
  int kslice = (K + S - 1) / S;
  kslice = (kslice + GBK - 1) / GBK * GBK;
  if (kslice < GBK) kslice = GBK;
  S = K > 0 ? (K + kslice - 1) / kslice : 1;
  double* P = nullptr;
  const long long pstride = (long long)M * N;
  if (S > 1) PCY_CUDA(pcy_malloc_async(&P, sizeof(double) * pstride * S, st));
  dim3 grid((unsigned)((N + GBN - 1) / GBN), (unsigned)((M + GBM - 1) / GBM), (unsigned)S);
  if (K <= 0) kslice = 0;
  switch ((ta ? 1 : 0) * 2 + (tb ? 1 : 0)) {
    case 0: k_gemm<0, 0><<<grid, 128, 0, st>>>(M, N, K, A, lda, B, ldb, kslice, P, pstride, alpha, beta, C, ldc, skip); break;
    case 1: k_gemm<0, 1><<<grid, 128, 0, st>>>(M, N, K, A, lda, B, ldb, kslice, P, pstride, alpha, beta, C, ldc, skip); break;
    case 2: k_gemm<1, 0><<<grid, 128, 0, st>>>(M, N, K, A, lda, B, ldb, kslice, P, pstride, alpha, beta, C, ldc, skip); break;
    default: k_gemm<1, 1><<<grid, 128, 0, st>>>(M, N, K, A, lda, B, ldb, kslice, P, pstride, alpha, beta, C, ldc, skip); break;
  }
  pcy_count_launch();
  if (S > 1) {
    const long long blocks = std::min<long long>((pstride + 255) / 256, 148LL * 8);
    k_gemm_reduce<<<(unsigned)blocks, 256, 0, st>>>(M, N, S, P, pstride, alpha, beta, C, ldc, skip);
    pcy_count_launch();
    cudaFreeAsync(P, st);
  }
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}
