// Shared device helpers for the piecy B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define PCY_FULL 0xffffffffu

// ---------------------------------------------------------------------------
// Error plumbing (host side).  Every C-ABI entry point returns 0 or a negative
// code and leaves a message in a thread-local buffer (pcy_last_error()).
// ---------------------------------------------------------------------------
#include "../../include/piecy_b200.h"   // C-ABI declarations and PCY_E* codes

void pcy_set_error(const char* fmt, ...);
void pcy_count_launch();
// Wait for all work queued on `st` by spinning on an event (no blocking-sync
// wake-up latency on the host thread).
cudaError_t pcy_spin_sync(cudaStream_t st);
// Device -> host copy of a small result through a thread-local pinned
// staging buffer, completed with pcy_spin_sync.
cudaError_t pcy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t st);
int pcy_launch_assign_d2_batch(const double* P, long long ldp, int n, const double* pn, const double* C, long long ldc,
                               const double* cn, int k, int d, int reps, const int* active, double* ppart, int* ppos,
                               int* assign, double* best, cudaStream_t st);
int pcy_launch_assign_d2(const double* P, long long ldp, int n, const double* pn, const double* C, long long ldc,
                         const double* cn, int k, int d, double* ppart, int* ppos, int* assign, double* best,
                         cudaStream_t st);
// split-TF32 distance contraction on tcgen05 (tc_dots.cu)
double pcy_tc_error_tau(int Kp);
int pcy_tc_pad(int d);
int pcy_tc_center(const double* src, const int* idx, long long ld, int d, double* center, cudaStream_t st);
// reference slots alive and not yet split for their creation index
// (done_idx) get the next live column (ncol ticket, col_of / col_slot) and
// their split in that row of hi / lo; nrm2 stays slot-indexed
int pcy_tc_split_slots(const double* src, long long ld, int d, long long nslots, const int* alive,
                       const long long* cidx, long long* done_idx, const double* center, float* hi, float* lo,
                       double* nrm2, int* col_of, int* col_slot, int* ncol, cudaStream_t st);
// rows_dev (nullable): device row count capping `rows` / `N`
int pcy_tc_split(const double* src, const int* idx, long long ld, int d, long long rows, const int* rows_dev,
                 const double* center, float* hi, float* lo, double* nrm2, cudaStream_t st);
int pcy_tc_dots(const float* Ahi, const float* Alo, long long a_cap, int M, const float* Bhi, const float* Blo,
                long long b_cap, int N, const int* n_dev, int Kp, float* out, long long ldo, cudaStream_t st);
// cudaMallocAsync from the device's default pool, whose memory is kept
// resident (release threshold raised once per device): per-call scratch of
// the projection and the engine then never re-maps physical memory.
cudaError_t pcy_malloc_async_raw(void** p, size_t bytes, cudaStream_t st);
template <class T>
inline cudaError_t pcy_malloc_async(T** p, size_t bytes, cudaStream_t st) {
  return pcy_malloc_async_raw((void**)p, bytes, st);
}
// DMMA distance contraction (distance.cu).  pcy_launch_gram of a block with
// itself (A == B) computes only the lower triangle (column <= row).
int pcy_launch_gram(const double* A, const int* aidx, long long lda, int M, const double* B, const int* bidx,
                    long long ldb, int N, int K, double* C, long long ldc, cudaStream_t st);
// the same self-Gram (lower triangle) with K split over S slices (scratch:
// S x M x ldc doubles), partials summed in slice order
int pcy_launch_gram_split(const double* A, const int* aidx, long long lda, int M, int K, double* C, long long ldc,
                          double* scratch, int S, cudaStream_t st);
int pcy_launch_parts(const double* A, const int* aidx, long long lda, int M, const double* B, const int* bidx,
                     long long ldb, const double* rn, int N, const int* n_dev, int K, double* C, long long ldc,
                     cudaStream_t st);
int pcy_launch_nearest(const double* A, const int* aidx, long long lda, int M, const double* B, const int* bidx,
                       long long ldb, const double* rn, int N, int K, double* ppart, int* ppos, int* out_pos,
                       double* out_part, cudaStream_t st);

// Per-kernel event timing (enabled by pcy_prof_enable).
enum { PCY_PROF_RESOLVE = 0, PCY_PROF_CHAIN = 1, PCY_PROF_REATTACH = 2, PCY_PROF_SEED = 3,
       PCY_PROF_LLOYD = 4, PCY_PROF_GEMM = 5, PCY_PROF_SLOTS = 8 };
struct PcyProfSlot { double ms = 0.0; long long count = 0; long long units = 0; };
bool pcy_prof_enabled();
void pcy_prof_add(int slot, double ms, long long units);

#define PCY_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      pcy_set_error("%s:%d: %s: %s", __FILE__, __LINE__, #call,              \
                    cudaGetErrorString(_e));                                  \
      return PCY_ECUDA;                                                       \
    }                                                                         \
  } while (0)

#define PCY_LAUNCH_CHECK()                                                    \
  do {                                                                        \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess) {                                                  \
      pcy_set_error("%s:%d: launch: %s", __FILE__, __LINE__,                  \
                    cudaGetErrorString(_e));                                  \
      return PCY_ECUDA;                                                       \
    }                                                                         \
  } while (0)

// ---------------------------------------------------------------------------
// Explicitly rounded fp64 arithmetic.  The reference evaluates every scalar
// decision expression as separately rounded IEEE operations (Python floats /
// numpy, no FMA); these wrappers keep nvcc from contracting them.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double rmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double radd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double rdiv(double a, double b) { return __ddiv_rn(a, b); }

// ---------------------------------------------------------------------------
// Warp reductions.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(PCY_FULL, v, o);
  return v;
}

// min of (value, position); ties resolve to the lower position.
__device__ __forceinline__ void warp_argmin(double& v, int& pos) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    double ov = __shfl_xor_sync(PCY_FULL, v, o);
    int op = __shfl_xor_sync(PCY_FULL, pos, o);
    if (ov < v || (ov == v && op < pos)) { v = ov; pos = op; }
  }
}

// Lane-strided fp64 dot of two length-d vectors, all lanes get the total.
// Lane-strided fp64 dot: lane l sums a[e] b[e] for e = l, l+32, ... in that
// order, then the warp tree.  Loads are issued 16 rows ahead (the FMA order
// is unchanged, so every caller sees bit-identical values at any d).
__device__ __forceinline__ double warp_dot(const double* __restrict__ a,
                                           const double* __restrict__ b, int d, int lane) {
  double acc = 0.0;
  int e = lane;
  for (; e + 15 * 32 < d; e += 16 * 32) {
    double av[16], bv[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) { av[q] = a[e + 32 * q]; bv[q] = b[e + 32 * q]; }
#pragma unroll
    for (int q = 0; q < 16; ++q) acc = fma(av[q], bv[q], acc);
  }
  for (; e < d; e += 32) acc = fma(a[e], b[e], acc);
  return warp_sum(acc);
}

// CTA-cooperative fp64 dot for one item per CTA (WPI warps): warp w sums the
// lane-strided elements e = 32 w + l + 32 WPI k in order, then the warp tree,
// then red[0] + red[1] + ... in warp order.  Deterministic; every warp of the
// CTA must call it (two __syncthreads).
template <int WPI>
__device__ __forceinline__ double cta_dot(const double* __restrict__ a, const double* __restrict__ b, int d,
                                          int lane, int warp, double* red) {
  double acc = 0.0;
  int e = warp * 32 + lane;
  constexpr int S = 32 * WPI;
  for (; e + 7 * S < d; e += 8 * S) {
    double av[8], bv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) { av[q] = a[e + S * q]; bv[q] = b[e + S * q]; }
#pragma unroll
    for (int q = 0; q < 8; ++q) acc = fma(av[q], bv[q], acc);
  }
  for (; e < d; e += S) acc = fma(a[e], b[e], acc);
  acc = warp_sum(acc);
  __syncthreads();
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  double t = red[0];
#pragma unroll
  for (int w = 1; w < WPI; ++w) t += red[w];
  return t;
}

// Transpose-reduce: lane l holds 32 partial sums acc[0..31] (one per member);
// afterwards acc[0] on lane l is the full sum for member l.  31 shuffles.
__device__ __forceinline__ double warp_transpose_reduce(double (&acc)[32], int lane) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int k = 0; k < s; ++k) {
      double send = upper ? acc[k] : acc[k + s];
      double keep = upper ? acc[k + s] : acc[k];
      acc[k] = keep + __shfl_xor_sync(PCY_FULL, send, s);
    }
  }
  return acc[0];
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27; z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

static inline int64_t pcy_round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
