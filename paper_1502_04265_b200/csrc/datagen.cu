// Paper instance families on the device (datagen.py:104-135).
//
// The reference draws every coordinate from numpy's Philox4x64-10 bit
// generator (datagen.py:15-16) as Generator.random(): u = (x >> 11) * 2^-53,
// one 64-bit output x per double.  numpy hands out the outputs of counter
// block c = 1, 2, ... in order (the counter is bumped before each block), so
// output t of a stream is word t % 4 of Philox(ctr = t / 4 + 1, key) -- any
// coordinate can be generated independently from its global draw index.
// Host code (datagen.py) keeps the draw bookkeeping (SWN's per-cluster
// permutations stay on numpy's own generator); these kernels write the
// (n x dim) float64 rows.
#include "common.cuh"

namespace {

__device__ __forceinline__ void mulhilo64(unsigned long long a, unsigned long long b, unsigned long long& hi,
                                          unsigned long long& lo) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

// Random123 / numpy philox4x64_R(10, ctr, key)
__device__ __forceinline__ void philox4x64_10(unsigned long long c0, unsigned long long c1, unsigned long long k0,
                                              unsigned long long k1, unsigned long long out[4]) {
  unsigned long long x0 = c0, x1 = c1, x2 = 0ull, x3 = 0ull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) { k0 += 0x9E3779B97F4A7C15ull; k1 += 0xBB67AE8584CAA73Bull; }
    unsigned long long hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ull, x0, hi0, lo0);
    mulhilo64(0xCA5A826395121157ull, x2, hi1, lo1);
    const unsigned long long y0 = hi1 ^ x1 ^ k0, y1 = lo1, y2 = hi0 ^ x3 ^ k1, y3 = lo0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

// Generator.random() value of global draw t (numpy's stream with key (k0, k1))
__device__ __forceinline__ double philox_uniform(unsigned long long t, unsigned long long k0, unsigned long long k1) {
  const unsigned long long blk = (t >> 2) + 1ull;   // numpy bumps the counter before each block
  unsigned long long w[4];
  philox4x64_10(blk, 0ull, k0, k1, w);
  const unsigned long long x = w[t & 3ull];
  return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

// (2u - 1) * scale as numpy evaluates it: 2.0 * u (exact), - 1.0, * scale
__device__ __forceinline__ double centred(double u, double scale) {
  return __dmul_rn(__dadd_rn(__dmul_rn(2.0, u), -1.0), scale);
}

// structured_with_noise (datagen.py:104-112): cluster c's points j = 0..ppc-1
// draw random(dim) (noise) then random(act) (signal at the permuted active
// dims).  base[c] = the global draw index of the cluster's first point;
// inv[c * dim + e] = position of dim e in the cluster's active list, or -1.
__global__ void k_gen_swn(double* __restrict__ out, long long ld, int clusters, long long ppc, int dim, int act,
                          unsigned long long k0, unsigned long long k1, const unsigned long long* __restrict__ base,
                          const int* __restrict__ inv, double noise, double spread) {
  const long long rows = (long long)clusters * ppc;
  const long long total = rows * dim;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / dim;
    const int col = (int)(e - r * dim);
    const int c = (int)(r / ppc);
    const long long j = r - (long long)c * ppc;
    const int a = inv[(long long)c * dim + col];
    const unsigned long long t = base[c] + (unsigned long long)j * (unsigned long long)(dim + act) +
                                 (unsigned long long)(a >= 0 ? dim + a : col);
    out[r * ld + col] = centred(philox_uniform(t, k0, k1), a >= 0 ? spread : noise);
  }
}

// random_cube (datagen.py:131-135): point i = random(n) from draw start + i*n
__global__ void k_gen_cube(double* __restrict__ out, long long ld, long long n, long long cols,
                           unsigned long long k0, unsigned long long k1, unsigned long long start, double spread) {
  const long long total = n * cols;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / cols, col = e - r * cols;
    out[r * ld + col] = centred(philox_uniform(start + (unsigned long long)e, k0, k1), spread);
  }
}

// lower_bound (datagen.py:115-128): point j of vertex i has spread at dim i
// and noise at dim k + i*(n/k) + j, zeros elsewhere.
__global__ void k_gen_lb(double* __restrict__ out, long long ld, int k, long long n, double spread, double noise) {
  const long long dim = k + n;
  const long long per = n / k;
  const long long total = n * dim;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / dim, col = e - r * dim;
    const long long v = r / per, j = r - v * per;
    double x = 0.0;
    if (col == v) x = spread;
    else if (col == k + v * per + j) x = noise;
    out[r * ld + col] = x;
  }
}

unsigned grid_for(long long total) {
  long long b = (total + 255) / 256;
  if (b > 148LL * 64) b = 148LL * 64;
  return (unsigned)(b > 0 ? b : 1);
}

}  // namespace

extern "C" {

int pcy_gen_swn(double* out, long long ld, int clusters, long long ppc, int dim, int act, unsigned long long key_lo,
                unsigned long long key_hi, const unsigned long long* base, const int* inv, double noise, double spread,
                void* stream) {
  if (clusters < 0 || ppc < 0 || dim < 1 || act < 1 || act > dim || ld < dim) {
    pcy_set_error("gen_swn: bad sizes"); return PCY_EINVAL;
  }
  const long long total = (long long)clusters * ppc * dim;
  if (total == 0) return PCY_OK;
  k_gen_swn<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(out, ld, clusters, ppc, dim, act, key_lo, key_hi, base,
                                                             inv, noise, spread);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

int pcy_gen_cube(double* out, long long ld, long long n, long long cols, unsigned long long key_lo,
                 unsigned long long key_hi, unsigned long long start, double spread, void* stream) {
  if (n < 0 || cols < 1 || ld < cols) { pcy_set_error("gen_cube: bad sizes"); return PCY_EINVAL; }
  if (n == 0) return PCY_OK;
  k_gen_cube<<<grid_for(n * cols), 256, 0, (cudaStream_t)stream>>>(out, ld, n, cols, key_lo, key_hi, start, spread);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

int pcy_gen_lower_bound(double* out, long long ld, int k, long long n, double spread, double noise, void* stream) {
  if (k < 2 || n < k || n % k != 0 || ld < k + n) { pcy_set_error("gen_lower_bound: bad sizes"); return PCY_EINVAL; }
  k_gen_lb<<<grid_for(n * (k + n)), 256, 0, (cudaStream_t)stream>>>(out, ld, k, n, spread, noise);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

}  // extern "C"
