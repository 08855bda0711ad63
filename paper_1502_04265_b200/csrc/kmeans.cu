// Weighted k-means++ seeding and weighted Lloyd on the coreset (sm_100a).
//
// Reference: /root/reference/pkg/src/piecy/evaluation.py
//   sq_distances  :39-46   d2 = ((-2 P C^T) + |p|^2) + |c|^2, clamped at 0
//   _draw         :49-53   first index with cumsum > u * total, clamped
//   kmeanspp_seed :56-82   D^2 rule with diff-form distances
//   lloyd_iterate :85-139  assignment, empty-cluster repair, cost, update
//   weighted_cost :142-149
// All sums are fixed-order (no float atomics) so repeated runs are bitwise
// deterministic, like the reference.
#include <cmath>
#include <vector>
#include "common.cuh"

namespace {

constexpr int KM_THREADS = 1024;

__device__ __forceinline__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = lane < nw ? red[lane] : 0.0;
  t = warp_sum(t);
  return t;
}

// Exclusive scan of per-thread values in thread order (Hillis-Steele over
// warp totals).  Returns the exclusive prefix; *total gets the block total.
__device__ __forceinline__ double block_exscan(double v, double* red, double* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(PCY_FULL, inc, o);
    if (lane >= o) inc += t;
  }
  __syncthreads();
  if (lane == 31) red[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    double wv = lane < nw ? red[lane] : 0.0, winc = wv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t = __shfl_up_sync(PCY_FULL, winc, o);
      if (lane >= o) winc += t;
    }
    if (lane < nw) red[32 + lane] = winc - wv;   // exclusive warp offsets
    if (lane == nw - 1) red[64] = winc;
  }
  __syncthreads();
  *total = red[64];
  return red[32 + wid] + (inc - v);
}

// _draw: first index i with cumsum(mass)[i] > u * cumsum[-1], clamped to n-1.
// Each thread owns a contiguous chunk; the running sum inside a chunk is
// sequential, chunk offsets come from the block scan.
__device__ int block_draw(const double* __restrict__ mass, long long n, double u, double* red, int* ired) {
  const long long per = (n + blockDim.x - 1) / blockDim.x;
  const long long a = (long long)threadIdx.x * per, b = min(n, a + per);
  double loc = 0.0;
  for (long long i = a; i < b; ++i) loc += mass[i];
  double total;
  const double pre = block_exscan(loc, red, &total);
  const double target = rmul(u, total);
  int cand = 0x7fffffff;
  double c = pre;
  for (long long i = a; i < b; ++i) {
    c += mass[i];
    if (c > target) { cand = (int)i; break; }
  }
  // min over threads
  int v = cand;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = min(v, __shfl_xor_sync(PCY_FULL, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) ired[threadIdx.x >> 5] = v;
  __syncthreads();
  int r = 0x7fffffff;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r = min(r, ired[k]);
  __syncthreads();
  return r == 0x7fffffff ? (int)(n - 1) : r;
}

// One CTA per repetition.  best[] and mass[] are per-rep scratch (n each).
__global__ void __launch_bounds__(KM_THREADS) k_seed(const double* __restrict__ P, const double* __restrict__ w,
                                                    long long n, int d, int k, const double* __restrict__ U,
                                                    double* __restrict__ centers, double* __restrict__ best_all,
                                                    double* __restrict__ mass_all, int* __restrict__ picks) {
  extern __shared__ double cv[];
  __shared__ double red[72];
  __shared__ int ired[32];
  __shared__ int s_pos;
  const int rep = blockIdx.x;
  const double* u = U + (long long)rep * k;
  double* best = best_all + (long long)rep * n;
  double* mass = mass_all + (long long)rep * n;
  double* C = centers + (long long)rep * k * d;
  for (int j = 0; j < k; ++j) {
    int idx;
    if (j == 0) {
      idx = block_draw(w, n, u[0], red, ired);
    } else {
      // mass = w * best; draw from it unless it sums to zero (:77-78).  The
      // sum of nonnegative terms is positive iff some term is positive.
      if (threadIdx.x == 0) s_pos = 0;
      __syncthreads();
      for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const double mv = rmul(w[i], best[i]);
        mass[i] = mv;
        if (mv > 0.0) s_pos = 1;
      }
      __syncthreads();
      idx = block_draw(s_pos ? mass : w, n, u[j], red, ired);
    }
    if (threadIdx.x == 0) picks[rep * k + j] = idx;
    for (int e = threadIdx.x; e < d; e += blockDim.x) {
      const double v = P[(long long)idx * d + e];
      cv[e] = v;
      C[(long long)j * d + e] = v;
    }
    __syncthreads();
    // best = min(best, |p - c|^2), diff form (:74-75, :80-81)
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
      const double* p = P + i * d;
      double acc = 0.0;
      for (int e = 0; e < d; ++e) { const double df = rsub(p[e], cv[e]); acc = fma(df, df, acc); }
      best[i] = j == 0 ? acc : fmin(best[i], acc);
    }
    __syncthreads();
  }
}

// Row squared norms (einsum 'ij,ij->i').
__global__ void k_rownorm(const double* __restrict__ X, long long n, int d, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  const double v = warp_dot(X + i * d, X + i * d, d, lane);
  if (lane == 0) out[i] = v;
}

// Assignment: warp per (point, rep).  d2 = max(((-2 g) + pn) + cn, 0),
// first minimum wins (:41-46, :105-107).
__global__ void k_assign(const double* __restrict__ P, const double* __restrict__ pn, long long n, int d, int k,
                         const double* __restrict__ centers, const double* __restrict__ cn,
                         const int* __restrict__ active, int* __restrict__ assign, double* __restrict__ bestd) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int rep = blockIdx.y;
  if (i >= n || (active && !active[rep])) return;
  const double* p = P + i * d;
  const double* C = centers + (long long)rep * k * d;
  const double* cnr = cn + (long long)rep * k;
  double bv = INFINITY; int bj = 0;
  for (int j = 0; j < k; ++j) {
    const double g = warp_dot(p, C + (long long)j * d, d, lane);
    double v = radd(radd(rmul(-2.0, g), pn[i]), cnr[j]);
    if (v < 0.0) v = 0.0;
    if (v < bv) { bv = v; bj = j; }
  }
  if (lane == 0) {
    assign[(long long)rep * n + i] = bj;
    bestd[(long long)rep * n + i] = bv;
  }
}

// Per rep: occupancy, empty-cluster repair (:109-124), cost = w . best (:126).
// One CTA per rep.  repair=0 computes only the cost (weighted_cost).
__global__ void __launch_bounds__(KM_THREADS) k_finish(const double* __restrict__ P, const double* __restrict__ w,
                                                      long long n, int d, int k, double* __restrict__ centers,
                                                      const int* __restrict__ active, int* __restrict__ assign_all,
                                                      double* __restrict__ best_all, int* __restrict__ counts_all,
                                                      double* __restrict__ cost_out, int repair) {
  __shared__ double red[72];
  __shared__ int s_empty, s_far;
  __shared__ double s_gmax;
  const int rep = blockIdx.x;
  if (active && !active[rep]) return;
  int* assign = assign_all + (long long)rep * n;
  double* best = best_all + (long long)rep * n;
  int* counts = counts_all + (long long)rep * k;
  double* C = centers + (long long)rep * k * d;
  if (repair) {
    for (;;) {
      for (int j = threadIdx.x; j < k; j += blockDim.x) counts[j] = 0;
      __syncthreads();
      for (long long i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&counts[assign[i]], 1);
      __syncthreads();
      if (threadIdx.x == 0) {
        s_empty = -1;
        for (int j = 0; j < k; ++j) if (counts[j] == 0) { s_empty = j; break; }
      }
      __syncthreads();
      if (s_empty < 0) break;
      // far = first argmax of w * best
      double gv = -INFINITY; long long gi = 0x7fffffffffffLL;
      for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const double g = rmul(w[i], best[i]);
        if (g > gv) { gv = g; gi = i; }
      }
      // block argmax with lowest index on ties
      for (int o = 16; o >= 1; o >>= 1) {
        const double og = __shfl_xor_sync(PCY_FULL, gv, o);
        const long long oi = __shfl_xor_sync(PCY_FULL, gi, o);
        if (og > gv || (og == gv && oi < gi)) { gv = og; gi = oi; }
      }
      __shared__ double wg[32]; __shared__ long long wi[32];
      if ((threadIdx.x & 31) == 0) { wg[threadIdx.x >> 5] = gv; wi[threadIdx.x >> 5] = gi; }
      __syncthreads();
      if (threadIdx.x == 0) {
        double bg = -INFINITY; long long bi = 0x7fffffffffffLL;
        for (int t = 0; t < (int)(blockDim.x >> 5); ++t)
          if (wg[t] > bg || (wg[t] == bg && wi[t] < bi)) { bg = wg[t]; bi = wi[t]; }
        s_gmax = bg; s_far = (int)bi;
      }
      __syncthreads();
      if (!(s_gmax > 0.0)) break;   // every point sits on a center
      const int emp = s_empty, far = s_far;
      for (int e = threadIdx.x; e < d; e += blockDim.x) C[(long long)emp * d + e] = P[(long long)far * d + e];
      __syncthreads();
      for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const double* p = P + i * d;
        const double* c = C + (long long)emp * d;
        double acc = 0.0;
        for (int e = 0; e < d; ++e) { const double df = rsub(p[e], c[e]); acc = fma(df, df, acc); }
        if (acc < best[i]) { assign[i] = emp; best[i] = acc; }
      }
      __syncthreads();
      if (threadIdx.x == 0) { assign[far] = emp; best[far] = 0.0; }
      __syncthreads();
    }
  }
  // cost = w . best in fixed order (chunked then tree)
  const long long per = (n + blockDim.x - 1) / blockDim.x;
  const long long a = (long long)threadIdx.x * per, b = min(n, a + per);
  double loc = 0.0;
  for (long long i = a; i < b; ++i) loc = fma(w[i], best[i], loc);
  const double tot = block_sum(loc, red);
  if (threadIdx.x == 0) cost_out[rep] = tot;
}

// Centroid update (:133-138): one CTA per (center, rep); points of the center
// summed in index order.  Empty centers keep their previous value.
__global__ void k_update(const double* __restrict__ P, const double* __restrict__ w, long long n, int d, int k,
                         const int* __restrict__ active, const int* __restrict__ assign_all,
                         double* __restrict__ centers) {
  extern __shared__ double acc_s[];
  __shared__ double s_mass;
  __shared__ int s_list[256];
  __shared__ int s_cnt;
  const int j = blockIdx.x, rep = blockIdx.y;
  if (active && !active[rep]) return;
  const int* assign = assign_all + (long long)rep * n;
  double* C = centers + (long long)rep * k * d;
  for (int e = threadIdx.x; e < d; e += blockDim.x) acc_s[e] = 0.0;
  if (threadIdx.x == 0) s_mass = 0.0;
  __syncthreads();
  for (long long base = 0; base < n; base += blockDim.x) {
    // compact this window's members (in index order) into s_list
    const long long i = base + threadIdx.x;
    const bool mine = i < n && assign[i] == j;
    const unsigned bal = __ballot_sync(PCY_FULL, mine);
    __shared__ int wcnt[32];
    if ((threadIdx.x & 31) == 0) wcnt[threadIdx.x >> 5] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { const int c = wcnt[q]; wcnt[q] = t; t += c; }
      s_cnt = t;
    }
    __syncthreads();
    if (mine) s_list[wcnt[threadIdx.x >> 5] + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = (int)(i - base);
    __syncthreads();
    const int cnt = s_cnt;
    for (int e = threadIdx.x; e < d; e += blockDim.x) {
      double a = acc_s[e];
      for (int t = 0; t < cnt; ++t) {
        const long long ii = base + s_list[t];
        a = fma(w[ii], P[ii * d + e], a);
      }
      acc_s[e] = a;
    }
    if (threadIdx.x == 0) { double mm = s_mass; for (int t = 0; t < cnt; ++t) mm += w[base + s_list[t]]; s_mass = mm; }
    __syncthreads();
  }
  if (s_mass > 0.0)
    for (int e = threadIdx.x; e < d; e += blockDim.x) C[(long long)j * d + e] = rdiv(acc_s[e], s_mass);
}

}  // namespace

// ==================================================================== C-ABI
extern "C" {

// Weighted D^2 seeding for `reps` independent repetitions.  U (device) holds
// reps x k uniforms, the exact rng.random() stream of each repetition.
int pcy_kmeanspp(const double* P, const double* w, long long n, int d, int k, int reps, const double* U,
                 double* centers, long long* picks_out, void* stream) {
  if (n < 1 || k < 1 || d < 1 || reps < 1) { pcy_set_error("kmeanspp: bad sizes"); return PCY_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  double *best = nullptr, *mass = nullptr; int* picks = nullptr;
  PCY_CUDA(pcy_malloc_async(&best, sizeof(double) * n * reps, st));
  PCY_CUDA(pcy_malloc_async(&mass, sizeof(double) * n * reps, st));
  PCY_CUDA(pcy_malloc_async(&picks, sizeof(int) * k * reps, st));
  const size_t sm = sizeof(double) * d;
  if (sm > 48 * 1024) PCY_CUDA(cudaFuncSetAttribute(k_seed, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  k_seed<<<reps, KM_THREADS, sm, st>>>(P, w, n, d, k, U, centers, best, mass, picks); pcy_count_launch();
  PCY_LAUNCH_CHECK();
  if (picks_out) {
    std::vector<int> h((size_t)k * reps);
    PCY_CUDA(pcy_d2h(h.data(), picks, sizeof(int) * k * reps, st));
    for (size_t i = 0; i < h.size(); ++i) picks_out[i] = h[i];
  }
  PCY_CUDA(cudaFreeAsync(best, st));
  PCY_CUDA(cudaFreeAsync(mass, st));
  PCY_CUDA(cudaFreeAsync(picks, st));
  return PCY_OK;
}

// Weighted Lloyd for `reps` center sets (centers updated in place).
// cost_log (host, reps x max_iters, nullable) receives the per-iteration
// costs; iters_out (host, reps) the number of logged costs.
int pcy_lloyd(const double* P, const double* w, long long n, int d, int k, int reps, double* centers,
              int max_iters, double tol, double* cost_log, int* iters_out, void* stream) {
  if (n < 1 || k < 1 || d < 1 || reps < 1) { pcy_set_error("lloyd: bad sizes"); return PCY_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  double *pn = nullptr, *cn = nullptr, *best = nullptr, *cost = nullptr; int *assign = nullptr, *counts = nullptr, *active = nullptr;
  PCY_CUDA(pcy_malloc_async(&pn, sizeof(double) * n, st));
  PCY_CUDA(pcy_malloc_async(&cn, sizeof(double) * k * reps, st));
  PCY_CUDA(pcy_malloc_async(&best, sizeof(double) * n * reps, st));
  PCY_CUDA(pcy_malloc_async(&assign, sizeof(int) * n * reps, st));
  PCY_CUDA(pcy_malloc_async(&counts, sizeof(int) * k * reps, st));
  PCY_CUDA(pcy_malloc_async(&cost, sizeof(double) * reps, st));
  PCY_CUDA(pcy_malloc_async(&active, sizeof(int) * reps, st));
  std::vector<int> act(reps, 1);
  std::vector<double> prev(reps, INFINITY), hc(reps);
  for (int r = 0; r < reps; ++r) iters_out[r] = 0;
  k_rownorm<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(P, n, d, pn); pcy_count_launch();
  const size_t usm = sizeof(double) * d;
  if (usm > 48 * 1024) PCY_CUDA(cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm));
  for (int it = 0; it < max_iters; ++it) {
    int nact = 0;
    for (int r = 0; r < reps; ++r) nact += act[r];
    if (!nact) break;
    PCY_CUDA(cudaMemcpyAsync(active, act.data(), sizeof(int) * reps, cudaMemcpyHostToDevice, st));
    k_rownorm<<<(unsigned)((k * reps + 7) / 8), 256, 0, st>>>(centers, (long long)k * reps, d, cn); pcy_count_launch();
    k_assign<<<dim3((unsigned)((n + 7) / 8), reps), 256, 0, st>>>(P, pn, n, d, k, centers, cn, active, assign, best); pcy_count_launch();
    k_finish<<<reps, KM_THREADS, 0, st>>>(P, w, n, d, k, centers, active, assign, best, counts, cost, 1); pcy_count_launch();
    PCY_LAUNCH_CHECK();
    PCY_CUDA(pcy_d2h(hc.data(), cost, sizeof(double) * reps, st));
    bool any_update = false;
    for (int r = 0; r < reps; ++r) {
      if (!act[r]) continue;
      if (cost_log) cost_log[(size_t)r * max_iters + it] = hc[r];
      iters_out[r] = it + 1;
      if (std::isfinite(prev[r]) && prev[r] - hc[r] <= tol * prev[r]) { act[r] = 0; continue; }
      prev[r] = hc[r];
      any_update = true;
    }
    if (!any_update) break;
    PCY_CUDA(cudaMemcpyAsync(active, act.data(), sizeof(int) * reps, cudaMemcpyHostToDevice, st));
    k_update<<<dim3(k, reps), 256, usm, st>>>(P, w, n, d, k, active, assign, centers); pcy_count_launch();
    PCY_LAUNCH_CHECK();
  }
  PCY_CUDA(pcy_spin_sync(st));
  cudaFreeAsync(pn, st); cudaFreeAsync(cn, st); cudaFreeAsync(best, st); cudaFreeAsync(assign, st);
  cudaFreeAsync(counts, st); cudaFreeAsync(cost, st); cudaFreeAsync(active, st);
  return PCY_OK;
}

// weighted_cost for `reps` center sets: costs (host, reps).
int pcy_weighted_cost(const double* P, const double* w, long long n, int d, int k, int reps,
                      const double* centers, double* costs, void* stream) {
  if (n < 1) { for (int r = 0; r < reps; ++r) costs[r] = 0.0; return PCY_OK; }
  cudaStream_t st = (cudaStream_t)stream;
  double *pn = nullptr, *cn = nullptr, *best = nullptr, *cost = nullptr; int *assign = nullptr;
  PCY_CUDA(pcy_malloc_async(&pn, sizeof(double) * n, st));
  PCY_CUDA(pcy_malloc_async(&cn, sizeof(double) * k * reps, st));
  PCY_CUDA(pcy_malloc_async(&best, sizeof(double) * n * reps, st));
  PCY_CUDA(pcy_malloc_async(&assign, sizeof(int) * n * reps, st));
  PCY_CUDA(pcy_malloc_async(&cost, sizeof(double) * reps, st));
  k_rownorm<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(P, n, d, pn); pcy_count_launch();
  k_rownorm<<<(unsigned)((k * reps + 7) / 8), 256, 0, st>>>(centers, (long long)k * reps, d, cn); pcy_count_launch();
  k_assign<<<dim3((unsigned)((n + 7) / 8), reps), 256, 0, st>>>(P, pn, n, d, k, centers, cn, nullptr, assign, best); pcy_count_launch();
  k_finish<<<reps, KM_THREADS, 0, st>>>(P, w, n, d, k, (double*)centers, nullptr, assign, best, nullptr, cost, 0); pcy_count_launch();
  PCY_LAUNCH_CHECK();
  PCY_CUDA(pcy_d2h(costs, cost, sizeof(double) * reps, st));
  cudaFreeAsync(pn, st); cudaFreeAsync(cn, st); cudaFreeAsync(best, st); cudaFreeAsync(assign, st);
  cudaFreeAsync(cost, st);
  return PCY_OK;
}

}  // extern "C"
