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
#include <algorithm>
#include <vector>
#include "common.cuh"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

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

// Cooperative k-means++ (all repetitions in one persistent launch).  CTA c
// of the G CTAs owns the rows [c n / G, (c+1) n / G) (equal ranges: every SM
// streams the same number of rows, no tail wave).  The cumulative mass of
// point i is  sum(range totals before its range) + running sum within its
// range up to i, every sum in a fixed order, so the draw is deterministic.
// Per centre:
//   draw (every CTA, one warp per repetition, identical results): _draw
//     (:49-53) from the range totals, falling back to the weights when the
//     mass is all zero (:77-78); CTA 0 records the picks and centre rows;
//   distance pass (all CTAs, two rows per warp): the diff-form distance of
//     each point to every repetition's newest centre (:74-75, :80-81), best =
//     min(best, dist), mass = w * best, the range totals; each point row is
//     read from HBM once for all repetitions (the HBM-bound pass);
// and one grid barrier.
constexpr int KS_THREADS = 512, KS_RMAX = 8;

__device__ __forceinline__ long long ks_lo(long long n, int c, int G) { return n * c / G; }

// Fixed-order total of vals[p0, p1): 32-element blocks, each an inclusive
// warp scan, added in block order -- the association warp_draw's in-range
// search uses, so the draw's running sum reaches exactly prefix + total at
// the end of a range.
__device__ __forceinline__ double warp_scan32(double v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(PCY_FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
// Loads are issued ahead of the dependent scans (KS_CMAX blocks of 32 values,
// KS_PMAX range totals per lane): one L2 round trip per draw level instead of
// one per block.  The arithmetic and its order are unchanged.
constexpr int KS_CMAX = 8, KS_PMAX = 16;
__device__ double warp_range_total(const double* vals, long long p0, long long p1, int lane) {
  double tb = 0.0;
  double raw[KS_CMAX];
#pragma unroll
  for (int q = 0; q < KS_CMAX; ++q) {
    const long long i = p0 + 32 * q + lane;
    raw[q] = i < p1 ? __ldcg(vals + i) : 0.0;
  }
#pragma unroll
  for (int q = 0; q < KS_CMAX; ++q) {
    if (p0 + 32 * q >= p1) break;
    const double v = warp_scan32(raw[q], lane);
    tb = tb + __shfl_sync(PCY_FULL, v, 31);
  }
  for (long long b0 = p0 + 32 * KS_CMAX; b0 < p1; b0 += 32) {
    const long long i = b0 + lane;
    const double v = warp_scan32(i < p1 ? __ldcg(vals + i) : 0.0, lane);
    tb = tb + __shfl_sync(PCY_FULL, v, 31);
  }
  return tb;
}

// Warp form of _draw (evaluation.py:49-53) over the G range totals `part`
// and the point values `vals`: the first i whose cumulative sum exceeds
// u * total, clamped to n - 1.  *total_out receives the grand total (lane-
// contiguous runs of range totals, then the warp scan).
__device__ long long warp_draw(const double* part, int G, const double* __restrict__ vals, long long n, double u,
                               int lane, double* total_out) {
  const int per = (G + 31) / 32;
  const int a = lane * per, b = min(G, a + per);
  const bool regs = per <= KS_PMAX;
  double pv[KS_PMAX];
#pragma unroll
  for (int t = 0; t < KS_PMAX; ++t) pv[t] = (regs && a + t < b) ? __ldcg(part + a + t) : 0.0;
  double loc = 0.0;
  if (regs) {
#pragma unroll
    for (int t = 0; t < KS_PMAX; ++t) if (a + t < b) loc += pv[t];
  } else {
    for (int c = a; c < b; ++c) loc += __ldcg(part + c);
  }
  const double inc = warp_scan32(loc, lane);
  const double total = __shfl_sync(PCY_FULL, inc, 31);
  *total_out = total;
  const double target = rmul(u, total);
  // the range holding the target: first c (lane order = range order)
  int cfound = 0x7fffffff;
  double cum = inc - loc, cstart = 0.0;
  if (regs) {
#pragma unroll
    for (int t = 0; t < KS_PMAX; ++t) {
      if (a + t < b && cfound == 0x7fffffff) {
        const double pc = pv[t];
        if (cum + pc > target) { cfound = a + t; cstart = cum; }
        else cum += pc;
      }
    }
  } else {
    for (int c = a; c < b; ++c) {
      const double pc = __ldcg(part + c);
      if (cum + pc > target) { cfound = c; cstart = cum; break; }
      cum += pc;
    }
  }
  const unsigned hit = __ballot_sync(PCY_FULL, cfound != 0x7fffffff);
  if (!hit) return n - 1;
  const int src = __ffs(hit) - 1;
  const int cs = __shfl_sync(PCY_FULL, cfound, src);
  cum = __shfl_sync(PCY_FULL, cstart, src);
  // in-range search, in the association of warp_range_total
  const long long p0 = ks_lo(n, cs, G), p1 = ks_lo(n, cs + 1, G);
  double tb = 0.0;
  double raw[KS_CMAX];
#pragma unroll
  for (int q = 0; q < KS_CMAX; ++q) {
    const long long i = p0 + 32 * q + lane;
    raw[q] = i < p1 ? __ldcg(vals + i) : 0.0;
  }
#pragma unroll
  for (int q = 0; q < KS_CMAX; ++q) {
    const long long b0 = p0 + 32 * q;
    if (b0 >= p1) break;
    const long long i = b0 + lane;
    const double v = warp_scan32(raw[q], lane);
    const unsigned over = __ballot_sync(PCY_FULL, i < p1 && cum + (tb + v) > target);
    if (over) return b0 + __ffs(over) - 1;
    tb = tb + __shfl_sync(PCY_FULL, v, 31);
  }
  for (long long b0 = p0 + 32 * KS_CMAX; b0 < p1; b0 += 32) {
    const long long i = b0 + lane;
    const double v = warp_scan32(i < p1 ? __ldcg(vals + i) : 0.0, lane);
    const unsigned over = __ballot_sync(PCY_FULL, i < p1 && cum + (tb + v) > target);
    if (over) return b0 + __ffs(over) - 1;
    tb = tb + __shfl_sync(PCY_FULL, v, 31);
  }
  return p1 - 1 < n - 1 ? p1 - 1 : n - 1;   // rounding guard: the range end
}

// Diff-form squared distances (evaluation.py:74-75, :80-81) of two point
// rows pa, pb to the rn staged centres cs (rn x d), lane partial sums in
// acc[row][centre].  Even d: 128-bit loads, 8 pairs in flight per row and
// lane; odd d: 8 elements per row and lane.
__device__ __forceinline__ void seed_rows2(const double* __restrict__ pa, const double* __restrict__ pb,
                                           const double* cs, int d, int rn, int lane, double (&acc)[2][KS_RMAX]) {
#pragma unroll
  for (int q = 0; q < KS_RMAX; ++q) { acc[0][q] = 0.0; acc[1][q] = 0.0; }
  if ((d & 1) == 0) {
    const double2* a2 = reinterpret_cast<const double2*>(pa);
    const double2* b2 = reinterpret_cast<const double2*>(pb);
    const int d2 = d >> 1;
    int e2 = lane;
    for (; e2 + 7 * 32 < d2; e2 += 8 * 32) {
      double2 av[8], bv[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) { av[t] = a2[e2 + 32 * t]; bv[t] = b2[e2 + 32 * t]; }
#pragma unroll
      for (int q = 0; q < KS_RMAX; ++q)
        if (q < rn) {
          const double2* cq = reinterpret_cast<const double2*>(cs + (long long)q * d) + e2;
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const double2 cv = cq[32 * t];
            double dx = rsub(av[t].x, cv.x), dy = rsub(av[t].y, cv.y);
            acc[0][q] = fma(dx, dx, acc[0][q]);
            acc[0][q] = fma(dy, dy, acc[0][q]);
            dx = rsub(bv[t].x, cv.x); dy = rsub(bv[t].y, cv.y);
            acc[1][q] = fma(dx, dx, acc[1][q]);
            acc[1][q] = fma(dy, dy, acc[1][q]);
          }
        }
    }
    for (int t = e2; t < d2; t += 32) {
      const double2 av = a2[t], bv = b2[t];
#pragma unroll
      for (int q = 0; q < KS_RMAX; ++q)
        if (q < rn) {
          const double2 cv = reinterpret_cast<const double2*>(cs + (long long)q * d)[t];
          double dx = rsub(av.x, cv.x), dy = rsub(av.y, cv.y);
          acc[0][q] = fma(dx, dx, acc[0][q]);
          acc[0][q] = fma(dy, dy, acc[0][q]);
          dx = rsub(bv.x, cv.x); dy = rsub(bv.y, cv.y);
          acc[1][q] = fma(dx, dx, acc[1][q]);
          acc[1][q] = fma(dy, dy, acc[1][q]);
        }
    }
    return;
  }
  int e = lane;
  for (; e + 7 * 32 < d; e += 8 * 32) {
    double av[8], bv[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) { av[t] = pa[e + 32 * t]; bv[t] = pb[e + 32 * t]; }
#pragma unroll
    for (int q = 0; q < KS_RMAX; ++q)
      if (q < rn) {
        const double* cq = cs + (long long)q * d + e;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const double c = cq[32 * t];
          const double da = rsub(av[t], c), db = rsub(bv[t], c);
          acc[0][q] = fma(da, da, acc[0][q]);
          acc[1][q] = fma(db, db, acc[1][q]);
        }
      }
  }
  for (; e < d; e += 32) {
    const double av = pa[e], bv = pb[e];
#pragma unroll
    for (int q = 0; q < KS_RMAX; ++q)
      if (q < rn) {
        const double c = cs[(long long)q * d + e];
        const double da = rsub(av, c), db = rsub(bv, c);
        acc[0][q] = fma(da, da, acc[0][q]);
        acc[1][q] = fma(db, db, acc[1][q]);
      }
  }
}

__global__ void __launch_bounds__(KS_THREADS) k_seed_coop(const double* __restrict__ P, const double* __restrict__ w,
                                                         long long n, int d, int k, int reps,
                                                         const double* __restrict__ U, double* __restrict__ centers,
                                                         double* __restrict__ best_all, double* __restrict__ mass_all,
                                                         double* __restrict__ part_all, double* __restrict__ wpart,
                                                         int* __restrict__ picks, int rg) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double ks_smem[];
  double* cs = ks_smem;                          // rg x d newest centres
  __shared__ long long s_idx[64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = KS_THREADS / 32;
  const int G = gridDim.x, c = blockIdx.x;
  const long long p0 = ks_lo(n, c, G), p1 = ks_lo(n, c + 1, G);
  // weight range totals (the first draw / fallback), fixed order
  if (warp == 0) {
    const double t = warp_range_total(w, p0, p1, lane);
    if (lane == 0) wpart[c] = t;
  }
  grid.sync();
  for (int j = 0; j < k; ++j) {
    // masses and range totals alternate between two buffers: centre j reads
    // those of centre j - 1 while faster CTAs already write centre j's
    const long long mstride = (long long)reps * n, pstride = (long long)reps * G;
    const double* mass_r = mass_all + ((j - 1) & 1) * mstride;
    const double* part_r = part_all + ((j - 1) & 1) * pstride;
    double* mass_w = mass_all + (j & 1) * mstride;
    double* part_w = part_all + (j & 1) * pstride;
    // draw centre j of every repetition, redundantly in every CTA
    for (int r = warp; r < reps; r += nwarp) {
      const double u = U[(long long)r * k + j];
      double tot = 0.0;
      long long idx;
      if (j == 0) {
        idx = warp_draw(wpart, G, w, n, u, lane, &tot);
      } else {
        idx = warp_draw(part_r + (long long)r * G, G, mass_r + (long long)r * n, n, u, lane, &tot);
        if (!(tot > 0.0)) idx = warp_draw(wpart, G, w, n, u, lane, &tot);
      }
      if (lane == 0) {
        s_idx[r] = idx;
        if (c == 0) picks[r * k + j] = (int)idx;
      }
    }
    __syncthreads();
    for (int r = c; r < reps; r += G) {   // repetition r's centre row: CTA r mod G
      double* C = centers + ((long long)r * k + j) * d;
      for (int e = threadIdx.x; e < d; e += blockDim.x) C[e] = P[s_idx[r] * d + e];
    }
    if (j == k - 1) break;
    // distances to the new centres, mass, range totals
    for (int r0 = 0; r0 < reps; r0 += rg) {
      const int rn = min(rg, reps - r0);
      for (int q = 0; q < rn; ++q)
        for (int e = threadIdx.x; e < d; e += blockDim.x) cs[(long long)q * d + e] = P[s_idx[r0 + q] * d + e];
      __syncthreads();
      // two rows per warp: every centre element read from shared memory
      // serves both rows, and twice the row bytes are in flight
      for (long long i = p0 + 2 * warp; i < p1; i += 2 * nwarp) {
        const long long ib = i + 1 < p1 ? i + 1 : -1;
        double acc[2][KS_RMAX];
        // lane q keeps repetition q's running minimum of both rows: loaded
        // before the distance pass, so the update below waits on nothing
        double bprev[2] = {0.0, 0.0}, wrow[2] = {0.0, 0.0};
        if (lane < rn) {
          const long long rb = (long long)(r0 + lane) * n;
          if (j > 0) { bprev[0] = best_all[rb + i]; if (ib >= 0) bprev[1] = best_all[rb + ib]; }
          wrow[0] = w[i]; if (ib >= 0) wrow[1] = w[ib];
        }
        seed_rows2(P + i * d, P + (ib >= 0 ? ib : i) * d, cs, d, rn, lane, acc);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const long long ii = h == 0 ? i : ib;
          if (ii < 0) break;
          double mine = 0.0;   // lane q: distance to repetition q's newest centre
#pragma unroll
          for (int q = 0; q < KS_RMAX; ++q) {
            if (q >= rn) break;
            const double a = warp_sum(acc[h][q]);
            if (lane == q) mine = a;
          }
          if (lane < rn) {
            const long long rb = (long long)(r0 + lane) * n;
            const double bb = j == 0 ? mine : fmin(bprev[h], mine);
            best_all[rb + ii] = bb;
            mass_w[rb + ii] = rmul(wrow[h], bb);
          }
        }
      }
      __syncthreads();
      // range totals, one warp per repetition (the association of warp_draw)
      for (int q = warp; q < rn; q += nwarp) {
        const double t = warp_range_total(mass_w + (long long)(r0 + q) * n, p0, p1, lane);
        if (lane == 0) part_w[(long long)(r0 + q) * G + c] = t;
      }
      __syncthreads();
    }
    grid.sync();
  }
}

__global__ void k_fill(double* __restrict__ p, long long n, double v) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) p[i] = v;
}

// Per-chunk sums of best (rows [c*chunk, (c+1)*chunk)), one CTA per chunk,
// fixed order (thread-chunked then tree) -- the reference's chunked running
// totals of evaluate_cost_multi (evaluation.py:172-179) group the same rows.
__global__ void __launch_bounds__(256) k_chunk_sums(const double* __restrict__ best, long long n, long long chunk,
                                                   double* __restrict__ out, long long out_stride) {
  __shared__ double red[72];
  const long long a0 = (long long)blockIdx.x * chunk, a1 = min(n, a0 + chunk);
  const long long per = (a1 - a0 + blockDim.x - 1) / blockDim.x;
  const long long a = a0 + (long long)threadIdx.x * per, b = min(a1, a + per);
  double loc = 0.0;
  for (long long i = a; i < b; ++i) loc += best[i];
  const double tot = block_sum(loc, red);
  if (threadIdx.x == 0) out[(long long)blockIdx.x * out_stride] = tot;
}

// Row squared norms (einsum 'ij,ij->i').
__global__ void k_rownorm(const double* __restrict__ X, long long n, int d, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  const double v = warp_dot(X + i * d, X + i * d, d, lane);
  if (lane == 0) out[i] = v;
}

// Empty-cluster repair (:109-124), one round for every repetition that needs
// it.  k_counts_empty (CTA per rep): occupancy counts; the first empty centre
// `emp`; far = first argmax of w * best; when that gain is positive the centre
// becomes P[far] and rep_state = {emp, far}, otherwise (or with no empty
// centre) the repetition's repair is over (emp = -1).
__global__ void __launch_bounds__(KM_THREADS) k_counts_empty(const double* __restrict__ P,
                                                            const double* __restrict__ w, long long n, int d, int k,
                                                            double* __restrict__ centers, const int* __restrict__ active,
                                                            const int* __restrict__ assign_all,
                                                            const double* __restrict__ best_all,
                                                            int* __restrict__ counts_all, int* __restrict__ rep_state) {
  __shared__ int s_empty, s_far;
  __shared__ double s_gmax;
  __shared__ double wg[32];
  __shared__ long long wi[32];
  const int rep = blockIdx.x;
  if (active && !active[rep]) { if (threadIdx.x == 0) rep_state[2 * rep] = -1; return; }
  const int* assign = assign_all + (long long)rep * n;
  const double* best = best_all + (long long)rep * n;
  int* counts = counts_all + (long long)rep * k;
  double* C = centers + (long long)rep * k * d;
  for (int j = threadIdx.x; j < k; j += blockDim.x) counts[j] = 0;
  __syncthreads();
  for (long long i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(&counts[assign[i]], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    s_empty = -1;
    for (int j = 0; j < k; ++j) if (counts[j] == 0) { s_empty = j; break; }
  }
  __syncthreads();
  if (s_empty < 0) { if (threadIdx.x == 0) rep_state[2 * rep] = -1; return; }
  double gv = -INFINITY; long long gi = 0x7fffffffffffLL;
  for (long long i = threadIdx.x; i < n; i += blockDim.x) {
    const double g = rmul(w[i], best[i]);
    if (g > gv) { gv = g; gi = i; }
  }
  for (int o = 16; o >= 1; o >>= 1) {
    const double og = __shfl_xor_sync(PCY_FULL, gv, o);
    const long long oi = __shfl_xor_sync(PCY_FULL, gi, o);
    if (og > gv || (og == gv && oi < gi)) { gv = og; gi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { wg[threadIdx.x >> 5] = gv; wi[threadIdx.x >> 5] = gi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double bg = -INFINITY; long long bi = 0x7fffffffffffLL;
    for (int t = 0; t < (int)(blockDim.x >> 5); ++t)
      if (wg[t] > bg || (wg[t] == bg && wi[t] < bi)) { bg = wg[t]; bi = wi[t]; }
    s_gmax = bg; s_far = (int)bi;
  }
  __syncthreads();
  if (!(s_gmax > 0.0)) { if (threadIdx.x == 0) rep_state[2 * rep] = -1; return; }   // every point on a centre
  const int emp = s_empty, far = s_far;
  for (int e = threadIdx.x; e < d; e += blockDim.x) C[(long long)emp * d + e] = P[(long long)far * d + e];
  if (threadIdx.x == 0) { rep_state[2 * rep] = emp; rep_state[2 * rep + 1] = far; }
}

// One Lloyd iteration's tail for every repetition, one CTA per repetition
// (KM_THREADS threads), no host round trip (evaluation.py:109-131):
//  * empty-cluster repair rounds until every centre is occupied or no point
//    has positive weighted distance: lowest empty centre <- first argmax of
//    w * best, points strictly closer (diff form) move to it, the far point
//    sits on it;
//  * cost = w . best (the fixed association of k_cost);
//  * the stop rule: the cost is logged, then prev - cost <= tol * prev clears
//    active (the centroid update of this iteration is skipped, as the
//    reference breaks before it); otherwise prev = cost.
// The last CTA to finish writes the number of still-active repetitions to
// flag[it] (mapped host memory) so the host can stop launching iterations.
__global__ void __launch_bounds__(KM_THREADS) k_lloyd_tail(const double* __restrict__ P, const double* __restrict__ w,
                                                          long long n, int d, int k, double* __restrict__ centers,
                                                          int* __restrict__ active, int* __restrict__ assign_all,
                                                          double* __restrict__ best_all, int* __restrict__ counts_all,
                                                          int use_smem_counts, double* __restrict__ prev,
                                                          double* __restrict__ logs, int* __restrict__ iters,
                                                          int max_iters, int it, double tol,
                                                          unsigned int* __restrict__ ticket,
                                                          volatile int* __restrict__ flag, int reps) {
  extern __shared__ int s_counts[];
  __shared__ int s_empty, s_far;
  __shared__ double s_gmax;
  __shared__ double wg[32];
  __shared__ long long wi[32];
  __shared__ double red[72];
  const int rep = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const bool act = active[rep] != 0;
  if (act) {
    int* assign = assign_all + (long long)rep * n;
    double* best = best_all + (long long)rep * n;
    int* counts = use_smem_counts ? s_counts : counts_all + (long long)rep * k;
    double* C = centers + (long long)rep * k * d;
    for (;;) {
      for (int j = tid; j < k; j += blockDim.x) counts[j] = 0;
      if (tid == 0) s_empty = 0x7fffffff;
      __syncthreads();
      for (long long i = tid; i < n; i += blockDim.x) atomicAdd(&counts[assign[i]], 1);
      __syncthreads();
      for (int j = tid; j < k; j += blockDim.x)
        if (counts[j] == 0) atomicMin(&s_empty, j);
      __syncthreads();
      if (s_empty == 0x7fffffff) break;
      double gv = -INFINITY; long long gi = 0x7fffffffffffLL;
      for (long long i = tid; i < n; i += blockDim.x) {
        const double g = rmul(w[i], best[i]);
        if (g > gv) { gv = g; gi = i; }
      }
      for (int o = 16; o >= 1; o >>= 1) {
        const double og = __shfl_xor_sync(PCY_FULL, gv, o);
        const long long oi = __shfl_xor_sync(PCY_FULL, gi, o);
        if (og > gv || (og == gv && oi < gi)) { gv = og; gi = oi; }
      }
      if (lane == 0) { wg[warp] = gv; wi[warp] = gi; }
      __syncthreads();
      if (tid == 0) {
        double bg = -INFINITY; long long bi = 0x7fffffffffffLL;
        for (int t = 0; t < nwarp; ++t)
          if (wg[t] > bg || (wg[t] == bg && wi[t] < bi)) { bg = wg[t]; bi = wi[t]; }
        s_gmax = bg; s_far = (int)bi;
      }
      __syncthreads();
      if (!(s_gmax > 0.0)) break;   // every point already sits on a centre
      const int emp = s_empty, far = s_far;
      for (int e = tid; e < d; e += blockDim.x) C[(long long)emp * d + e] = P[(long long)far * d + e];
      __syncthreads();
      const double* c = C + (long long)emp * d;
      for (long long i = warp; i < n; i += nwarp) {
        const double* p = P + i * d;
        double acc = 0.0;
        for (int e = lane; e < d; e += 32) { const double df = rsub(p[e], c[e]); acc = fma(df, df, acc); }
        acc = warp_sum(acc);
        if (lane == 0) {
          if (i == far) { assign[i] = emp; best[i] = 0.0; }
          else if (acc < best[i]) { assign[i] = emp; best[i] = acc; }
        }
      }
      __syncthreads();
    }
    // cost (same association as k_cost)
    const long long per = (n + blockDim.x - 1) / blockDim.x;
    const long long a = (long long)tid * per, b = min(n, a + per);
    double loc = 0.0;
    for (long long i = a; i < b; ++i) loc = fma(w[i], best[i], loc);
    const double cost = block_sum(loc, red);
    if (tid == 0) {
      logs[(long long)rep * max_iters + it] = cost;
      iters[rep] = it + 1;
      const double pv = prev[rep];
      if (isfinite(pv) && pv - cost <= tol * pv) active[rep] = 0;
      else prev[rep] = cost;
    }
  }
  if (tid == 0) {
    __threadfence();
    const unsigned int t = atomicAdd(ticket, 1u);
    if (t == (unsigned)reps - 1) {   // last repetition of this iteration: publish
      __threadfence();
      int na = 0;
      for (int r = 0; r < reps; ++r) na += ((volatile int*)active)[r] != 0;
      *ticket = 0u;
      flag[it] = na;
      __threadfence_system();
    }
  }
}

// Points closer to the re-seeded centre move to it (diff form); the far point
// itself sits on it.  Grid over points x repetitions, warp per point.
__global__ void k_repair_dist(const double* __restrict__ P, long long n, int d, int k,
                              const double* __restrict__ centers, const int* __restrict__ rep_state,
                              int* __restrict__ assign_all, double* __restrict__ best_all) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int rep = blockIdx.y;
  const int emp = rep_state[2 * rep], far = rep_state[2 * rep + 1];
  if (i >= n || emp < 0) return;
  const double* p = P + i * d;
  const double* c = centers + ((long long)rep * k + emp) * d;
  double acc = 0.0;
  for (int e = lane; e < d; e += 32) { const double df = rsub(p[e], c[e]); acc = fma(df, df, acc); }
  acc = warp_sum(acc);
  if (lane == 0) {
    int* assign = assign_all + (long long)rep * n;
    double* best = best_all + (long long)rep * n;
    if (i == far) { assign[i] = emp; best[i] = 0.0; }
    else if (acc < best[i]) { assign[i] = emp; best[i] = acc; }
  }
}

// cost = w . best per repetition (:126), fixed order (chunked then tree).
__global__ void __launch_bounds__(KM_THREADS) k_cost(const double* __restrict__ w, long long n,
                                                    const int* __restrict__ active,
                                                    const double* __restrict__ best_all, double* __restrict__ cost_out) {
  __shared__ double red[72];
  const int rep = blockIdx.x;
  if (active && !active[rep]) return;
  const double* best = best_all + (long long)rep * n;
  const long long per = (n + blockDim.x - 1) / blockDim.x;
  const long long a = (long long)threadIdx.x * per, b = min(n, a + per);
  double loc = 0.0;
  for (long long i = a; i < b; ++i) loc = fma(w[i], best[i], loc);
  const double tot = block_sum(loc, red);
  if (threadIdx.x == 0) cost_out[rep] = tot;
}

// Centroid update (:133-138): one CTA per (center, rep); the members of the
// center are compacted in index order, 4096 assignments per window (16 per
// thread, one block scan per window), and their weighted rows summed in index
// order.  Empty centers keep their previous value.
constexpr int KU_THREADS = 256, KU_PER = 16, KU_WIN = KU_THREADS * KU_PER;
__global__ void __launch_bounds__(KU_THREADS) k_update(const double* __restrict__ P, const double* __restrict__ w,
                                                       long long n, int d, int k, const int* __restrict__ active,
                                                       const int* __restrict__ assign_all, double* __restrict__ centers) {
  extern __shared__ double acc_s[];
  __shared__ int s_list[KU_WIN];
  __shared__ int wtot[KU_THREADS / 32 + 1];
  __shared__ double s_mass;
  const int j = blockIdx.x, rep = blockIdx.y;
  if (active && !active[rep]) return;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int* assign = assign_all + (long long)rep * n;
  double* C = centers + (long long)rep * k * d;
  for (int e = threadIdx.x; e < d; e += blockDim.x) acc_s[e] = 0.0;
  if (threadIdx.x == 0) s_mass = 0.0;
  __syncthreads();
  for (long long base = 0; base < n; base += KU_WIN) {
    // my 16 consecutive assignments
    const long long i0 = base + (long long)threadIdx.x * KU_PER;
    unsigned mine = 0u;
#pragma unroll
    for (int t = 0; t < KU_PER; ++t) {
      const long long i = i0 + t;
      if (i < n && assign[i] == j) mine |= 1u << t;
    }
    const int c = __popc(mine);
    // exclusive scan of the counts in thread order
    int inc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(PCY_FULL, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31) wtot[wid] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int q = 0; q < KU_THREADS / 32; ++q) { const int v = wtot[q]; wtot[q] = run; run += v; }
      wtot[KU_THREADS / 32] = run;
    }
    __syncthreads();
    int pos = wtot[wid] + inc - c;
    for (int t = 0; t < KU_PER; ++t)
      if ((mine >> t) & 1u) s_list[pos++] = (int)(i0 + t - base);
    __syncthreads();
    const int cnt = wtot[KU_THREADS / 32];
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
  double *best = nullptr, *mass = nullptr, *part = nullptr, *wpart = nullptr; int* picks = nullptr;
  // centres of rg repetitions per shared-memory pass (<= 200 KB)
  const size_t budget = 200 * 1024;
  int rg = (int)std::min<long long>(std::min(reps, KS_RMAX), (long long)(budget / (sizeof(double) * d)));
  if (rg < 1) { pcy_set_error("kmeanspp: dimension too large for the seeding kernel"); return PCY_EINVAL; }
  if (reps > 64) { pcy_set_error("kmeanspp: at most 64 repetitions per call"); return PCY_EINVAL; }
  const size_t sm = sizeof(double) * (size_t)rg * d;
  PCY_CUDA(cudaFuncSetAttribute(k_seed_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_seed_coop, KS_THREADS, sm);
  const long long max_blocks = (long long)sms * (per > 0 ? per : 1);
  // one row range per CTA, at least 32 rows each
  const long long blocks = std::max<long long>(1, std::min<long long>(max_blocks, (n + 31) / 32));
  int nb = (int)blocks;
  PCY_CUDA(pcy_malloc_async(&best, sizeof(double) * n * reps, st));
  PCY_CUDA(pcy_malloc_async(&mass, sizeof(double) * 2 * n * reps, st));
  PCY_CUDA(pcy_malloc_async(&part, sizeof(double) * 2 * blocks * reps, st));
  PCY_CUDA(pcy_malloc_async(&wpart, sizeof(double) * blocks, st));
  PCY_CUDA(pcy_malloc_async(&picks, sizeof(int) * k * reps, st));
  long long n_ = n; int d_ = d, k_ = k, reps_ = reps;
  void* args[] = {(void*)&P, (void*)&w, &n_, &d_, &k_, &reps_, (void*)&U, &centers, &best, &mass, &part, &wpart, &picks, &rg};
  const bool prof = pcy_prof_enabled();
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (prof) { cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventRecord(e0, st); }
  PCY_CUDA(cudaLaunchCooperativeKernel((const void*)k_seed_coop, dim3(nb), dim3(KS_THREADS), args, sm, st));
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  if (prof) {
    // algorithmic bytes: per distance pass the point rows once (n d 8) and, per
    // repetition, best read + write and mass write (24 n); weights n 8
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    const double bytes = (double)(k - 1) * ((double)n * d * 8.0 + (double)n * reps * 24.0 + (double)n * 8.0);
    pcy_prof_add(PCY_PROF_SEED, t, (long long)bytes);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
  }
  if (picks_out) {
    std::vector<int> h((size_t)k * reps);
    PCY_CUDA(pcy_d2h(h.data(), picks, sizeof(int) * k * reps, st));
    for (size_t i = 0; i < h.size(); ++i) picks_out[i] = h[i];
  }
  PCY_CUDA(cudaFreeAsync(best, st));
  PCY_CUDA(cudaFreeAsync(mass, st));
  PCY_CUDA(cudaFreeAsync(part, st));
  PCY_CUDA(cudaFreeAsync(wpart, st));
  PCY_CUDA(cudaFreeAsync(picks, st));
  return PCY_OK;
}

// Weighted Lloyd for `reps` center sets (centers updated in place).
// cost_log (host, reps x max_iters, nullable) receives the per-iteration
// costs; iters_out (host, reps) the number of logged costs.
// Per iteration: centre norms, one batched assignment launch for all
// repetitions (DMMA + argmin), k_lloyd_tail (repair, cost, stop rule on the
// device) and the centroid update -- the host never reads device state inside
// the loop; it polls the mapped per-iteration active count LAG iterations
// behind and stops launching once every repetition has converged (the at most
// LAG extra iterations find no active repetition and exit at once).
int pcy_lloyd(const double* P, const double* w, long long n, int d, int k, int reps, double* centers,
              int max_iters, double tol, double* cost_log, int* iters_out, void* stream) {
  if (n < 1 || k < 1 || d < 1 || reps < 1) { pcy_set_error("lloyd: bad sizes"); return PCY_EINVAL; }
  cudaStream_t st = (cudaStream_t)stream;
  for (int r = 0; r < reps; ++r) iters_out[r] = 0;
  if (max_iters <= 0) return PCY_OK;
  const int ntiles = (k + 63) / 64;
  double *pn = nullptr, *cn = nullptr, *best = nullptr, *prev = nullptr, *logs = nullptr, *ppart = nullptr;
  int *assign = nullptr, *counts = nullptr, *active = nullptr, *iters = nullptr, *ppos = nullptr;
  unsigned int* ticket = nullptr;
  int* flag_h = nullptr;
  int* flag_d = nullptr;
  cudaEvent_t pe0 = nullptr, pe1 = nullptr;
  const bool smem_counts = (size_t)k * sizeof(int) <= 64 * 1024;
  auto body = [&]() -> int {
    PCY_CUDA(pcy_malloc_async(&pn, sizeof(double) * n, st));
    PCY_CUDA(pcy_malloc_async(&cn, sizeof(double) * k * reps, st));
    PCY_CUDA(pcy_malloc_async(&best, sizeof(double) * n * reps, st));
    PCY_CUDA(pcy_malloc_async(&assign, sizeof(int) * n * reps, st));
    if (!smem_counts) PCY_CUDA(pcy_malloc_async(&counts, sizeof(int) * k * reps, st));
    PCY_CUDA(pcy_malloc_async(&active, sizeof(int) * reps, st));
    PCY_CUDA(pcy_malloc_async(&prev, sizeof(double) * reps, st));
    PCY_CUDA(pcy_malloc_async(&logs, sizeof(double) * reps * max_iters, st));
    PCY_CUDA(pcy_malloc_async(&iters, sizeof(int) * reps, st));
    PCY_CUDA(pcy_malloc_async(&ticket, sizeof(unsigned int), st));
    PCY_CUDA(pcy_malloc_async(&ppart, sizeof(double) * n * ntiles * reps, st));
    PCY_CUDA(pcy_malloc_async(&ppos, sizeof(int) * n * ntiles * reps, st));
    {   // per-thread mapped flag buffer, kept across calls (no host-alloc per call)
      static thread_local int* fbuf = nullptr;
      static thread_local int fcap = 0;
      if (fcap < max_iters) {
        if (fbuf) cudaFreeHost(fbuf);
        fbuf = nullptr; fcap = 0;
        int c = 128; while (c < max_iters) c *= 2;
        PCY_CUDA(cudaHostAlloc((void**)&fbuf, sizeof(int) * c, cudaHostAllocMapped | cudaHostAllocPortable));
        fcap = c;
      }
      flag_h = fbuf;
    }
    for (int t = 0; t < max_iters; ++t) flag_h[t] = -1;
    PCY_CUDA(cudaHostGetDevicePointer((void**)&flag_d, flag_h, 0));
    {
      std::vector<int> one(reps, 1);
      std::vector<double> inf(reps, INFINITY);
      PCY_CUDA(cudaMemcpyAsync(active, one.data(), sizeof(int) * reps, cudaMemcpyHostToDevice, st));
      PCY_CUDA(cudaMemcpyAsync(prev, inf.data(), sizeof(double) * reps, cudaMemcpyHostToDevice, st));
      PCY_CUDA(cudaMemsetAsync(iters, 0, sizeof(int) * reps, st));
      PCY_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned int), st));
      PCY_CUDA(cudaStreamSynchronize(st));   // the host vectors go out of scope
    }
    PCY_CUDA(cudaEventCreate(&pe0));
    PCY_CUDA(cudaEventCreate(&pe1));
    k_rownorm<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(P, n, d, pn); pcy_count_launch();
    const size_t usm = sizeof(double) * d;
    PCY_CUDA(cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)usm));
    const size_t tsm = smem_counts ? sizeof(int) * (size_t)k : 0;
    if (tsm > 48 * 1024) PCY_CUDA(cudaFuncSetAttribute(k_lloyd_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
    const bool prof = pcy_prof_enabled();
    float t_assign = 0.f;
    long long n_assign = 0;
    constexpr int LAG = 2;
    for (int it = 0; it < max_iters; ++it) {
      if (it >= LAG) {   // iteration it - LAG has finished once its flag is set
        volatile int* f = flag_h + (it - LAG);
        for (long long spins = 0; *f < 0; ++spins) {
          if ((spins & 1023) == 1023) {
            const cudaError_t e = cudaStreamQuery(st);
            if (e != cudaSuccess && e != cudaErrorNotReady) { pcy_set_error("lloyd: %s", cudaGetErrorString(e)); return PCY_ECUDA; }
          }
        }
        if (*f == 0) break;   // every repetition stopped
      }
      k_rownorm<<<(unsigned)((k * reps + 7) / 8), 256, 0, st>>>(centers, (long long)k * reps, d, cn); pcy_count_launch();
      if (prof) cudaEventRecord(pe0, st);
      int rc = pcy_launch_assign_d2_batch(P, d, (int)n, pn, centers, d, cn, k, d, reps, active, ppart, ppos, assign,
                                          best, st);
      if (rc) return rc;
      if (prof) {
        cudaEventRecord(pe1, st);
        cudaEventSynchronize(pe1);
        float t = 0.f;
        cudaEventElapsedTime(&t, pe0, pe1);
        t_assign += t;
        n_assign += reps;   // launched repetitions (inactive ones exit at once)
      }
      k_lloyd_tail<<<reps, KM_THREADS, tsm, st>>>(P, w, n, d, k, centers, active, assign, best, counts,
                                                  smem_counts ? 1 : 0, prev, logs, iters, max_iters, it, tol, ticket,
                                                  flag_d, reps);
      pcy_count_launch();
      k_update<<<dim3(k, reps), KU_THREADS, usm, st>>>(P, w, n, d, k, active, assign, centers); pcy_count_launch();
      PCY_LAUNCH_CHECK();
    }
    if (prof) pcy_prof_add(PCY_PROF_LLOYD, t_assign, (long long)(2.0 * (double)n * k * d * (double)n_assign));
    std::vector<double> hl((size_t)reps * max_iters);
    std::vector<int> hi(reps);
    PCY_CUDA(pcy_d2h(hl.data(), logs, sizeof(double) * hl.size(), st));
    PCY_CUDA(pcy_d2h(hi.data(), iters, sizeof(int) * reps, st));
    for (int r = 0; r < reps; ++r) {
      iters_out[r] = hi[r];
      if (cost_log)
        for (int t = 0; t < hi[r]; ++t) cost_log[(size_t)r * max_iters + t] = hl[(size_t)r * max_iters + t];
    }
    return PCY_OK;
  };
  const int rc = body();
  cudaFreeAsync(pn, st); cudaFreeAsync(cn, st); cudaFreeAsync(best, st); cudaFreeAsync(assign, st);
  if (counts) cudaFreeAsync(counts, st);
  cudaFreeAsync(active, st); cudaFreeAsync(prev, st); cudaFreeAsync(logs, st); cudaFreeAsync(iters, st);
  cudaFreeAsync(ticket, st); cudaFreeAsync(ppart, st); cudaFreeAsync(ppos, st);
  if (pe0) cudaEventDestroy(pe0);
  if (pe1) cudaEventDestroy(pe1);
  return rc;
}

// weighted_cost for `reps` center sets into device memory: costs_dev (device,
// reps) -- no host synchronisation (the streaming evaluation accumulates
// chunk costs on the device).  w (device, fp64) may be null for unit weights.
int pcy_weighted_cost_dev(const double* P, const double* w, long long n, int d, int k, int reps,
                          const double* centers, double* costs_dev, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1) { PCY_CUDA(cudaMemsetAsync(costs_dev, 0, sizeof(double) * reps, st)); return PCY_OK; }
  double *pn = nullptr, *cn = nullptr, *best = nullptr, *ones = nullptr; int *assign = nullptr;
  PCY_CUDA(pcy_malloc_async(&pn, sizeof(double) * n, st));
  PCY_CUDA(pcy_malloc_async(&cn, sizeof(double) * k * reps, st));
  PCY_CUDA(pcy_malloc_async(&best, sizeof(double) * n * reps, st));
  PCY_CUDA(pcy_malloc_async(&assign, sizeof(int) * n * reps, st));
  if (!w) {
    PCY_CUDA(pcy_malloc_async(&ones, sizeof(double) * n, st));
    k_fill<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 8), 256, 0, st>>>(ones, n, 1.0); pcy_count_launch();
    w = ones;
  }
  k_rownorm<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(P, n, d, pn); pcy_count_launch();
  k_rownorm<<<(unsigned)((k * reps + 7) / 8), 256, 0, st>>>(centers, (long long)k * reps, d, cn); pcy_count_launch();
  const int ntiles = (k + 63) / 64;
  double* ppart = nullptr; int* ppos = nullptr;
  PCY_CUDA(pcy_malloc_async(&ppart, sizeof(double) * n * ntiles, st));
  PCY_CUDA(pcy_malloc_async(&ppos, sizeof(int) * n * ntiles, st));
  int rc = PCY_OK;
  for (int r = 0; r < reps && rc == PCY_OK; ++r)
    rc = pcy_launch_assign_d2(P, d, (int)n, pn, centers + (long long)r * k * d, d, cn + (long long)r * k, k, d,
                              ppart, ppos, assign + (long long)r * n, best + (long long)r * n, st);
  if (rc == PCY_OK) { k_cost<<<reps, KM_THREADS, 0, st>>>(w, n, nullptr, best, costs_dev); pcy_count_launch(); }
  PCY_LAUNCH_CHECK();
  cudaFreeAsync(pn, st); cudaFreeAsync(cn, st); cudaFreeAsync(best, st); cudaFreeAsync(assign, st);
  cudaFreeAsync(ppart, st); cudaFreeAsync(ppos, st);
  if (ones) cudaFreeAsync(ones, st);
  return rc;
}

// Streaming evaluation block (evaluate_cost_multi, evaluation.py:157-180):
// rows P (device, n x d fp64, n a multiple of `chunk` except at the stream
// end) against one centre set C (device, k x d): out (device) receives the
// unweighted chunk sums of the first-min GEMM-form distances at
// out[c * out_stride], c = 0 .. ceil(n/chunk)-1.  Scratch is allocated once
// per call; 5 launches per call whatever n is.
int pcy_cost_chunks(const double* P, long long n, int d, const double* C, int k, long long chunk, double* out,
                    long long out_stride, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1) return PCY_OK;
  if (chunk < 1 || k < 1) { pcy_set_error("cost_chunks: bad sizes"); return PCY_EINVAL; }
  const int ntiles = (k + 63) / 64;
  double *pn = nullptr, *cn = nullptr, *best = nullptr, *ppart = nullptr; int *assign = nullptr, *ppos = nullptr;
  PCY_CUDA(pcy_malloc_async(&pn, sizeof(double) * n, st));
  PCY_CUDA(pcy_malloc_async(&cn, sizeof(double) * k, st));
  PCY_CUDA(pcy_malloc_async(&best, sizeof(double) * n, st));
  PCY_CUDA(pcy_malloc_async(&assign, sizeof(int) * n, st));
  PCY_CUDA(pcy_malloc_async(&ppart, sizeof(double) * n * ntiles, st));
  PCY_CUDA(pcy_malloc_async(&ppos, sizeof(int) * n * ntiles, st));
  k_rownorm<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(P, n, d, pn); pcy_count_launch();
  k_rownorm<<<(unsigned)((k + 7) / 8), 256, 0, st>>>(C, k, d, cn); pcy_count_launch();
  int rc = pcy_launch_assign_d2(P, d, (int)n, pn, C, d, cn, k, d, ppart, ppos, assign, best, st);
  if (rc == PCY_OK) {
    k_chunk_sums<<<(unsigned)((n + chunk - 1) / chunk), 256, 0, st>>>(best, n, chunk, out, out_stride);
    pcy_count_launch();
  }
  PCY_LAUNCH_CHECK();
  cudaFreeAsync(pn, st); cudaFreeAsync(cn, st); cudaFreeAsync(best, st); cudaFreeAsync(assign, st);
  cudaFreeAsync(ppart, st); cudaFreeAsync(ppos, st);
  return rc;
}

// weighted_cost for `reps` center sets: costs (host, reps).
int pcy_weighted_cost(const double* P, const double* w, long long n, int d, int k, int reps,
                      const double* centers, double* costs, void* stream) {
  if (n < 1) { for (int r = 0; r < reps; ++r) costs[r] = 0.0; return PCY_OK; }
  cudaStream_t st = (cudaStream_t)stream;
  double* cost = nullptr;
  PCY_CUDA(pcy_malloc_async(&cost, sizeof(double) * reps, st));
  int rc = pcy_weighted_cost_dev(P, w, n, d, k, reps, centers, cost, stream);
  if (rc == PCY_OK) PCY_CUDA(pcy_d2h(costs, cost, sizeof(double) * reps, st));
  cudaFreeAsync(cost, st);
  return rc;
}

}  // extern "C"
