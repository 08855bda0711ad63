// BICO clustering-feature engine on B200 (sm_100a).
//
// Reference semantics: /root/reference/pkg/src/piecy/coreset.py (BicoEngine).
// Layout and kernel roles are described in DESIGN.md §3-§4:
//   k_stage    -- upcast/copy a block, x_sq, validation, exact-bytes hash
//   k_boot_*   -- bootstrap buffering (coreset.py:283-295): parallel scan, same result as in order
//   k_mp_*     -- T0 = min positive pairwise sq. distance * m / 16 (:297-299, :479-489)
//   k_snapshot -- freeze group counts for the chain kernel
//   k_chain    -- K1: every item's capacity-free nearest-reference chain against
//                 the snapshot, all items in parallel (warp per item)
//   k_resolve  -- K3: in-order resolve (:307-377): re-tests members opened since
//                 the snapshot, closed-form capacity, CF update (K2), open
//   k_rb_*     -- K4: rebuild (:381-421): T*=2, order (-w, index), reattach
//   k_dfs/k_gather_* -- features()/extract_coreset() (:425-451)
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <mutex>
#include <cstddef>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include "engine.cuh"

static thread_local char g_err[512];
void pcy_set_error(const char* fmt, ...) {
  va_list ap; va_start(ap, fmt); vsnprintf(g_err, sizeof(g_err), fmt, ap); va_end(ap);
}
extern "C" const char* pcy_last_error(void) { return g_err; }

// Launch counter (bench.py's gpu_launches) and optional per-kernel event
// timing of the engine's sequential kernels (bench.py's roofline).
static std::atomic<long long> g_launches{0};
static std::atomic<long long> g_counters[6];   // summed over destroyed engines
void pcy_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static std::atomic<int> g_prof_on{0};
static std::mutex g_prof_mu;
static PcyProfSlot g_prof[PCY_PROF_SLOTS];
bool pcy_prof_enabled() { return g_prof_on.load(std::memory_order_relaxed) != 0; }
void pcy_prof_add(int slot, double ms, long long units) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof[slot].ms += ms; g_prof[slot].count += 1; g_prof[slot].units += units;
}
cudaError_t pcy_spin_sync(cudaStream_t st) {
  static thread_local cudaEvent_t ev = nullptr;
  cudaError_t e;
  if (!ev && (e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaEventRecord(ev, st)) != cudaSuccess) return e;
  for (;;) {
    e = cudaEventQuery(ev);
    if (e != cudaErrorNotReady) return e;
  }
}
cudaError_t pcy_malloc_async_raw(void** p, size_t bytes, cudaStream_t st) {
  static std::once_flag once[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::call_once(once[dev & 63], [dev] {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      unsigned long long keep = ~0ULL;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
  return cudaMallocAsync(p, bytes, st);
}

cudaError_t pcy_d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  static thread_local void* buf = nullptr;
  static thread_local size_t cap = 0;
  cudaError_t e;
  if (bytes > cap) {
    if (buf) cudaFreeHost(buf);
    size_t c = 4096; while (c < bytes) c *= 2;
    if ((e = cudaMallocHost(&buf, c)) != cudaSuccess) { buf = nullptr; cap = 0; return e; }
    cap = c;
  }
  if ((e = cudaMemcpyAsync(buf, src, bytes, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = pcy_spin_sync(st)) != cudaSuccess) return e;
  memcpy(dst, buf, bytes);
  return cudaSuccess;
}
extern "C" long long pcy_launch_count(void) { return g_launches.load(); }
extern "C" int pcy_prof_enable(int on) { g_prof_on.store(on); return 0; }
extern "C" int pcy_prof_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& p : g_prof) p = PcyProfSlot{};
  return 0;
}
extern "C" int pcy_prof_read(int slot, double* ms, long long* count, long long* units) {
  if (slot < 0 || slot >= PCY_PROF_SLOTS) return PCY_EINVAL;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  *ms = g_prof[slot].ms; *count = g_prof[slot].count; *units = g_prof[slot].units;
  return 0;
}

// ----------------------------------------------------------------- helpers
__device__ __forceinline__ bool rows_equal(const double* a, const double* b, int d, int lane) {
  bool eq = true;
  for (int e = lane; e < d; e += 32)
    eq &= (__double_as_longlong(a[e]) == __double_as_longlong(b[e]));
  return __all_sync(PCY_FULL, eq);
}

__device__ __forceinline__ unsigned long long row_hash(const double* x, int d, int lane) {
  unsigned long long h = 0;
  for (int e = lane; e < d; e += 32)
    h += mix64((unsigned long long)__double_as_longlong(x[e]) + 0x9E3779B97F4A7C15ULL * (unsigned long long)(e + 1));
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) h += __shfl_xor_sync(PCY_FULL, h, o);
  return mix64(h);
}

// Append `node` to group g (warp-uniform call).  Returns false on arena overflow.
__device__ bool grp_append(const EngDev& E, int g, int node, long long& A_alloc, int lane) {
  int cnt = E.g_count[g], cap = E.g_cap[g], base = E.g_base[g];
  if (cnt == cap) {
    int ncap = cap ? 2 * cap : PCY_GROUP_MIN_CAP;
    long long nb = A_alloc;
    if (nb + ncap > E.AC) return false;
    A_alloc += ncap;
    for (int p = lane; p < cnt; p += 32) E.arena[nb + p] = E.arena[base + p];
    base = (int)nb; cap = ncap;
    if (lane == 0) { E.g_base[g] = base; E.g_cap[g] = cap; }
  }
  if (lane == 0) { E.arena[base + cnt] = node; E.g_count[g] = cnt + 1; }
  __syncwarp();
  return true;
}

// Nearest among members [lo, hi) of the arena segment `mem`, against vector xv
// (shared memory).  Lane-per-member transposed dots.  Returns the part
// |r|^2 - 2 r.x and the position (lowest position wins ties), on all lanes.
__device__ __forceinline__ void scan_members(const EngDev& E, const int* __restrict__ mem,
                                             int lo, int hi, const double* __restrict__ xv,
                                             int lane, double& bp, int& bpos) {
  const int d = E.d, ld = E.ld;
  bp = INFINITY; bpos = 0x7fffffff;
  for (int c0 = lo; c0 < hi; c0 += 32) {
    const int nm = min(32, hi - c0);
    const int myid = lane < nm ? mem[c0 + lane] : -1;
    double acc[32];
#pragma unroll
    for (int mm = 0; mm < 32; ++mm) {
      const int id = __shfl_sync(PCY_FULL, myid, mm);
      double a = 0.0;
      if (id >= 0) {
        const double* __restrict__ rr = E.r + (long long)id * ld;
        for (int e = lane; e < d; e += 32) a = fma(rr[e], xv[e], a);
      }
      acc[mm] = a;
    }
    const double dt = warp_transpose_reduce(acc, lane);
    double part = INFINITY; int pos = 0x7fffffff;
    if (lane < nm) { part = radd(E.rn[myid], rmul(dt, -2.0)); pos = c0 + lane; }
    warp_argmin(part, pos);
    if (part < bp) { bp = part; bpos = pos; }
  }
}

// Nearest among members [0, cnt) of a small group, d <= 256 (visited-groups
// K1): lane-per-member fp64 dots.  Each lane issues its member's whole
// reference row (16-byte loads, up to 64 elements per pass) before the FMAs,
// so a chunk of 32 members costs one L2 round trip instead of 32 dependent
// warp reductions.  Part |r|^2 - 2 r.x as in coreset.py:173-176, lowest
// position on ties.  xv: the point in shared memory (entries < d are read).
__device__ __forceinline__ void scan_members_lane(const EngDev& E, const int* __restrict__ mem, int cnt,
                                                  const double* __restrict__ xv, int lane, double& bp, int& bpos) {
  const int d = E.d, ld = E.ld;
  bp = INFINITY; bpos = 0x7fffffff;
  for (int c0 = 0; c0 < cnt; c0 += 32) {
    const int p = c0 + lane;
    double part = INFINITY;
    int pos = 0x7fffffff;
    if (p < cnt) {
      const int id = mem[p];
      const double2* __restrict__ rr = reinterpret_cast<const double2*>(E.r + (long long)id * ld);
      const double rn = E.rn[id];
      double acc = 0.0;
      for (int e0 = 0; e0 < d; e0 += 64) {
        double2 v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = (e0 + 2 * q < ld) ? __ldg(rr + (e0 >> 1) + q) : make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          if (e0 + 2 * q < d) acc = fma(v[q].x, xv[e0 + 2 * q], acc);
          if (e0 + 2 * q + 1 < d) acc = fma(v[q].y, xv[e0 + 2 * q + 1], acc);
        }
      }
      part = radd(rn, rmul(acc, -2.0));
      pos = p;
    }
    warp_argmin(part, pos);
    if (part < bp) { bp = part; bpos = pos; }
  }
}

// scan_members_lane plus the winner's slot and statistics: every lane also
// loads its member's (w, q, sn, child) in the same round trip as the row, and
// the winning lane's values are shuffled out -- the chain walk then needs no
// further dependent load before it can fetch the next level's group.
struct LaneWinner { int id, child; long long w; double q, sn; };
__device__ __forceinline__ void scan_members_lane_w(const EngDev& E, const int* __restrict__ mem, int cnt,
                                                    const double* __restrict__ xv, int lane, double& bp, int& bpos,
                                                    LaneWinner& win) {
  const int d = E.d, ld = E.ld;
  bp = INFINITY; bpos = 0x7fffffff;
  win = LaneWinner{-1, -1, 0, 0.0, 0.0};
  for (int c0 = 0; c0 < cnt; c0 += 32) {
    const int p = c0 + lane;
    double part = INFINITY;
    int pos = 0x7fffffff;
    LaneWinner mine{-1, -1, 0, 0.0, 0.0};
    if (p < cnt) {
      const int id = mem[p];
      const double2* __restrict__ rr = reinterpret_cast<const double2*>(E.r + (long long)id * ld);
      const double rn = E.rn[id];
      mine = LaneWinner{id, E.child[id], E.w[id], E.q[id], E.sn[id]};
      double acc = 0.0;
      for (int e0 = 0; e0 < d; e0 += 64) {
        double2 v[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = (e0 + 2 * q < ld) ? __ldg(rr + (e0 >> 1) + q) : make_double2(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          if (e0 + 2 * q < d) acc = fma(v[q].x, xv[e0 + 2 * q], acc);
          if (e0 + 2 * q + 1 < d) acc = fma(v[q].y, xv[e0 + 2 * q + 1], acc);
        }
      }
      part = radd(rn, rmul(acc, -2.0));
      pos = p;
    }
    warp_argmin(part, pos);
    if (part < bp) {
      bp = part; bpos = pos;
      const int src = pos - c0;
      win.id = __shfl_sync(PCY_FULL, mine.id, src);
      win.child = __shfl_sync(PCY_FULL, mine.child, src);
      win.w = __shfl_sync(PCY_FULL, mine.w, src);
      win.q = __shfl_sync(PCY_FULL, mine.q, src);
      win.sn = __shfl_sync(PCY_FULL, mine.sn, src);
    }
  }
}

// Nearest among members [0, cnt) using a precomputed parts row (full-set K1;
// columns are the live columns, gathered per member through col_of).
__device__ __forceinline__ void scan_parts(const double* __restrict__ prow, const int* __restrict__ col_of,
                                           const int* __restrict__ mem, int cnt, int lane, double& bp, int& bpos) {
  bp = INFINITY; bpos = 0x7fffffff;
  for (int c0 = 0; c0 < cnt; c0 += 32) {
    const int p = c0 + lane;
    double v = INFINITY; int ps = 0x7fffffff;
    if (p < cnt) { v = prow[col_of[mem[p]]]; ps = p; }
    warp_argmin(v, ps);
    if (v < bp) { bp = v; bpos = ps; }
  }
}

// Nearest among members [0, cnt) from the tensor-core dots row of item i:
// approximate centred parts a_j = |r_j-c|^2 - 2 dot_j carry the rigorous
// error e_j = 2 tau |r_j-c| |x-c|; every member with a_j - e_j <= min(a + e)
// is re-decided with its exact fp64 part (first position on ties), so the
// result is the fp64 argmin.  *nre counts the exact re-decisions.
template <class RDot>
__device__ __forceinline__ void scan_parts_tc(const EngDev& E, long long i, int g, const int* __restrict__ mem,
                                              int cnt, RDot rdot, int lane, double& bp, int& bpos, int& nre,
                                              int pbase = -1) {
  // pbase < 0: columns are live columns (k_tc_split_slots), gathered per
  // member through col_of, norms slot-indexed.  pbase >= 0: the group's members
  // are the panel columns pbase + position (k_publish_panel), norms by column.
  // Four chunks of 32 members in flight per pass.
  const float* __restrict__ dots = E.tc_dots + i * E.tc_ldo;
  const double* __restrict__ rnc = E.tc_rnc;
  const int* __restrict__ col_of = E.col_of;
  const double xn = sqrt(E.tc_xn2[i]);
  const double tau2 = 2.0 * E.tc_tau * (1.0 + 1e-9);
  double U = INFINITY;
  for (int c0 = 0; c0 < cnt; c0 += 128) {
    int jj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) { const int p = c0 + 32 * q + lane; jj[q] = p < cnt ? mem[p] : -1; }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (jj[q] >= 0) {
        const int col = pbase >= 0 ? pbase + c0 + 32 * q + lane : col_of[jj[q]];
        const double rc = rnc[pbase >= 0 ? col : jj[q]];
        U = fmin(U, rc - 2.0 * (double)dots[col] + tau2 * sqrt(rc) * xn + 1e-300);
      }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) U = fmin(U, __shfl_xor_sync(PCY_FULL, U, o));
  bp = INFINITY; bpos = 0x7fffffff;
  int ncand = 0;
  for (int c0 = 0; c0 < cnt; c0 += 128) {
    int jj[4];
    bool cand[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) { const int p = c0 + 32 * q + lane; jj[q] = p < cnt ? mem[p] : -1; }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      cand[q] = false;
      if (jj[q] >= 0) {
        const int col = pbase >= 0 ? pbase + c0 + 32 * q + lane : col_of[jj[q]];
        const double rc = rnc[pbase >= 0 ? col : jj[q]];
        cand[q] = rc - 2.0 * (double)dots[col] - tau2 * sqrt(rc) * xn <= U;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      unsigned m = __ballot_sync(PCY_FULL, cand[q]);
      while (m) {   // position order
        const int b = __ffs(m) - 1;
        m &= m - 1;
        const int j = __shfl_sync(PCY_FULL, jj[q], b);
        const double part = radd(E.rn[j], rmul(rdot(j), -2.0));
        if (part < bp) { bp = part; bpos = c0 + 32 * q + b; }
        ++ncand;
      }
    }
  }
  if (ncand > 1) nre += ncand - 1;   // members re-decided beyond the winner
}

// CTA form (WPI warps walk one item together, k_chain2<WPI>): the members are
// split over the CTA's threads for both passes; the candidates gather in a
// shared list (clist[0] = count) and are re-decided together with the CTA
// dot, the lowest position winning exact ties as in the warp form.
constexpr int TC_CAND_MAX = 256;
template <int WPI, class RDot>
__device__ __forceinline__ void scan_parts_tc_cta(const EngDev& E, long long i, const int* __restrict__ mem, int cnt,
                                                  RDot rdot, int lane, int wib, double* red, int* clist, double& bp,
                                                  int& bpos, int& nre) {
  const float* __restrict__ dots = E.tc_dots + i * E.tc_ldo;
  const double* __restrict__ rnc = E.tc_rnc;
  const int* __restrict__ col_of = E.col_of;
  const double xn = sqrt(E.tc_xn2[i]);
  const double tau2 = 2.0 * E.tc_tau * (1.0 + 1e-9);
  constexpr int T = 32 * WPI;
  const int t = wib * 32 + lane;
  double U = INFINITY;
  for (int p0 = t; p0 < cnt; p0 += 4 * T) {
    int jj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) { const int p = p0 + T * q; jj[q] = p < cnt ? mem[p] : -1; }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (jj[q] >= 0) {
        const double rc = rnc[jj[q]];
        U = fmin(U, rc - 2.0 * (double)dots[col_of[jj[q]]] + tau2 * sqrt(rc) * xn + 1e-300);
      }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) U = fmin(U, __shfl_xor_sync(PCY_FULL, U, o));
  __syncthreads();
  if (lane == 0) red[wib] = U;
  if (t == 0) clist[0] = 0;
  __syncthreads();
#pragma unroll
  for (int w = 0; w < WPI; ++w) U = fmin(U, red[w]);
  for (int p0 = t; p0 < cnt; p0 += 4 * T) {
    int jj[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) { const int p = p0 + T * q; jj[q] = p < cnt ? mem[p] : -1; }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (jj[q] >= 0) {
        const double rc = rnc[jj[q]];
        if (rc - 2.0 * (double)dots[col_of[jj[q]]] - tau2 * sqrt(rc) * xn <= U) {
          const int k = atomicAdd(&clist[0], 1);
          if (k < TC_CAND_MAX) clist[1 + k] = p0 + T * q;
        }
      }
  }
  __syncthreads();
  const int nc = clist[0];
  bp = INFINITY; bpos = 0x7fffffff;
  if (nc <= TC_CAND_MAX) {
    for (int c = 0; c < nc; ++c) {
      const int p = clist[1 + c];
      const double part = radd(E.rn[mem[p]], rmul(rdot(mem[p]), -2.0));
      if (part < bp || (part == bp && p < bpos)) { bp = part; bpos = p; }
    }
  } else {   // very wide near-tie window: every member exactly, position order
    for (int p = 0; p < cnt; ++p) {
      const double part = radd(E.rn[mem[p]], rmul(rdot(mem[p]), -2.0));
      if (part < bp) { bp = part; bpos = p; }
    }
  }
  if (nc > 1) nre += nc - 1;
  __syncthreads();   // clist / red reuse
}

#include "resolve_fast.cuh"
#include "reattach_fast.cuh"
#include "resolve_smem.cuh"

// Column order of the full-set contraction (one CTA): gofs[g] = exclusive
// prefix sum of the group member counts, *cnt = total.  Group g's members
// then occupy columns [gofs[g], gofs[g] + g_count[g]), so the chain walk reads
// its parts / dots row contiguously, with no slot indirection.
__global__ void __launch_bounds__(1024) k_group_offsets(const int* __restrict__ gcount, long long ng,
                                                        int* __restrict__ gofs, int* __restrict__ cnt) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (long long base = 0; base < ng; base += 1024) {
    const long long g = base + tid;
    const int c = g < ng ? gcount[g] : 0;
    int v = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) { const int t = __shfl_up_sync(PCY_FULL, v, o); if (lane >= o) v += t; }
    if (lane == 31) wsum[warp] = v;
    __syncthreads();
    if (warp == 0) {
      int u = wsum[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) { const int t = __shfl_up_sync(PCY_FULL, u, o); if (lane >= o) u += t; }
      wsum[lane] = u;   // inclusive over warps
    }
    __syncthreads();
    if (g < ng) gofs[g] = carry + (warp ? wsum[warp - 1] : 0) + v - c;
    __syncthreads();
    if (tid == 0) carry += wsum[31];
    __syncthreads();
  }
  if (tid == 0) *cnt = carry;
}

// list[gofs[g] + p] = member p of group g (one warp per group)
__global__ void k_group_scatter(EngDev E, long long ng, int* __restrict__ list) {
  const int lane = threadIdx.x & 31;
  const long long g = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (g >= ng) return;
  const int c = E.g_count[g], b = E.g_base[g], o = E.fs_gofs[g];
  for (int p = lane; p < c; p += 32) list[o + p] = E.arena[b + p];
}

// ------------------------------------------------------------------ stage
// One warp per row: fp32/fp64 -> fp64 padded row, x_sq, validation, hash.
__global__ void k_stage(EngDev E, const void* __restrict__ src, int dtype, long long stride,
                        const long long* __restrict__ wsrc, long long n, int dohash) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  const int d = E.d, ld = E.ld;
  double* __restrict__ dst = E.xb + i * ld;
  double acc = 0.0; bool fin = true;
  for (int e = lane; e < ld; e += 32) {
    double v = 0.0;
    if (e < d) {
      v = dtype == 1 ? (double)((const float*)src)[i * stride + e] : ((const double*)src)[i * stride + e];
      fin &= isfinite(v);
      acc = fma(v, v, acc);
    }
    dst[e] = v;
  }
  const double xs = warp_sum(acc);
  const bool allfin = __all_sync(PCY_FULL, fin);
  __syncwarp();
  unsigned long long h = dohash ? row_hash(dst, d, lane) : 0ULL;
  if (lane == 0) {
    const long long wv = wsrc ? wsrc[i] : 1LL;
    int code = 0;
    if (wv < 1) code = 3;
    else if (!isfinite(xs)) code = allfin ? 2 : 1;
    E.xsq[i] = xs; E.wb[i] = wv; E.bad[i] = code;
    if (dohash) E.hsh[i] = h;
  }
}

// x_sq for rows already in engine layout (pending replay).
__global__ void k_rowsq(const double* __restrict__ X, int d, int ld, long long n, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  const double* x = X + i * ld;
  double acc = 0.0;
  for (int e = lane; e < d; e += 32) acc = fma(x[e], x[e], acc);
  acc = warp_sum(acc);
  if (lane == 0) out[i] = acc;
}

// --------------------------------------------------------------- bootstrap
// Parallel bootstrap (coreset.py:283-295: exactly the one-at-a-time result).  The last
// pending entry always holds the previous row's key, so row i starts a new
// pending entry iff it differs from row i-1 (from the last entry for the
// first row); a row is a new distinct key iff it is not in the table and no
// earlier row of the block has its bytes.  A prefix scan over the block then
// places the stop (invalid row, pending buffer full, budget + 1 distinct) and
// the pending / distinct positions.
struct BootScratch {
  int* flags;    // per row: bit0 starts a pending entry, bit1 new distinct key
  int* spos;     // per row: scratch-table slot
  int* ppos;     // per row: pending position (rows starting an entry)
  int* dpos;     // per row: distinct position (new keys)
  int* skey;     // scratch table: first claiming row (-1 empty)
  int* sfirst;   // scratch table: lowest row with those bytes
  long long scap;
};

__global__ void k_boot_scan_rows(EngDev E, BootScratch B, long long start, long long n) {
  const int lane = threadIdx.x & 31;
  const long long i = start + (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n) return;
  const int d = E.d, ld = E.ld;
  const double* x = E.xb + i * ld;
  const long long npend0 = E.ctl->npend;
  bool newp;
  if (i == start) newp = !(npend0 > 0 && rows_equal(E.pend_x + (npend0 - 1) * ld, x, d, lane));
  else newp = !rows_equal(E.xb + (i - 1) * ld, x, d, lane);
  // known key?
  const unsigned long long mask = (unsigned long long)E.hcap - 1ULL;
  unsigned long long slot = E.hsh[i] & mask;
  bool found = false;
  for (;;) {
    const int k = E.htab[slot];
    if (k < 0) break;
    if (rows_equal(E.dist_x + (long long)k * ld, x, d, lane)) { found = true; break; }
    slot = (slot + 1) & mask;
  }
  int sp = -1;
  if (!found) {
    // first row of the block with these bytes
    const unsigned long long smask = (unsigned long long)B.scap - 1ULL;
    unsigned long long ss = E.hsh[i] & smask;
    for (;;) {
      int k = 0;
      if (lane == 0) k = atomicCAS(&B.skey[ss], -1, (int)(i - start));
      k = __shfl_sync(PCY_FULL, k, 0);
      if (k == -1 || rows_equal(E.xb + (start + k) * ld, x, d, lane)) break;
      ss = (ss + 1) & smask;
    }
    sp = (int)ss;
    if (lane == 0) atomicMin(&B.sfirst[ss], (int)(i - start));
  }
  if (lane == 0) { B.flags[i - start] = newp ? 1 : 0; B.spos[i - start] = sp; }
}

// One CTA: flags -> stop, positions, counters.
__global__ void __launch_bounds__(1024) k_boot_plan(EngDev E, BootScratch B, long long start, long long n) {
  __shared__ long long red[2][33];
  __shared__ long long s_stop;
  __shared__ int s_status;
  __shared__ long long s_np, s_nd, s_w;
  EngCtl* C = E.ctl;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long cnt = n - start;
  if (tid == 0) { s_stop = cnt; s_status = ST_DONE; s_np = C->npend; s_nd = C->ndist; s_w = 0; C->err = 0; }
  __syncthreads();
  for (long long c0 = 0; c0 < cnt; c0 += blockDim.x) {
    const long long r = c0 + tid;
    const bool in = r < cnt && r < s_stop;
    int fl = 0;
    if (in) {
      fl = B.flags[r];
      if (B.spos[r] >= 0 && B.sfirst[B.spos[r]] == (int)r) fl |= 2;
    }
    const long long np_in = (fl & 1), nd_in = (fl >> 1) & 1;
    // inclusive scans of (new pending, new distinct) in row order
    long long a = np_in, b = nd_in;
    for (int o = 1; o < 32; o <<= 1) {
      const long long ta = __shfl_up_sync(PCY_FULL, a, o), tb = __shfl_up_sync(PCY_FULL, b, o);
      if (lane >= o) { a += ta; b += tb; }
    }
    if (lane == 31) { red[0][wid] = a; red[1][wid] = b; }
    __syncthreads();
    if (wid == 0) {
      long long wa = lane < (int)(blockDim.x >> 5) ? red[0][lane] : 0, wb = lane < (int)(blockDim.x >> 5) ? red[1][lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const long long ta = __shfl_up_sync(PCY_FULL, wa, o), tb = __shfl_up_sync(PCY_FULL, wb, o);
        if (lane >= o) { wa += ta; wb += tb; }
      }
      red[0][lane] = wa; red[1][lane] = wb;   // inclusive warp totals
    }
    __syncthreads();
    const long long pa = (wid ? red[0][wid - 1] : 0) + a, pb = (wid ? red[1][wid - 1] : 0) + b;   // inclusive
    const long long np0 = s_np, nd0 = s_nd;
    // per-row events in stream order: invalid (row not taken), pending full
    // (row not taken), then the row is taken and may be the budget + 1-th key
    long long ev = 0x7fffffffffffLL; int st = ST_DONE;
    if (in) {
      const int bad = E.bad[start + r];
      if (bad) { ev = 2 * r; st = ST_INVALID; }
      else if (np_in && np0 + pa - 1 >= E.pend_cap) { ev = 2 * r; st = ST_GROW; }
      else if (nd_in && nd0 + pb > E.m) { ev = 2 * r + 1; st = ST_BUILD; }
    }
    // earliest event of the chunk
    long long evm = ev;
    for (int o = 16; o >= 1; o >>= 1) evm = min(evm, __shfl_xor_sync(PCY_FULL, evm, o));
    __syncthreads();
    if (lane == 0) red[0][wid] = evm;
    __syncthreads();
    if (tid == 0) {
      long long e = 0x7fffffffffffLL;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) e = min(e, red[0][q]);
      red[1][32] = e;
    }
    __syncthreads();
    const long long eall = red[1][32];
    if (in && eall != 0x7fffffffffffLL && ev == eall) {   // the event's (unique) row
      s_status = st;
      s_stop = r;
      C->err = st == ST_INVALID ? E.bad[start + r] : 0;
    }
    __syncthreads();
    const long long lim = eall == 0x7fffffffffffLL ? cnt : (eall >> 1) + (eall & 1);   // rows taken in this chunk range
    const bool take = in && r < lim;
    if (take) {
      if (np_in) B.ppos[r] = (int)(np0 + pa - 1);
      if (nd_in) B.dpos[r] = (int)(nd0 + pb - 1);
    }
    // counters over taken rows
    long long wsum = take ? E.wb[start + r] : 0;
    long long tnp = take ? np_in : 0, tnd = take ? nd_in : 0;
    for (int o = 16; o >= 1; o >>= 1) {
      wsum += __shfl_xor_sync(PCY_FULL, wsum, o);
      tnp += __shfl_xor_sync(PCY_FULL, tnp, o);
      tnd += __shfl_xor_sync(PCY_FULL, tnd, o);
    }
    __syncthreads();
    if (lane == 0) { red[0][wid] = wsum; red[1][wid] = tnp * 65536LL + tnd; }
    __syncthreads();
    if (tid == 0) {
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { s_w += red[0][q]; s_np += red[1][q] >> 16; s_nd += red[1][q] & 65535; }
    }
    __syncthreads();
    if (eall != 0x7fffffffffffLL) break;
  }
  if (tid == 0) {
    C->npend = s_np; C->ndist = s_nd; C->total_w += s_w;
    C->status = s_status; C->stop = start + (s_status == ST_DONE ? cnt : s_stop);
    B.flags[cnt] = (int)(s_status == ST_DONE ? cnt : s_stop + (s_status == ST_BUILD ? 1 : 0));   // rows taken
  }
}

// Rows taken: pending rows and weights (a run of equal rows sums into its
// first), new keys into the distinct rows and the table.
__global__ void k_boot_apply(EngDev E, BootScratch B, long long start, long long n, long long npend0) {
  const int lane = threadIdx.x & 31;
  const long long r = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long taken = B.flags[n - start];
  if (r >= taken) return;
  const int d = E.d, ld = E.ld;
  const double* x = E.xb + (start + r) * ld;
  const int fl = B.flags[r];
  if ((fl & 1) || r == 0) {
    // weight of the run starting here (the leading run continues the last entry)
    long long q = r;
    long long wsum = E.wb[start + q];
    for (++q; q < taken && !(B.flags[q] & 1); ++q) wsum += E.wb[start + q];
    if (fl & 1) {
      const long long p = B.ppos[r];
      double* pr = E.pend_x + p * ld;
      for (int e = lane; e < ld; e += 32) pr[e] = x[e];
      if (lane == 0) { E.pend_w[p] = wsum; E.pend_xsq[p] = E.xsq[start + r]; }
    } else if (lane == 0) {
      E.pend_w[npend0 - 1] += wsum;   // leading run of the previous entry's key
    }
  }
  if (B.spos[r] >= 0 && B.sfirst[B.spos[r]] == (int)r) {
    const long long p = B.dpos[r];
    double* dr = E.dist_x + p * ld;
    for (int e = lane; e < ld; e += 32) dr[e] = x[e];
    if (lane == 0) {
      const unsigned long long mask = (unsigned long long)E.hcap - 1ULL;
      unsigned long long slot = E.hsh[start + r] & mask;
      while (atomicCAS(&E.htab[slot], -1, (int)p) != -1) slot = (slot + 1) & mask;
    }
  }
}

// ---------------------------------------------- min pairwise (threshold T0)
__global__ void k_mp_norms(EngDev E, long long ns, double* __restrict__ nrm) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= ns) return;
  const double* x = E.dist_x + i * E.ld;
  double v = warp_dot(x, x, E.d, lane);
  if (lane == 0) {
    nrm[i] = v;
    atomicMax(E.minbits + 1, (unsigned long long)__double_as_longlong(v));
  }
}

// 32x32 tile of the sample Gram; v = (n_i + n_j) - 2 G_ij, min over v > 0, i < j.
__global__ void k_mp_tiles(EngDev E, long long ns, const double* __restrict__ nrm) {
  __shared__ double As[32][33], Bs[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
  const long long i0 = (long long)blockIdx.y * 32, j0 = (long long)blockIdx.x * 32;
  if (j0 + 31 < i0) return;
  const int d = E.d, ld = E.ld;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int e0 = 0; e0 < d; e0 += 32) {
    for (int r = ty; r < 32; r += 8) {
      const long long ia = i0 + r, jb = j0 + r;
      As[r][tx] = (ia < ns && e0 + tx < d) ? E.dist_x[ia * ld + e0 + tx] : 0.0;
      Bs[r][tx] = (jb < ns && e0 + tx < d) ? E.dist_x[jb * ld + e0 + tx] : 0.0;
    }
    __syncthreads();
    const int ne = min(32, d - e0);
    for (int e = 0; e < ne; ++e) {
      const double b = Bs[tx][e];
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[k] = fma(As[ty + 8 * k][e], b, acc[k]);
    }
    __syncthreads();
  }
  unsigned long long best = 0x7ff0000000000000ULL;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const long long i = i0 + ty + 8 * k, j = j0 + tx;
    if (i < ns && j < ns && i < j) {
      const double v = rsub(radd(nrm[i], nrm[j]), rmul(2.0, acc[k]));
      if (v > 0.0) best = min(best, (unsigned long long)__double_as_longlong(v));
    }
  }
  if (best != 0x7ff0000000000000ULL) atomicMin(E.minbits, best);
}

__global__ void k_mp_finish(EngDev E, long long ns) {
  if (threadIdx.x || blockIdx.x) return;
  double mn;
  if (ns < 2) mn = 1.0;
  else if (E.minbits[0] == 0x7ff0000000000000ULL) {
    const double nmax = __longlong_as_double((long long)E.minbits[1]);
    mn = rmul(1e-12, nmax > 1.0 ? nmax : 1.0);
  } else mn = __longlong_as_double((long long)E.minbits[0]);
  E.ctl->T = rdiv(rmul(mn, (double)E.m), 16.0);
}

// ------------------------------------------------------- host publication
// Live columns of the full-set contraction (DMMA path; the tensor-core path
// assigns them in k_tc_split_slots): every slot that holds a node without a
// column for its creation index takes the next column.  Between rebuilds no
// node dies, so the columns are exactly the live nodes; after a rebuild the
// engine recompacts (done = -1, ncol = 0), and the contraction spans F
// columns instead of every slot ever allocated.
__global__ void k_assign_cols(const int* __restrict__ alive, const long long* __restrict__ cidx, long long n,
                              long long* __restrict__ done, int* __restrict__ col_of, int* __restrict__ col_slot,
                              int* __restrict__ ncol) {
  const long long s = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool need = s < n && alive[s] && done[s] != cidx[s];
  const unsigned msk = __ballot_sync(PCY_FULL, need);
  if (!msk) return;
  const int leader = __ffs(msk) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(ncol, __popc(msk));
  base = __shfl_sync(PCY_FULL, base, leader);
  if (need) {
    const int c = base + __popc(msk & ((1u << lane) - 1u));
    col_of[s] = c; col_slot[c] = (int)s; done[s] = cidx[s];
  }
}

__global__ void k_publish(EngCtl* __restrict__ src, EngCtl* dst, long long seq, const int* g_count,
                          const int* g_base) {
  const int lane = threadIdx.x;
  if (lane == 0) { src->root_count = g_count[0]; src->root_base = g_base[0]; }
  __syncwarp();
  const int words = (int)(offsetof(EngCtl, seq) / sizeof(long long));
  const long long* s = reinterpret_cast<const long long*>(src);
  volatile long long* t = reinterpret_cast<volatile long long*>(dst);
  for (int k = lane; k < words; k += 32) t[k] = s[k];
  __threadfence_system();
  __syncwarp();
  if (lane == 0) t[words] = seq;
}

// Publication with the visited-groups panel (d <= 256, one CTA of 1024
// threads): groups of at least PCY_PANEL_MIN members -- visited by many items
// of the next K1 batch -- get consecutive panel columns in group-index order
// (fs_gofs[g], -1 for the groups the chain walk scans directly), their member
// slots go to fs_list in position order, and panel_n is published with the
// counters.  The tree does not change between this publication and the next
// K1 launch, so the panel is that launch's snapshot.
constexpr int PCY_PANEL_MAXG = 2048;   // listed big groups (later ones are scanned directly)
__global__ void __launch_bounds__(1024) k_publish_panel(EngDev E, EngCtl* dst, long long seq) {
  __shared__ int wsc[32], wsb[32];
  __shared__ int big[PCY_PANEL_MAXG];
  __shared__ int carry_c, carry_b;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  EngCtl* src = E.ctl;
  const long long G = src->G_alloc;
  if (tid == 0) { carry_c = 0; carry_b = 0; }
  __syncthreads();
  for (long long base = 0; base < G; base += 1024) {
    const long long g = base + tid;
    const int c = g < G ? E.g_count[g] : 0;
    const int isb = c >= PCY_PANEL_MIN ? 1 : 0;
    int vc = isb ? c : 0, vb = isb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int tc = __shfl_up_sync(PCY_FULL, vc, o), tb = __shfl_up_sync(PCY_FULL, vb, o);
      if (lane >= o) { vc += tc; vb += tb; }
    }
    if (lane == 31) { wsc[warp] = vc; wsb[warp] = vb; }
    __syncthreads();
    if (warp == 0) {
      int uc = wsc[lane], ub = wsb[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int tc = __shfl_up_sync(PCY_FULL, uc, o), tb = __shfl_up_sync(PCY_FULL, ub, o);
        if (lane >= o) { uc += tc; ub += tb; }
      }
      wsc[lane] = uc; wsb[lane] = ub;   // inclusive over warps
    }
    __syncthreads();
    const int rank = carry_b + (warp ? wsb[warp - 1] : 0) + vb - isb;   // big groups before g
    const int ofs = carry_c + (warp ? wsc[warp - 1] : 0) + vc - (isb ? c : 0);
    if (g < G) {
      const bool listed = isb && rank < PCY_PANEL_MAXG;
      E.fs_gofs[g] = listed ? ofs : -1;
      if (listed) big[rank] = (int)g;
    }
    __syncthreads();
    if (tid == 0) {
      // columns stop at the last listed group: later big groups are scanned directly
      const int tb = wsb[31], tcnt = wsc[31];
      if (carry_b + tb <= PCY_PANEL_MAXG) carry_c += tcnt;
      else if (carry_b < PCY_PANEL_MAXG) {
        int acc = 0;   // columns of the listed groups of this tile
        for (int k = carry_b; k < PCY_PANEL_MAXG; ++k) acc += E.g_count[big[k]];
        carry_c += acc;
      }
      carry_b += tb;
    }
    __syncthreads();
  }
  const int nbig = carry_b < PCY_PANEL_MAXG ? carry_b : PCY_PANEL_MAXG;
  for (int b = warp; b < nbig; b += 32) {
    const int g = big[b];
    const int c = E.g_count[g], bs = E.g_base[g], o = E.fs_gofs[g];
    for (int p = lane; p < c; p += 32) E.fs_list[o + p] = E.arena[bs + p];
  }
  if (tid == 0) { src->panel_n = carry_c; src->root_count = E.g_count[0]; src->root_base = E.g_base[0]; }
  __syncthreads();
  if (warp == 0) {
    const int words = (int)(offsetof(EngCtl, seq) / sizeof(long long));
    const long long* s = reinterpret_cast<const long long*>(src);
    volatile long long* t = reinterpret_cast<volatile long long*>(dst);
    for (int k = lane; k < words; k += 32) t[k] = s[k];
    __threadfence_system();
    __syncwarp();
    if (lane == 0) t[words] = seq;
  }
}

// ------------------------------------------------------------- tree reset
__global__ void k_tree_reset(EngDev E) {
  if (threadIdx.x || blockIdx.x) return;
  EngCtl* C = E.ctl;
  C->G_alloc = 1; C->A_alloc = 0; C->F = 0; C->maxg = 0;
  E.g_count[0] = 0; E.g_cap[0] = 0; E.g_base[0] = 0;
}

__global__ void k_snapshot(EngDev E) {
  const long long G = E.ctl->G_alloc;
  for (long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x; g < G; g += (long long)gridDim.x * blockDim.x) {
    E.g_bs[g] = E.g_count[g];
    E.g_bsbase[g] = E.g_base[g];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) E.ctl->G_snap = G;
}

// ------------------------------------------------------------- K1: chains
// One warp per item: walk the snapshot tree along nearest references while
// the admission radius holds (coreset.py:325-329, :369-372), ignoring
// capacity.  Records (node, part) per level; the final recorded level is the
// one where the chain leaves (outside radius or empty group).
__global__ void k_chain(EngDev E, const double* __restrict__ X, const double* __restrict__ XS,
                        long long n) {
  extern __shared__ double sm_x[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  if (i >= n) return;
  const int d = E.d, ld = E.ld;
  double* xv = sm_x + (long long)wib * ld;
  const double xs = XS[i];
  if (!isfinite(xs)) { if (lane == 0) E.ch_len[i] = 0; return; }   // rejected by k_resolve
  for (int e = lane; e < d; e += 32) xv[e] = X[i * ld + e];
  __syncwarp();
  const long long Gsnap = E.ctl->G_snap;
  double radius = E.ctl->T;
  int g = 0, L = 0;
  int* cn = E.ch_node + i * PCY_MAXL;
  double* cp = E.ch_part + i * PCY_MAXL;
  for (;;) {
    const int cnt = g < Gsnap ? E.g_bs[g] : 0;
    double bp; int bpos;
    scan_members(E, E.arena + (cnt ? E.g_bsbase[g] : 0), 0, cnt, xv, lane, bp, bpos);
    const int bj = (cnt && bpos < cnt) ? E.arena[E.g_bsbase[g] + bpos] : -1;
    if (lane == 0) { cn[L] = bj; cp[L] = bp; }
    ++L;
    if (bj < 0 || radd(bp, xs) > radius) break;
    const int c = E.child[bj];
    if (c < 0 || c >= Gsnap) {
      if (L < PCY_MAXL) { if (lane == 0) { cn[L] = -1; cp[L] = INFINITY; } ++L; }
      break;
    }
    if (L >= PCY_MAXL) break;   // truncated: k_resolve scans directly below
    g = c;
    radius = rmul(radius, 0.25);
  }
  if (lane == 0) E.ch_len[i] = L;
}

// ------------------------------------------------------------- K3: resolve
// One warp, items in stream order.  Per level: the chain's snapshot winner is
// compared with members appended after the snapshot (or all members in
// direct mode), then the closed-form capacity (coreset.py:336-356) decides
// how many copies stay; CF statistics update in place (:357-368).
__global__ void k_resolve(EngDev E, const double* __restrict__ X, const double* __restrict__ XS,
                          const long long* __restrict__ W, const int* __restrict__ BAD,
                          long long n, long long start, long long first_rem, int countw) {
  extern __shared__ double xv[];
  const int lane = threadIdx.x;
  EngCtl* C = E.ctl;
  const int d = E.d, ld = E.ld;
  const long long m = E.m;
  const double T = C->T;
  long long F = C->F, Falloc = C->F_alloc, freen = C->free_n, Galloc = C->G_alloc;
  long long Aalloc = C->A_alloc, nidx = C->next_index, totw = C->total_w, maxdepth = C->max_depth;
  const long long Gsnap = C->G_snap;
  int status = ST_DONE, err = 0; long long stop = n, remaining = 0;

  for (long long i = start; i < n; ++i) {
    if (BAD && BAD[i]) { status = ST_INVALID; err = BAD[i]; stop = i; break; }
    const bool resume = (i == start && first_rem >= 0);
    const long long wi = W ? W[i] : 1LL;
    long long rem = resume ? first_rem : wi;
    if (countw && !resume) totw += wi;
    for (int e = lane; e < d; e += 32) xv[e] = X[i * ld + e];
    __syncwarp();
    const double xs = XS[i];
    const int len = E.ch_len[i];
    const int* cn = E.ch_node + i * PCY_MAXL;
    const double* cp = E.ch_part + i * PCY_MAXL;
    int g = 0, L = 0;
    double radius = T;
    bool direct = false;
    for (;;) {
      int bj = -1; double bp = INFINITY;
      if (!direct) {
        if (L < len) { bj = cn[L]; bp = cp[L]; }
        else direct = true;
      }
      const int cnt = E.g_count[g];
      const int lo = direct ? 0 : (g < Gsnap ? E.g_bs[g] : 0);
      bool newwin = false;
      if (cnt > lo) {
        double np_; int npos;
        const int* mem = E.arena + E.g_base[g];
        scan_members(E, mem, lo, cnt, xv, lane, np_, npos);
        if (npos < cnt && (np_ < bp || bj < 0)) {
          bp = np_; bj = mem[npos]; newwin = true;
        }
      }
      if (bj < 0 || radd(bp, xs) > radius) {
        // _open (coreset.py:329-335, :374-377)
        const bool full = F >= m;
        const long long wopen = full ? 1LL : rem;
        long long slot;
        if (freen > 0) slot = E.free_ids[--freen];
        else slot = Falloc++;
        double* rr = E.r + slot * ld;
        double* ss = E.s + slot * ld;
        const double fw = (double)wopen;
        for (int e = lane; e < d; e += 32) { rr[e] = xv[e]; ss[e] = rmul(fw, xv[e]); }
        if (lane == 0) {
          E.w[slot] = wopen;
          E.q[slot] = rmul(fw, xs);
          E.sn[slot] = rmul((double)(wopen * wopen), xs);
          E.rn[slot] = xs;
          E.idx[slot] = nidx;
          E.child[slot] = -1;
          E.alive[slot] = 1;
        }
        ++nidx;
        __syncwarp();
        if (!grp_append(E, g, (int)slot, Aalloc, lane)) { status = ST_ARENA; stop = i; break; }
        ++F;
        if (L + 1 > maxdepth) maxdepth = L + 1;
        rem -= wopen;
        if (full) { status = ST_REBUILD; stop = i; remaining = rem; }
        break;
      }
      // capacity on the winner (coreset.py:336-356)
      const long long nn = E.w[bj];
      const double fn = (double)nn;
      const double nrm = rdiv(E.sn[bj], fn);
      double errv = rsub(E.q[bj], nrm);
      if (errv < 0.0) errv = 0.0;
      double* ss = E.s + (long long)bj * ld;
      const double dt = warp_dot(ss, xv, d, lane);
      double dist = rsub(xs, rdiv(rsub(rmul(2.0, dt), nrm), fn));
      if (dist < 0.0) dist = 0.0;
      const double slack = radd(rsub(rmul(fn, dist), T), errv);
      long long take;
      if (slack <= 0.0) take = rem;
      else {
        const double limit = rdiv(rsub(rmul(fn, T), rmul(fn, errv)), slack);
        if (limit >= (double)rem) take = rem;
        else if (limit > 0.0) take = (long long)limit;
        else take = 0;
      }
      if (take > 0) {
        const double ft = (double)take;
        if (take == 1) { for (int e = lane; e < d; e += 32) ss[e] = radd(ss[e], xv[e]); }
        else { for (int e = lane; e < d; e += 32) ss[e] = radd(ss[e], rmul(ft, xv[e])); }
        if (lane == 0) {
          E.w[bj] = nn + take;
          E.q[bj] = radd(E.q[bj], rmul(ft, xs));
          E.sn[bj] = radd(E.sn[bj], radd(rmul(rmul(2.0, ft), dt), rmul((double)(take * take), xs)));
        }
        __syncwarp();
        rem -= take;
        if (rem == 0) { if (L + 1 > maxdepth) maxdepth = L + 1; break; }
      }
      if (newwin) direct = true;
      int c = E.child[bj];
      if (c < 0) {
        c = (int)Galloc++;
        if (lane == 0) { E.g_count[c] = 0; E.g_cap[c] = 0; E.g_base[c] = 0; E.child[bj] = c; }
        __syncwarp();
      }
      g = c;
      radius = rmul(radius, 0.25);
      ++L;
    }
    __syncwarp();
    if (status != ST_DONE) break;
  }
  if (lane == 0) {
    C->F = F; C->F_alloc = Falloc; C->free_n = freen; C->G_alloc = Galloc;
    C->A_alloc = Aalloc; C->next_index = nidx; C->total_w = totw; C->max_depth = maxdepth;
    C->status = status; C->err = err; C->stop = stop; C->remaining = remaining;
  }
}

// ------------------------------------------------------------ K4: rebuild
// Order live slots by (-weight, creation index) (coreset.py:454-455).
__global__ void k_rb_rank(EngDev E, long long nslots) {
  __shared__ long long sw[256], si[256];
  __shared__ int sa[256];
  const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool mine = u < nslots && E.alive[u];
  const long long wu = mine ? E.w[u] : 0, iu = mine ? E.idx[u] : 0;
  long long rank = 0;
  for (long long t0 = 0; t0 < nslots; t0 += 256) {
    const long long v = t0 + threadIdx.x;
    sa[threadIdx.x] = v < nslots ? E.alive[v] : 0;
    sw[threadIdx.x] = v < nslots ? E.w[v] : 0;
    si[threadIdx.x] = v < nslots ? E.idx[v] : 0;
    __syncthreads();
    if (mine) {
      const int nt = (int)min(256LL, nslots - t0);
      for (int k = 0; k < nt; ++k)
        rank += sa[k] && (sw[k] > wu || (sw[k] == wu && si[k] < iu));
    }
    __syncthreads();
  }
  if (mine) E.order[rank] = (int)u;
}

// Sliced form of k_rb_rank: blockIdx.y counts over one slice of the
// candidates and adds its count into rank[u] (zeroed before); the scatter
// k_rb_scatter then places each alive node.  The (-weight, index) keys are
// distinct among alive nodes, so the ranks are a permutation, as above.
constexpr int RB_SLICES = 16;
__global__ void __launch_bounds__(256) k_rb_rank_sliced(EngDev E, long long nslots, int* __restrict__ rank) {
  __shared__ long long sw[256], si[256];
  __shared__ int sa[256];
  const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const bool mine = u < nslots && E.alive[u];
  const long long wu = mine ? E.w[u] : 0, iu = mine ? E.idx[u] : 0;
  const long long per = ((nslots + RB_SLICES - 1) / RB_SLICES + 255) / 256 * 256;
  const long long lo = (long long)blockIdx.y * per, hi = min(nslots, lo + per);
  int cnt = 0;
  for (long long t0 = lo; t0 < hi; t0 += 256) {
    const long long v = t0 + threadIdx.x;
    sa[threadIdx.x] = v < hi ? E.alive[v] : 0;
    sw[threadIdx.x] = v < hi ? E.w[v] : 0;
    si[threadIdx.x] = v < hi ? E.idx[v] : 0;
    __syncthreads();
    if (mine) {
      const int nt = (int)min(256LL, hi - t0);
      for (int k = 0; k < nt; ++k)
        cnt += sa[k] && (sw[k] > wu || (sw[k] == wu && si[k] < iu));
    }
    __syncthreads();
  }
  if (mine && cnt) atomicAdd(&rank[u], cnt);
}

__global__ void k_rb_scatter(EngDev E, long long nslots, const int* __restrict__ rank) {
  const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (u < nslots && E.alive[u]) E.order[rank[u]] = (int)u;
}

// T *= 2; detach every subtree; fresh roots (coreset.py:386-391).
__global__ void k_rb_reset(EngDev E, long long nslots) {
  const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (u < nslots) E.child[u] = -1;
  if (u == 0) {
    EngCtl* C = E.ctl;
    C->T = rmul(C->T, 2.0);
    C->G_alloc = 1; C->A_alloc = 0; C->F = 0; C->maxg = 0;
    E.g_count[0] = 0; E.g_cap[0] = 0; E.g_base[0] = 0;
  }
}

// Reattach nodes in rank order (coreset.py:395-421).  One CTA of 32 warps;
// the member scan of each level is split across warps.
__global__ void __launch_bounds__(512) k_rb_reattach(EngDev E, long long nodes) {
  extern __shared__ double refv[];
  __shared__ double red_p[32];
  __shared__ int red_pos[32];
  __shared__ int s_dec, s_host;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  EngCtl* C = E.ctl;
  const int d = E.d, ld = E.ld;
  const double T = C->T;
  long long F = 0, Galloc = 1, Aalloc = 0, freen = C->free_n;
  for (long long k = 0; k < nodes; ++k) {
    const int u = E.order[k];
    for (int e = threadIdx.x; e < d; e += blockDim.x) refv[e] = E.r[(long long)u * ld + e];
    __syncthreads();
    const double rsq = E.rn[u];
    int g = 0;
    double radius = T;
    for (;;) {
      const int cnt = E.g_count[g];
      const int* mem = E.arena + E.g_base[g];
      double bp = INFINITY; int bpos = 0x7fffffff;
      for (int c0 = wid * 32; c0 < cnt; c0 += nw * 32) {
        double p; int ps;
        scan_members(E, mem, c0, min(cnt, c0 + 32), refv, lane, p, ps);
        if (p < bp) { bp = p; bpos = ps; }
      }
      if (lane == 0) { red_p[wid] = bp; red_pos[wid] = bpos; }
      __syncthreads();
      if (wid == 0) {
        double p = lane < nw ? red_p[lane] : INFINITY;
        int ps = lane < nw ? red_pos[lane] : 0x7fffffff;
        warp_argmin(p, ps);
        int dec;   // 0 add, 1 merged, 2 descend
        int h = -1;
        if (cnt == 0 || radd(p, rsq) > radius) {
          dec = 0;
          if (!grp_append(E, g, u, Aalloc, lane)) dec = 3;
          ++F;
        } else {
          h = mem[ps];
          const long long mw = E.w[h] + E.w[u];
          const double* sh = E.s + (long long)h * ld;
          const double* su = E.s + (long long)u * ld;
          double acc = 0.0;
          for (int e = lane; e < d; e += 32) { const double v = radd(sh[e], su[e]); acc = fma(v, v, acc); }
          const double mnorm = warp_sum(acc);
          const double mq = radd(E.q[h], E.q[u]);
          if (rsub(mq, rdiv(mnorm, (double)mw)) <= T) {
            double* shw = E.s + (long long)h * ld;
            for (int e = lane; e < d; e += 32) shw[e] = radd(shw[e], su[e]);
            if (lane == 0) {
              E.w[h] = mw; E.q[h] = mq; E.sn[h] = mnorm;
              E.alive[u] = 0; E.free_ids[freen] = u;
            }
            ++freen;
            dec = 1;
          } else {
            dec = 2;
            int c = E.child[h];
            if (c < 0) {
              c = (int)Galloc++;
              if (lane == 0) { E.g_count[c] = 0; E.g_cap[c] = 0; E.g_base[c] = 0; E.child[h] = c; }
            }
            h = c;
          }
        }
        if (lane == 0) { s_dec = dec; s_host = h; }
      }
      __syncthreads();
      const int dec = s_dec;
      if (dec != 2) break;
      g = s_host;
      radius = rmul(radius, 0.25);
      __syncthreads();
    }
    __syncthreads();
    if (s_dec == 3) break;
  }
  if (threadIdx.x == 0) {
    C->F = F; C->G_alloc = Galloc; C->A_alloc = Aalloc; C->free_n = freen;
    C->status = s_dec == 3 ? ST_ARENA : ST_DONE;
  }
}

// ------------------------------------------------------------- extraction
// DFS pre-order over groups (coreset.py:433-440).  Single thread; the output
// order drives the parallel gathers below.
__global__ void k_dfs(EngDev E) {
  if (threadIdx.x || blockIdx.x) return;
  long long cnt = 0; int depth = 0;
  E.stk_g[0] = 0; E.stk_p[0] = 0;
  while (depth >= 0) {
    const int g = E.stk_g[depth], p = E.stk_p[depth];
    if (p >= E.g_count[g]) { --depth; continue; }
    E.stk_p[depth] = p + 1;
    const int u = E.arena[E.g_base[g] + p];
    E.order[cnt] = u; E.lvl[cnt] = depth + 1; ++cnt;
    const int c = E.child[u];
    if (c >= 0 && E.g_count[c] > 0) { ++depth; E.stk_g[depth] = c; E.stk_p[depth] = 0; }
  }
  E.ctl->stop = cnt;
}

// features(): level, weight, linear sum, square sum, reference.
__global__ void k_gather_features(EngDev E, long long cnt, int* __restrict__ lv, long long* __restrict__ wo,
                                  double* __restrict__ so, double* __restrict__ qo, double* __restrict__ ro) {
  const int lane = threadIdx.x & 31;
  const long long k = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= cnt) return;
  const int u = E.order[k], d = E.d, ld = E.ld;
  if (so) for (int e = lane; e < d; e += 32) so[k * d + e] = E.s[(long long)u * ld + e];
  if (ro) for (int e = lane; e < d; e += 32) ro[k * d + e] = E.r[(long long)u * ld + e];
  if (lane == 0) {
    if (lv) lv[k] = E.lvl[k];
    if (wo) wo[k] = E.w[u];
    if (qo) qo[k] = E.q[u];
  }
}

// extract_coreset(): row = s / n (coreset.py:449).
__global__ void k_gather_points(EngDev E, long long cnt, double* __restrict__ po, long long* __restrict__ wo) {
  const int lane = threadIdx.x & 31;
  const long long k = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= cnt) return;
  const int u = E.order[k], d = E.d, ld = E.ld;
  const double fw = (double)E.w[u];
  for (int e = lane; e < d; e += 32) po[k * d + e] = rdiv(E.s[(long long)u * ld + e], fw);
  if (lane == 0 && wo) wo[k] = E.w[u];
}

// Bootstrap-time features: pending aggregated per exact location in
// first-occurrence order (coreset.py:429-432, :466-476).  The distinct table
// is in first-seen order, so aggregation is a keyed weight sum.
__global__ void k_boot_aggregate(EngDev E, long long* __restrict__ aggw) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= E.ctl->npend) return;
  const double* x = E.pend_x + i * E.ld;
  const unsigned long long mask = (unsigned long long)E.hcap - 1ULL;
  unsigned long long slot = row_hash(x, E.d, lane) & mask;
  for (;;) {
    const int k = E.htab[slot];
    if (k < 0) return;   // unreachable: every pending row was registered
    if (rows_equal(E.dist_x + (long long)k * E.ld, x, E.d, lane)) {
      if (lane == 0) atomicAdd((unsigned long long*)&aggw[k], (unsigned long long)E.pend_w[i]);
      return;
    }
    slot = (slot + 1) & mask;
  }
}

__global__ void k_boot_gather(EngDev E, long long cnt, const long long* __restrict__ aggw, int* __restrict__ lv,
                              long long* __restrict__ wo, double* __restrict__ so, double* __restrict__ qo,
                              double* __restrict__ ro, double* __restrict__ po) {
  const int lane = threadIdx.x & 31;
  const long long k = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= cnt) return;
  const int d = E.d;
  const double* x = E.dist_x + k * E.ld;
  const long long wk = aggw[k];
  const double fw = (double)wk;
  double acc = 0.0;
  for (int e = lane; e < d; e += 32) {
    const double sv = rmul(fw, x[e]);
    if (so) so[k * d + e] = sv;
    if (ro) ro[k * d + e] = x[e];
    if (po) po[k * d + e] = rdiv(sv, fw);
    acc = fma(x[e], x[e], acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) {
    if (lv) lv[k] = 1;
    if (wo) wo[k] = wk;
    if (qo) qo[k] = rmul(fw, acc);
  }
}

// ====================================================================== host
namespace {

// Mapped pinned control mirrors are recycled across engines: cudaFreeHost
// would synchronise the device whenever an engine is destroyed.
static std::mutex g_ctl_mu;
static std::vector<EngCtl*> g_ctl_pool;
static EngCtl* ctl_pool_get() {
  {
    std::lock_guard<std::mutex> lk(g_ctl_mu);
    if (!g_ctl_pool.empty()) { EngCtl* c = g_ctl_pool.back(); g_ctl_pool.pop_back(); return c; }
  }
  EngCtl* c = nullptr;
  if (cudaHostAlloc(&c, sizeof(EngCtl), cudaHostAllocMapped) != cudaSuccess) return nullptr;
  return c;
}
static void ctl_pool_put(EngCtl* c) {
  std::lock_guard<std::mutex> lk(g_ctl_mu);
  g_ctl_pool.push_back(c);
}

// Launch with the programmatic-serialization attribute: the kernel may be
// scheduled before its predecessor in the stream has finished and orders
// itself with pdl_wait() (engine.cuh).
template <class... KArgs, class... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid; cfg.blockDim = block; cfg.dynamicSmemBytes = smem; cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, KArgs(args)...);
}

struct Engine {
  int dev = 0, d = 0, ld = 0;
  long long m = 0, sample_cap = 0, NC = 0, GC = 0, AC = 0, Bmax = 0;
  bool built = false;
  EngDev E{};
  EngCtl* ctl_h = nullptr;   // mapped pinned mirror (host view)
  // Engine buffers come from the stream-ordered pool on `own`; destruction
  // waits (on the device) for the last public call's stream through `done_ev`
  // and frees asynchronously -- no device-wide synchronisation.
  cudaStream_t own = nullptr;
  cudaEvent_t done_ev = nullptr;
  bool done_rec = false;
  EngCtl* ctl_map_d = nullptr;   // device view of the mirror
  long long seq = 0, plan_seq = 0, tl_early = 0;
  long long* aggw = nullptr;
  double* mp_nrm = nullptr;
  cudaEvent_t ev[8] = {};
  // Side stream (highest priority) for the batch Gram of k_plan's conflict
  // test: it depends only on the batch rows and runs beside the chain walk;
  // evk1 (rows / previous window done) and evk3 (Gram done) order it.
  cudaStream_t hi = nullptr;
  cudaEvent_t evk1 = nullptr, evk3 = nullptr;
  bool gemm_timed = false;           // ev[6..7] bracket the last full-set contraction
  double gemm_flops = 0.0;
  ChainHdr* chh = nullptr;
  ChainLvl* chr = nullptr;
  double* parts = nullptr;                             // full-set parts matrix (1024 x NC)
  double* gram = nullptr;                              // block Gram (K3 with rows in HBM)
  double* gram_b = nullptr;                            // second Gram buffer: run-ahead batches alternate
  int gram_flip = 0;
  double* gram_part = nullptr;                         // split-K partials of the block Gram (large d)
  int gram_split = 1;
  bool use_tc = false;                                 // full-set K1 on tcgen05 (split TF32 + recheck)
  bool panel = false;                                  // visited-groups K1 (d <= 256): big-group panel + direct scans
  double exec_tensor_flops = 0.0;                      // tensor-pipe flops of the panel contractions (3 TF32 products)
  long long panel_launches = 0;
  int Kp = 0;
  double tc_tau = 0.0;
  float *tc_ahi = nullptr, *tc_alo = nullptr, *tc_bhi = nullptr, *tc_blo = nullptr, *tc_dots = nullptr;
  double *tc_rnc = nullptr, *tc_xn2 = nullptr, *tc_c = nullptr;
  long long* tc_done = nullptr;   // creation index each slot's column (and split) was made for
  int* col_slot = nullptr;        // live column -> slot
  int* rb_rank = nullptr;         // rebuild order: rank of each slot (k_rb_rank_sliced)
  int* ncol = nullptr;            // device count of live columns
  bool cols_reset = true;         // recompact the live columns at the next contraction
  BootScratch bs{};            // parallel bootstrap scratch
  size_t plan_smem = 0;        // k_plan dynamic shared memory
  ParCtl* parctl = nullptr;    // k_plan output (subtree-parallel resolve)
  long long kbatch = 1024;     // K1 rows per launch when k3par
  bool k3par = false;         // subtree-parallel resolve / reattach enabled
  int nper = 0;          // resolve kernel: 1..8 register rows, 100/101 shared-memory rows, 0 generic
  int nnew_cap = 0, rea_cap = 0;   // new-node table sizes of K3 and of the reattach
  int rea_cap_t = 0;               // reattach table with reference rows (no batch Gram)
  int rea_ts_cap = 0;              // entries of the Gram-scored table whose s rows stay in shared memory
  bool rea_gram = false;           // k_reattach2 takes new-entry dots from the batch Gram
  size_t rea_smem_t = 0, rea_smem_g = 0;
  size_t res_smem = 0, rea_smem = 0;
  std::vector<void*> allocs;

  template <class T> int alloc(T*& p, long long count) {
    void* q = nullptr;
    cudaError_t e = pcy_malloc_async_raw(&q, sizeof(T) * (size_t)(count > 0 ? count : 1), own);
    if (e != cudaSuccess) { pcy_set_error("cudaMallocAsync(%lld x %zu): %s", count, sizeof(T), cudaGetErrorString(e)); return PCY_ENOMEM; }
    allocs.push_back(q);
    p = (T*)q;
    return PCY_OK;
  }
  void release(void* p) {   // caller guarantees no pending use (it synchronised)
    for (auto& a : allocs) if (a == p) { cudaFreeAsync(a, own); a = nullptr; }
  }
  void touch(cudaStream_t st) { if (cudaEventRecord(done_ev, st) == cudaSuccess) done_rec = true; }
  ~Engine() {
#ifdef PCY_TIMELINE
    {   // build-time diagnostics: mean phase durations / gaps of the insertion windows (us)
      cudaDeviceSynchronize();
      unsigned int cnt = 0;
      cudaMemcpyFromSymbol(&cnt, g_tl_n, sizeof(cnt));
      if (cnt > PCY_TL_CAP) cnt = PCY_TL_CAP;
      std::vector<unsigned long long> h(cnt);
      if (cnt) cudaMemcpyFromSymbol(h.data(), g_tl, sizeof(unsigned long long) * cnt);
      const unsigned int zero = 0;
      cudaMemcpyToSymbol(g_tl_n, &zero, sizeof(zero));
      std::sort(h.begin(), h.end());
      double sum[8] = {}; long long num[8] = {};
      // transitions: 1->2 chain (+hop), 2->3 plan, 3->4 plan->resolve gap, 4->5 resolve, 5->1 resolve end -> next chain
      for (size_t i = 1; i < h.size(); ++i) {
        const int a = (int)(h[i - 1] & 15), b = (int)(h[i] & 15);
        const double dt = (double)((h[i] >> 4) - (h[i - 1] >> 4)) * 1e-3;
        int k = -1;
        if (a == 1 && b == 2) k = 0; else if (a == 2 && b == 3) k = 1; else if (a == 3 && b == 4) k = 2;
        else if (a == 4 && b == 5) k = 3; else if (a == 5 && b == 1) k = 4;
        if (k >= 0 && dt < 5000.0) { sum[k] += dt; ++num[k]; }
      }
      {
        unsigned int cc = 0;
        cudaMemcpyFromSymbol(&cc, g_tlc_n, sizeof(cc));
        if (cc > PCY_TL_CAP) cc = PCY_TL_CAP;
        std::vector<unsigned long long> hc(cc);
        if (cc) cudaMemcpyFromSymbol(hc.data(), g_tlc, sizeof(unsigned long long) * cc);
        cudaMemcpyToSymbol(g_tlc_n, &zero, sizeof(zero));
        // cycles by item-count bucket, and the slowest CTAs
        double cs[8] = {}, it[8] = {}, sl[8] = {}, nn[8] = {}; long long cn[8] = {};
        for (auto v : hc) {
          const long long items = v & 0xffff, nnew = (v >> 16) & 0xfff, slow = (v >> 28) & 0xfff, cyc = v >> 40;
          int b = items <= 2 ? 0 : items <= 4 ? 1 : items <= 8 ? 2 : items <= 12 ? 3 : items <= 16 ? 4 : items <= 24 ? 5 : items <= 48 ? 6 : 7;
          cs[b] += (double)cyc; it[b] += (double)items; sl[b] += (double)slow; nn[b] += (double)nnew; ++cn[b];
        }
        const char* bn[8] = {"<=2", "<=4", "<=8", "<=12", "<=16", "<=24", "<=48", ">48"};
        fprintf(stderr, "[timeline-cta] %u resolve CTAs:", cc);
        for (int b = 0; b < 8; ++b)
          if (cn[b]) fprintf(stderr, " | items %s: n %lld mean items %.1f new %.1f slow %.1f cycles %.0f", bn[b], cn[b], it[b] / cn[b], nn[b] / cn[b], sl[b] / cn[b], cs[b] / cn[b]);
        fprintf(stderr, "\n");
        unsigned long long ts[8][8];
        cudaMemcpyFromSymbol(ts, g_tls, sizeof(ts));
        unsigned long long tz[8][8] = {};
        cudaMemcpyToSymbol(g_tls, tz, sizeof(tz));
        fprintf(stderr, "[timeline-split]");
        for (int b = 0; b < 8; ++b)
          if (ts[b][0]) fprintf(stderr, " | items %s: wait %.0f slow %.0f start %.0f clean %.0f demand %.0f fast %.0f", bn[b], (double)ts[b][1] / ts[b][0], (double)ts[b][2] / ts[b][0],
                                (double)ts[b][3] / ts[b][0], (double)ts[b][4] / ts[b][0], (double)ts[b][5] / ts[b][0], (double)ts[b][6] / ts[b][0]);
        fprintf(stderr, "\n");
        unsigned long long t2[8][8];
        cudaMemcpyFromSymbol(t2, g_tls2, sizeof(t2));
        cudaMemcpyToSymbol(g_tls2, tz, sizeof(tz));
        fprintf(stderr, "[timeline-split2]");
        for (int b = 0; b < 8; ++b)
          if (ts[b][0]) fprintf(stderr, " | items %s: direct-scan %.0f (n %.1f) new-members %.0f (n %.1f) capacity %.0f levels %.1f clean %.1f", bn[b], (double)t2[b][1] / ts[b][0], (double)t2[b][4] / ts[b][0],
                                (double)t2[b][2] / ts[b][0], (double)t2[b][5] / ts[b][0], (double)t2[b][3] / ts[b][0], (double)t2[b][6] / ts[b][0], (double)t2[b][7] / ts[b][0]);
        fprintf(stderr, "\n");
      }
      {
        unsigned long long tr[8][8], tz2[8][8] = {};
        cudaMemcpyFromSymbol(tr, g_tlr, sizeof(tr));
        cudaMemcpyToSymbol(g_tlr, tz2, sizeof(tz2));
        const char* rb[8] = {"<=8", "<=16", "<=32", "<=64", "<=128", "<=256", "<=512", ">512"};
        fprintf(stderr, "[timeline-rea]");
        for (int b = 0; b < 8; ++b)
          if (tr[b][0]) fprintf(stderr, " | items %s: n %llu mean items %.1f cycles %.0f stage-wait %.0f adds %.1f levels %.1f scan %.0f", rb[b], tr[b][0], (double)tr[b][2] / tr[b][0],
                                (double)tr[b][1] / tr[b][0], (double)tr[b][3] / tr[b][0], (double)tr[b][4] / tr[b][0], (double)tr[b][5] / tr[b][0], (double)tr[b][6] / tr[b][0]);
        fprintf(stderr, "\n");
        unsigned long long t2[8][12], tz3[8][12] = {};
        cudaMemcpyFromSymbol(t2, g_tlr2, sizeof(t2));
        cudaMemcpyToSymbol(g_tlr2, tz3, sizeof(tz3));
        fprintf(stderr, "[timeline-rea2]");
        for (int b = 0; b < 8; ++b)
          if (tr[b][0]) {
            const double c = (double)tr[b][0];
            fprintf(stderr, " | items %s: dirscan n %.1f head cyc %.0f newscan n %.1f cyc %.0f merge rec %.1f glob %.1f smem %.1f cyc %.0f tail cyc %.0f", rb[b], t2[b][0] / c, t2[b][1] / c,
                    t2[b][2] / c, t2[b][3] / c, t2[b][4] / c, t2[b][5] / c, t2[b][6] / c, t2[b][7] / c, t2[b][8] / c);
          }
        fprintf(stderr, "\n");
      }
      {
        unsigned long long tp[10], tzp[10] = {};
        cudaMemcpyFromSymbol(tp, g_tlp, sizeof(tp));
        cudaMemcpyToSymbol(g_tlp, tzp, sizeof(tzp));
        const char* pn[10] = {"", "init", "pass1", "conflicts", "budget", "domains", "tickets", "balance", "ranks", "tail"};
        fprintf(stderr, "[timeline-plan] n %llu cycles:", tp[0]);
        for (int k = 1; k < 10; ++k) fprintf(stderr, " %s %.0f", pn[k], tp[0] ? (double)tp[k] / tp[0] : 0.0);
        fprintf(stderr, "\n");
      }
      const char* nm[5] = {"chain start->plan start", "plan", "plan end->resolve start", "resolve", "resolve end->next chain start"};
      fprintf(stderr, "[timeline] %u stamps, %lld run-ahead K1 launches", cnt, tl_early);
      for (int k = 0; k < 5; ++k) fprintf(stderr, " | %s: n %lld mean %.2f us total %.2f ms", nm[k], num[k], num[k] ? sum[k] / num[k] : 0.0, sum[k] * 1e-3);
      fprintf(stderr, "\n");
    }
#endif
    if (ctl_h) {
      g_counters[0] += ctl_h->cnt_levels; g_counters[1] += ctl_h->cnt_direct; g_counters[2] += ctl_h->cnt_demand;
      g_counters[3] += ctl_h->cnt_slow; g_counters[4] += ctl_h->cnt_items;
      long long md = g_counters[5].load();
      while (ctl_h->max_depth > md && !g_counters[5].compare_exchange_weak(md, ctl_h->max_depth)) {}
    }
    if (own && done_rec) cudaStreamWaitEvent(own, done_ev, 0);
    for (void* a : allocs) if (a) cudaFreeAsync(a, own);
    if (hi) cudaStreamDestroy(hi);
    if (evk1) cudaEventDestroy(evk1);
    if (evk3) cudaEventDestroy(evk3);
    for (auto& e : ev) if (e) cudaEventDestroy(e);
    if (done_ev) cudaEventDestroy(done_ev);
    if (own) cudaStreamDestroy(own);
    if (ctl_h) ctl_pool_put(ctl_h);
  }

  // Publish the device counters into the mapped host mirror and spin on its
  // sequence number: no stream synchronisation, no wake-up latency.
  int sync_ctl(cudaStream_t st) {
    const long long want = ++seq;
    if (panel) k_publish_panel<<<1, 1024, 0, st>>>(E, ctl_map_d, want);
    else k_publish<<<1, 32, 0, st>>>(E.ctl, ctl_map_d, want, E.g_count, E.g_base);
    pcy_count_launch();
    PCY_LAUNCH_CHECK();
    return wait_seq(st, want);
  }
  // The window kernels publish themselves while no group is in the K1 panel
  // (k_resolve2x & co.); the panel publication is a separate launch.
  bool self_publish() const { return !panel || ctl_h->maxg < PCY_PANEL_MIN; }
  // k_plan's early publication (mirror words after `seq`)
  int wait_plan(cudaStream_t st, long long want) {
    volatile long long* sp = &ctl_h->plan_seq;
    for (long long spins = 0; *sp != want; ++spins) {
      if ((spins & 1023) == 1023) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e != cudaSuccess && e != cudaErrorNotReady) {
          pcy_set_error("engine kernel failed: %s", cudaGetErrorString(e));
          return PCY_ECUDA;
        }
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return PCY_OK;
  }
  int wait_seq(cudaStream_t st, long long want) {
    volatile long long* sp = &ctl_h->seq;
    for (long long spins = 0; *sp != want; ++spins) {
      if ((spins & 1023) == 1023) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e != cudaSuccess && e != cudaErrorNotReady) {
          pcy_set_error("engine kernel failed: %s", cudaGetErrorString(e));
          return PCY_ECUDA;
        }
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return PCY_OK;
  }

  int init(int device, int dim, long long budget, long long bootstrap_cap, long long block_rows) {
    dev = device; d = dim; m = budget;
    ld = (int)pcy_round_up(d, 4);
    sample_cap = budget + 1 < bootstrap_cap ? budget + 1 : bootstrap_cap;
    NC = m + 2; GC = NC + 2; AC = 24 * NC + 4096;
    // rows staged per block: windows run ahead of the host only inside a
    // block, so small-d engines stage whole pieces (about 64 MB of rows)
    if (block_rows > 0) Bmax = block_rows;
    else {
      const long long fit = ((long long)64 << 20) / (8LL * ld);
      Bmax = fit < 4096 ? 4096 : fit > 16384 ? 16384 : fit / 1024 * 1024;
    }
    PCY_CUDA(cudaSetDevice(dev));
    PCY_CUDA(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
    PCY_CUDA(cudaEventCreateWithFlags(&done_ev, cudaEventDisableTiming));
    PCY_CUDA(cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    PCY_CUDA(cudaFuncSetAttribute(k_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    PCY_CUDA(cudaFuncSetAttribute(k_rb_reattach, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    E.d = d; E.ld = ld; E.m = m; E.NC = NC; E.GC = GC; E.AC = AC;
    int rc;
#define A_(p, n) if ((rc = alloc(p, n))) return rc
    A_(E.w, NC); A_(E.q, NC); A_(E.sn, NC); A_(E.rn, NC); A_(E.idx, NC);
    A_(E.child, NC); A_(E.alive, NC); A_(E.free_ids, NC);
    A_(E.fs_list, NC); A_(E.fs_gofs, GC); A_(E.fs_cnt, 1);
    { int* co = nullptr; A_(co, NC); E.col_of = co; }
    A_(col_slot, NC); A_(ncol, 1); A_(tc_done, NC); A_(rb_rank, NC);
    A_(E.pathj, Bmax * 16);
    A_(E.s, NC * ld); A_(E.r, NC * ld);
    A_(E.g_base, GC); A_(E.g_count, GC); A_(E.g_cap, GC); A_(E.g_bs, GC); A_(E.g_bsbase, GC);
    A_(E.arena, AC);
    A_(E.ctl, 1);
    A_(E.xb, Bmax * ld); A_(E.xsq, Bmax); A_(E.wb, Bmax); A_(E.hsh, Bmax); A_(E.bad, Bmax);
    A_(E.ch_node, Bmax * PCY_MAXL); A_(E.ch_part, Bmax * PCY_MAXL); A_(E.ch_len, Bmax);
    A_(chh, Bmax); A_(chr, Bmax * PCY_FMAXL);
    A_(gram, (long long)1024 * 1024);
    A_(gram_b, (long long)1024 * 1024);
    gram_split = d >= 2048 ? 8 : d >= 512 ? 4 : 1;   // K slices of >= 128-512 elements
    if (gram_split > 1) A_(gram_part, (long long)gram_split * 1024 * 1024);
    E.pend_cap = m + 2;
    A_(E.pend_x, E.pend_cap * ld); A_(E.pend_w, E.pend_cap); A_(E.pend_xsq, E.pend_cap);
    A_(E.dist_x, (m + 2) * ld);
    E.hcap = 1; while (E.hcap < 2 * (m + 2)) E.hcap <<= 1;
    A_(E.htab, E.hcap);
    A_(E.order, NC); A_(E.lvl, NC); A_(E.stk_g, NC + 1); A_(E.stk_p, NC + 1);
    A_(E.minbits, 2);
    A_(aggw, m + 2); A_(mp_nrm, sample_cap + 1);
    bs.scap = 1; while (bs.scap < 2 * Bmax) bs.scap <<= 1;
    A_(bs.flags, Bmax + 1); A_(bs.spos, Bmax); A_(bs.ppos, Bmax); A_(bs.dpos, Bmax); A_(bs.skey, bs.scap); A_(bs.sfirst, bs.scap);
    A_(parctl, 1);
#undef A_
    PCY_CUDA(cudaMemsetAsync(parctl, 0, sizeof(ParCtl), own));   // ParCtl::ready starts below every launch number
    for (auto& e : ev) PCY_CUDA(cudaEventCreate(&e));
    {
      int least = 0, greatest = 0;
      PCY_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
      PCY_CUDA(cudaStreamCreateWithPriority(&hi, cudaStreamNonBlocking, greatest));
      PCY_CUDA(cudaEventCreateWithFlags(&evk1, cudaEventDisableTiming));
      PCY_CUDA(cudaEventCreateWithFlags(&evk3, cudaEventDisableTiming));
    }
    {
      use_tc = d >= 256;
      Kp = pcy_tc_pad(d);
      tc_tau = pcy_tc_error_tau(Kp);
    }
    const size_t maxsm = 227 * 1024;
    PCY_CUDA(cudaFuncSetAttribute(k_chain2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    PCY_CUDA(cudaFuncSetAttribute(k_chain2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    PCY_CUDA(cudaFuncSetAttribute(k_rchain, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    if (ld <= 256 && !getenv("PCY_SMEM_RESOLVE")) {
      nper = ld <= 32 ? 1 : ld <= 64 ? 2 : ld <= 128 ? 4 : 8;
      const size_t base = resolve_smem_bytes(ld, 0, NC, GC);
      long long cap = maxsm > base ? (long long)((maxsm - base) / (sizeof(double) * (2 * ld + 1))) : 0;
      if (cap > PCY_NNEW_FAST) cap = PCY_NNEW_FAST;
      nnew_cap = (int)cap;
      res_smem = resolve_smem_bytes(ld, nnew_cap, NC, GC);
      // reattach table: with the batch Gram (subtree-parallel mode) the new
      // entries need no reference rows in shared memory; without it they do
      const size_t rbase = reattach_smem_bytes(ld, 0, NC, GC);
      long long rcap = maxsm > rbase ? (long long)((maxsm - rbase) / (sizeof(double) * (ld | 1))) : 0;
      if (rcap > PCY_NNEW_REA) rcap = PCY_NNEW_REA;
      rea_cap_t = (int)rcap;
      rea_smem_t = reattach_smem_bytes(ld, rea_cap_t, NC, GC);
      rea_smem_g = reattach_smem_bytes(ld, PCY_NNEW_REA, NC, GC, false);
      {   // s rows of the first entries in what is left of shared memory
        const long long left = maxsm > rea_smem_g ? (long long)((maxsm - rea_smem_g) / (sizeof(double) * ld)) : 0;
        rea_ts_cap = (int)(left > PCY_NNEW_REA ? PCY_NNEW_REA : left);
        rea_smem_g += sizeof(double) * (size_t)ld * rea_ts_cap;
      }
      rea_cap = rea_cap_t;
      rea_smem = rea_smem_t > rea_smem_g ? rea_smem_t : rea_smem_g;   // attribute: either variant fits
      if (nnew_cap < 8) { nper = 0; use_tc = false; }
      switch (nper) {
        case 1: PCY_CUDA(cudaFuncSetAttribute(k_resolve2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_resolve2x<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_reattach2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_reattach2x<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem)); break;
        case 2: PCY_CUDA(cudaFuncSetAttribute(k_resolve2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_resolve2x<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_reattach2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_reattach2x<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem)); break;
        case 4: PCY_CUDA(cudaFuncSetAttribute(k_resolve2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_resolve2x<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_reattach2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_reattach2x<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem)); break;
        case 8: PCY_CUDA(cudaFuncSetAttribute(k_resolve2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_resolve2x<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_reattach2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem));
                PCY_CUDA(cudaFuncSetAttribute(k_reattach2x<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem)); break;
        default: break;
      }
    }
    if (!nper) {
      // rows in shared memory, any dimension
      const size_t base_t = resolve3_smem_bytes<2048>(ld, 0, true, NC, GC, 2);
      long long cap = maxsm > base_t ? (long long)((maxsm - base_t) / (sizeof(double) * (2 * ld + 1))) : 0;
      if (cap > PCY_NNEW_MAX) cap = PCY_NNEW_MAX;
      if (cap >= 16) {
        nper = 100; nnew_cap = (int)cap;
        res_smem = resolve3_smem_bytes<2048>(ld, nnew_cap, true, NC, GC, 0);
        rea_smem = resolve3_smem_bytes<2048>(ld, nnew_cap, true, NC, GC, 2);
        PCY_CUDA(cudaFuncSetAttribute(k_resolve3<true, 2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
        PCY_CUDA(cudaFuncSetAttribute(k_reattach3<true, 2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem));
        PCY_CUDA(cudaFuncSetAttribute(k_resolve3x<true, 2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
        PCY_CUDA(cudaFuncSetAttribute(k_reattach3x<true, 2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem));
      } else if (resolve3_smem_bytes<512>(ld, 0, false, NC, GC, 2) <= maxsm) {
        nper = 101; nnew_cap = PCY_NNEW_MAX;
        res_smem = resolve3_smem_bytes<512>(ld, 0, false, NC, GC, 0);
        rea_smem = resolve3_smem_bytes<512>(ld, 0, false, NC, GC, 2);
        PCY_CUDA(cudaFuncSetAttribute(k_resolve3<false, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
        PCY_CUDA(cudaFuncSetAttribute(k_reattach3<false, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem));
        PCY_CUDA(cudaFuncSetAttribute(k_resolve3x<false, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)res_smem));
        PCY_CUDA(cudaFuncSetAttribute(k_reattach3x<false, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)rea_smem));
      }
    }
    plan_smem = plan_smem_bytes((int)(NC / 32 + 1));
    {
      const char* pe = getenv("PCY_K3PAR");
      k3par = nper >= 1 && (!pe || atoi(pe) != 0) && plan_smem <= maxsm;
      if (k3par) PCY_CUDA(cudaFuncSetAttribute(k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan_smem));
      if (nper >= 1 && nper <= 8) {
        const bool g = k3par;
        rea_cap = g ? PCY_NNEW_REA : rea_cap_t;
        rea_smem = g ? rea_smem_g : rea_smem_t;
        rea_gram = g;
      }
    }
    // visited-groups K1 for d <= 256: small groups by direct fp64 scans, groups
    // of >= PCY_PANEL_MIN members by a tcgen05 split-TF32 panel contraction
    panel = nper >= 1 && nper <= 8 && !use_tc;
    E.panel_gofs = panel ? E.fs_gofs : nullptr;
    if (!(ctl_h = ctl_pool_get())) { pcy_set_error("cudaHostAlloc of the control mirror failed"); return PCY_ENOMEM; }
    memset(ctl_h, 0, sizeof(EngCtl));
    PCY_CUDA(cudaHostGetDevicePointer((void**)&ctl_map_d, ctl_h, 0));
    PCY_CUDA(cudaMemcpyAsync(E.ctl, ctl_h, sizeof(EngCtl), cudaMemcpyHostToDevice, own));
    PCY_CUDA(cudaMemsetAsync(E.htab, 0xff, sizeof(int) * E.hcap, own));
    PCY_CUDA(cudaMemsetAsync(E.alive, 0, sizeof(int) * NC, own));
    PCY_CUDA(cudaMemsetAsync(E.g_count, 0, sizeof(int) * GC, own));
    PCY_CUDA(cudaMemsetAsync(E.g_base, 0, sizeof(int) * GC, own));
    PCY_CUDA(cudaMemsetAsync(E.fs_gofs, 0xff, sizeof(int) * GC, own));
    PCY_CUDA(cudaMemsetAsync(E.s, 0, sizeof(double) * NC * ld, own));
    PCY_CUDA(cudaMemsetAsync(E.r, 0, sizeof(double) * NC * ld, own));
    PCY_CUDA(cudaStreamSynchronize(own));   // buffers ready for any stream
    return PCY_OK;
  }

  // Full-set K1: one DMMA contraction of the block against every allocated
  // reference slot gives the parts matrix; the chain walk then only gathers
  // parts of the visited groups' members.  Used once the tree is large.
  bool full_set(const double* A, const int* aidx, long long M, cudaStream_t st, int* rc) {
    *rc = PCY_OK;
    E.tc_dots = nullptr;
    if (panel) {   // visited-groups K1: only the big groups' members are contracted
      const long long NP = ctl_h->panel_n;   // published with the tree this launch walks
      if (NP <= 0) return false;
      const long long acap = 1024, bcap = (NC + 127) / 128 * 128;
      if (!tc_dots) {
        if ((*rc = alloc(tc_ahi, acap * Kp)) || (*rc = alloc(tc_alo, acap * Kp)) || (*rc = alloc(tc_bhi, bcap * Kp)) ||
            (*rc = alloc(tc_blo, bcap * Kp)) || (*rc = alloc(tc_dots, acap * NC)) || (*rc = alloc(tc_rnc, NC)) ||
            (*rc = alloc(tc_xn2, acap)) || (*rc = alloc(tc_c, (long long)Kp)))
          return false;
        if (cudaMemsetAsync(tc_bhi, 0, sizeof(float) * bcap * Kp, st) != cudaSuccess ||
            cudaMemsetAsync(tc_blo, 0, sizeof(float) * bcap * Kp, st) != cudaSuccess ||
            cudaMemsetAsync(tc_ahi, 0, sizeof(float) * acap * Kp, st) != cudaSuccess ||
            cudaMemsetAsync(tc_alo, 0, sizeof(float) * acap * Kp, st) != cudaSuccess) {
          pcy_set_error("tc buffer init failed"); *rc = PCY_ECUDA; return false;
        }
        if ((*rc = pcy_tc_center(A, aidx, ld, d, tc_c, st))) return false;   // the engine's centre
      }
      if ((*rc = pcy_tc_split(A, aidx, ld, d, M, nullptr, tc_c, tc_ahi, tc_alo, tc_xn2, st))) return false;
      if ((*rc = pcy_tc_split(E.r, E.fs_list, ld, d, NP, nullptr, tc_c, tc_bhi, tc_blo, tc_rnc, st))) return false;
      const bool prof = pcy_prof_enabled();
      if (prof) PCY_CUDA(cudaEventRecord(ev[6], st));
      if ((*rc = pcy_tc_dots(tc_ahi, tc_alo, acap, (int)M, tc_bhi, tc_blo, bcap, (int)NP, nullptr, Kp, tc_dots, NP, st)))
        return false;
      if (prof) { PCY_CUDA(cudaEventRecord(ev[7], st)); gemm_timed = true; gemm_flops = 2.0 * (double)M * (double)NP * d; }
      exec_tensor_flops += 3.0 * 2.0 * (double)((M + 127) / 128 * 128) * (double)((NP + 127) / 128 * 128) * Kp;
      ++panel_launches;
      E.tc_dots = tc_dots; E.tc_ldo = NP; E.tc_rnc = tc_rnc; E.tc_xn2 = tc_xn2; E.tc_tau = tc_tau;
      return false;
    }
    const long long N = ctl_h->F_alloc;   // upper bound on the live columns (device count in ncol)
    if (!nper || N < 256) return false;
    if (cols_reset) {   // recompact: every live node takes a fresh column below
      if (cudaMemsetAsync(tc_done, 0xff, sizeof(long long) * NC, st) != cudaSuccess ||
          cudaMemsetAsync(ncol, 0, sizeof(int), st) != cudaSuccess) {
        pcy_set_error("live-column reset failed"); *rc = PCY_ECUDA; return false;
      }
      cols_reset = false;
    }
    if (use_tc) {
      // tensor cores: split-TF32 dots against the reference slots.  The slots
      // keep their split (fixed engine centre, re-split only when a slot gets a
      // new reference), so a launch splits only the block rows.
      if (!tc_dots) {
        const long long acap = 1024, bcap = (NC + 127) / 128 * 128;
        if ((*rc = alloc(tc_ahi, acap * Kp)) || (*rc = alloc(tc_alo, acap * Kp)) || (*rc = alloc(tc_bhi, bcap * Kp)) ||
            (*rc = alloc(tc_blo, bcap * Kp)) || (*rc = alloc(tc_dots, acap * NC)) || (*rc = alloc(tc_rnc, NC)) ||
            (*rc = alloc(tc_xn2, acap)) || (*rc = alloc(tc_c, (long long)Kp)))
          return false;
        if (cudaMemsetAsync(tc_bhi, 0, sizeof(float) * bcap * Kp, st) != cudaSuccess ||
            cudaMemsetAsync(tc_blo, 0, sizeof(float) * bcap * Kp, st) != cudaSuccess) {
          pcy_set_error("tc buffer init failed"); *rc = PCY_ECUDA; return false;
        }
        if ((*rc = pcy_tc_center(A, aidx, ld, d, tc_c, st))) return false;   // the engine's centre
      }
      if ((*rc = pcy_tc_split(A, aidx, ld, d, M, nullptr, tc_c, tc_ahi, tc_alo, tc_xn2, st))) return false;
      if ((*rc = pcy_tc_split_slots(E.r, ld, d, N, E.alive, E.idx, tc_done, tc_c, tc_bhi, tc_blo, tc_rnc,
                                    const_cast<int*>(E.col_of), col_slot, ncol, st)))
        return false;
      const bool prof = pcy_prof_enabled();
      if (prof) PCY_CUDA(cudaEventRecord(ev[6], st));
      if ((*rc = pcy_tc_dots(tc_ahi, tc_alo, 1024, (int)M, tc_bhi, tc_blo, (NC + 127) / 128 * 128, (int)N, ncol,
                             Kp, tc_dots, N, st)))
        return false;
      if (prof) { PCY_CUDA(cudaEventRecord(ev[7], st)); gemm_timed = true; gemm_flops = 2.0 * (double)M * (double)N * d; }
      exec_tensor_flops += 3.0 * 2.0 * (double)((M + 127) / 128 * 128) * (double)((N + 127) / 128 * 128) * Kp;
      ++panel_launches;
      E.tc_dots = tc_dots; E.tc_ldo = N; E.tc_rnc = tc_rnc; E.tc_xn2 = tc_xn2; E.tc_tau = tc_tau;
      return false;   // no fp64 parts matrix: K1 reads E.tc_dots
    }
    if (!parts) { if ((*rc = alloc(parts, (long long)1024 * NC))) return false; }
    const bool prof = pcy_prof_enabled();
    if (prof) { cudaEventRecord(ev[6], st); }
    // columns = live columns (B rows gathered through col_slot; CTAs past ncol exit)
    k_assign_cols<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(E.alive, E.idx, N, tc_done, const_cast<int*>(E.col_of),
                                                               col_slot, ncol);
    pcy_count_launch();
    *rc = pcy_launch_parts(A, aidx, ld, (int)M, E.r, col_slot, ld, E.rn, (int)N, ncol, d, parts, N, st);
    if (prof) { cudaEventRecord(ev[7], st); gemm_timed = true; gemm_flops = 2.0 * (double)M * (double)N * d; }
    return true;
  }

  int grow_pending(cudaStream_t st) {
    const long long nc = E.pend_cap * 2;
    double *nx = nullptr, *nq = nullptr; long long* nw = nullptr;
    int rc;
    if ((rc = alloc(nx, nc * ld)) || (rc = alloc(nw, nc)) || (rc = alloc(nq, nc))) return rc;
    PCY_CUDA(cudaMemcpyAsync(nx, E.pend_x, sizeof(double) * E.pend_cap * ld, cudaMemcpyDeviceToDevice, st));
    PCY_CUDA(cudaMemcpyAsync(nw, E.pend_w, sizeof(long long) * E.pend_cap, cudaMemcpyDeviceToDevice, st));
    PCY_CUDA(cudaMemcpyAsync(nq, E.pend_xsq, sizeof(double) * E.pend_cap, cudaMemcpyDeviceToDevice, st));
    PCY_CUDA(pcy_spin_sync(st));
    release(E.pend_x); release(E.pend_w); release(E.pend_xsq);
    E.pend_x = nx; E.pend_w = nw; E.pend_xsq = nq; E.pend_cap = nc;
    return PCY_OK;
  }

  int rebuild(cudaStream_t st) {
    // precondition: ctl_h mirrors the device counters
    while (ctl_h->F > m) {
      const long long nslots = ctl_h->F_alloc;
      const long long nodes = ctl_h->F;
      if (nslots >= 4096) {   // one thread per node is too few CTAs: slice the candidates
        PCY_CUDA(cudaMemsetAsync(rb_rank, 0, sizeof(int) * nslots, st));
        k_rb_rank_sliced<<<dim3((unsigned)((nslots + 255) / 256), RB_SLICES), 256, 0, st>>>(E, nslots, rb_rank);
        pcy_count_launch();
        k_rb_scatter<<<(unsigned)((nslots + 255) / 256), 256, 0, st>>>(E, nslots, rb_rank); pcy_count_launch();
      } else {
        k_rb_rank<<<(unsigned)((nslots + 255) / 256), 256, 0, st>>>(E, nslots); pcy_count_launch();
      }
      k_rb_reset<<<(unsigned)((nslots + 255) / 256), 256, 0, st>>>(E, nslots); pcy_count_launch();
      ctl_h->root_count = 0;   // fresh roots; the mirror refreshes at the next publication
      if (panel) {   // the reattach K1 needs the panel of the emptied tree
        // no group is listed until one reaches the panel size again (the
        // publications in between are skipped, see self_publish)
        PCY_CUDA(cudaMemsetAsync(E.fs_gofs, 0xff, sizeof(int) * GC, st));
        const int prc = sync_ctl(st);
        if (prc) return prc;
      }
      const bool prof = pcy_prof_enabled();
      if (prof) PCY_CUDA(cudaEventRecord(ev[3], st));
      int rc;
      if (nper) {
        // K1 rows per reattach launch, adapted to where launches stop.  The
        // first launches meet an empty tree (one domain: every node is a root
        // or competes for one), so they stay short until roots exist.
        long long off = 0, batch = k3par ? 64 : 1024;
        const int wpc = ld <= 512 ? 8 : (ld <= 2048 ? 4 : 2);
        while (off < nodes) {
          const long long nb = nodes - off < batch ? nodes - off : batch;
          int grc;
          // the batch Gram depends only on the batch's references: a side
          // stream computes it beside the contraction and the chain walk
          const bool gram_early = k3par && nper <= 8 && hi;   // small d only: at large d the Gram competes with the K1 contraction
          if (gram_early) {
            PCY_CUDA(cudaEventRecord(evk1, st)); PCY_CUDA(cudaStreamWaitEvent(hi, evk1, 0));
            grc = pcy_launch_gram_split(E.r, E.order + off, ld, (int)nb, d, gram, nb, gram_part, gram_split, hi);
            if (grc) return grc;
            PCY_CUDA(cudaEventRecord(evk3, hi));
          }
          const bool use_p = full_set(E.r, E.order + off, nb, st, &grc);
          if (grc) return grc;
          k_rchain<<<(unsigned)((nb + wpc - 1) / wpc), wpc * 32, sizeof(double) * wpc * ld, st>>>(
              E, E.order + off, nb, chh, chr, use_p ? parts : nullptr, ctl_h->F_alloc); pcy_count_launch();
          if (nper == 101 && !gram_early) {
            grc = pcy_launch_gram_split(E.r, E.order + off, ld, (int)nb, d, gram, nb, gram_part, gram_split, st);
            if (grc) return grc;
          }
          if (gram_early) PCY_CUDA(cudaStreamWaitEvent(st, evk3, 0));
          ParCtl* pp = nullptr;
          bool selfp = false; long long pseq = 0;
          const double* rg = rea_gram ? gram : nullptr;   // the batch Gram exists exactly when k3par
          if (k3par) {
            if (nper != 101 && !gram_early) {   // opener rows against the batch (k_plan's conflict test)
              grc = pcy_launch_gram_split(E.r, E.order + off, ld, (int)nb, d, gram, nb, gram_part, gram_split, st);
              if (grc) return grc;
            }
            k_plan<<<1, PCY_PAR_MAXITEMS, plan_smem, st>>>(E, nullptr, nullptr, nullptr, nb, -1, nper <= 8 ? rea_cap : nnew_cap,
                                                   16, chh, chr, parctl, (int)(NC / 32 + 1), E.order + off,
                                                   gram, nb, nullptr, 0);
            pcy_count_launch();
            pp = parctl;
            // one launch serves either choice of k_plan and, while no group is
            // in the K1 panel, publishes the counters itself
            selfp = self_publish();
            pseq = selfp ? ++seq : 0;
            EngCtl* pb = selfp ? ctl_map_d : nullptr;
            switch (nper) {
              case 1: k_reattach2x<1><<<PCY_PAR_MAXCTA, 32, rea_smem, st>>>(E, E.order + off, nb, rea_cap, chh, chr, pp, rg, nb, pb, pseq, rg ? rea_ts_cap : 0); break;
              case 2: k_reattach2x<2><<<PCY_PAR_MAXCTA, 32, rea_smem, st>>>(E, E.order + off, nb, rea_cap, chh, chr, pp, rg, nb, pb, pseq, rg ? rea_ts_cap : 0); break;
              case 4: k_reattach2x<4><<<PCY_PAR_MAXCTA, 32, rea_smem, st>>>(E, E.order + off, nb, rea_cap, chh, chr, pp, rg, nb, pb, pseq, rg ? rea_ts_cap : 0); break;
              case 8: k_reattach2x<8><<<PCY_PAR_MAXCTA, 32, rea_smem, st>>>(E, E.order + off, nb, rea_cap, chh, chr, pp, rg, nb, pb, pseq, rg ? rea_ts_cap : 0); break;
              case 100: k_reattach3x<true, 2048><<<PCY_PAR_MAXCTA, 32, rea_smem, st>>>(E, E.order + off, nb, nnew_cap, chh, chr, nullptr, 0, 0, pp, pb, pseq); break;
              default: k_reattach3x<false, 512><<<PCY_PAR_MAXCTA, 32, rea_smem, st>>>(E, E.order + off, nb, nnew_cap, chh, chr, gram, nb, 0, pp, pb, pseq); break;
            }
            pcy_count_launch();
          } else {
            switch (nper) {
              case 1: k_reattach2<1><<<1, 32, rea_smem, st>>>(E, E.order + off, nb, rea_cap, chh, chr, pp, rg, nb); break;
              case 2: k_reattach2<2><<<1, 32, rea_smem, st>>>(E, E.order + off, nb, rea_cap, chh, chr, pp, rg, nb); break;
              case 4: k_reattach2<4><<<1, 32, rea_smem, st>>>(E, E.order + off, nb, rea_cap, chh, chr, pp, rg, nb); break;
              case 8: k_reattach2<8><<<1, 32, rea_smem, st>>>(E, E.order + off, nb, rea_cap, chh, chr, pp, rg, nb); break;
              case 100: k_reattach3<true, 2048><<<1, 32, rea_smem, st>>>(E, E.order + off, nb, nnew_cap, chh, chr, nullptr, 0, 0, pp); break;
              default: k_reattach3<false, 512><<<1, 32, rea_smem, st>>>(E, E.order + off, nb, nnew_cap, chh, chr, gram, nb, 0, pp); break;
            }
            pcy_count_launch();
          }
          PCY_LAUNCH_CHECK();
          rc = selfp ? wait_seq(st, pseq) : sync_ctl(st); if (rc) return rc;
          if (selfp && !self_publish()) { rc = sync_ctl(st); if (rc) return rc; }   // a group reached the panel size
          if (ctl_h->status == ST_ARENA) { pcy_set_error("member arena exhausted in rebuild"); return PCY_ESTATE; }
          if (ctl_h->status == ST_PAR_BROKEN) {
            pcy_set_error("subtree-parallel reattach met an excluded stop (inner status %d, window %lld, F %lld, m %lld)",
                          ctl_h->err, ctl_h->stop, ctl_h->F, m);
            return PCY_ESTATE;
          }
#ifdef PCY_TRACE
          {   // build-time diagnostics only (PCY_NVCC_EXTRA=-DPCY_TRACE)
            int pm[2] = {-1, 0};
            if (k3par) cudaMemcpy(pm, parctl, sizeof(pm), cudaMemcpyDeviceToHost);
            fprintf(stderr, "[rea] nodes %lld off %lld nb %lld status %d stop %lld mode %d P %d\n", nodes, off, nb,
                    ctl_h->status, ctl_h->stop, pm[0], pm[1]);
          }
#endif
          if (ctl_h->status == ST_FULL) {
            if (ctl_h->stop == 0) { pcy_set_error("reattach made no progress"); return PCY_ESTATE; }
            off += ctl_h->stop;
            batch = std::min<long long>(1024, std::max<long long>(128, 2 * ctl_h->stop));
          } else {
            off += nb;
            batch = batch * 4 > 1024 ? 1024 : batch * 4;
          }
        }
      } else {
        k_rb_reattach<<<1, 512, sizeof(double) * ld, st>>>(E, nodes); pcy_count_launch();
      }
      if (prof) PCY_CUDA(cudaEventRecord(ev[4], st));
      cols_reset = true;   // merged nodes left dead columns
      PCY_LAUNCH_CHECK();
      rc = sync_ctl(st); if (rc) return rc;
      if (ctl_h->status == ST_ARENA) { pcy_set_error("member arena exhausted in rebuild"); return PCY_ESTATE; }
      if (prof) {
        float t = 0.f;
        PCY_CUDA(cudaEventElapsedTime(&t, ev[3], ev[4]));
        pcy_prof_add(PCY_PROF_REATTACH, t, nodes);
      }
      if (ctl_h->status == ST_ARENA) { pcy_set_error("member arena exhausted in rebuild"); return PCY_ESTATE; }
    }
    return PCY_OK;
  }

  // Live insertion of rows X (engine layout, stride ld) with x_sq XS, weights W
  // (nullable = unit), validation codes BAD (nullable).  Returns PCY_OK and
  // sets *bad_at = -1, or the index of the first invalid row.
  int live(const double* X, const double* XS, const long long* W, const int* BAD, long long n,
           int countw, cudaStream_t st, long long* bad_at, int* bad_code) {
    *bad_at = -1;
    const int wpc = ld <= 512 ? 8 : (ld <= 2048 ? 4 : 2);
    const bool gram_early = k3par && nper <= 8 && hi;   // small d only: at large d the Gram competes with the K1 contraction
    // K1 of rows [s0, s0 + kn): the batch Gram for k_plan's open-conflict test
    // (it depends only on the rows: on the K3 stream, beside the chain walk),
    // the panel contraction and the chain walk.  Nothing here needs the host
    // to know the tree (the panel size is the last publication's).
    // The batch Grams alternate between two buffers: with `ahead` (run-ahead
    // batch) the side stream waits only for the event recorded before the
    // current window's k_plan -- the buffer's last reader is the k_plan before
    // that one -- so nothing sits between the resolve kernel and this chain
    // walk in the stream and the walk is launched programmatically.
    double* gram_k1 = gram;   // the buffer of the batch enqueued last
    auto enqueue_k1 = [&](long long s0, long long kn, bool prof, bool ahead, long long wait_seq) -> int {
      const double* Xs = X + s0 * ld;
      const double* XSs = XS + s0;
      const long long* Ws = W ? W + s0 : nullptr;
      if (!nper) { k_snapshot<<<64, 256, 0, st>>>(E); pcy_count_launch(); }
      if (prof) PCY_CUDA(cudaEventRecord(ev[0], st));
      if (gram_early) {
        gram_flip ^= 1;
        gram_k1 = gram_flip ? gram_b : gram;
        if (!ahead) PCY_CUDA(cudaEventRecord(evk1, st));
        PCY_CUDA(cudaStreamWaitEvent(hi, evk1, 0));
        const int grc = pcy_launch_gram_split(Xs, nullptr, ld, (int)kn, d, gram_k1, kn, gram_part, gram_split, hi);
        if (grc) return grc;
        PCY_CUDA(cudaEventRecord(evk3, hi));   // k_plan waits for it
      }
      if (nper) {
        int grc;
        const bool use_p = full_set(Xs, nullptr, kn, st, &grc);
        if (grc) return grc;
        if (ld > 512)   // one item per CTA, dots split over 4 warps
          k_chain2<4><<<(unsigned)(kn), 128, sizeof(double) * (ld + 8) + sizeof(int) * (TC_CAND_MAX + 4), st>>>(
              E, Xs, XSs, Ws, kn, chh, chr, use_p ? parts : nullptr, ctl_h->F_alloc);
        else if (ahead)
          PCY_CUDA(launch_pdl(k_chain2<1>, dim3((unsigned)((kn + wpc - 1) / wpc)), dim3(wpc * 32), sizeof(double) * wpc * ld, st,
                              E, Xs, XSs, Ws, kn, chh, chr, (const double*)(use_p ? parts : nullptr), (long long)ctl_h->F_alloc, wait_seq));
        else
          k_chain2<1><<<(unsigned)((kn + wpc - 1) / wpc), wpc * 32, sizeof(double) * wpc * ld, st>>>(
              E, Xs, XSs, Ws, kn, chh, chr, use_p ? parts : nullptr, ctl_h->F_alloc);
        pcy_count_launch();
        if (nper == 101 && !gram_early) {
          const int grc2 = pcy_launch_gram_split(Xs, nullptr, ld, (int)(kn), d, gram, kn, gram_part, gram_split, st);
          if (grc2) return grc2;
        }
      } else {
        k_chain<<<(unsigned)((kn + wpc - 1) / wpc), wpc * 32, sizeof(double) * wpc * ld, st>>>(E, Xs, XSs, kn); pcy_count_launch();
      }
      PCY_LAUNCH_CHECK();
      return PCY_OK;
    };
    long long off = 0;
    while (off < n) {
      // without the subtree-parallel planner one K3 launch absorbs about 1024 items
      const long long sub = k3par ? n : (nper ? (long long)1024 : Bmax);
      const long long nb = n - off < sub ? n - off : sub;
      long long start = 0, first_rem = -1;
      long long k1_kn = 0;   // > 0: K1 of rows [start, start + k1_kn) is already enqueued
      while (start < nb) {
        // K1 chains kn rows; with the subtree-parallel resolve the batch follows
        // where the windows stop, so rows are not re-chained many times
        const long long kn = k1_kn > 0 ? k1_kn : (k3par && nb - start > kbatch ? kbatch : nb - start);
        const double* Xs = X + (off + start) * ld;
        const double* XSs = XS + off + start;
        const bool prof = pcy_prof_enabled();
        const long long* Ws = W ? W + off + start : nullptr;
        const int* Bs = BAD ? BAD + off + start : nullptr;
        if (k1_kn == 0) { const int rc1 = enqueue_k1(off + start, kn, prof, false, 0); if (rc1) return rc1; }
        k1_kn = 0;
        double* const gram_w = gram_early ? gram_k1 : gram;   // this window's batch Gram
        // K1, k_plan and the resolve kernel share the caller's stream (no
        // cross-stream hop on the window's critical path); only the batch Gram
        // runs beside the chain walk on the side stream
        cudaStream_t rs = st;
        if (gram_early) {
          PCY_CUDA(cudaStreamWaitEvent(st, evk3, 0));
          PCY_CUDA(cudaEventRecord(evk1, st));   // a run-ahead batch's Gram may start from here (other buffer)
        }
        if (prof) PCY_CUDA(cudaEventRecord(ev[1], rs));
        ParCtl* pp = nullptr;
        bool selfp = false; long long pseq = 0, planseq = 0;
        if (k3par) {
          // k_plan picks a subtree-parallel window or a sequential stretch
          if (nper != 101 && !gram_early) {   // opener rows against the batch (k_plan's conflict test)
            const int grc = pcy_launch_gram_split(Xs, nullptr, ld, (int)kn, d, gram, kn, gram_part, gram_split, rs);
            if (grc) return grc;
          }
          planseq = ++plan_seq;
          k_plan<<<1, PCY_PAR_MAXITEMS, plan_smem, rs>>>(E, XSs, Ws, Bs, kn, first_rem, nnew_cap, 16, chh, chr, parctl,
                                                 (int)(NC / 32 + 1), nullptr, gram_w, kn, ctl_map_d, planseq);
          pcy_count_launch();
          pp = parctl;
          // one launch serves either choice of k_plan and, while no group is
          // in the K1 panel, publishes the counters itself
          selfp = self_publish();
          pseq = selfp ? ++seq : 0;
          EngCtl* pb = selfp ? ctl_map_d : nullptr;
          switch (nper) {
            case 1: PCY_CUDA(launch_pdl(k_resolve2x<1>, dim3(PCY_PAR_MAXCTA), dim3(64), res_smem, rs, E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, (const ChainHdr*)chh, (const ChainLvl*)chr, pp, pb, pseq, planseq)); break;
            case 2: PCY_CUDA(launch_pdl(k_resolve2x<2>, dim3(PCY_PAR_MAXCTA), dim3(64), res_smem, rs, E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, (const ChainHdr*)chh, (const ChainLvl*)chr, pp, pb, pseq, planseq)); break;
            case 4: PCY_CUDA(launch_pdl(k_resolve2x<4>, dim3(PCY_PAR_MAXCTA), dim3(64), res_smem, rs, E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, (const ChainHdr*)chh, (const ChainLvl*)chr, pp, pb, pseq, planseq)); break;
            case 8: PCY_CUDA(launch_pdl(k_resolve2x<8>, dim3(PCY_PAR_MAXCTA), dim3(64), res_smem, rs, E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, (const ChainHdr*)chh, (const ChainLvl*)chr, pp, pb, pseq, planseq)); break;
            case 100: k_resolve3x<true, 2048><<<PCY_PAR_MAXCTA, 32, res_smem, rs>>>(E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, chh, chr, nullptr, 0, 0, pp, pb, pseq); break;
            case 101: k_resolve3x<false, 512><<<PCY_PAR_MAXCTA, 32, res_smem, rs>>>(E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, chh, chr, gram, kn, 0, pp, pb, pseq); break;
          }
          pcy_count_launch();
        } else {
          switch (nper) {
            case 1: k_resolve2<1><<<1, 64, res_smem, rs>>>(E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, chh, chr, pp); pcy_count_launch(); break;
            case 2: k_resolve2<2><<<1, 64, res_smem, rs>>>(E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, chh, chr, pp); pcy_count_launch(); break;
            case 4: k_resolve2<4><<<1, 64, res_smem, rs>>>(E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, chh, chr, pp); pcy_count_launch(); break;
            case 8: k_resolve2<8><<<1, 64, res_smem, rs>>>(E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, chh, chr, pp); pcy_count_launch(); break;
            case 100: k_resolve3<true, 2048><<<1, 32, res_smem, rs>>>(E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, chh, chr, nullptr, 0, 0, pp); pcy_count_launch(); break;
            case 101: k_resolve3<false, 512><<<1, 32, res_smem, rs>>>(E, Xs, XSs, Ws, Bs, kn, first_rem, countw, nnew_cap, chh, chr, gram, kn, 0, pp); pcy_count_launch(); break;
            default:
              k_resolve<<<1, 32, sizeof(double) * ld, rs>>>(E, Xs, XSs, Ws, Bs, kn, 0, first_rem, countw); pcy_count_launch();
          }
        }
        if (prof) PCY_CUDA(cudaEventRecord(ev[2], rs));
        PCY_LAUNCH_CHECK();
        // Run-ahead: k_plan publishes the window it chose before the resolve
        // kernel runs.  A parallel window of n_win items ends at start + n_win
        // whatever the resolve does (its only other outcomes are fatal), so the
        // next batch's K1 is enqueued now and the host round trip hides behind
        // the resolve kernel.  Needs the self-published counters (no panel
        // launch between the windows) and a K1 that takes nothing from the host
        // mirror (panel mode with an empty panel).
        long long nstart = -1, nkn = 0, nkb = kbatch;
#ifndef PCY_TRACE
        if (selfp && panel && hi && !prof && first_rem < 0) {
          int rcp = wait_plan(rs, planseq); if (rcp) return rcp;
          if (ctl_h->plan_mode == 0) {
            const long long nwin = ctl_h->plan_nwin;
            if (nwin == kn) nkb = kbatch * 2 > 1024 ? 1024 : kbatch * 2;
            else { const long long b2 = 2 * nwin; nkb = b2 < 128 ? 128 : b2 > 1024 ? 1024 : b2; }
            nstart = start + nwin;
            if (nwin > 0 && nstart < nb) {
              nkn = nb - nstart > nkb ? nkb : nb - nstart;
              rcp = enqueue_k1(off + nstart, nkn, false, true, pseq); if (rcp) return rcp;
#ifdef PCY_TIMELINE
              ++tl_early;
#endif
            }
          }
        }
#endif
        int rc = selfp ? wait_seq(rs, pseq) : sync_ctl(rs);
        if (!rc && selfp && !self_publish()) rc = sync_ctl(rs);   // a group reached the panel size
        if (rc) return rc;
        if (prof) {
          float t1 = 0.f, t2 = 0.f;
          PCY_CUDA(cudaEventSynchronize(ev[2]));   // recorded after the self-publishing kernel
          PCY_CUDA(cudaEventElapsedTime(&t1, ev[0], ev[1]));
          PCY_CUDA(cudaEventElapsedTime(&t2, ev[1], ev[2]));
          const long long done = ctl_h->status == ST_DONE ? kn : ctl_h->stop + (ctl_h->status == ST_FULL ? 0 : 1);
          pcy_prof_add(PCY_PROF_CHAIN, t1, kn);
          pcy_prof_add(PCY_PROF_RESOLVE, t2, done);
          if (gemm_timed) {
            float tg = 0.f;
            PCY_CUDA(cudaEventElapsedTime(&tg, ev[6], ev[7]));
            pcy_prof_add(PCY_PROF_GEMM, tg, (long long)gemm_flops);
            gemm_timed = false;
          }
        }
#ifdef PCY_TRACE
        {   // build-time diagnostics only (PCY_NVCC_EXTRA=-DPCY_TRACE)
          int pm[2] = {-1, 0}, dbg[3] = {0, 0, 0};
          if (k3par) {
            cudaMemcpy(pm, parctl, sizeof(pm), cudaMemcpyDeviceToHost);
            cudaMemcpy(dbg, &parctl->dbg_sets, sizeof(dbg), cudaMemcpyDeviceToHost);
          }
          fprintf(stderr, "[ins] start %lld kn %lld status %d stop %lld mode %d P %d F %lld sets %d maxset %d maxcta %d\n", off + start, kn,
                  ctl_h->status, ctl_h->stop, pm[0], pm[1], ctl_h->F, dbg[0], dbg[1], dbg[2]);
        }
#endif
        const int status = ctl_h->status;
        if (status == ST_DONE) {
          if (k3par) kbatch = kbatch * 2 > 1024 ? 1024 : kbatch * 2;
          if (kn < nb - start) {
            start += kn; first_rem = -1;
            if (nkn > 0 && nstart == start) k1_kn = nkn;
            continue;
          }
          break;
        }
        if (status == ST_INVALID) { *bad_at = off + start + ctl_h->stop; *bad_code = ctl_h->err; return PCY_OK; }
        if (status == ST_ARENA) { pcy_set_error("member arena exhausted"); return PCY_ESTATE; }
        if (status == ST_PAR_BROKEN) {
          pcy_set_error("subtree-parallel resolve met an excluded stop (inner status %d, window %lld of %lld, F %lld, m %lld, weighted %d)",
                        ctl_h->err, ctl_h->stop, kn, ctl_h->F, m, W ? 1 : 0);
          return PCY_ESTATE;
        }
        if (status == ST_FULL) {
          if (ctl_h->stop == 0) { pcy_set_error("resolve made no progress"); return PCY_ESTATE; }
          start += ctl_h->stop; first_rem = -1;
          if (k3par) { const long long b2 = 2 * ctl_h->stop; kbatch = b2 < 128 ? 128 : b2 > 1024 ? 1024 : b2; }
          if (nkn > 0 && nstart == start) k1_kn = nkn;
          continue;
        }
        if (status == ST_REBUILD) {
          const long long at = start + ctl_h->stop;
          const long long r = ctl_h->remaining;
          rc = rebuild(st); if (rc) return rc;
          if (r > 0) { start = at; first_rem = r; }
          else { start = at + 1; first_rem = -1; }
          continue;
        }
        pcy_set_error("unexpected resolve status %d", status);
        return PCY_ESTATE;
      }
      off += nb;
    }
    return PCY_OK;
  }

  int build(cudaStream_t st) {
    const long long ns = ctl_h->ndist < sample_cap ? ctl_h->ndist : sample_cap;
    unsigned long long init[2] = {0x7ff0000000000000ULL, 0ULL};
    PCY_CUDA(cudaMemcpyAsync(E.minbits, init, sizeof(init), cudaMemcpyHostToDevice, st));
    k_mp_norms<<<(unsigned)((ns + 7) / 8), 256, 0, st>>>(E, ns, mp_nrm); pcy_count_launch();
    dim3 grid((unsigned)((ns + 31) / 32), (unsigned)((ns + 31) / 32));
    if (ns >= 2) { k_mp_tiles<<<grid, dim3(32, 8), 0, st>>>(E, ns, mp_nrm); pcy_count_launch(); }
    k_mp_finish<<<1, 1, 0, st>>>(E, ns); pcy_count_launch();
    k_tree_reset<<<1, 1, 0, st>>>(E); pcy_count_launch();
    PCY_LAUNCH_CHECK();
    int rc = sync_ctl(st); if (rc) return rc;
    built = true;
    const long long np = ctl_h->npend;
    long long bad_at; int code;
    rc = live(E.pend_x, E.pend_xsq, E.pend_w, nullptr, np, 0, st, &bad_at, &code);
    return rc;
  }

  int insert(const void* x, int dtype, long long stride, const long long* w, long long n,
             cudaStream_t st, long long* consumed, int* bad_code) {
    *consumed = n; *bad_code = 0;
    if (dtype != 0 && dtype != 1) { pcy_set_error("dtype must be 0 (f64) or 1 (f32)"); return PCY_EINVAL; }
    const size_t esz = dtype == 1 ? 4 : 8;
    long long pos = 0;
    while (pos < n) {
      const long long nb = n - pos < Bmax ? n - pos : Bmax;
      k_stage<<<(unsigned)((nb + 7) / 8), 256, 0, st>>>(E, (const char*)x + (size_t)pos * stride * esz,
                                                         dtype, stride, w ? w + pos : nullptr, nb, built ? 0 : 1); pcy_count_launch();
      PCY_LAUNCH_CHECK();
      long long i = 0;
      while (i < nb) {
        if (!built) {
          {
            PCY_CUDA(cudaMemsetAsync(bs.skey, 0xff, sizeof(int) * bs.scap, st));
            PCY_CUDA(cudaMemsetAsync(bs.sfirst, 0x7f, sizeof(int) * bs.scap, st));
            const unsigned g8 = (unsigned)((nb - i + 7) / 8);
            k_boot_scan_rows<<<g8, 256, 0, st>>>(E, bs, i, nb); pcy_count_launch();
            k_boot_plan<<<1, 1024, 0, st>>>(E, bs, i, nb); pcy_count_launch();
            k_boot_apply<<<g8, 256, 0, st>>>(E, bs, i, nb, ctl_h->npend); pcy_count_launch();
          }
          PCY_LAUNCH_CHECK();
          int rc = sync_ctl(st); if (rc) return rc;
          const int status = ctl_h->status;
          if (status == ST_DONE) { i = nb; break; }
          if (status == ST_INVALID) { *consumed = pos + ctl_h->stop; *bad_code = ctl_h->err; return PCY_OK; }
          if (status == ST_GROW) { i = ctl_h->stop; rc = grow_pending(st); if (rc) return rc; continue; }
          if (status == ST_BUILD) { i = ctl_h->stop + 1; rc = build(st); if (rc) return rc; continue; }
          pcy_set_error("unexpected bootstrap status %d", status);
          return PCY_ESTATE;
        } else {
          long long bad_at; int code = 0;
          int rc = live(E.xb + i * ld, E.xsq + i, E.wb + i, E.bad + i, nb - i, 1, st, &bad_at, &code);
          if (rc) return rc;
          if (bad_at >= 0) { *consumed = pos + i + bad_at; *bad_code = code; return PCY_OK; }
          i = nb;
        }
      }
      pos += nb;
    }
    return PCY_OK;
  }

  int count(cudaStream_t st, long long* cnt) {
    int rc = sync_ctl(st); if (rc) return rc;
    if (!built) { *cnt = ctl_h->ndist; return PCY_OK; }
    k_dfs<<<1, 1, 0, st>>>(E); pcy_count_launch();
    PCY_LAUNCH_CHECK();
    rc = sync_ctl(st); if (rc) return rc;
    *cnt = ctl_h->stop;
    return PCY_OK;
  }

  int features(int* lv, long long* wo, double* so, double* qo, double* ro, double* po,
               long long cap, long long* cnt, cudaStream_t st) {
    int rc = count(st, cnt); if (rc) return rc;
    const long long n = *cnt < cap ? *cnt : cap;
    if (n <= 0) return PCY_OK;
    if (!built) {
      PCY_CUDA(cudaMemsetAsync(aggw, 0, sizeof(long long) * (ctl_h->ndist + 1), st));
      k_boot_aggregate<<<(unsigned)((ctl_h->npend + 7) / 8), 256, 0, st>>>(E, aggw); pcy_count_launch();
      k_boot_gather<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(E, n, aggw, lv, wo, so, qo, ro, po); pcy_count_launch();
    } else {
      if (po) { k_gather_points<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(E, n, po, wo); pcy_count_launch(); }
      if (lv || so || qo || ro || (wo && !po)) {
        k_gather_features<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(E, n, lv, wo, so, qo, ro); pcy_count_launch();
      }
    }
    PCY_LAUNCH_CHECK();
    return PCY_OK;
  }
};

}  // namespace

// ==================================================================== C-ABI
extern "C" {

int pcy_engine_create(int device, int dim, long long budget, long long bootstrap_cap,
                      long long block_rows, void** out) {
  *out = nullptr;
  if (dim < 1) { pcy_set_error("dim must be >= 1"); return PCY_EINVAL; }
  if (budget < 1) { pcy_set_error("budget must be >= 1"); return PCY_EINVAL; }
  if (budget > (1LL << 28)) { pcy_set_error("budget too large"); return PCY_EINVAL; }
  Engine* e = new Engine();
  int rc = e->init(device, dim, budget, bootstrap_cap, block_rows);
  if (rc) { delete e; return rc; }
  *out = e;
  return PCY_OK;
}

int pcy_engine_destroy(void* h) {
  delete (Engine*)h;
  return PCY_OK;
}

int pcy_engine_insert(void* h, const void* x, int dtype, long long stride, const long long* w,
                      long long n, void* stream, long long* consumed, int* bad_code) {
  Engine* e = (Engine*)h;
  if (!e) { pcy_set_error("null engine"); return PCY_EINVAL; }
  if (n <= 0) { *consumed = 0; *bad_code = 0; return PCY_OK; }
  const int rc = e->insert(x, dtype, stride, w, n, (cudaStream_t)stream, consumed, bad_code);
  e->touch((cudaStream_t)stream);
  return rc;
}

int pcy_engine_stats(void* h, long long* num_features, double* threshold, long long* total_weight,
                     int* built, void* stream) {
  Engine* e = (Engine*)h;
  int rc = e->sync_ctl((cudaStream_t)stream);
  e->touch((cudaStream_t)stream);
  if (rc) return rc;
  *num_features = e->built ? e->ctl_h->F : e->ctl_h->ndist;
  *threshold = e->ctl_h->T;
  *total_weight = e->ctl_h->total_w;
  *built = e->built ? 1 : 0;
  return PCY_OK;
}

// Engine instrumentation counters: [levels, direct scans, demand loads,
// full capacity evaluations, items, max depth].
int pcy_engine_counters(void* h, long long* out6) {
  Engine* e = (Engine*)h;
  out6[0] = e->ctl_h->cnt_levels; out6[1] = e->ctl_h->cnt_direct; out6[2] = e->ctl_h->cnt_demand;
  out6[3] = e->ctl_h->cnt_slow; out6[4] = e->ctl_h->cnt_items; out6[5] = e->ctl_h->max_depth;
  return PCY_OK;
}

// K1 work of this engine's chain walks (insertion and rebuild reattach):
// out[0] member visits (the reference's own nearest-reference work,
// coreset.py:172: one d-length dot per visited member), out[1] the visits
// served by direct fp64 scans, out[2] tensor-pipe flops executed by the
// panel contractions (3 TF32 products, padded tiles), out[3] panel launches.
int pcy_engine_work(void* h, double* out4) {
  Engine* e = (Engine*)h;
  out4[0] = (double)e->ctl_h->cnt_vis; out4[1] = (double)e->ctl_h->cnt_vis_direct;
  out4[2] = e->exec_tensor_flops; out4[3] = (double)e->panel_launches;
  return PCY_OK;
}

// Same counters summed over every engine destroyed so far in this process.
int pcy_engine_counters_total(long long* out6) {
  for (int k = 0; k < 6; ++k) out6[k] = g_counters[k].load();
  return PCY_OK;
}

int pcy_engine_features(void* h, int* level, long long* weight, double* lsum, double* sqsum,
                        double* ref, long long cap, long long* count, void* stream) {
  Engine* e = (Engine*)h;
  const int rc = e->features(level, weight, lsum, sqsum, ref, nullptr, cap, count, (cudaStream_t)stream);
  e->touch((cudaStream_t)stream);
  return rc;
}

int pcy_engine_extract(void* h, double* points, long long* weights, long long cap, long long* count,
                       void* stream) {
  Engine* e = (Engine*)h;
  const int rc = e->features(nullptr, weights, nullptr, nullptr, nullptr, points, cap, count, (cudaStream_t)stream);
  e->touch((cudaStream_t)stream);
  return rc;
}

}  // extern "C"
