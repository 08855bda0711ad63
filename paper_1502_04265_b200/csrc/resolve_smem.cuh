// K3 / K4-reattach with rows in shared memory (any d), included by engine.cu
// after resolve_fast.cuh and reattach_fast.cuh.
//
// Same algorithm as k_resolve2 / k_reattach2 (see resolve_fast.cuh), but the
// item's x row and the predicted node's s row live in double-buffered shared
// memory and are prefetched one item ahead with cp.async (no register
// staging), so one code path serves d = 2 .. several thousand.  When the
// dimension is too large for a shared-memory new-node table (TROWS = false),
// rows of nodes opened in the launch live in HBM at their slot.
#pragma once


// ld doubles (ld % 4 == 0, 32-B aligned rows) global -> shared, asynchronous
__device__ __forceinline__ void row_fetch(double* dst, const double* src, int ld, int lane) {
  for (int c = lane; c < ld / 2; c += 32) cp_async16(dst + 2 * c, src + 2 * c);
}

// Whole rows global -> shared with one bulk (TMA) copy each, completed on an
// mbarrier (expect_tx = all bytes of the batch).  All lanes first fence the
// generic proxy against the async proxy (earlier plain stores to the source
// rows in HBM and to the destination buffers in shared memory), then lane 0
// issues.  rows_wait spins on the barrier's current phase.
__device__ __forceinline__ void rows_issue(unsigned long long* bar, int lane, unsigned bytes, double* d0,
                                           const double* s0, double* d1, const double* s1, double* d2,
                                           const double* s2) {
  asm volatile("fence.proxy.async;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    const unsigned total = bytes * (unsigned)(1 + (s1 != nullptr) + (s2 != nullptr));
    const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(total) : "memory");
    double* ds[3] = {d0, d1, d2};
    const double* ss[3] = {s0, s1, s2};
#pragma unroll
    for (int q = 0; q < 3; ++q)
      if (ss[q])
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         (unsigned)__cvta_generic_to_shared(ds[q])),
                     "l"(ss[q]), "r"(bytes), "r"(b)
                     : "memory");
  }
}
__device__ __forceinline__ void rows_wait(unsigned long long* bar, unsigned& phase) {
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "RW_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra RW_DONE;\n\t"
      "bra RW_WAIT;\n"
      "RW_DONE:\n\t}" ::"r"(b),
      "r"(phase)
      : "memory");
  phase ^= 1u;
}
// Row prefetch: bulk copies for long rows (>= 16 KB, where one TMA copy per
// row beats 512+ cp.async per lane and the proxy fence), cp.async otherwise.
__device__ __forceinline__ void rows_fetch(bool bulk, unsigned long long* bar, int lane, int ld, double* d0,
                                           const double* s0, double* d1, const double* s1, double* d2,
                                           const double* s2) {
  if (bulk) {
    rows_issue(bar, lane, (unsigned)(sizeof(double) * ld), d0, s0, d1, s1, d2, s2);
  } else {
    row_fetch(d0, s0, ld, lane);
    if (s1) row_fetch(d1, s1, ld, lane);
    if (s2) row_fetch(d2, s2, ld, lane);
  }
}

__device__ __forceinline__ void rows_bar_init(unsigned long long* bar, int n, int lane) {
  if (lane == 0) {
    for (int q = 0; q < n; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(bar + q)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
}
// lane-strided fp64 dot in warp_dot order (shared with K1's snapshot dots)
__device__ __forceinline__ double row_dot(const double* a, const double* b, int d, int lane) {
  return warp_dot(a, b, d, lane);   // same lane-strided order, loads issued ahead
}

// s += take * x over one row (lane-strided), written to the smem copy and to
// HBM: 8 elements in flight per lane; the same rounded operations as
// element-at-a-time (radd / rmul per element), so the values are identical.
__device__ __forceinline__ void row_absorb(double* __restrict__ prow, const double* __restrict__ x,
                                           double* __restrict__ dst, int d, int lane, long long take) {
  const double ft = (double)take;
  int e = lane;
  if (take == 1) {
    for (; e + 7 * 32 < d; e += 8 * 32) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = radd(prow[e + 32 * q], x[e + 32 * q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) { prow[e + 32 * q] = v[q]; if (dst) dst[e + 32 * q] = v[q]; }
    }
    for (; e < d; e += 32) { const double v = radd(prow[e], x[e]); prow[e] = v; if (dst) dst[e] = v; }
  } else {
    for (; e + 7 * 32 < d; e += 8 * 32) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = radd(prow[e + 32 * q], rmul(ft, x[e + 32 * q]));
#pragma unroll
      for (int q = 0; q < 8; ++q) { prow[e + 32 * q] = v[q]; if (dst) dst[e + 32 * q] = v[q]; }
    }
    for (; e < d; e += 32) { const double v = radd(prow[e], rmul(ft, x[e])); prow[e] = v; if (dst) dst[e] = v; }
  }
}

template <int MS>
struct ResolveSmemT {
  ChainLvl rb[2][PCY_FMAXL];
  int mkey[MS], mchild[MS];
  long long mw[MS];
  double mq[MS], msn[MS];
  int gkey[PCY_GMAP_SLOTS], ghead[PCY_GMAP_SLOTS], gtail[PCY_GMAP_SLOTS];
  int tid[PCY_NNEW_MAX], tgrp[PCY_NNEW_MAX], tchild[PCY_NNEW_MAX], tnext[PCY_NNEW_MAX];
  int tk[PCY_NNEW_MAX], tfirst[PCY_NNEW_MAX], tcnt[PCY_NNEW_MAX], tbase[PCY_NNEW_MAX], tcap[PCY_NNEW_MAX];
  int titem[PCY_NNEW_MAX];   // Gram row of the item that placed the entry
  long long tw[PCY_NNEW_MAX];
  double trn[PCY_NNEW_MAX], tq[PCY_NNEW_MAX], tsn[PCY_NNEW_MAX];
  unsigned long long rbar[2];   // bulk row copies into buffer 0 / 1
  int modcount;
};

// dynamic tail: xb[2][ld], pb[2][ld], (sb[2][ld] reattach), tref[nnew][ld|1], ts[nnew][ld] (TROWS), mbits, gbits
template <int MS>
__host__ __device__ inline size_t resolve3_smem_bytes(int ld, int nnew, bool trows, long long NC, long long GC,
                                                      int extra_rows) {
  return ((sizeof(ResolveSmemT<MS>) + 15) & ~size_t(15)) +
         sizeof(double) * (size_t)ld * (4 + (size_t)extra_rows) +
         (trows ? sizeof(double) * (size_t)nnew * ((size_t)(ld | 1) + ld) : 0) +
         sizeof(unsigned) * (size_t)(NC / 32 + 1 + GC / 32 + 1);
}

template <int MS>
__device__ __forceinline__ int map3_slot(int id) { return (int)(((unsigned)id * 2654435761u) >> 20) & (MS - 1); }

template <int MS>
__device__ __forceinline__ int map3_find(const ResolveSmemT<MS>& S, int id) {
  int s = map3_slot<MS>(id);
  for (;;) {
    const int k = S.mkey[s];
    if (k == id) return s;
    if (k < 0) return -1;
    s = (s + 1) & (MS - 1);
  }
}

template <int MS>
__device__ __forceinline__ int map3_put(ResolveSmemT<MS>& S, unsigned* mbits, int id, long long w, double q,
                                        double sn, int child, int lane) {
  int s = map3_slot<MS>(id);
  while (S.mkey[s] >= 0 && S.mkey[s] != id) s = (s + 1) & (MS - 1);
  if (lane == 0) {
    if (S.mkey[s] < 0) { S.modcount++; mbits[id >> 5] |= 1u << (id & 31); }
    S.mkey[s] = id; S.mw[s] = w; S.mq[s] = q; S.msn[s] = sn; S.mchild[s] = child;
  }
  __syncwarp();
  return s;
}

template <int MS>
__device__ __forceinline__ int gmap3_find(const ResolveSmemT<MS>& S, int g) {
  int s = (int)(((unsigned)g * 2654435761u) >> 24) & (PCY_GMAP_SLOTS - 1);
  for (;;) {
    const int k = S.gkey[s];
    if (k == g) return s;
    if (k < 0) return -1;
    s = (s + 1) & (PCY_GMAP_SLOTS - 1);
  }
}

// append table entry t to group g's chain of new members (lane 0 writes)
template <int MS>
__device__ __forceinline__ void gchain_append(ResolveSmemT<MS>& S, unsigned* gbits, int g, int t, int lane) {
  const bool had = ((gbits[g >> 5] >> (g & 31)) & 1u) != 0;
  int gs;
  if (had) gs = gmap3_find<MS>(S, g);
  else {
    gs = (int)(((unsigned)g * 2654435761u) >> 24) & (PCY_GMAP_SLOTS - 1);
    while (S.gkey[gs] >= 0) gs = (gs + 1) & (PCY_GMAP_SLOTS - 1);
  }
  if (lane == 0) {
    S.tnext[t] = -1;
    if (had) { S.tnext[S.gtail[gs]] = t; S.gtail[gs] = t; }
    else { S.gkey[gs] = g; S.ghead[gs] = t; S.gtail[gs] = t; gbits[g >> 5] |= 1u << (g & 31); }
  }
}

// nearest among the launch's new members of group g (position order)
template <bool TROWS, int MS>
__device__ __forceinline__ void scan_new(const EngDev& E, const ResolveSmemT<MS>& S, const unsigned* gbits,
                                         const double* tref, int lds, const double* xsm, int g, int nnew,
                                         int lane, double& bp, int& bj, int& bt,
                                         const double* gram, long long gld, long long gq) {
  if (!((gbits[g >> 5] >> (g & 31)) & 1u)) return;
  const int d = E.d, ld = E.ld;
  if (!TROWS && gram) {
    // same-launch members are rows of this block: their dots come from the
    // block Gram computed on the tensor pipe before the launch
    double np_ = INFINITY; int nt = 0x7fffffff;
    for (int c0 = 0; c0 < nnew; c0 += 32) {
      const int t = c0 + lane;
      if (t < nnew && S.tgrp[t] == g) {
        // (current item, earlier item): the lower triangle pcy_launch_gram computes
        const double part = radd(S.trn[t], rmul(gram[gq * gld + S.titem[t]], -2.0));
        if (part < np_) { np_ = part; nt = t; }
      }
    }
    warp_argmin(np_, nt);
    if (nt != 0x7fffffff && (np_ < bp || bj < 0)) { bp = np_; bt = nt; bj = S.tid[nt]; }
    return;
  }
  if (TROWS) {
    double np_ = INFINITY; int nt = 0x7fffffff;
    for (int c0 = 0; c0 < nnew; c0 += 32) {
      const int t = c0 + lane;
      if (t < nnew && S.tgrp[t] == g) {
        const double* rr = tref + (long long)t * lds;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;   // 4 chains: ILP over d
        int e = 0;
        for (; e + 3 < d; e += 4) {
          a0 = fma(rr[e], xsm[e], a0); a1 = fma(rr[e + 1], xsm[e + 1], a1);
          a2 = fma(rr[e + 2], xsm[e + 2], a2); a3 = fma(rr[e + 3], xsm[e + 3], a3);
        }
        for (; e < d; ++e) a0 = fma(rr[e], xsm[e], a0);
        const double acc = (a0 + a1) + (a2 + a3);
        const double part = radd(S.trn[t], rmul(acc, -2.0));
        if (part < np_) { np_ = part; nt = t; }
      }
    }
    warp_argmin(np_, nt);
    if (nt != 0x7fffffff && (np_ < bp || bj < 0)) { bp = np_; bt = nt; bj = S.tid[nt]; }
  } else {
    for (int tt = S.ghead[gmap3_find<MS>(S, g)]; tt >= 0; tt = S.tnext[tt]) {
      const double part = radd(S.trn[tt], rmul(row_dot(E.r + (long long)S.tid[tt] * ld, xsm, d, lane), -2.0));
      if (part < bp || bj < 0) { bp = part; bt = tt; bj = S.tid[tt]; }
    }
  }
}

// memberships of the launch's table entries -> arena, position order (both kernels)
template <int MS>
__device__ bool table_cleanup(const EngDev& E, ResolveSmemT<MS>& S, int nnew, long long& Aalloc, int lane,
                              ParCtl* par = nullptr) {
  for (int t = lane; t < nnew; t += 32) {
    const int g = S.tgrp[t];
    int k = 0, f = t;
    for (int u = t - 1; u >= 0; --u) if (S.tgrp[u] == g) { ++k; f = u; }
    S.tk[t] = k; S.tfirst[t] = f;
    S.tcnt[t] = E.g_count[g]; S.tcap[t] = E.g_cap[g]; S.tbase[t] = E.g_base[g];
  }
  __syncwarp();
  bool ok = true;
  for (int t = 0; t < nnew; ++t) {
    if (S.tfirst[t] != t) continue;
    const int g = S.tgrp[t];
    int total = 0;
    for (int u = t; u < nnew; ++u) total += (S.tgrp[u] == g);
    const int cnt = S.tcnt[t], cap = S.tcap[t], base = S.tbase[t];
    int nb = base, ncap = cap;
    if (cnt + total > cap) {
      ncap = cap ? 2 * cap : PCY_GROUP_MIN_CAP;
      while (ncap < cnt + total) ncap *= 2;
      if (par) {   // subtree-parallel launch: arena extents by ticket
        unsigned long long at = 0;
        if (lane == 0) at = atomicAdd(&par->a_ticket, (unsigned long long)ncap);
        const long long a0 = par->Aalloc0 + (long long)__shfl_sync(PCY_FULL, at, 0);
        if (a0 + ncap > E.AC) { ok = false; break; }
        nb = (int)a0;
      } else {
        if (Aalloc + ncap > E.AC) { ok = false; break; }
        nb = (int)Aalloc; Aalloc += ncap;
      }
      for (int p = lane; p < cnt; p += 32) E.arena[nb + p] = E.arena[base + p];
    }
    if (lane == 0) {
      S.tbase[t] = nb; S.tcap[t] = ncap;
      E.g_base[g] = nb; E.g_cap[g] = ncap; E.g_count[g] = cnt + total;
    }
    __syncwarp();
  }
  if (ok)
    for (int t = lane; t < nnew; t += 32) {
      const int f = S.tfirst[t];
      E.arena[S.tbase[f] + S.tcnt[f] + S.tk[t]] = S.tid[t];
    }
  __syncwarp();
  return ok;
}

constexpr int REC3_CHUNKS = PCY_FMAXL * (int)sizeof(ChainLvl) / 16;

// PAR / par: as k_resolve2 (k_plan windows, one CTA per subtree list).
template <bool TROWS, int MS, bool PAR>
__device__ __forceinline__ void resolve3_body(const EngDev& E, const double* __restrict__ X,
                                              const double* __restrict__ XS, const long long* __restrict__ W,
                                              const int* __restrict__ BAD, long long n, long long first_rem,
                                              int countw, int nnew_cap, const ChainHdr* __restrict__ H,
                                              const ChainLvl* __restrict__ R, const double* __restrict__ gram,
                                              long long gld, long long goff, ParCtl* __restrict__ par,
                                              EngCtl* pub, long long pseq) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ResolveSmemT<MS>& S = *reinterpret_cast<ResolveSmemT<MS>*>(smraw);
  const int lane = threadIdx.x;
  const int* ilist = nullptr;
  if constexpr (PAR) {
    if (par->mode != 0 || (int)blockIdx.x >= par->P) return;
    const int o0 = par->off[blockIdx.x];
    ilist = par->list + o0;
    n = par->off[blockIdx.x + 1] - o0;
    first_rem = -1;
  } else {
    if (par) {
      if (par->mode != 1) return;
      n = par->n_win;
    }
  }
  auto gix = [&](long long j) -> long long {
    if constexpr (PAR) return (long long)ilist[j];
    else return j;
  };
  const int d = E.d, ld = E.ld;
  double* xb = reinterpret_cast<double*>(smraw + ((sizeof(ResolveSmemT<MS>) + 15) & ~size_t(15)));
  double* pb = xb + 2 * (long long)ld;
  const int lds = ld | 1;
  double* tref = pb + 2 * (long long)ld;
  double* ts = tref + (TROWS ? (long long)nnew_cap * lds : 0);
  unsigned* mbits = reinterpret_cast<unsigned*>(ts + (TROWS ? (long long)nnew_cap * ld : 0));
  const int mwords = (int)(E.NC / 32 + 1);
  unsigned* gbits = mbits + mwords;
  const int gwords = (int)(E.GC / 32 + 1);
  EngCtl* C = E.ctl;
  const long long m = E.m;
  const double T = C->T;
  long long F = C->F, Falloc = C->F_alloc, freen = C->free_n, Galloc = C->G_alloc;
  long long Aalloc = C->A_alloc, nidx = C->next_index, totw = C->total_w, maxdepth = C->max_depth;
  long long c_lv = 0, c_dir = 0, c_dem = 0, c_slow = 0, c_it = 0;
  long long G0 = Galloc, opened = 0;
  if constexpr (PAR) { G0 = par->Galloc0; totw = 0; maxdepth = 0; freen = 0; }
  auto new_group = [&]() -> int {
    if constexpr (PAR) {
      unsigned long long t = 0;
      if (lane == 0) t = atomicAdd(&par->g_ticket, 1ULL);
      return (int)(par->Galloc0 + (long long)__shfl_sync(PCY_FULL, t, 0));
    } else {
      return (int)Galloc++;
    }
  };
  int status = ST_DONE, err = 0; long long stop = n, remaining = 0;

  for (int s2 = lane; s2 < MS; s2 += 32) S.mkey[s2] = -1;
  for (int s2 = lane; s2 < PCY_GMAP_SLOTS; s2 += 32) S.gkey[s2] = -1;
  for (int s2 = lane; s2 < mwords; s2 += 32) mbits[s2] = 0u;
  for (int s2 = lane; s2 < gwords; s2 += 32) gbits[s2] = 0u;
  if (lane == 0) S.modcount = 0;
  int nnew = 0;
  int free_top = freen > 0 ? E.free_ids[freen - 1] : -1;

  int bad_c = (n > 0 && BAD) ? BAD[gix(0)] : 0;
  long long w_c = (n > 0 && W) ? W[gix(0)] : 1LL;
  double xs_c = n > 0 ? XS[gix(0)] : 0.0;
  ChainHdr hc = n > 0 ? H[gix(0)] : ChainHdr{0, 0, -1, 0};
  ChainHdr hn = n > 1 ? H[gix(1)] : ChainHdr{0, 0, -1, 0};
  rows_bar_init(S.rbar, 2, lane);
  unsigned rph[2] = {0u, 0u};
  const bool bulk = ld >= 2048;
  if (n > 0) {
    rows_fetch(bulk, &S.rbar[0], lane, ld, xb, X + gix(0) * ld, pb,
               hc.predj >= 0 ? E.s + (long long)hc.predj * ld : nullptr, nullptr, nullptr);
    const uint4* src = reinterpret_cast<const uint4*>(R + gix(0) * PCY_FMAXL);
    uint4* dst = reinterpret_cast<uint4*>(&S.rb[0][0]);
    for (int c = lane; c < REC3_CHUNKS; c += 32) cp_async16(dst + c, src + c);
    cp_async_commit();
    cp_async_wait_all();
    if (bulk) rows_wait(&S.rbar[0], rph[0]);
  }
  __syncwarp();
  int cur = 0;
  int prnode = hc.predj;   // node whose current s row is in pb[cur]

  for (long long i = 0; i < n; ++i) {
    if (bad_c) { status = ST_INVALID; err = bad_c; stop = i; break; }
    if (nnew >= nnew_cap || S.modcount >= MS / 2) { status = ST_FULL; stop = i; break; }
    double* xsm = xb + (long long)cur * ld;
    double* prow = pb + (long long)cur * ld;
    // ---- prefetch item i+1 into the other buffers
    const bool has_next = i + 1 < n;
    ChainHdr h2 = ChainHdr{0, 0, -1, 0};
    int bad_n = 0; long long w_n = 1; double xs_n = 0.0;
    if (has_next) {
      const long long gn = gix(i + 1);
      bad_n = BAD ? BAD[gn] : 0;
      w_n = W ? W[gn] : 1LL;
      xs_n = XS[gn];
      rows_fetch(bulk, &S.rbar[cur ^ 1], lane, ld, xb + (long long)(cur ^ 1) * ld, X + gn * ld,
                 pb + (long long)(cur ^ 1) * ld, hn.predj >= 0 ? E.s + (long long)hn.predj * ld : nullptr,
                 nullptr, nullptr);
      const uint4* src = reinterpret_cast<const uint4*>(R + gn * PCY_FMAXL);
      uint4* dst = reinterpret_cast<uint4*>(&S.rb[cur ^ 1][0]);
      for (int c = lane; c < REC3_CHUNKS; c += 32) cp_async16(dst + c, src + c);
      cp_async_commit();
      if (i + 2 < n) h2 = H[gix(i + 2)];
    }
    // ---- item i
    const bool resume = (i == 0 && first_rem >= 0);
    const long long wi = w_c;
    long long rem = resume ? first_rem : wi;
    if (countw && !resume) totw += wi;
    const double xs = xs_c;
    const int len = hc.len;
    int g = 0, L = 0;
    double radius = T;
    bool direct = false;
    int lastmod = -1, nmod = 0;
    int modl[4] = {-1, -1, -1, -1};

    auto load_prow = [&](int node) {
      const double* src = E.s + (long long)node * ld;
      for (int e = lane; e < ld; e += 32) prow[e] = src[e];
      __syncwarp();
      prnode = node;
      ++c_dem;
    };
    auto do_open = [&](int gg, int LL) -> bool {
      const bool full = !PAR && F >= m;   // k_plan: F0 + window <= m
      const long long wopen = full ? 1LL : rem;
      long long slot, nid = nidx;
      if constexpr (PAR) {
        unsigned long long tk = 0;
        if (lane == 0) tk = atomicAdd(&par->open_ticket, 1ULL);
        const long long tt = (long long)__shfl_sync(PCY_FULL, tk, 0);
        if (par->F0 + tt >= E.m) return true;   // k_plan's budget bound violated (never expected): report
        slot = tt < par->freen0 ? (long long)E.free_ids[par->freen0 - 1 - tt] : par->Falloc0 + (tt - par->freen0);
        nid = par->nidx0 + gix(i);
        ++opened;
      } else {
        if (freen > 0) { slot = free_top; --freen; free_top = freen > 0 ? E.free_ids[freen - 1] : -1; }
        else slot = Falloc++;
      }
      const int t = nnew++;
      const double fw = (double)wopen;
      double* rr = TROWS ? tref + (long long)t * lds : E.r + slot * ld;
      double* sr = TROWS ? ts + (long long)t * ld : E.s + slot * ld;
      for (int e = lane; e < ld; e += 32) { rr[e] = xsm[e]; sr[e] = rmul(fw, xsm[e]); }
      gchain_append<MS>(S, gbits, gg, t, lane);
      if (lane == 0) {
        S.titem[t] = (int)(goff + gix(i));
        S.tid[t] = (int)slot; S.tgrp[t] = gg; S.tchild[t] = -1; S.tw[t] = wopen;
        S.tq[t] = rmul(fw, xs); S.tsn[t] = rmul((double)(wopen * wopen), xs); S.trn[t] = xs;
        E.idx[slot] = nid; E.alive[slot] = 1; E.child[slot] = -1;
      }
      ++nidx; ++F;
      if (LL + 1 > maxdepth) maxdepth = LL + 1;
      rem -= wopen;
      __syncwarp();
      return full;
    };
    auto absorb_snapshot = [&](int bj, long long take, long long nw2, double nq, double nsn, int child_now) {
      const double ft = (double)take;
      if (bj != prnode) load_prow(bj);
      (void)ft;
      row_absorb(prow, xsm, E.s + (long long)bj * ld, d, lane, take);
      __syncwarp();
      const int ms = map3_put<MS>(S, mbits, bj, nw2, nq, nsn, child_now, lane);
      if (lane == 0) { E.w[bj] = nw2; E.q[bj] = nq; E.sn[bj] = nsn; }
      if (nmod < 4) modl[nmod] = bj;
      ++nmod;
      lastmod = bj;
      return ms;
    };

    // ---- verified fast path (see k_resolve2)
    bool done_fast = false;
    unsigned cleanmask = 0u;   // unchanged levels above K1's action level (see k_resolve2)
    if (!resume && len > 0 && !hc.trunc) {
      const int pl = hc.pred;
      bool ok = pl >= 0 && pl < len;
      if (ok) {
        bool cl = false;
        if (lane < pl) {
          const ChainLvl& rl = S.rb[cur][lane];
          const int g2 = rl.g, j2 = rl.j;
          const bool bad = (g2 >= 0 && ((gbits[g2 >> 5] >> (g2 & 31)) & 1u)) || (j2 >= 0 && ((mbits[j2 >> 5] >> (j2 & 31)) & 1u));
          cl = !bad && g2 >= 0 && j2 >= 0 && rl.child >= 0 && rl.take == 0;
        }
        cleanmask = __ballot_sync(PCY_FULL, cl);
      }
      for (int L2 = 0; ok && L2 <= pl; ++L2) {
        const int g2 = S.rb[cur][L2].g, j2 = S.rb[cur][L2].j;
        if (g2 >= 0 && ((gbits[g2 >> 5] >> (g2 & 31)) & 1u)) ok = false;
        if (j2 >= 0 && ((mbits[j2 >> 5] >> (j2 & 31)) & 1u)) ok = false;
      }
      if (ok) {
        const ChainLvl& rp = S.rb[cur][pl];
        if (rp.take > 0 && rp.take == rem) {
          absorb_snapshot(rp.j, rp.take, rp.w + rp.take, rp.nq, rp.nsn, rp.child);
          rem = 0;
          if (pl + 1 > maxdepth) maxdepth = pl + 1;
          c_lv += pl + 1;
          done_fast = true;
        } else if (rp.take == 0) {
          int gg = rp.g;
          if (gg < 0) {
            const ChainLvl& pp = S.rb[cur][pl - 1];
            gg = new_group();
            if (lane == 0) { E.g_count[gg] = 0; E.g_cap[gg] = 0; E.g_base[gg] = 0; E.child[pp.j] = gg; }
            map3_put<MS>(S, mbits, pp.j, pp.w, pp.q, pp.sn, gg, lane);
          }
          if (do_open(gg, pl)) { status = ST_REBUILD; stop = i; remaining = rem; }
          c_lv += pl + 1;
          done_fast = true;
        }
      }
    }
    if (!done_fast) for (;;) {
      if (!direct && rem == wi && ((cleanmask >> L) & 1u)) {   // unchanged level: K1's descent stands
        g = S.rb[cur][L].child;
        radius = rmul(radius, 0.25);
        ++L; ++c_lv;
        continue;
      }
      int bj = -1, li = -1;
      double bp = INFINITY;
      if (!direct) {
        if (L < len) { li = L; bj = S.rb[cur][L].j; bp = S.rb[cur][L].part; }
        else direct = true;
      }
      ++c_lv;
      if (direct && g < G0) {
        ++c_dir;
        const int cnt = E.g_count[g];
        if (cnt > 0) {
          double p; int ps;
          const int* mem = E.arena + E.g_base[g];
          scan_members(E, mem, 0, cnt, xsm, lane, p, ps);
          if (ps < cnt) { bj = mem[ps]; bp = p; }
        }
      }
      int bt = -1;
      scan_new<TROWS, MS>(E, S, gbits, tref, lds, xsm, g, nnew, lane, bp, bj, bt, gram, gld, goff + gix(i));
      if (bj < 0 || radd(bp, xs) > radius) {
        if (do_open(g, L)) { status = ST_REBUILD; stop = i; remaining = rem; }
        break;
      }
      long long nn, take, nw2 = 0;
      double qv, snv, nq = 0.0, nsn = 0.0;
      int ms = -1;
      const bool touched = bt < 0 && ((mbits[bj >> 5] >> (bj & 31)) & 1u);
      double* trow = nullptr;
      if (bt >= 0) trow = TROWS ? ts + (long long)bt * ld : E.s + (long long)S.tid[bt] * ld;
      if (bt < 0 && li >= 0 && !touched && rem == wi && !resume) {
        const ChainLvl& rc = S.rb[cur][li];
        nn = rc.w; qv = rc.q; snv = rc.sn; take = rc.take;
        if (take > 0) { nw2 = nn + take; nq = rc.nq; nsn = rc.nsn; }
      } else {
        double dt;
        ++c_slow;
        if (bt >= 0) {
          nn = S.tw[bt]; qv = S.tq[bt]; snv = S.tsn[bt];
          dt = row_dot(trow, xsm, d, lane);
        } else {
          if (touched) { ms = map3_find<MS>(S, bj); nn = S.mw[ms]; qv = S.mq[ms]; snv = S.msn[ms]; }
          else if (li >= 0) { const ChainLvl& rc = S.rb[cur][li]; nn = rc.w; qv = rc.q; snv = rc.sn; }
          else { nn = E.w[bj]; qv = E.q[bj]; snv = E.sn[bj]; }
          if (!touched && li >= 0) dt = S.rb[cur][li].dot;
          else {
            if (bj != prnode) load_prow(bj);
            dt = row_dot(prow, xsm, d, lane);
          }
        }
        take = capacity(nn, qv, snv, dt, xs, T, rem);
        if (take > 0) {
          const double ft = (double)take;
          nw2 = nn + take;
          nq = radd(qv, rmul(ft, xs));
          nsn = radd(snv, radd(rmul(rmul(2.0, ft), dt), rmul((double)(take * take), xs)));
        }
      }
      if (take > 0) {
        const double ft = (double)take;
        if (bt >= 0) {
          row_absorb(trow, xsm, nullptr, d, lane, take);
          if (lane == 0) { S.tw[bt] = nw2; S.tq[bt] = nq; S.tsn[bt] = nsn; }
          __syncwarp();
        } else {
          int child_now;
          if (touched) { if (ms < 0) ms = map3_find<MS>(S, bj); child_now = S.mchild[ms]; }
          else child_now = li >= 0 ? S.rb[cur][li].child : E.child[bj];
          ms = absorb_snapshot(bj, take, nw2, nq, nsn, child_now);
        }
        rem -= take;
        if (rem == 0) { if (L + 1 > maxdepth) maxdepth = L + 1; break; }
      }
      int c;
      if (bt >= 0) {
        c = S.tchild[bt];
        if (c < 0) {
          c = new_group();
          if (lane == 0) { S.tchild[bt] = c; E.g_count[c] = 0; E.g_cap[c] = 0; E.g_base[c] = 0; }
          __syncwarp();
        }
        direct = true;
      } else {
        const bool tnow = ((mbits[bj >> 5] >> (bj & 31)) & 1u) != 0;
        if (tnow && ms < 0) ms = map3_find<MS>(S, bj);
        c = tnow ? S.mchild[ms] : (li >= 0 ? S.rb[cur][li].child : E.child[bj]);
        if (c < 0) {
          c = new_group();
          if (lane == 0) { E.g_count[c] = 0; E.g_cap[c] = 0; E.g_base[c] = 0; E.child[bj] = c; }
          if (tnow) { if (lane == 0) S.mchild[ms] = c; __syncwarp(); }
          else ms = map3_put<MS>(S, mbits, bj, nn, qv, snv, c, lane);
        }
      }
      g = c;
      radius = rmul(radius, 0.25);
      ++L;
    }
    __syncwarp();
    ++c_it;
    if (status != ST_DONE) { if (has_next && bulk) rows_wait(&S.rbar[cur ^ 1], rph[cur ^ 1]); break; }
    if (has_next) {
      cp_async_wait_all();
      if (bulk) rows_wait(&S.rbar[cur ^ 1], rph[cur ^ 1]);
      __syncwarp();
      int nextnode = hn.predj;
      bool hit = nmod > 4 || nextnode == lastmod;
#pragma unroll
      for (int q = 0; q < 4; ++q) hit |= (modl[q] >= 0 && modl[q] == nextnode);
      if (nextnode >= 0 && hit) {
        if (nextnode == lastmod && prnode == lastmod) {
          double* nxt = pb + (long long)(cur ^ 1) * ld;
          for (int e = lane; e < ld; e += 32) nxt[e] = prow[e];
        } else {
          nextnode = -1;
        }
      }
      prnode = nextnode;
      hc = hn; hn = h2;
      bad_c = bad_n; w_c = w_n; xs_c = xs_n;
      cur ^= 1;
    }
    __syncwarp();
  }
  cp_async_wait_all();
  __syncwarp();

  // ---- cleanup
  if (TROWS) {
    for (int t = 0; t < nnew; ++t) {
      const int node = S.tid[t];
      const double* rr = tref + (long long)t * lds;
      const double* sr = ts + (long long)t * ld;
      for (int e = lane; e < ld; e += 32) { E.r[(long long)node * ld + e] = rr[e]; E.s[(long long)node * ld + e] = sr[e]; }
    }
  }
  for (int t = lane; t < nnew; t += 32) {
    const int node = S.tid[t];
    E.w[node] = S.tw[t]; E.q[node] = S.tq[t]; E.sn[node] = S.tsn[t]; E.rn[node] = S.trn[t];
    E.child[node] = S.tchild[t];
  }
  __syncwarp();
  if (!table_cleanup<MS>(E, S, nnew, Aalloc, lane, PAR ? par : nullptr)) status = ST_ARENA;
  if constexpr (PAR) {
    int lastf = 0;   // this CTA finished the window: its warp publishes
    if (lane == 0) {
      using ull = unsigned long long;
      if (status != ST_DONE) { atomicExch(&par->arena_fail, status == ST_ARENA ? ST_ARENA : ST_PAR_BROKEN); par->pad = status; }
      atomicAdd((ull*)&C->F, (ull)opened);
      atomicAdd((ull*)&C->total_w, (ull)totw);
      atomicMax(&C->max_depth, maxdepth);
      atomicAdd((ull*)&C->cnt_levels, (ull)c_lv); atomicAdd((ull*)&C->cnt_direct, (ull)c_dir);
      atomicAdd((ull*)&C->cnt_demand, (ull)c_dem); atomicAdd((ull*)&C->cnt_slow, (ull)c_slow);
      atomicAdd((ull*)&C->cnt_items, (ull)c_it);
      __threadfence();
      const ull ticket = atomicAdd(&par->done, 1ULL);
      if (ticket == (ull)par->P - 1) {
        __threadfence();
        const long long opens = (long long)*(volatile ull*)&par->open_ticket;
        const long long fr = par->freen0;
        C->free_n = opens < fr ? fr - opens : 0;
        C->F_alloc = par->Falloc0 + (opens > fr ? opens - fr : 0);
        C->G_alloc = par->Galloc0 + (long long)*(volatile ull*)&par->g_ticket;
        C->A_alloc = par->Aalloc0 + (long long)*(volatile ull*)&par->a_ticket;
        C->next_index = par->nidx0 + par->n_win;
        const int fail = *(volatile int*)&par->arena_fail;
        C->status = fail ? fail : (par->n_win < par->n_total ? ST_FULL : ST_DONE);
        C->err = fail ? par->pad : 0; C->stop = par->n_win; C->remaining = 0;
        __threadfence();
        lastf = 1;
      }
    }
    lastf = __shfl_sync(PCY_FULL, lastf, 0);
    if (lastf && pub) ctl_publish_warp(E, pub, pseq, lane);
    return;
  }
  if (par && status == ST_DONE && n < par->n_total) { status = ST_FULL; stop = n; }   // k_plan's sequential stretch
  if (lane == 0) {
    C->F = F; C->F_alloc = Falloc; C->free_n = freen; C->G_alloc = Galloc;
    C->A_alloc = Aalloc; C->next_index = nidx; C->total_w = totw; C->max_depth = maxdepth;
    C->status = status; C->err = err; C->stop = stop; C->remaining = remaining;
    C->cnt_levels += c_lv; C->cnt_direct += c_dir; C->cnt_demand += c_dem; C->cnt_slow += c_slow;
    C->cnt_items += c_it;
    __threadfence();
  }
  __syncwarp();
  if (pub) ctl_publish_warp(E, pub, pseq, lane);
}

template <bool TROWS, int MS, bool PAR = false>
__global__ void __launch_bounds__(32, 1) k_resolve3(EngDev E, const double* __restrict__ X,
                                                    const double* __restrict__ XS, const long long* __restrict__ W,
                                                    const int* __restrict__ BAD, long long n, long long first_rem,
                                                    int countw, int nnew_cap, const ChainHdr* __restrict__ H,
                                                    const ChainLvl* __restrict__ R, const double* __restrict__ gram,
                                                    long long gld, long long goff, ParCtl* __restrict__ par = nullptr) {
  resolve3_body<TROWS, MS, PAR>(E, X, XS, W, BAD, n, first_rem, countw, nnew_cap, H, R, gram, gld, goff, par, nullptr, 0);
}

// One launch for either choice of k_plan (as k_resolve2x).
template <bool TROWS, int MS>
__global__ void __launch_bounds__(32, 1) k_resolve3x(EngDev E, const double* __restrict__ X,
                                                     const double* __restrict__ XS, const long long* __restrict__ W,
                                                     const int* __restrict__ BAD, long long n, long long first_rem,
                                                     int countw, int nnew_cap, const ChainHdr* __restrict__ H,
                                                     const ChainLvl* __restrict__ R, const double* __restrict__ gram,
                                                     long long gld, long long goff, ParCtl* __restrict__ par,
                                                     EngCtl* pub, long long pseq) {
  pdl_wait();   // k_plan has finished (programmatic launch)
  if (par->mode == 0)
    resolve3_body<TROWS, MS, true>(E, X, XS, W, BAD, n, first_rem, countw, nnew_cap, H, R, gram, gld, goff, par, pub, pseq);
  else if (blockIdx.x == 0)
    resolve3_body<TROWS, MS, false>(E, X, XS, W, BAD, n, first_rem, countw, nnew_cap, H, R, gram, gld, goff, par, pub, pseq);
}

// ------------------------------------------------------------- reattach
template <bool TROWS, int MS, bool PAR>
__device__ __forceinline__ void reattach3_body(const EngDev& E, const int* __restrict__ order, long long n,
                                               int nnew_cap, const ChainHdr* __restrict__ H,
                                               const ChainLvl* __restrict__ R, const double* __restrict__ gram,
                                               long long gld, long long goff, ParCtl* __restrict__ par,
                                               EngCtl* pub, long long pseq) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ResolveSmemT<MS>& S = *reinterpret_cast<ResolveSmemT<MS>*>(smraw);
  const int lane = threadIdx.x;
  const int* ilist = nullptr;
  if constexpr (PAR) {
    if (par->mode != 0 || (int)blockIdx.x >= par->P) return;
    const int o0 = par->off[blockIdx.x];
    ilist = par->list + o0;
    n = par->off[blockIdx.x + 1] - o0;
  } else {
    if (par) {
      if (par->mode != 1) return;
      n = par->n_win;
    }
  }
  auto gix = [&](long long j) -> long long {
    if constexpr (PAR) return (long long)ilist[j];
    else return j;
  };
  const int d = E.d, ld = E.ld;
  double* xb = reinterpret_cast<double*>(smraw + ((sizeof(ResolveSmemT<MS>) + 15) & ~size_t(15)));
  double* pb = xb + 2 * (long long)ld;     // [2][ld]: predicted host rows
  double* sb = pb + 2 * (long long)ld;     // [2][ld]: the item's own s row
  const int lds = ld | 1;
  double* tref = sb + 2 * (long long)ld;
  unsigned* mbits = reinterpret_cast<unsigned*>(tref + (TROWS ? (long long)nnew_cap * (lds + ld) : 0));
  const int mwords = (int)(E.NC / 32 + 1);
  unsigned* gbits = mbits + mwords;
  const int gwords = (int)(E.GC / 32 + 1);
  EngCtl* C = E.ctl;
  const double T = C->T;
  long long F = C->F, freen = C->free_n, Galloc = C->G_alloc, Aalloc = C->A_alloc;
  long long G0 = Galloc;
  if constexpr (PAR) { G0 = par->Galloc0; F = 0; freen = 0; }
  auto new_group = [&]() -> int {
    if constexpr (PAR) {
      unsigned long long t = 0;
      if (lane == 0) t = atomicAdd(&par->g_ticket, 1ULL);
      return (int)(par->Galloc0 + (long long)__shfl_sync(PCY_FULL, t, 0));
    } else {
      return (int)Galloc++;
    }
  };
  int status = ST_DONE; long long stop = n;

  for (int s2 = lane; s2 < MS; s2 += 32) S.mkey[s2] = -1;
  for (int s2 = lane; s2 < PCY_GMAP_SLOTS; s2 += 32) S.gkey[s2] = -1;
  for (int s2 = lane; s2 < mwords; s2 += 32) mbits[s2] = 0u;
  for (int s2 = lane; s2 < gwords; s2 += 32) gbits[s2] = 0u;
  if (lane == 0) S.modcount = 0;
  int nnew = 0;

  int u_c = n > 0 ? order[gix(0)] : 0;
  int u_n = n > 1 ? order[gix(1)] : 0;
  ChainHdr hc = n > 0 ? H[gix(0)] : ChainHdr{0, 0, -1, 0};
  ChainHdr hn = n > 1 ? H[gix(1)] : ChainHdr{0, 0, -1, 0};
  long long wu_c = 0; double qu_c = 0.0, snu_c = 0.0, rsq_c = 0.0;
  rows_bar_init(S.rbar, 2, lane);
  unsigned rph[2] = {0u, 0u};
  const bool bulk = ld >= 2048;
  if (n > 0) {
    rows_fetch(bulk, &S.rbar[0], lane, ld, xb, E.r + (long long)u_c * ld, sb, E.s + (long long)u_c * ld, pb,
               hc.predj >= 0 ? E.s + (long long)hc.predj * ld : nullptr);
    wu_c = E.w[u_c]; qu_c = E.q[u_c]; snu_c = E.sn[u_c]; rsq_c = E.rn[u_c];
    const uint4* src = reinterpret_cast<const uint4*>(R + gix(0) * PCY_FMAXL);
    uint4* dst = reinterpret_cast<uint4*>(&S.rb[0][0]);
    for (int c = lane; c < REC3_CHUNKS; c += 32) cp_async16(dst + c, src + c);
    cp_async_commit();
    cp_async_wait_all();
    if (bulk) rows_wait(&S.rbar[0], rph[0]);
  }
  __syncwarp();
  int cur = 0;
  int prnode = hc.predj;

  for (long long i = 0; i < n; ++i) {
    if (nnew >= nnew_cap || S.modcount >= MS / 2) { status = ST_FULL; stop = i; break; }
    double* xsm = xb + (long long)cur * ld;
    double* prow = pb + (long long)cur * ld;
    const double* su = sb + (long long)cur * ld;
    const bool has_next = i + 1 < n;
    ChainHdr h2 = ChainHdr{0, 0, -1, 0};
    int u2 = 0;
    long long wu_n = 0; double qu_n = 0.0, snu_n = 0.0, rsq_n = 0.0;
    if (has_next) {
      rows_fetch(bulk, &S.rbar[cur ^ 1], lane, ld, xb + (long long)(cur ^ 1) * ld, E.r + (long long)u_n * ld,
                 sb + (long long)(cur ^ 1) * ld, E.s + (long long)u_n * ld, pb + (long long)(cur ^ 1) * ld,
                 hn.predj >= 0 ? E.s + (long long)hn.predj * ld : nullptr);
      const uint4* src = reinterpret_cast<const uint4*>(R + gix(i + 1) * PCY_FMAXL);
      uint4* dst = reinterpret_cast<uint4*>(&S.rb[cur ^ 1][0]);
      for (int c = lane; c < REC3_CHUNKS; c += 32) cp_async16(dst + c, src + c);
      cp_async_commit();
      wu_n = E.w[u_n]; qu_n = E.q[u_n]; snu_n = E.sn[u_n]; rsq_n = E.rn[u_n];
      if (i + 2 < n) { h2 = H[gix(i + 2)]; u2 = order[gix(i + 2)]; }
    }
    const int u = u_c;
    const int len = hc.len;
    int g = 0, L = 0;
    double radius = T;
    bool direct = false;
    int lastmod = -1;
    unsigned cleanmask = 0u;   // unchanged levels above K1's action level (see k_reattach2)
    if (!hc.trunc && hc.pred > 0 && hc.pred < len) {
      bool cl = false;
      if (lane < hc.pred) {
        const ChainLvl& rl = S.rb[cur][lane];
        const int g2 = rl.g, j2 = rl.j;
        const bool bad = (g2 >= 0 && ((gbits[g2 >> 5] >> (g2 & 31)) & 1u)) || (j2 >= 0 && ((mbits[j2 >> 5] >> (j2 & 31)) & 1u));
        cl = !bad && g2 >= 0 && j2 >= 0 && rl.child >= 0 && rl.take == 0;
      }
      cleanmask = __ballot_sync(PCY_FULL, cl);
    }
    for (;;) {
      if (!direct && ((cleanmask >> L) & 1u)) {   // unchanged level: K1's descent stands
        g = S.rb[cur][L].child;
        radius = rmul(radius, 0.25);
        ++L;
        continue;
      }
      int bj = -1, li = -1;
      double bp = INFINITY;
      if (!direct) {
        if (L < len) { li = L; bj = S.rb[cur][L].j; bp = S.rb[cur][L].part; }
        else direct = true;
      }
      if (direct && g < G0) {
        const int cnt = E.g_count[g];
        if (cnt > 0) {
          double p; int ps;
          const int* mem = E.arena + E.g_base[g];
          scan_members(E, mem, 0, cnt, xsm, lane, p, ps);
          if (ps < cnt) { bj = mem[ps]; bp = p; }
        }
      }
      int bt = -1;
      scan_new<TROWS, MS>(E, S, gbits, tref, lds, xsm, g, nnew, lane, bp, bj, bt, gram, gld, goff + gix(i));
      if (bj < 0 || radd(bp, rsq_c) > radius) {
        // group.add(node): u keeps its statistics (coreset.py:403-406)
        const int t = nnew++;
        if (TROWS) {
          double* rr = tref + (long long)t * lds;
          for (int e = lane; e < ld; e += 32) rr[e] = xsm[e];
        }
        gchain_append<MS>(S, gbits, g, t, lane);
        if (lane == 0) {
          S.titem[t] = (int)(goff + gix(i));
          S.tid[t] = u; S.tgrp[t] = g; S.tchild[t] = -1;
          S.tw[t] = wu_c; S.tq[t] = qu_c; S.tsn[t] = snu_c; S.trn[t] = rsq_c;
        }
        ++F;
        __syncwarp();
        break;
      }
      const bool touched = bt < 0 && ((mbits[bj >> 5] >> (bj & 31)) & 1u);
      int ms = -1;
      bool merge;
      long long mw; double mq, mnorm, hq, hsn; long long hw;
      if (bt < 0 && li >= 0 && !touched) {
        const ChainLvl& rc = S.rb[cur][li];
        hw = rc.w; hq = rc.q; hsn = rc.sn;
        merge = rc.take != 0; mw = rc.w + wu_c; mq = rc.nq; mnorm = rc.nsn;
      } else {
        if (bt >= 0) { hw = S.tw[bt]; hq = S.tq[bt]; hsn = S.tsn[bt]; }
        else if (touched) { ms = map3_find<MS>(S, bj); hw = S.mw[ms]; hq = S.mq[ms]; hsn = S.msn[ms]; }
        else { hw = E.w[bj]; hq = E.q[bj]; hsn = E.sn[bj]; }
        if (bj != prnode) {
          const double* src = E.s + (long long)bj * ld;
          for (int e = lane; e < ld; e += 32) prow[e] = src[e];
          __syncwarp();
          prnode = bj;
        }
        double acc = 0.0;
        for (int e = lane; e < d; e += 32) { const double v = radd(prow[e], su[e]); acc = fma(v, v, acc); }
        mnorm = warp_sum(acc);
        mw = hw + wu_c; mq = radd(hq, qu_c);
        merge = rsub(mq, rdiv(mnorm, (double)mw)) <= T;
      }
      if (merge) {
        if (bj != prnode) {
          const double* src = E.s + (long long)bj * ld;
          for (int e = lane; e < ld; e += 32) prow[e] = src[e];
          __syncwarp();
          prnode = bj;
        }
        double* dst = E.s + (long long)bj * ld;
        row_absorb(prow, su, dst, d, lane, 1);
        __syncwarp();
        if (bt >= 0) {
          if (lane == 0) { S.tw[bt] = mw; S.tq[bt] = mq; S.tsn[bt] = mnorm; }
          __syncwarp();
        } else {
          int child_now;
          if (touched) { if (ms < 0) ms = map3_find<MS>(S, bj); child_now = S.mchild[ms]; }
          else child_now = li >= 0 ? S.rb[cur][li].child : E.child[bj];
          ms = map3_put<MS>(S, mbits, bj, mw, mq, mnorm, child_now, lane);
          if (lane == 0) { E.w[bj] = mw; E.q[bj] = mq; E.sn[bj] = mnorm; }
        }
        if constexpr (PAR) {
          if (lane == 0) {
            E.alive[u] = 0;
            const unsigned long long tk = atomicAdd(&par->open_ticket, 1ULL);   // free-stack pushes
            E.free_ids[par->freen0 + (long long)tk] = u;
          }
        } else {
          if (lane == 0) { E.alive[u] = 0; E.free_ids[freen] = u; }
          ++freen;
        }
        lastmod = bj;
        __syncwarp();
        break;
      }
      int c;
      if (bt >= 0) {
        c = S.tchild[bt];
        if (c < 0) {
          c = new_group();
          if (lane == 0) { S.tchild[bt] = c; E.g_count[c] = 0; E.g_cap[c] = 0; E.g_base[c] = 0; }
          __syncwarp();
        }
        direct = true;
      } else {
        const bool tnow = ((mbits[bj >> 5] >> (bj & 31)) & 1u) != 0;
        if (tnow && ms < 0) ms = map3_find<MS>(S, bj);
        c = tnow ? S.mchild[ms] : (li >= 0 ? S.rb[cur][li].child : E.child[bj]);
        if (c < 0) {
          c = new_group();
          if (lane == 0) { E.g_count[c] = 0; E.g_cap[c] = 0; E.g_base[c] = 0; E.child[bj] = c; }
          if (tnow) { if (lane == 0) S.mchild[ms] = c; __syncwarp(); }
          else ms = map3_put<MS>(S, mbits, bj, hw, hq, hsn, c, lane);
        }
      }
      g = c;
      radius = rmul(radius, 0.25);
      ++L;
    }
    __syncwarp();
    if (has_next) {
      cp_async_wait_all();
      if (bulk) rows_wait(&S.rbar[cur ^ 1], rph[cur ^ 1]);
      __syncwarp();
      int nextnode = hn.predj;
      if (nextnode >= 0 && nextnode == lastmod) {
        if (prnode == lastmod) {
          double* nxt = pb + (long long)(cur ^ 1) * ld;
          for (int e = lane; e < ld; e += 32) nxt[e] = prow[e];
        } else nextnode = -1;
      }
      prnode = nextnode;
      hc = hn; hn = h2;
      u_c = u_n; u_n = u2;
      wu_c = wu_n; qu_c = qu_n; snu_c = snu_n; rsq_c = rsq_n;
      cur ^= 1;
    }
    __syncwarp();
  }
  cp_async_wait_all();
  __syncwarp();
  for (int t = lane; t < nnew; t += 32) {
    const int node = S.tid[t];
    E.w[node] = S.tw[t]; E.q[node] = S.tq[t]; E.sn[node] = S.tsn[t];
    E.child[node] = S.tchild[t];
  }
  __syncwarp();
  if (!table_cleanup<MS>(E, S, nnew, Aalloc, lane, PAR ? par : nullptr)) status = ST_ARENA;
  if constexpr (PAR) {
    int lastf = 0;   // this CTA finished the window: its warp publishes
    if (lane == 0) {
      using ull = unsigned long long;
      if (status != ST_DONE) { atomicExch(&par->arena_fail, status == ST_ARENA ? ST_ARENA : ST_PAR_BROKEN); par->pad = status; }
      atomicAdd((ull*)&C->F, (ull)F);
      __threadfence();
      const ull ticket = atomicAdd(&par->done, 1ULL);
      if (ticket == (ull)par->P - 1) {
        __threadfence();
        C->free_n = par->freen0 + (long long)*(volatile ull*)&par->open_ticket;
        C->G_alloc = par->Galloc0 + (long long)*(volatile ull*)&par->g_ticket;
        C->A_alloc = par->Aalloc0 + (long long)*(volatile ull*)&par->a_ticket;
        const int fail = *(volatile int*)&par->arena_fail;
        C->status = fail ? fail : (par->n_win < par->n_total ? ST_FULL : ST_DONE);
        C->stop = par->n_win;
        __threadfence();
        lastf = 1;
      }
    }
    lastf = __shfl_sync(PCY_FULL, lastf, 0);
    if (lastf && pub) ctl_publish_warp(E, pub, pseq, lane);
    return;
  }
  if (par && status == ST_DONE && n < par->n_total) { status = ST_FULL; stop = n; }   // k_plan's sequential stretch
  if (lane == 0) {
    C->F = F; C->free_n = freen; C->G_alloc = Galloc; C->A_alloc = Aalloc;
    C->status = status; C->stop = stop;
    __threadfence();
  }
  __syncwarp();
  if (pub) ctl_publish_warp(E, pub, pseq, lane);
}

template <bool TROWS, int MS, bool PAR = false>
__global__ void __launch_bounds__(32, 1) k_reattach3(EngDev E, const int* __restrict__ order, long long n,
                                                     int nnew_cap, const ChainHdr* __restrict__ H,
                                                     const ChainLvl* __restrict__ R, const double* __restrict__ gram,
                                                     long long gld, long long goff, ParCtl* __restrict__ par = nullptr) {
  reattach3_body<TROWS, MS, PAR>(E, order, n, nnew_cap, H, R, gram, gld, goff, par, nullptr, 0);
}

// One launch for either choice of k_plan (as k_resolve2x).
template <bool TROWS, int MS>
__global__ void __launch_bounds__(32, 1) k_reattach3x(EngDev E, const int* __restrict__ order, long long n,
                                                      int nnew_cap, const ChainHdr* __restrict__ H,
                                                      const ChainLvl* __restrict__ R, const double* __restrict__ gram,
                                                      long long gld, long long goff, ParCtl* __restrict__ par,
                                                      EngCtl* pub, long long pseq) {
  pdl_wait();   // k_plan has finished (programmatic launch)
  if (par->mode == 0) reattach3_body<TROWS, MS, true>(E, order, n, nnew_cap, H, R, gram, gld, goff, par, pub, pseq);
  else if (blockIdx.x == 0) reattach3_body<TROWS, MS, false>(E, order, n, nnew_cap, H, R, gram, gld, goff, par, pub, pseq);
}
