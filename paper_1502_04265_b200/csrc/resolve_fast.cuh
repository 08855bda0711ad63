// K1/K3 fast path for ld <= 256 (included by engine.cu after its helpers).
//
// k_chain2 (K1, warp per item, all items in parallel) records for every level
// of an item's capacity-free chain the snapshot winner, its part, the snapshot
// scalars (w, q, sn) of that node and the direct dot <s_j, x>, plus the level
// at which the snapshot statistics say the item would stop (pred).
//
// k_resolve2 (K3, one warp, items in order) re-decides every level with the
// *current* state.  State changed inside the launch lives in shared memory:
//   * new-node table: nodes opened in this launch (ref row, s row, scalars,
//     group, child) -- these are the only members appended since the snapshot;
//   * modified map:   current (w, q, sn, child) of snapshot nodes touched in
//     this launch (their s rows are written through to HBM).
// Snapshot values from K1 are used whenever a node is untouched, so the common
// item needs no HBM round trip on its critical path: its x row, chain record
// and the s row of its predicted node are prefetched one item ahead.
// <s, x> is always the same lane-strided fp64 dot (warp_dot order), whether
// K1 or K3 evaluates it, so both produce identical values.
#pragma once

#define PCY_FMAXL 16
#define PCY_MOD_SLOTS 2048
#define PCY_NNEW_MAX 96    // new-node table of the large-d kernels (resolve_smem.cuh)
#define PCY_NNEW_FAST 160  // new-node table of k_resolve2 (d <= 256), capped by shared memory
#define PCY_NNEW_REA 320   // new-node table of k_reattach2 (Gram dots: no reference rows in shared memory)
#define PCY_GMAP_SLOTS 256

struct __align__(16) ChainLvl {
  double part, dot, q, sn;   // snapshot winner: part, <s_j, x>, q_j, sn_j
  double nq, nsn;            // post-update q / sn when take > 0 (snapshot statistics)
  long long w, take;         // snapshot weight; copies taken at this level (rem = W[i])
  int j, g, child, pad;      // winner node, group of the level, snapshot child group
};
struct __align__(16) ChainHdr { int len, pred, predj, trunc; };

__device__ __forceinline__ ChainLvl empty_level() {
  ChainLvl t;
  t.part = INFINITY; t.dot = 0.0; t.q = 0.0; t.sn = 0.0; t.nq = 0.0; t.nsn = 0.0;
  t.w = 0; t.take = 0; t.j = -1; t.g = -1; t.child = -1; t.pad = 0;
  return t;
}

// Closed-form capacity (coreset.py:336-356, inlined max_insertable_copies).
__device__ __forceinline__ long long capacity(long long nn, double qv, double snv, double dt, double xs,
                                              double T, long long rem) {
  const double fn = (double)nn;
  const double nrm = rdiv(snv, fn);
  double errv = rsub(qv, nrm);
  if (errv < 0.0) errv = 0.0;
  double dist = rsub(xs, rdiv(rsub(rmul(2.0, dt), nrm), fn));
  if (dist < 0.0) dist = 0.0;
  const double slack = radd(rsub(rmul(fn, dist), T), errv);
  if (slack <= 0.0) return rem;
  const double limit = rdiv(rsub(rmul(fn, T), rmul(fn, errv)), slack);
  if (limit >= (double)rem) return rem;
  if (limit > 0.0) return (long long)limit;
  return 0;
}

// ------------------------------------------------------------------- K1
template <int WPI>
__global__ void k_chain2(EngDev E, const double* __restrict__ X, const double* __restrict__ XS,
                         const long long* __restrict__ W, long long n, ChainHdr* __restrict__ H,
                         ChainLvl* __restrict__ R, const double* __restrict__ P, long long ldp,
                         long long wait_seq = 0) {
  // WPI == 1: one warp per item, several items per CTA.  WPI > 1: one item per
  // CTA; every warp walks the same chain (identical decisions) and the fp64
  // dots are split over the warps (cta_dot), for large d.
  extern __shared__ double sm_x[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // run-ahead launch: the previous window's resolve kernel has finished its
  // tree writes (wait_seq: its publication number) / has completed
  if (wait_seq > 0) flag_wait(&E.ctl->win_done, wait_seq);
  else pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) PCY_TL(1);
  const long long i = WPI == 1 ? (long long)blockIdx.x * (blockDim.x >> 5) + wib : (long long)blockIdx.x;
  if (i >= n) return;
  const int d = E.d, ld = E.ld;
  double* xv = WPI == 1 ? sm_x + (long long)wib * ld : sm_x;
  double* red = sm_x + ld;
  const bool writer = lane == 0 && (WPI == 1 || wib == 0);
  auto xdot = [&](const double* row) -> double {
    if constexpr (WPI == 1) return warp_dot(row, xv, d, lane);
    else return cta_dot<WPI>(row, xv, d, lane, wib, red);
  };
  const double xs = XS[i];
  ChainLvl* rec = R + i * PCY_FMAXL;
  if (!isfinite(xs)) { if (writer) H[i] = ChainHdr{0, 0, -1, 0}; return; }
  if constexpr (WPI == 1) {
    for (int e = lane; e < d; e += 32) xv[e] = X[i * ld + e];
    __syncwarp();
  } else {
    for (int e = threadIdx.x; e < d; e += blockDim.x) xv[e] = X[i * ld + e];
    __syncthreads();
  }
  const double T = E.ctl->T;
  const long long rem = W ? W[i] : 1LL;
  double radius = T;
  int g = 0, L = 0, pred = -1, predj = -1, trunc = 0, nre = 0;
  long long vis = 0, vdir = 0;   // member visits (all / direct scans)
  // the next level's group (count, base, panel column) is loaded as soon as
  // its id is known, overlapping the <s_j, x> dot of the current level
  int cnt = E.g_count[0], base = E.g_base[0];
  int pb = E.panel_gofs ? E.panel_gofs[0] : -1;
  for (;;) {
    double bp; int bpos;
    LaneWinner win{-1, -1, 0, 0.0, 0.0};
    bool have_win = false;
    // visited-groups K1 (panel mode, d <= 256): big groups from the tensor-core
    // panel, the others by direct fp64 scans; otherwise the full-set contraction
    vis += cnt;
    if (E.panel_gofs) {
      if constexpr (WPI == 1) {
        if (E.tc_dots && pb >= 0)
          scan_parts_tc(E, i, g, E.arena + base, cnt, [&](int jj) { return xdot(E.r + (long long)jj * ld); }, lane,
                        bp, bpos, nre, pb);
        else { scan_members_lane_w(E, E.arena + base, cnt, xv, lane, bp, bpos, win); vdir += cnt; have_win = true; }
      }
    } else if (E.tc_dots) {   // tensor-core dots + near-tie recheck
      if constexpr (WPI == 1)
        scan_parts_tc(E, i, g, E.arena + base, cnt, [&](int jj) { return xdot(E.r + (long long)jj * ld); }, lane, bp,
                      bpos, nre);
      else
        scan_parts_tc_cta<WPI>(E, i, E.arena + base, cnt, [&](int jj) { return xdot(E.r + (long long)jj * ld); },
                               lane, wib, red, reinterpret_cast<int*>(red + 8), bp, bpos, nre);
    }
    else if (P) scan_parts(P + i * ldp, E.col_of, E.arena + base, cnt, lane, bp, bpos);   // DMMA parts
    else { scan_members(E, E.arena + base, 0, cnt, xv, lane, bp, bpos); vdir += cnt; }
    const int j = have_win ? (bpos < cnt ? win.id : -1) : (bpos < cnt ? E.arena[base + bpos] : -1);
    ChainLvl c = empty_level();
    c.part = bp; c.j = j; c.g = g;
    int ncnt = 0, nbase = 0, npb = -1;
    if (j >= 0) {
      if (have_win) { c.w = win.w; c.q = win.q; c.sn = win.sn; c.child = win.child; }
      else { c.w = E.w[j]; c.q = E.q[j]; c.sn = E.sn[j]; c.child = E.child[j]; }
      if (c.child >= 0) {   // issued before the dot: both round trips overlap
        ncnt = E.g_count[c.child]; nbase = E.g_base[c.child];
        npb = E.panel_gofs ? E.panel_gofs[c.child] : -1;
      }
      c.dot = xdot(E.s + (long long)j * ld);
    }
    ++L;
    const bool outside = j < 0 || radd(bp, xs) > radius;
    if (!outside) {
      c.take = capacity(c.w, c.q, c.sn, c.dot, xs, T, rem);
      if (c.take > 0) {
        const double ft = (double)c.take;
        c.nq = radd(c.q, rmul(ft, xs));
        c.nsn = radd(c.sn, radd(rmul(rmul(2.0, ft), c.dot), rmul((double)(c.take * c.take), xs)));
        if (pred < 0) { pred = L - 1; predj = j; }
      }
    }
    if (writer) { rec[L - 1] = c; E.pathj[i * PCY_FMAXL + L - 1] = c.j; }
    if (outside) { if (pred < 0) pred = L - 1; break; }
    if (c.child < 0) {
      if (L < PCY_FMAXL) {
        if (writer) { rec[L] = empty_level(); E.pathj[i * PCY_FMAXL + L] = -1; }
        ++L;
        if (pred < 0) pred = L - 1;
      } else trunc = 1;
      break;
    }
    if (L >= PCY_FMAXL) { trunc = 1; break; }
    g = c.child;
    cnt = ncnt; base = nbase; pb = npb;
    radius = rmul(radius, 0.25);
  }
  if (pred < 0) pred = L - 1;
  if (writer) H[i] = ChainHdr{L, pred, predj, trunc};
  if (writer && nre > 0) atomicAdd((unsigned long long*)&E.ctl->cnt_direct, (unsigned long long)nre);
  if (writer) {
    atomicAdd((unsigned long long*)&E.ctl->cnt_vis, (unsigned long long)vis);
    if (vdir) atomicAdd((unsigned long long*)&E.ctl->cnt_vis_direct, (unsigned long long)vdir);
  }
}

// ------------------------------------------------------------------- K3
template <int NT>
struct ResolveSmemN {
  ChainLvl rb[4][PCY_FMAXL];                 // chain records: staging ring (k_resolve2) / double buffer
  int mkey[PCY_MOD_SLOTS], mchild[PCY_MOD_SLOTS];   // touched snapshot nodes
  long long mw[PCY_MOD_SLOTS];
  double mq[PCY_MOD_SLOTS], msn[PCY_MOD_SLOTS];
  int gkey[PCY_GMAP_SLOTS], ghead[PCY_GMAP_SLOTS], gtail[PCY_GMAP_SLOTS];  // groups with new members
  int tid[NT], tgrp[NT], tchild[NT], tnext[NT];
  int tk[NT], tfirst[NT], tcnt[NT], tbase[NT], tcap[NT];
  int titem[NT];   // k_reattach2: batch row of the node that placed the entry (its Gram row)
  int tgn[NT];     // k_reattach2: new entries of the group, at the group's first entry
  int tdirty[NT];  // k_reattach2: the entry's shared-memory s row took a merge
  long long tw[NT];
  double trn[NT], tq[NT], tsn[NT];
  // item staging ring of k_resolve2 (producer warp -> decision warp), K3_SLOTS slots
  ChainHdr shdr[4];
  long long sw[4];
  double sxs[4];
  int sbad[4];
  int stop_flag;
  int modcount;
};
using ResolveSmem = ResolveSmemN<PCY_NNEW_FAST>;
using ReattachSmem = ResolveSmemN<PCY_NNEW_REA>;
// dynamic tail: double slotx[4][ld], slotp[4][ld]; double tref[nnew][ld|1]; double ts[nnew][ld];
// (k_reattach2 keeps a single xsm[ld] and no ts, see reattach_smem_bytes)
//               unsigned mbits[NC/32+1]; unsigned gbits[GC/32+1]

__host__ __device__ inline size_t resolve_smem_bytes(int ld, int nnew, long long NC, long long GC) {
  return ((sizeof(ResolveSmem) + 15) & ~size_t(15)) + sizeof(double) * ((size_t)8 * ld + (size_t)nnew * ((size_t)(ld | 1) + ld)) +
         ((sizeof(unsigned) * (size_t)(NC / 32 + 1 + GC / 32 + 1) + 15) & ~size_t(15));
}
// k_reattach2 keeps only the reference rows of its new entries (no s rows),
// and none when the batch Gram gives their dots (trows = false)
__host__ __device__ inline size_t reattach_smem_bytes(int ld, int nnew, long long NC, long long GC, bool trows = true) {
  // without reference rows the current and the next item's batch-Gram rows are staged instead
  return ((sizeof(ReattachSmem) + 15) & ~size_t(15)) + sizeof(double) * ((size_t)ld + (trows ? (size_t)nnew * (size_t)(ld | 1) : 0)) +
         ((sizeof(unsigned) * (size_t)(NC / 32 + 1 + GC / 32 + 1) + 15) & ~size_t(15)) +
         (trows ? 0 : sizeof(double) * 2 * PCY_PAR_MAXITEMS);
}

__device__ __forceinline__ int map_slot(int id) { return (int)(((unsigned)id * 2654435761u) >> 21) & (PCY_MOD_SLOTS - 1); }

template <class SM>
__device__ __forceinline__ int map_find(const SM& S, int id) {
  int s = map_slot(id);
  for (;;) {
    const int k = S.mkey[s];
    if (k == id) return s;
    if (k < 0) return -1;
    s = (s + 1) & (PCY_MOD_SLOTS - 1);
  }
}

// insert-or-update; lane 0 writes; caller syncs.  *fresh (nullable, every
// lane) is incremented when the key was not present.
template <class SM>
__device__ __forceinline__ int map_put(SM& S, unsigned* mbits, int id, long long w, double q, double sn,
                                       int child, int lane, int* fresh = nullptr) {
  int s = map_slot(id);
  while (S.mkey[s] >= 0 && S.mkey[s] != id) s = (s + 1) & (PCY_MOD_SLOTS - 1);
  if (fresh && S.mkey[s] < 0) ++*fresh;
  __syncwarp();
  if (lane == 0) {
    if (S.mkey[s] < 0) { S.modcount++; mbits[id >> 5] |= 1u << (id & 31); }
    S.mkey[s] = id; S.mw[s] = w; S.mq[s] = q; S.msn[s] = sn; S.mchild[s] = child;
  }
  __syncwarp();
  return s;
}

template <class SM>
__device__ __forceinline__ int gmap_find(const SM& S, int g) {
  int s = (int)(((unsigned)g * 2654435761u) >> 24) & (PCY_GMAP_SLOTS - 1);
  for (;;) {
    const int k = S.gkey[s];
    if (k == g) return s;
    if (k < 0) return -1;
    s = (s + 1) & (PCY_GMAP_SLOTS - 1);
  }
}

template <int NPER>
__device__ __forceinline__ double reg_dot(const double (&a)[NPER], const double (&b)[NPER]) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < NPER; ++k) acc = fma(a[k], b[k], acc);
  return warp_sum(acc);
}

template <int NPER>
__device__ __forceinline__ double smem_dot(const double* __restrict__ row, const double (&x)[NPER], int d, int lane) {
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < NPER; ++k) { const int e = lane + 32 * k; if (e < d) acc = fma(row[e], x[k], acc); }
  return warp_sum(acc);
}

template <int NPER>
__device__ __forceinline__ void load_row(double (&r)[NPER], const double* __restrict__ src, int d, int lane) {
#pragma unroll
  for (int k = 0; k < NPER; ++k) { const int e = lane + 32 * k; r[k] = e < d ? src[e] : 0.0; }
}

template <int NPER>
__device__ __forceinline__ void store_row(double* __restrict__ dst, const double (&r)[NPER], int d, int lane) {
#pragma unroll
  for (int k = 0; k < NPER; ++k) { const int e = lane + 32 * k; if (e < d) dst[e] = r[k]; }
}

constexpr int REC_CHUNKS = PCY_FMAXL * (int)sizeof(ChainLvl) / 16;   // uint4 per record

// named barriers between the decision warp and the staging warp of k_resolve2
__device__ __forceinline__ void nbar_sync(int id, int cnt) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
__device__ __forceinline__ void nbar_arrive(int id, int cnt) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
constexpr int K3_SLOTS = 4, K3_BAR_FULL = 1, K3_BAR_EMPTY = 1 + K3_SLOTS;   // + slot

// PAR = false: one CTA resolves items 0..n-1 in stream order (with `par`
// non-null it runs only when k_plan chose the sequential mode, for
// par->n_win items).  PAR = true: CTA b resolves the items of root subtree
// list b of k_plan's window (see ParCtl), allocating through the tickets.
// pub / pseq (k_resolve2x only): the CTA that finishes the window copies the
// counters to the host mirror itself (no separate publication launch).
template <int NPER, bool PAR>
__device__ __forceinline__ void resolve2_body(const EngDev& E, const double* __restrict__ X,
                                              const double* __restrict__ XS, const long long* __restrict__ W,
                                              const int* __restrict__ BAD, long long n, long long first_rem,
                                              int countw, int nnew_cap, const ChainHdr* __restrict__ H,
                                              const ChainLvl* __restrict__ R, ParCtl* __restrict__ par,
                                              EngCtl* pub, long long pseq) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ResolveSmem& S = *reinterpret_cast<ResolveSmem*>(smraw);
  const int lane = threadIdx.x & 31;
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
  // window position of local item j (the block row K1 chained)
  auto gix = [&](long long j) -> long long {
    if constexpr (PAR) return (long long)ilist[j];
    else return j;
  };
  const int d = E.d, ld = E.ld;
  double* slotx = reinterpret_cast<double*>(smraw + ((sizeof(ResolveSmem) + 15) & ~size_t(15)));   // [K3_SLOTS][ld]
  double* slotp = slotx + K3_SLOTS * ld;                                                             // [K3_SLOTS][ld]
  const int lds = ld | 1;   // odd stride: conflict-free lane-per-row reads
  double* tref = slotp + K3_SLOTS * ld;
  double* ts = tref + (long long)nnew_cap * lds;
  unsigned* mbits = reinterpret_cast<unsigned*>(ts + (long long)nnew_cap * ld);
  const int mwords = (int)(E.NC / 32 + 1);
  unsigned* gbits = mbits + mwords;
  const int gwords = (int)(E.GC / 32 + 1);

  if (threadIdx.x >= 32) {
    // ---- staging warp: item j's header, scalars, x row, chain levels and
    // predicted s row into slot j&1, once the decision warp has finished item
    // j-2 (the slot's previous user).  Rows of nodes the decision warp rewrites
    // meanwhile may be read stale or torn here; the decision warp never uses a
    // predicted row of a node that the previous item rewrote.
    // software pipeline: item j+1's rows are in registers while item j is
    // stored; headers run two items ahead (a record's length and predicted
    // node are needed to issue its loads)
    constexpr int RQ = (REC_CHUNKS + 31) / 32;
    struct Stage { double x[NPER], p[NPER]; uint4 r[RQ]; ChainHdr h; int bad; long long w; double xs; };
    auto fetch = [&](Stage& t, long long jl, const ChainHdr& h) {
      const long long j = gix(jl);
      t.h = h;
      t.bad = BAD ? BAD[j] : 0; t.w = W ? W[j] : 1LL; t.xs = XS[j];
      load_row<NPER>(t.x, X + j * ld, d, lane);
      if (h.predj >= 0) load_row<NPER>(t.p, E.s + (long long)h.predj * ld, d, lane);
      const uint4* src = reinterpret_cast<const uint4*>(R + j * PCY_FMAXL);
      const int nch = h.len * (int)(sizeof(ChainLvl) / 16);
#pragma unroll
      for (int q = 0; q < RQ; ++q) { const int c = lane + 32 * q; if (c < nch) t.r[q] = src[c]; }
    };
    Stage cur_st, nxt_st;
    ChainHdr h_ahead = n > 1 ? H[gix(1)] : ChainHdr{0, 0, -1, 0};
    if (n > 0) fetch(cur_st, 0, H[gix(0)]);
    for (long long j = 0; j < n; ++j) {
      const int sl = (int)(j & (K3_SLOTS - 1));
      if (j >= K3_SLOTS) {
        nbar_sync(K3_BAR_EMPTY + sl, 64);
        if (*(volatile int*)&S.stop_flag) break;
      }
      if (j + 1 < n) {
        const ChainHdr h1 = h_ahead;
        if (j + 2 < n) h_ahead = H[gix(j + 2)];
        fetch(nxt_st, j + 1, h1);
      }
      // store item j into its slot
      if (lane == 0) { S.shdr[sl] = cur_st.h; S.sbad[sl] = cur_st.bad; S.sw[sl] = cur_st.w; S.sxs[sl] = cur_st.xs; }
      store_row<NPER>(slotx + sl * ld, cur_st.x, ld, lane);
      if (cur_st.h.predj >= 0) store_row<NPER>(slotp + sl * ld, cur_st.p, ld, lane);
      uint4* dst = reinterpret_cast<uint4*>(&S.rb[sl][0]);
      const int nch = cur_st.h.len * (int)(sizeof(ChainLvl) / 16);
#pragma unroll
      for (int q = 0; q < RQ; ++q) { const int c = lane + 32 * q; if (c < nch) dst[c] = cur_st.r[q]; }
      __threadfence_block();
      __syncwarp();
      nbar_arrive(K3_BAR_FULL + sl, 64);
      cur_st = nxt_st;
    }
    return;
  }

#ifdef PCY_TIMELINE
  const long long tl_t0 = clock64();
  long long tl_wait = 0, tl_slow = 0, tl_start = 0, tl_clean = 0, tl_dem = 0, tl_fast = 0, tl_dir = 0, tl_new = 0, tl_cap = 0, tl_ndir = 0, tl_nnew = 0, tl_nlev = 0, tl_ncl = 0;
#endif
  EngCtl* C = E.ctl;
  const long long m = E.m;
  const double T = C->T;
  long long F = C->F, Falloc = C->F_alloc, freen = C->free_n, Galloc = C->G_alloc;
  long long Aalloc = C->A_alloc, nidx = C->next_index, totw = C->total_w, maxdepth = C->max_depth;
  long long c_lv = 0, c_dir = 0, c_dem = 0, c_slow = 0, c_it = 0, c_demf = 0, c_tch = 0;
  long long G0 = Galloc, opened = 0;
  if constexpr (PAR) { G0 = par->Galloc0; totw = 0; maxdepth = 0; freen = 0; }
  // a fresh child group (coreset.py:369-371); lane-uniform
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

  for (int s2 = lane; s2 < PCY_MOD_SLOTS; s2 += 32) S.mkey[s2] = -1;
  for (int s2 = lane; s2 < PCY_GMAP_SLOTS; s2 += 32) S.gkey[s2] = -1;
  for (int s2 = lane; s2 < mwords; s2 += 32) mbits[s2] = 0u;
  for (int s2 = lane; s2 < gwords; s2 += 32) gbits[s2] = 0u;
  if (lane == 0) { S.modcount = 0; S.stop_flag = 0; }
  int nnew = 0, mcount = 0;   // mcount: touched-node map entries (register copy, every lane)
  int free_top = freen > 0 ? E.free_ids[freen - 1] : -1;

  double pr[NPER];
  int prnode = -1;               // node whose current s row is held in pr[]
  // rewrites of the last K3_SLOTS items: the staging warp reads item i's
  // predicted row once item i-K3_SLOTS-1 is done (one item ahead of its slot
  // store), so any of items i-K3_SLOTS .. i-1 may have rewritten it since
  int rec_mod[K3_SLOTS];
#pragma unroll
  for (int q = 0; q < K3_SLOTS; ++q) rec_mod[q] = -1;
  int multi_left = 0;            // items left in the window since one rewrote several nodes
  // a stop (FULL / REBUILD / INVALID) releases the staging warp
  auto signal_stop = [&](int sl) {
    if (lane == 0) S.stop_flag = 1;
    __threadfence_block();
    __syncwarp();
    nbar_arrive(K3_BAR_EMPTY + sl, 64);
  };

  for (long long i = 0; i < n; ++i) {
    const int sl = (int)(i & (K3_SLOTS - 1));
    const int cur = sl;
#ifdef PCY_TIMELINE
    const long long tl_w0 = clock64();
    if (i == 0) tl_start = tl_w0 - tl_t0;
#endif
    nbar_sync(K3_BAR_FULL + sl, 64);
#ifdef PCY_TIMELINE
    tl_wait += clock64() - tl_w0;
#endif
    const ChainHdr hc = S.shdr[sl];
    const int bad_c = S.sbad[sl];
    const long long w_c = S.sw[sl];
    const double xs_c = S.sxs[sl];
    double* xsm = slotx + sl * ld;
    double xr[NPER];
#pragma unroll
    for (int k = 0; k < NPER; ++k) { const int e = lane + 32 * k; xr[k] = e < d ? xsm[e] : 0.0; }
    {
      // staged predicted row: usable unless the previous item rewrote that node
      const int np_ = hc.predj;
      bool recent = multi_left > 0;
#pragma unroll
      for (int q = 0; q < K3_SLOTS; ++q) recent |= rec_mod[q] == np_;
      if (np_ >= 0 && np_ != prnode && !recent) {
        const double* pd = slotp + sl * ld;
#pragma unroll
        for (int k = 0; k < NPER; ++k) { const int e = lane + 32 * k; pr[k] = e < d ? pd[e] : 0.0; }
        prnode = np_;
      }
    }
    if (bad_c) { status = ST_INVALID; err = bad_c; stop = i; signal_stop(sl); break; }
    if (nnew >= nnew_cap || mcount >= PCY_MOD_SLOTS / 2) { status = ST_FULL; stop = i; signal_stop(sl); break; }
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
    int lastmod = -1;      // last snapshot node this item rewrote (its row is in pr)
    bool multi = false;    // the item rewrote more than one snapshot node
    // current row of snapshot node bj into pr (HBM unless it is the held row)
    auto fetch_row = [&](int bj) {
      if (bj == prnode) return;
#ifdef PCY_TIMELINE
      const long long tl_d0 = clock64();
#endif
      load_row<NPER>(pr, E.s + (long long)bj * ld, d, lane);
#ifdef PCY_TIMELINE
      if (__shfl_sync(PCY_FULL, pr[0], 0) == 1.2345e-300) ++c_dem;   // wait for the row
      tl_dem += clock64() - tl_d0;
#endif
      ++c_dem;
      prnode = bj;
    };
    // _open (coreset.py:329-335, :374-377) into group g at level L; returns true when full (rebuild)
    auto do_open = [&](int g, int L) -> bool {
        const bool full = !PAR && F >= m;   // k_plan: F0 + window <= m
        const long long wopen = full ? 1LL : rem;
        long long slot, nid = nidx;
        if constexpr (PAR) {
          // the t-th open of the window pops the free stack, then bumps F_alloc;
          // creation index = window position (same order as one-at-a-time)
          unsigned long long t = 0;
          if (lane == 0) t = atomicAdd(&par->open_ticket, 1ULL);
          const long long tt = (long long)__shfl_sync(PCY_FULL, t, 0);
          // k_plan's budget bound guarantees F0 + tt < m; a violation (never
          // expected) would need a rebuild here: report it, write nothing
          if (par->F0 + tt >= E.m) return true;
          slot = tt < par->freen0 ? (long long)E.free_ids[par->freen0 - 1 - tt] : par->Falloc0 + (tt - par->freen0);
          nid = par->nidx0 + gix(i);
          ++opened;
        } else {
          if (freen > 0) { slot = free_top; --freen; free_top = freen > 0 ? E.free_ids[freen - 1] : -1; }
          else slot = Falloc++;
        }
        const int t = nnew++;
        const double fw = (double)wopen;
        double* rr = tref + (long long)t * lds;
        double* sr = ts + (long long)t * ld;
#pragma unroll
        for (int k = 0; k < NPER; ++k) {
          const int e = lane + 32 * k;
          if (e < ld) { rr[e] = xr[k]; sr[e] = rmul(fw, xr[k]); }
        }
        const bool had = ((gbits[g >> 5] >> (g & 31)) & 1u) != 0;
        int gs = -1;
        if (had) gs = gmap_find(S, g);
        else {
          gs = (int)(((unsigned)g * 2654435761u) >> 24) & (PCY_GMAP_SLOTS - 1);
          while (S.gkey[gs] >= 0) gs = (gs + 1) & (PCY_GMAP_SLOTS - 1);
        }
        if (lane == 0) {
          S.tid[t] = (int)slot; S.tgrp[t] = g; S.tchild[t] = -1; S.tnext[t] = -1; S.tw[t] = wopen;
          S.tq[t] = rmul(fw, xs); S.tsn[t] = rmul((double)(wopen * wopen), xs); S.trn[t] = xs;
          if (had) { S.tnext[S.gtail[gs]] = t; S.gtail[gs] = t; }
          else { S.gkey[gs] = g; S.ghead[gs] = t; S.gtail[gs] = t; gbits[g >> 5] |= 1u << (g & 31); }
          E.idx[slot] = nid; E.alive[slot] = 1; E.child[slot] = -1;
        }
        ++nidx; ++F;
        if (L + 1 > maxdepth) maxdepth = L + 1;
        rem -= wopen;
        __syncwarp();
        return full;
    };
    // ---- verified fast path: nothing on K1's path changed in this launch, so
    // every decision along it is K1's (same statistics, dots, members).
    bool done_fast = false;
    // levels above K1's action level where nothing changed in this launch and
    // K1 descended (no take) into an existing child group: the slow path below
    // steps over them, as K1 did
    unsigned cleanmask = 0u;
#ifdef PCY_TIMELINE
    const long long tl_f0 = clock64();
#endif
    if (!resume && len > 0 && !hc.trunc) {
      const int pl = hc.pred;
      bool ok = pl >= 0 && pl < len;
      if (ok) {
        // one level per lane: a group that gained a member or a touched node fails
        bool bad = false, cl = false;
        if (lane <= pl) {
          const ChainLvl& rl = S.rb[cur][lane];
          const int g2 = rl.g, j2 = rl.j;
          bad = (g2 >= 0 && ((gbits[g2 >> 5] >> (g2 & 31)) & 1u)) || (j2 >= 0 && ((mbits[j2 >> 5] >> (j2 & 31)) & 1u));
          cl = !bad && lane < pl && j2 >= 0 && rl.child >= 0 && rl.take == 0;
        }
        ok = !__any_sync(PCY_FULL, bad);
        cleanmask = __ballot_sync(PCY_FULL, cl);
      }
      if (ok) {
        const ChainLvl& rp = S.rb[cur][pl];
        if (rp.take > 0 && rp.take == rem) {
          const int bj = rp.j;
          const long long take = rp.take;
          const double ft = (double)take;
          if (bj != prnode) ++c_demf;
          fetch_row(bj);
#pragma unroll
          for (int k = 0; k < NPER; ++k) pr[k] = take == 1 ? radd(pr[k], xr[k]) : radd(pr[k], rmul(ft, xr[k]));
          store_row<NPER>(E.s + (long long)bj * ld, pr, d, lane);
          const long long nw2 = rp.w + take;
          map_put(S, mbits, bj, nw2, rp.nq, rp.nsn, rp.child, lane, &mcount);
          if (lane == 0) { E.w[bj] = nw2; E.q[bj] = rp.nq; E.sn[bj] = rp.nsn; }
          lastmod = bj;
          rem = 0;
          if (pl + 1 > maxdepth) maxdepth = pl + 1;
          c_lv += pl + 1;
          done_fast = true;
        } else if (rp.take == 0) {
          int g = rp.g;
          if (g < 0) {
            // the snapshot parent had no child group: create it (coreset.py:369-371)
            const ChainLvl& pp = S.rb[cur][pl - 1];
            g = new_group();
            if (lane == 0) { E.g_count[g] = 0; E.g_cap[g] = 0; E.g_base[g] = 0; E.child[pp.j] = g; }
            map_put(S, mbits, pp.j, pp.w, pp.q, pp.sn, g, lane, &mcount);
          }
          if (do_open(g, pl)) { status = ST_REBUILD; stop = i; remaining = rem; }
          c_lv += pl + 1;
          done_fast = true;
        }
      }
    }
#ifdef PCY_TIMELINE
    const long long tl_s0 = clock64();
    tl_fast += tl_s0 - tl_f0;
#endif
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
        else direct = true;   // truncated chain
      }
      ++c_lv;
#ifdef PCY_TIMELINE
      const long long tl_l0 = clock64();
      ++tl_nlev;
#endif
      if (direct && g < G0) {
#ifdef PCY_TIMELINE
        ++tl_ndir;
#endif
        // members present at launch start, scanned directly (truncated chains only)
        ++c_dir;
        const int cnt = E.g_count[g];
        if (cnt > 0) {
          double p; int ps;
          const int* mem = E.arena + E.g_base[g];
          scan_members(E, mem, 0, cnt, xsm, lane, p, ps);
          if (ps < cnt) { bj = mem[ps]; bp = p; }
        }
      }
      // members opened in this launch, in position order
      int bt = -1;
#ifdef PCY_TIMELINE
      const long long tl_l1 = clock64();
      tl_dir += tl_l1 - tl_l0;
      if ((gbits[g >> 5] >> (g & 31)) & 1u) ++tl_nnew;
#endif
      if ((gbits[g >> 5] >> (g & 31)) & 1u) {
        // one new member per lane: sequential dot over the padded smem row
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
      }
#ifdef PCY_TIMELINE
      const long long tl_l2 = clock64();
      tl_new += tl_l2 - tl_l1;
#endif
      // admission radius (coreset.py:329)
      if (bj < 0 || radd(bp, xs) > radius) {
        if (do_open(g, L)) { status = ST_REBUILD; stop = i; remaining = rem; }
        break;
      }
      // capacity on the winner (coreset.py:336-356)
      long long nn, take, nw2 = 0;
      double qv, snv, nq = 0.0, nsn = 0.0;
      int ms = -1;
      const bool touched = bt < 0 && ((mbits[bj >> 5] >> (bj & 31)) & 1u);
      if (bt < 0 && li >= 0 && !touched && rem == wi && !resume) {
        // untouched snapshot node on the first descent: K1's decision is exact
#ifdef PCY_TIMELINE
        if (!((gbits[g >> 5] >> (g & 31)) & 1u)) ++tl_ncl;
#endif
        const ChainLvl& rc = S.rb[cur][li];
        nn = rc.w; qv = rc.q; snv = rc.sn; take = rc.take;
        if (take > 0) { nw2 = nn + take; nq = rc.nq; nsn = rc.nsn; }
      } else {
        double dt;
        ++c_slow;
        if (bt >= 0) {
          nn = S.tw[bt]; qv = S.tq[bt]; snv = S.tsn[bt];
          dt = smem_dot<NPER>(ts + (long long)bt * ld, xr, d, lane);
        } else {
          if (touched) { ms = map_find(S, bj); nn = S.mw[ms]; qv = S.mq[ms]; snv = S.msn[ms]; }
          else if (li >= 0) { const ChainLvl& rc = S.rb[cur][li]; nn = rc.w; qv = rc.q; snv = rc.sn; }
          else { nn = E.w[bj]; qv = E.q[bj]; snv = E.sn[bj]; }
          if (!touched && li >= 0) dt = S.rb[cur][li].dot;
          else {
            fetch_row(bj);
            dt = reg_dot<NPER>(pr, xr);
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
#ifdef PCY_TIMELINE
      tl_cap += clock64() - tl_l2;
#endif
      if (take > 0) {
        const double ft = (double)take;
        if (bt >= 0) {
          double* srow = ts + (long long)bt * ld;
#pragma unroll
          for (int k = 0; k < NPER; ++k) {
            const int e = lane + 32 * k;
            if (e < d) srow[e] = take == 1 ? radd(srow[e], xr[k]) : radd(srow[e], rmul(ft, xr[k]));
          }
          if (lane == 0) { S.tw[bt] = nw2; S.tq[bt] = nq; S.tsn[bt] = nsn; }
          __syncwarp();
        } else {
          if (touched && ms < 0) ms = map_find(S, bj);
          fetch_row(bj);
#pragma unroll
          for (int k = 0; k < NPER; ++k) pr[k] = take == 1 ? radd(pr[k], xr[k]) : radd(pr[k], rmul(ft, xr[k]));
          store_row<NPER>(E.s + (long long)bj * ld, pr, d, lane);
          int child_now;
          if (touched) child_now = S.mchild[ms];
          else child_now = li >= 0 ? S.rb[cur][li].child : E.child[bj];
          ms = map_put(S, mbits, bj, nw2, nq, nsn, child_now, lane, &mcount);
          if (lane == 0) { E.w[bj] = nw2; E.q[bj] = nq; E.sn[bj] = nsn; }
          if (lastmod >= 0 && lastmod != bj) multi = true;
          lastmod = bj;
        }
        rem -= take;
        if (rem == 0) { if (L + 1 > maxdepth) maxdepth = L + 1; break; }
      }
      // descend (coreset.py:369-372)
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
        if (tnow && ms < 0) ms = map_find(S, bj);
        c = tnow ? S.mchild[ms] : (li >= 0 ? S.rb[cur][li].child : E.child[bj]);
        if (c < 0) {
          c = new_group();
          if (lane == 0) { E.g_count[c] = 0; E.g_cap[c] = 0; E.g_base[c] = 0; E.child[bj] = c; }
          if (tnow) { if (lane == 0) S.mchild[ms] = c; __syncwarp(); }
          else { ms = map_put(S, mbits, bj, nn, qv, snv, c, lane, &mcount); ++c_tch; }   // untouched: current stats
        }
      }
      g = c;
      radius = rmul(radius, 0.25);
      ++L;
    }
    __syncwarp();
#ifdef PCY_TIMELINE
    if (!done_fast) tl_slow += clock64() - tl_s0;
#endif
    ++c_it;
#pragma unroll
    for (int q = K3_SLOTS - 1; q > 0; --q) rec_mod[q] = rec_mod[q - 1];
    rec_mod[0] = lastmod;
    multi_left = multi ? K3_SLOTS : (multi_left > 0 ? multi_left - 1 : 0);
    if (status != ST_DONE) { signal_stop(sl); break; }
    __threadfence_block();
    nbar_arrive(K3_BAR_EMPTY + sl, 64);
  }

  // ---- cleanup: new nodes and their memberships to HBM (position order per group)
  __syncwarp();
#ifdef PCY_TIMELINE
  tl_clean = clock64();
#endif
  for (int t = 0; t < nnew; ++t) {
    const int node = S.tid[t];
    const double* rr = tref + (long long)t * lds;
    const double* sr = ts + (long long)t * ld;
    for (int e = lane; e < ld; e += 32) { E.r[(long long)node * ld + e] = rr[e]; E.s[(long long)node * ld + e] = sr[e]; }
  }
  for (int t = lane; t < nnew; t += 32) {
    const int node = S.tid[t];
    E.w[node] = S.tw[t]; E.q[node] = S.tq[t]; E.sn[node] = S.tsn[t]; E.rn[node] = S.trn[t];
    E.child[node] = S.tchild[t];
    const int g = S.tgrp[t];
    int k = 0, f = t;
    for (int u = t - 1; u >= 0; --u) if (S.tgrp[u] == g) { ++k; f = u; }
    S.tk[t] = k; S.tfirst[t] = f;
    S.tcnt[t] = E.g_count[g]; S.tcap[t] = E.g_cap[g]; S.tbase[t] = E.g_base[g];
  }
  __syncwarp();
  bool arena_ok = true;
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
      if constexpr (PAR) {
        unsigned long long at = 0;
        if (lane == 0) at = atomicAdd(&par->a_ticket, (unsigned long long)ncap);
        const long long a0 = par->Aalloc0 + (long long)__shfl_sync(PCY_FULL, at, 0);
        if (a0 + ncap > E.AC) { arena_ok = false; break; }
        nb = (int)a0;
      } else {
        if (Aalloc + ncap > E.AC) { arena_ok = false; break; }
        nb = (int)Aalloc; Aalloc += ncap;
      }
      for (int p = lane; p < cnt; p += 32) E.arena[nb + p] = E.arena[base + p];
    }
    if (lane == 0) {
      S.tbase[t] = nb; S.tcap[t] = ncap;
      E.g_base[g] = nb; E.g_cap[g] = ncap; E.g_count[g] = cnt + total;
      if (cnt + total >= PCY_PANEL_MIN) atomicMax(&C->maxg, (long long)(cnt + total));
    }
    __syncwarp();
  }
  if (arena_ok) {
    for (int t = lane; t < nnew; t += 32) {
      const int f = S.tfirst[t];
      E.arena[S.tbase[f] + S.tcnt[f] + S.tk[t]] = S.tid[t];
    }
  } else {
    status = ST_ARENA;
  }
  __syncwarp();
  if constexpr (PAR) {
    // deltas of this subtree, then the last CTA publishes the window
    int lastf = 0;   // this CTA finished the window: its warp publishes
#ifdef PCY_TIMELINE
    if (lane == 0) { tl_cta(n, nnew, c_slow, clock64() - tl_t0); tl_split(n, tl_wait, tl_slow, tl_start, clock64() - tl_clean, tl_dem, tl_fast); tl_split2(n, tl_dir, tl_new, tl_cap, tl_ndir, tl_nnew, tl_nlev, tl_ncl); }
#endif
    if (lane == 0) {
      using ull = unsigned long long;
      if (status != ST_DONE) { atomicExch(&par->arena_fail, status == ST_ARENA ? ST_ARENA : ST_PAR_BROKEN); par->pad = status; }
      atomicAdd((ull*)&C->F, (ull)opened);
      atomicAdd((ull*)&C->total_w, (ull)totw);
      atomicMax(&C->max_depth, maxdepth);
      atomicAdd((ull*)&C->cnt_levels, (ull)c_lv); atomicAdd((ull*)&C->cnt_direct, (ull)c_dir);
      atomicAdd((ull*)&C->cnt_demand, (ull)c_dem); atomicAdd((ull*)&C->cnt_slow, (ull)c_slow);
      atomicAdd((ull*)&C->cnt_items, (ull)c_it); atomicAdd((ull*)&C->cnt_dem_fast, (ull)c_demf);
      atomicAdd((ull*)&C->cnt_touch_child, (ull)c_tch);
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
        if (pub) *(volatile long long*)&C->win_done = pseq;   // the run-ahead chain walk may start
        PCY_TL(5);
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
    C->cnt_items += c_it; C->cnt_dem_fast += c_demf; C->cnt_touch_child += c_tch;
    __threadfence();
    if (pub) { *(volatile long long*)&C->win_done = pseq; PCY_TL(5); }
  }
  __syncwarp();
  if (pub) ctl_publish_warp(E, pub, pseq, lane);
}

template <int NPER, bool PAR = false>
__global__ void __launch_bounds__(64, 1) k_resolve2(EngDev E, const double* __restrict__ X,
                                                    const double* __restrict__ XS, const long long* __restrict__ W,
                                                    const int* __restrict__ BAD, long long n, long long first_rem,
                                                    int countw, int nnew_cap, const ChainHdr* __restrict__ H,
                                                    const ChainLvl* __restrict__ R, ParCtl* __restrict__ par = nullptr) {
  resolve2_body<NPER, PAR>(E, X, XS, W, BAD, n, first_rem, countw, nnew_cap, H, R, par, nullptr, 0);
}

// One launch for either choice of k_plan: the subtree-parallel window (every
// CTA with a list) or the sequential stretch (CTA 0).
template <int NPER>
__global__ void __launch_bounds__(64, 1) k_resolve2x(EngDev E, const double* __restrict__ X,
                                                     const double* __restrict__ XS, const long long* __restrict__ W,
                                                     const int* __restrict__ BAD, long long n, long long first_rem,
                                                     int countw, int nnew_cap, const ChainHdr* __restrict__ H,
                                                     const ChainLvl* __restrict__ R, ParCtl* __restrict__ par,
                                                     EngCtl* pub, long long pseq, long long planseq) {
  flag_wait(&par->ready, planseq);   // k_plan has written its window
  pdl_launch_dependents();   // the next batch's chain walk may be scheduled; it waits for this grid
  if (blockIdx.x == 0 && threadIdx.x == 0) PCY_TL(4);
  if (par->mode == 0) resolve2_body<NPER, true>(E, X, XS, W, BAD, n, first_rem, countw, nnew_cap, H, R, par, pub, pseq);
  else if (blockIdx.x == 0) resolve2_body<NPER, false>(E, X, XS, W, BAD, n, first_rem, countw, nnew_cap, H, R, par, pub, pseq);
}

// ------------------------------------------------------------- K3 planner
// k_plan (one CTA, thread per item of the K1 batch) chooses how the batch's
// next stretch is resolved and writes the ParCtl the two resolve launches read.
//
// Window: the longest prefix with no invalid row, at most m - F0 items (every
// item opens at most one feature without a rebuild, so F < m before each of
// them, coreset.py:330-332) and no conflicting root open (below).
//
// Domains.  From K1's record every item has a predicted action: absorb at node
// a (coreset.py:336-368, take > 0) or open into the child group of a parent P
// (coreset.py:329-335; P = ROOT for group 0).  Items are grouped into domains
// that own disjoint state:
//   SUB(v)  node v, its statistics and everything below it;
//   OPEN(P) the membership of P's child group (its opens, in stream order).
// v is a domain root when some window item absorbs at v, or when an earlier
// window open into the group containing v would be preferred by an item whose
// K1 winner there is v (the opener's row against the item, from the batch
// Gram, below the recorded part plus a rounding margin): then the opener and
// that item may interact, and OPEN(P) is united with SUB(v).  An item joins
// the first domain on its path (an opener that meets none joins OPEN(P)), and
// every further domain below it on its path, or its open group, is united
// with that one (nested state).  Above its domain an item sees no absorbs and
// no preferred new members, so by induction over stream order it follows K1
// there; the united domains partition the window's writes, so one CTA per
// domain set resolves the window exactly.  A conflicting root open ends the
// window.  With a weighted item in the window the domains stay at the roots
// and every root open ends the window (K1 does not follow partial takes).
//
// Domain sets get CTAs in order of first appearance (mod PCY_PAR_MAXCTA); each
// CTA list keeps stream order and holds at most cap items (its tables cannot
// fill).  A window shorter than theta goes to the sequential kernel.
// With `order` (rebuild reattach, coreset.py:395-421) the items are the
// collected nodes in rebuild order: a merge is the absorb, a group add the open.
constexpr int PLAN_HASH = 4096;
constexpr int PLAN_ROOT = -2;
// dynamic shared memory of k_plan: the hash / union-find tables, per-item xs
// and opener links, and the active-node bitmap (nwords words)
__host__ __device__ inline size_t plan_smem_bytes(int nwords) {
  return sizeof(int) * 6 * PLAN_HASH + sizeof(double) * PCY_PAR_MAXITEMS + sizeof(int) * PCY_PAR_MAXITEMS +
         sizeof(unsigned) * (size_t)nwords;
}
__device__ __forceinline__ int ph_slot(int key) { return (int)(((unsigned)key * 2654435761u) >> 20) & (PLAN_HASH - 1); }
__device__ __forceinline__ int ph_insert(int* hkey, int key) {
  int s = ph_slot(key);
  for (;;) {
    const int prev = atomicCAS(&hkey[s], -1, key);
    if (prev == -1 || prev == key) return s;
    s = (s + 1) & (PLAN_HASH - 1);
  }
}
__device__ __forceinline__ int ph_find(const int* hkey, int key) {
  int s = ph_slot(key);
  for (;;) {
    const int k = *(volatile const int*)&hkey[s];
    if (k == key) return s;
    if (k == -1) return -1;
    s = (s + 1) & (PLAN_HASH - 1);
  }
}
__device__ __forceinline__ int uf_find(int* uf, int a) {
  for (;;) {
    const int p = *(volatile int*)&uf[a];
    if (p == a) return a;
    a = p;
  }
}
__device__ __forceinline__ void uf_union(int* uf, int a, int b) {
  for (;;) {
    a = uf_find(uf, a); b = uf_find(uf, b);
    if (a == b) return;
    if (a > b) { const int t = a; a = b; b = t; }
    if (atomicCAS(&uf[b], b, a) == b) return;   // link the larger root under the smaller
  }
}

__global__ void __launch_bounds__(PCY_PAR_MAXITEMS) k_plan(EngDev E, const double* __restrict__ XS,
                                                           const long long* __restrict__ W,
                                                           const int* __restrict__ BAD, long long n,
                                                           long long first_rem, int cap_items, int theta,
                                                           const ChainHdr* __restrict__ H,
                                                           const ChainLvl* __restrict__ R, ParCtl* __restrict__ par,
                                                           int nwords,
                                                           const int* __restrict__ order, const double* __restrict__ gram,
                                                           long long gld, EngCtl* pub, long long planseq) {
  extern __shared__ int plan_sm[];
  int* hkey = plan_sm;                    // domain keys: SUB(v) = v, OPEN(P) = NC + P, OPEN(ROOT) = 2 NC
  int* uf = plan_sm + PLAN_HASH;          // union-find over hash slots
  int* ohead = plan_sm + 2 * PLAN_HASH;   // OPEN(P): list of its openers; later: set tickets
  int* hfirst = plan_sm + 3 * PLAN_HASH;  // first item of each domain set
  double* xs_s = reinterpret_cast<double*>(plan_sm + 4 * PLAN_HASH);   // per item: |x|^2 (rn of the node)
  int* onext = reinterpret_cast<int*>(xs_s + PCY_PAR_MAXITEMS);        // opener list links, by item
  unsigned* act_bits = reinterpret_cast<unsigned*>(onext + PCY_PAR_MAXITEMS);   // active nodes
  int* tkey = reinterpret_cast<int*>(act_bits + nwords);   // budget bound: node / group keys ...
  int* tmin = tkey + PLAN_HASH;                            // ... and the first item that may touch them
  __shared__ unsigned char s_unc[PCY_PAR_MAXITEMS];       // item may open (or is invalid)
  __shared__ int ccnt[PCY_PAR_MAXITEMS / 32][PCY_PAR_MAXCTA];
  __shared__ int ctot[PCY_PAR_MAXCTA];
  __shared__ int wsum[32];
  __shared__ int s_c, s_last, s_heavy, s_cut, s_P;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#ifdef PCY_TIMELINE
  long long plan_t[10];
  plan_t[0] = clock64();
#define PLAN_T(k) plan_t[k] = clock64()
#else
#define PLAN_T(k) ((void)0)
#endif
  pdl_launch_dependents();   // the resolve kernel's CTAs may be scheduled; they wait for this grid
  if (tid == 0 && !order) PCY_TL(2);
  const EngCtl* C = E.ctl;
  const long long F0 = C->F;
  const int NC = (int)E.NC;
  const int nn = (int)(n < PCY_PAR_MAXITEMS ? n : PCY_PAR_MAXITEMS);
  long long room = E.m - F0;
  if (room < 0) room = 0;
  if (order) room = n;   // rebuild reattach: merges and adds never exceed the budget
  for (int h = tid; h < PLAN_HASH; h += blockDim.x) {
    hkey[h] = -1; uf[h] = h; ohead[h] = -1; hfirst[h] = 0x7fffffff; tkey[h] = -1;
  }
  if (tid < PCY_PAR_MAXITEMS) s_unc[tid] = 0;
  for (int q = tid; q < (PCY_PAR_MAXITEMS / 32) * PCY_PAR_MAXCTA; q += blockDim.x) (&ccnt[0][0])[q] = 0;
  for (int q = tid; q < nwords; q += blockDim.x) act_bits[q] = 0u;
  if (tid == 0) {
    // the budget cut (no item may find F == m) is placed after the predictions:
    // weighted windows take `room` items, unit windows as many as keep the
    // number of items that may open within `room` (see below)
    s_c = nn;
    if (first_rem >= 0) s_c = 0;
    s_last = -1; s_heavy = 0; s_cut = 0x7fffffff; s_P = 0;
  }
  __syncthreads();
  PLAN_T(1);
  // pass 1: invalid rows, weighted items, predicted actions
  ChainHdr h = ChainHdr{0, 0, -1, 0};
  const ChainLvl* rec = R + (long long)tid * PCY_FMAXL;
  double xs = 0.0;
  int pl = -1, alev = -1, absorb = -1, target = -1;   // absorb at `absorb` (level alev), or open under `target`
  bool opener = false;
  int pj[PCY_FMAXL];   // K1 winner per level (E.pathj: 64 contiguous bytes per item)
#pragma unroll
  for (int l = 0; l < PCY_FMAXL; ++l) pj[l] = -1;
  if (tid < nn) {
    h = H[tid];
    const int4* src = reinterpret_cast<const int4*>(E.pathj + (long long)tid * PCY_FMAXL);
#pragma unroll
    for (int q = 0; q < PCY_FMAXL / 4; ++q) {
      const int4 v = src[q];
      pj[4 * q] = v.x; pj[4 * q + 1] = v.y; pj[4 * q + 2] = v.z; pj[4 * q + 3] = v.w;
    }
    const bool invalid = (BAD && BAD[tid]) || h.len == 0;
    if (!invalid) {
      xs = order ? E.rn[order[tid]] : XS[tid];
      xs_s[tid] = xs;
      pl = h.pred < h.len ? h.pred : h.len - 1;
      if (h.trunc) alev = h.len - 1;   // acts somewhere below the record
      else if (rec[pl].take > 0) alev = pl;
      else opener = true;
#pragma unroll
      for (int l = 0; l < PCY_FMAXL; ++l) {
        if (l == alev) absorb = pj[l];
        if (opener && l + 1 == pl) target = pj[l];
      }
      if (opener && pl == 0) target = PLAN_ROOT;
    } else {
      atomicMin(&s_c, tid);
      if (tid < 64) atomicMax(&s_last, tid);
      s_unc[tid] = 1;
    }
    if (opener) s_unc[tid] = 1;
    if (W && W[tid] > 1) s_heavy = 1;
  }
  __syncthreads();
  PLAN_T(2);
  const bool heavy = s_heavy != 0;
  if (tid == 0 && (heavy || order) && room < nn) atomicMin(&s_c, (int)room);
  auto open_key = [&](int P) { return NC + (P == PLAN_ROOT ? NC : P); };
  if (heavy) {
    if (tid < nn && opener && target == PLAN_ROOT) {   // root opens end the window
      atomicMin(&s_c, tid);
      if (tid < 64) atomicMax(&s_last, tid);
    }
  } else {
    // opener lists per open group
    if (tid < s_c && opener) {
      const int so = ph_insert(hkey, open_key(target));
      onext[tid] = atomicExch(&ohead[so], tid);
    }
    __syncthreads();
    // conflicts: an earlier opener y of a group x visits (at a level <= its
    // action) whose row x would prefer to its K1 winner there
    if (tid < s_c) {
      const int lmax = opener ? pl : alev;
#pragma unroll
      for (int l = 0; l < PCY_FMAXL; ++l) {
        if (l > lmax) break;
        const int P = l == 0 ? PLAN_ROOT : pj[l - 1];
        if (opener && P == target) break;   // x opens there itself: same domain
        const int so = ph_find(hkey, open_key(P));
        if (so < 0) continue;
        const double prec = rec[l].part;
        for (int y = ohead[so]; y >= 0; y = onext[y]) {
          if (y >= tid) continue;
          const double xsy = xs_s[y];
          const double pnew = radd(xsy, rmul(gram[(long long)tid * gld + y], -2.0));
          if (pnew < prec + 1e-10 * (xs + xsy) + 1e-300) {
            s_unc[tid] = 1;   // its decisions may change: it may open
            if (P == PLAN_ROOT) {
              // x would prefer the earlier root opener y: the window ends
              // before x (y's open stays in the window, in the OPEN(ROOT)
              // domain; items before x do not prefer any new root, so their
              // root winners -- and domains -- stand)
              atomicMin(&s_c, tid);
              if (tid < 64) atomicMax(&s_last, tid);
            } else {
              const int v = pj[l];
              atomicOr(&act_bits[v >> 5], 1u << (v & 31));
              uf_union(uf, so, ph_insert(hkey, v));
            }
          }
        }
      }
    }
  }
  __syncthreads();
  PLAN_T(3);
  // Budget bound of unit windows (coreset.py:330-335: an open at F == m opens
  // one copy and rebuilds, which a parallel window cannot do).  Only items that
  // may open count against room = m - F0: predicted openers, conflicting
  // items, and absorbers whose K1 decision may not hold -- their absorb node
  // may be touched by an earlier item of the window, or an earlier item that
  // may open (not predicted) could add a member to a group on their path.
  // "May touch" is every path node of an uncertain item (it may absorb at any
  // level of its chain) and only the absorb node of a certain one; the sets
  // are iterated to a fixpoint (uncertainty only grows).  A certain absorber
  // follows its K1 chain and absorbs, so the window is safe when the count of
  // uncertain items before its end is <= room.
  if (!heavy && !order && room < nn && s_c > 0) {
    const int cmax = s_c;
    const bool live = tid < cmax;
    int gk[PCY_FMAXL];   // group key per level: OPEN(parent)
#pragma unroll
    for (int l = 0; l < PCY_FMAXL; ++l) gk[l] = open_key(l == 0 ? PLAN_ROOT : pj[l > 0 ? l - 1 : 0]);
    // The may-touch minima only decrease as items turn uncertain, so the table
    // is filled incrementally: certain absorbers enter their absorb node once,
    // an item enters its whole path when it turns uncertain (same tables and
    // decisions as recomputing them every round).
    for (int hh = tid; hh < PLAN_HASH; hh += blockDim.x) tmin[hh] = 0x7fffffff;
    __syncthreads();
    bool unc = live && s_unc[tid];
    bool pending = unc;   // uncertain, path not entered yet
    if (live && !unc && absorb >= 0) atomicMin(&tmin[ph_insert(tkey, absorb)], tid);
    for (int it = 0; it < 16; ++it) {
      if (pending) {
#pragma unroll
        for (int l = 0; l < PCY_FMAXL; ++l)
          if (l < h.len && pj[l] >= 0) atomicMin(&tmin[ph_insert(tkey, pj[l])], tid);
        if (!opener && h.len > 0) atomicMin(&tmin[ph_insert(tkey, gk[h.len - 1 < PCY_FMAXL ? h.len - 1 : 0])], tid);
        pending = false;
      }
      __syncthreads();
      int changed = 0;
      if (live && !unc) {
        bool u = false;
        if (absorb >= 0) { const int so = ph_find(tkey, absorb); u = so >= 0 && tmin[so] < tid; }
#pragma unroll
        for (int l = 0; l < PCY_FMAXL; ++l) {
          if (l > alev) break;
          const int so = ph_find(tkey, gk[l]);
          if (so >= 0 && tmin[so] < tid) u = true;
        }
        if (u) { s_unc[tid] = 1; unc = true; pending = true; changed = 1; }
      }
      if (!__syncthreads_or(changed)) break;
    }
    // window end: the first item whose inclusive count of uncertain items exceeds room
    const int u = live && s_unc[tid] ? 1 : 0;
    int inc = u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(PCY_FULL, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      const int v = wsum[lane];
      int wi = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(PCY_FULL, wi, o);
        if (lane >= o) wi += t;
      }
      wsum[lane] = wi - v;
    }
    __syncthreads();
    const int cum = wsum[wid] + inc;
    if (u && cum > room && cum - 1 <= room) {   // the (room+1)-th possible opener
      atomicMin(&s_c, tid);
      if (tid < 64) atomicMax(&s_last, tid);
    }
    __syncthreads();
  }
  const int c0 = s_c;
  PLAN_T(4);
  if (c0 < theta) {
    if (tid == 0) {
      par->mode = 1; par->P = 0; par->n_total = n;
      long long ns = n;
      // through the stoppers among the next 64 items (invalid rows, root opens)
      if (first_rem < 0 && room >= theta && c0 < nn) ns = (s_last > c0 ? s_last : c0) + 1;
      if (ns > n) ns = n;
      par->n_win = ns;
      if (!order) PCY_TL(3);
      __threadfence();
      *(volatile long long*)&par->ready = planseq;   // the resolve CTAs may go (flag_wait)
      if (pub) {   // early publication: the host may enqueue the next K1 batch now
        volatile long long* t = &pub->plan_mode;
        t[0] = 1; t[1] = ns;
        __threadfence_system();
        t[2] = planseq;
      }
    }
    return;
  }
  const bool act = tid < c0;
  if (act && absorb >= 0) atomicOr(&act_bits[absorb >> 5], 1u << (absorb & 31));
  __syncthreads();
  // the item's first domain, united with every further domain on its path
  int k1 = -1;
  if (act) {
    if (heavy) k1 = ph_insert(hkey, pj[0] >= 0 ? pj[0] : 2 * NC + 1);
    else {
      const int lmax = opener ? pl : alev;
#pragma unroll
      for (int l = 0; l < PCY_FMAXL; ++l) {
        if (l > lmax) break;
        int ks = -1;
        if (opener && l == pl) ks = ph_insert(hkey, open_key(target));
        else {
          const int j = pj[l];
          if (j >= 0 && ((act_bits[j >> 5] >> (j & 31)) & 1u)) ks = ph_insert(hkey, j);
        }
        if (ks >= 0) {
          if (k1 < 0) k1 = ks;
          else uf_union(uf, k1, ks);
        }
      }
    }
  }
  __syncthreads();
  PLAN_T(5);
  const int root = act ? uf_find(uf, k1) : -1;
  if (act) atomicMin(&hfirst[root], tid);
  __syncthreads();
  const int isfirst = act && hfirst[root] == tid;
#ifdef PCY_TRACE
  {   // build-time diagnostics: set sizes
    __shared__ int s_dbg[2];
    if (tid < 2) s_dbg[tid] = 0;
    for (int hh = tid; hh < PLAN_HASH; hh += blockDim.x) tmin[hh] = 0;
    __syncthreads();
    if (act) atomicAdd(&tmin[root], 1);
    __syncthreads();
    if (isfirst) { atomicAdd(&s_dbg[0], 1); atomicMax(&s_dbg[1], tmin[root]); }
    __syncthreads();
    if (tid == 0) { par->dbg_sets = s_dbg[0]; par->dbg_maxset = s_dbg[1]; }
  }
#endif
  // exclusive scan of isfirst in item order: set tickets
  const unsigned bal = __ballot_sync(PCY_FULL, isfirst);
  if (lane == 0) wsum[wid] = __popc(bal);
  __syncthreads();
  if (wid == 0) {   // exclusive scan of the 32 warp counts
    const int v = wsum[lane];
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(PCY_FULL, inc, o);
      if (lane >= o) inc += t;
    }
    wsum[lane] = inc - v;
  }
  __syncthreads();
  if (isfirst) ohead[root] = wsum[wid] + __popc(bal & ((1u << lane) - 1u));
  __syncthreads();
  PLAN_T(6);
  // Balanced CTA lists.  A window of 1024 items has ~800 domain sets, most of
  // one or two items and a few of tens; the resolve launch lasts as long as
  // its longest list.  Sets of >= PLAN_BIG items are dealt out largest first
  // in snake order; the small sets then fill the CTAs, in stream order, up to
  // a common level (water-filling over the big sets' loads).  Deterministic.
  constexpr int PLAN_BIG = 4, PLAN_NBIG = PCY_PAR_MAXITEMS / PLAN_BIG;
  __shared__ int s_load[PCY_PAR_MAXCTA], s_cap[PCY_PAR_MAXCTA + 1];
  __shared__ int s_bsz[PLAN_NBIG], s_broot[PLAN_NBIG];
  __shared__ int s_nbig;
  int* scnt = tmin;   // items per set (by hash slot); the budget bound is done with these tables
  int* scta = tkey;   // CTA of each set
  for (int hh = tid; hh < PLAN_HASH; hh += blockDim.x) scnt[hh] = 0;
  if (tid < PCY_PAR_MAXCTA) s_load[tid] = 0;
  __syncthreads();
  if (act) atomicAdd(&scnt[root], 1);
  __syncthreads();
  const int ssz = isfirst ? scnt[root] : 0;
  const bool bigf = isfirst && ssz >= PLAN_BIG;
  {
    // big sets compacted in stream order; small sets' item prefix in stream order
    const unsigned bb = __ballot_sync(PCY_FULL, bigf);
    int sv = (isfirst && !bigf) ? ssz : 0, sinc = sv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(PCY_FULL, sinc, o);
      if (lane >= o) sinc += t;
    }
    __shared__ int wbig[32], wsml[32];
    if (lane == 31) wsml[wid] = sinc;
    if (lane == 0) wbig[wid] = __popc(bb);
    __syncthreads();
    if (wid == 0) {
      const int vb = wbig[lane], vs = wsml[lane];
      int ib = vb, is = vs;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int tb = __shfl_up_sync(PCY_FULL, ib, o), ts2 = __shfl_up_sync(PCY_FULL, is, o);
        if (lane >= o) { ib += tb; is += ts2; }
      }
      wbig[lane] = ib - vb; wsml[lane] = is - vs;
      if (lane == 31) s_nbig = ib;
    }
    __syncthreads();
    if (bigf) { const int kk = wbig[wid] + __popc(bb & ((1u << lane) - 1u)); s_bsz[kk] = ssz; s_broot[kk] = root; }
    sinc = wsml[wid] + sinc - sv;   // exclusive prefix of small-set items before this item
    __syncthreads();
    const int nbig = s_nbig;
    if (tid < nbig) {
      const int mysz = s_bsz[tid];
      int rk = 0;
      for (int kk = 0; kk < nbig; ++kk) { const int o = s_bsz[kk]; rk += (o > mysz) || (o == mysz && kk < tid); }
      const int pos = rk % (2 * PCY_PAR_MAXCTA);
      const int cc = pos < PCY_PAR_MAXCTA ? pos : 2 * PCY_PAR_MAXCTA - 1 - pos;
      scta[s_broot[tid]] = cc;
      atomicAdd(&s_load[cc], mysz);
    }
    __syncthreads();
    if (wid == 0) {
      int bigsum = 0;
      for (int q = lane; q < PCY_PAR_MAXCTA; q += 32) bigsum += s_load[q];
      bigsum = __reduce_add_sync(PCY_FULL, bigsum);
      const int small = c0 - bigsum;
      int lo = 0, hi = PCY_PAR_MAXITEMS + 1;   // least level whose free room holds the small sets
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        int f = 0;
        for (int q = lane; q < PCY_PAR_MAXCTA; q += 32) f += max(0, mid - s_load[q]);
        f = __reduce_add_sync(PCY_FULL, f);
        if (f >= small) hi = mid; else lo = mid + 1;
      }
      int carry = 0;
      for (int base = 0; base < PCY_PAR_MAXCTA; base += 32) {
        const int q = base + lane;
        const int v = q < PCY_PAR_MAXCTA ? max(0, lo - s_load[q]) : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(PCY_FULL, inc, o);
          if (lane >= o) inc += t;
        }
        if (q < PCY_PAR_MAXCTA) s_cap[q] = carry + inc - v;
        carry += __shfl_sync(PCY_FULL, inc, 31);
      }
      if (lane == 0) s_cap[PCY_PAR_MAXCTA] = carry;
    }
    __syncthreads();
    if (isfirst && !bigf) {
      int lo = 0, hi = PCY_PAR_MAXCTA - 1;   // last CTA whose room starts at or before this set
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_cap[mid] <= sinc) lo = mid; else hi = mid - 1;
      }
      scta[root] = lo;
    }
    __syncthreads();
  PLAN_T(7);
  }
  const int cta = act ? scta[root] : -1 - lane;
  // rank of each item within its CTA (stream order): per-warp chunk counts
  const unsigned grp = __match_any_sync(PCY_FULL, cta);
  const int rin = __popc(grp & ((1u << lane) - 1u));
  if (act && rin == 0) ccnt[wid][cta] = __popc(grp);
  __syncthreads();
  for (int q = tid; q < PCY_PAR_MAXCTA; q += blockDim.x) {
    int run = 0;
    for (int w2 = 0; w2 < PCY_PAR_MAXITEMS / 32; ++w2) { const int v = ccnt[w2][q]; ccnt[w2][q] = run; run += v; }
    ctot[q] = 0;
  }
  __syncthreads();
  // items per CTA: the new-node table (one open per item) and, for weighted
  // items (partial takes at up to PCY_FMAXL levels), the touched-node map
  const int cap = heavy ? min((PCY_MOD_SLOTS / 2) / (PCY_FMAXL + 2), cap_items) : cap_items;
  const int rank = act ? ccnt[wid][cta] + rin : 0;
  if (act && rank >= cap) atomicMin(&s_cut, tid);
  __syncthreads();
  const int c = c0 < s_cut ? c0 : s_cut;
  if (tid < c) atomicMax(&ctot[cta], rank + 1);
  __syncthreads();
  PLAN_T(8);
  // list offsets: exclusive scan of the CTA counts (warps 0..4), P = last CTA with items + 1
  constexpr int SCAN_T = (PCY_PAR_MAXCTA + 1 + 31) / 32 * 32;
  int cv = 0, cinc = 0;
  if (tid < SCAN_T) {
    cv = tid < PCY_PAR_MAXCTA ? ctot[tid] : 0;
    cinc = cv;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(PCY_FULL, cinc, o);
      if (lane >= o) cinc += t;
    }
    if (lane == 31) wsum[wid] = cinc;
    if (cv > 0) atomicMax(&s_P, tid + 1);
#ifdef PCY_TRACE
    if (tid == 0) par->dbg_maxcta = 0;
#endif
  }
#ifdef PCY_TRACE
  __syncthreads();
  if (tid < PCY_PAR_MAXCTA) atomicMax(&par->dbg_maxcta, cv);
#endif
  __syncthreads();
  if (tid < SCAN_T) {
    int base = 0;
    for (int q = 0; q < wid; ++q) base += wsum[q];
    const int ex = base + cinc - cv;
    if (tid < PCY_PAR_MAXCTA) ctot[tid] = ex;
    if (tid <= PCY_PAR_MAXCTA) par->off[tid] = ex;   // off[P] = window size
  }
  __syncthreads();
  if (tid < c) { par->list[ctot[cta] + rank] = tid; __threadfence(); }
  __syncthreads();
  if (tid == 0) {
    const int P = s_P;
    par->mode = 0; par->P = P; par->n_win = c; par->n_total = n;
    par->F0 = F0; par->Falloc0 = C->F_alloc; par->freen0 = C->free_n; par->Galloc0 = C->G_alloc;
    par->Aalloc0 = C->A_alloc; par->nidx0 = C->next_index;
    par->open_ticket = 0; par->g_ticket = 0; par->a_ticket = 0; par->done = 0; par->opens = 0;
    par->arena_fail = 0;
    __threadfence();
    *(volatile long long*)&par->ready = planseq;   // the resolve CTAs may go (flag_wait)
#ifdef PCY_TIMELINE
    plan_t[9] = clock64();
    if (!order) { for (int k = 1; k < 10; ++k) atomicAdd(&g_tlp[k], (unsigned long long)(plan_t[k] - plan_t[k - 1])); atomicAdd(&g_tlp[0], 1ULL); }
#endif
    if (!order) PCY_TL(3);
    if (pub) {   // early publication: the host may enqueue the next K1 batch now
      volatile long long* t = &pub->plan_mode;
      t[0] = 0; t[1] = c;
      __threadfence_system();
      t[2] = planseq;
    }
  }
}
