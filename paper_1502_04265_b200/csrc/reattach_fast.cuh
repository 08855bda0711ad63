// K4 rebuild reattach, batched (included by engine.cu after resolve_fast.cuh).
//
// _reattach (coreset.py:395-421) re-inserts the collected nodes in (-weight,
// index) order.  Like insertion, a node's nearest-reference chain depends only
// on the references already placed, so it is computed for a whole batch in
// parallel against the partially rebuilt tree (k_rchain, one warp per node),
// together with the merge test under the snapshot statistics.  k_reattach2
// then walks the batch in order on one warp, re-testing only against nodes
// placed earlier in the same launch (shared-memory table) and recomputing the
// merge test for hosts touched in the launch.

__global__ void k_rchain(EngDev E, const int* __restrict__ order, long long n, ChainHdr* __restrict__ H,
                         ChainLvl* __restrict__ R, const double* __restrict__ P, long long ldp) {
  extern __shared__ double sm_x[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  if (i >= n) return;
  const int d = E.d, ld = E.ld;
  const int u = order[i];
  double* xv = sm_x + (long long)wib * ld;
  for (int e = lane; e < d; e += 32) xv[e] = E.r[(long long)u * ld + e];
  __syncwarp();
  const double rsq = E.rn[u];
  const long long wu = E.w[u];
  const double qu = E.q[u];
  const double* su = E.s + (long long)u * ld;
  const double T = E.ctl->T;
  ChainLvl* rec = R + i * PCY_FMAXL;
  double radius = T;
  int g = 0, L = 0, pred = -1, predj = -1, trunc = 0, nre = 0;
  long long vis = 0, vdir = 0;
  int cnt = E.g_count[0], base = E.g_base[0];
  int pb = E.panel_gofs ? E.panel_gofs[0] : -1;
  for (;;) {
    double bp; int bpos;
    LaneWinner win{-1, -1, 0, 0.0, 0.0};
    bool have_win = false;
    vis += cnt;
    if (E.panel_gofs) {   // visited-groups K1: panel for big groups, direct fp64 scans otherwise
      if (E.tc_dots && pb >= 0)
        scan_parts_tc(E, i, g, E.arena + base, cnt,
                      [&](int jj) { return warp_dot(E.r + (long long)jj * ld, xv, d, lane); }, lane, bp, bpos, nre, pb);
      else { scan_members_lane_w(E, E.arena + base, cnt, xv, lane, bp, bpos, win); vdir += cnt; have_win = true; }
    } else if (E.tc_dots)   // tensor-core dots + near-tie recheck
      scan_parts_tc(E, i, g, E.arena + base, cnt, [&](int jj) { return warp_dot(E.r + (long long)jj * ld, xv, d, lane); },
                    lane, bp, bpos, nre);
    else if (P) scan_parts(P + i * ldp, E.col_of, E.arena + base, cnt, lane, bp, bpos);   // parts from the DMMA contraction
    else { scan_members(E, E.arena + base, 0, cnt, xv, lane, bp, bpos); vdir += cnt; }
    const int j = have_win ? (bpos < cnt ? win.id : -1) : (bpos < cnt ? E.arena[base + bpos] : -1);
    ChainLvl c = empty_level();
    c.part = bp; c.j = j; c.g = g;
    ++L;
    const bool outside = j < 0 || radd(bp, rsq) > radius;
    int ncnt = 0, nbase = 0, npb = -1;
    if (!outside) {
      if (have_win) { c.w = win.w; c.q = win.q; c.sn = win.sn; c.child = win.child; }
      else { c.w = E.w[j]; c.q = E.q[j]; c.sn = E.sn[j]; c.child = E.child[j]; }
      if (c.child >= 0) {   // next level's group, overlapping the merge-norm dot
        ncnt = E.g_count[c.child]; nbase = E.g_base[c.child];
        npb = E.panel_gofs ? E.panel_gofs[c.child] : -1;
      }
      const double* sh = E.s + (long long)j * ld;
      double acc = 0.0;
      for (int e = lane; e < d; e += 32) { const double v = radd(sh[e], su[e]); acc = fma(v, v, acc); }
      const double mnorm = warp_sum(acc);
      const long long mw = c.w + wu;
      const double mq = radd(c.q, qu);
      c.nq = mq; c.nsn = mnorm;
      c.take = rsub(mq, rdiv(mnorm, (double)mw)) <= T ? 1 : 0;
      if (c.take && pred < 0) { pred = L - 1; predj = j; }
    }
    if (lane == 0) { rec[L - 1] = c; E.pathj[i * PCY_FMAXL + L - 1] = c.j; }
    if (outside) { if (pred < 0) pred = L - 1; break; }
    if (c.child < 0) {
      if (L < PCY_FMAXL) {
        if (lane == 0) { rec[L] = empty_level(); E.pathj[i * PCY_FMAXL + L] = -1; }
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
  if (lane == 0) H[i] = ChainHdr{L, pred, predj, trunc};
  if (lane == 0 && nre > 0) atomicAdd((unsigned long long*)&E.ctl->cnt_direct, (unsigned long long)nre);
  if (lane == 0) {
    atomicAdd((unsigned long long*)&E.ctl->cnt_vis, (unsigned long long)vis);
    if (vdir) atomicAdd((unsigned long long*)&E.ctl->cnt_vis_direct, (unsigned long long)vdir);
  }
}

// PAR = true: CTA b reattaches the nodes of k_plan's subtree list b (the same
// partition argument as the resolve: merges change only the host, adds only
// the group of the parent); PAR = false with `par`: k_plan's sequential stretch.
template <int NPER, bool PAR>
__device__ __forceinline__ void reattach2_body(const EngDev& E, const int* __restrict__ order, long long n,
                                               int nnew_cap, const ChainHdr* __restrict__ H,
                                               const ChainLvl* __restrict__ R, ParCtl* __restrict__ par,
                                               const double* __restrict__ gram, long long gld,
                                               EngCtl* pub, long long pseq, int ts_cap) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ReattachSmem& S = *reinterpret_cast<ReattachSmem*>(smraw);
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
  double* xsm = reinterpret_cast<double*>(smraw + ((sizeof(ReattachSmem) + 15) & ~size_t(15)));
  const int lds = ld | 1;   // odd stride: conflict-free lane-per-row reads
  double* tref = xsm + ld;
  unsigned* mbits = reinterpret_cast<unsigned*>(tref + (gram ? 0LL : (long long)nnew_cap * lds));   // layout: reattach_smem_bytes
  const int mwords = (int)(E.NC / 32 + 1);
  unsigned* gbits = mbits + mwords;
  const int gwords = (int)(E.GC / 32 + 1);
  // batch-Gram rows of the current and the next item (lower triangle: the
  // columns of earlier items), staged with cp.async one item ahead so the
  // scans of same-launch entries read shared memory
  double* growb = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(mbits) +
                                            ((sizeof(unsigned) * (size_t)(mwords + gwords) + 15) & ~size_t(15)));
  // Only the columns the scans read are staged, by entry: the batch rows of the
  // entries placed so far (nn of them) and of the item being processed while
  // this copy is in flight (it may place entry nn).  Entries come from earlier
  // items of this list, so their columns are in the row's lower triangle.
  auto stage_grow = [&](int buf, long long it, int nn, long long placing) {
    if (!gram) return;
    const double* src = gram + it * gld;
    double* dst = growb + buf * PCY_PAR_MAXITEMS;
    for (int t = lane; t < nn; t += 32) cp_async8(dst + t, src + S.titem[t]);
    if (lane == 0 && placing >= 0) cp_async8(dst + nn, src + placing);
    cp_async_commit();
  };
  // s rows of the first ts_cap entries placed in this launch: in a fresh tree
  // most hosts are such entries, and the merge test (coreset.py:407-417) then
  // reads and updates shared memory instead of waiting on an HBM row per level
  double* tsr = growb + 2 * PCY_PAR_MAXITEMS;
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
#ifdef PCY_TIMELINE
  const long long tl_t0 = clock64();
  long long tl_wait = 0, tl_lev = 0, tl_scan = 0, tl_nd = 0, tl_cd = 0, tl_nn = 0, tl_cn = 0, tl_nrec = 0, tl_nglob = 0, tl_cm = 0, tl_nsm = 0, tl_ctail = 0, tl_head = 0;
#endif

  for (int s2 = lane; s2 < PCY_MOD_SLOTS; s2 += 32) S.mkey[s2] = -1;
  for (int s2 = lane; s2 < PCY_GMAP_SLOTS; s2 += 32) S.gkey[s2] = -1;
  for (int s2 = lane; s2 < mwords; s2 += 32) mbits[s2] = 0u;
  for (int s2 = lane; s2 < gwords; s2 += 32) gbits[s2] = 0u;
  if (lane == 0) S.modcount = 0;
  int nnew = 0;

  // ---- prologue: item 0
  double xr[NPER], su[NPER], pr[NPER];
  // window positions of items i .. i+2 in registers (list entries are read
  // three items ahead: no list load sits on an item's critical path)
  long long gq0 = n > 0 ? gix(0) : 0, gq1 = n > 1 ? gix(1) : 0, gq2 = n > 2 ? gix(2) : 0;
  int u_c = n > 0 ? order[gq0] : 0;
  int u_n = n > 1 ? order[gq1] : 0;
  ChainHdr hc = n > 0 ? H[gq0] : ChainHdr{0, 0, -1, 0};
  ChainHdr hn = n > 1 ? H[gq1] : ChainHdr{0, 0, -1, 0};
  long long wu_c = 0; double qu_c = 0.0, snu_c = 0.0, rsq_c = 0.0;
  if (n > 0) {
    load_row<NPER>(xr, E.r + (long long)u_c * ld, d, lane);
    load_row<NPER>(su, E.s + (long long)u_c * ld, d, lane);
    if (hc.predj >= 0) load_row<NPER>(pr, E.s + (long long)hc.predj * ld, d, lane);
    wu_c = E.w[u_c]; qu_c = E.q[u_c]; snu_c = E.sn[u_c]; rsq_c = E.rn[u_c];
    const uint4* src = reinterpret_cast<const uint4*>(R + gq0 * PCY_FMAXL);
    uint4* dst = reinterpret_cast<uint4*>(&S.rb[0][0]);
    for (int c = lane; c < REC_CHUNKS; c += 32) dst[c] = src[c];
    stage_grow(0, gq0, 0, -1);
    cp_async_wait_all();
  }
  __syncwarp();
  int cur = 0;
  int prnode = hc.predj;

  for (long long i = 0; i < n; ++i) {
#ifdef PCY_TIMELINE
    const long long tl_h0 = clock64();
#endif
    if (nnew >= nnew_cap || S.modcount >= PCY_MOD_SLOTS / 2) { status = ST_FULL; stop = i; break; }
    // ---- prefetch item i+1
    double xn[NPER], sun[NPER], pn[NPER];
    uint4 rpf[(REC_CHUNKS + 31) / 32];
    const bool has_next = i + 1 < n;
    ChainHdr h2 = ChainHdr{0, 0, -1, 0};
    int u2 = 0;
    long long wu_n = 0; double qu_n = 0.0, snu_n = 0.0, rsq_n = 0.0;
    const long long gq3 = i + 3 < n ? gix(i + 3) : 0;
    if (has_next) {
      load_row<NPER>(xn, E.r + (long long)u_n * ld, d, lane);
      load_row<NPER>(sun, E.s + (long long)u_n * ld, d, lane);
      wu_n = E.w[u_n]; qu_n = E.q[u_n]; snu_n = E.sn[u_n]; rsq_n = E.rn[u_n];
      const uint4* src = reinterpret_cast<const uint4*>(R + gq1 * PCY_FMAXL);
#pragma unroll
      for (int q = 0; q < (REC_CHUNKS + 31) / 32; ++q) { const int c = lane + 32 * q; if (c < REC_CHUNKS) rpf[q] = src[c]; }
      if (hn.predj >= 0) load_row<NPER>(pn, E.s + (long long)hn.predj * ld, d, lane);
      if (i + 2 < n) { h2 = H[gq2]; u2 = order[gq2]; }
      stage_grow(cur ^ 1, gq1, nnew, gq0);
    }
    // ---- item i: node u
    const int u = u_c;
    const int len = hc.len;
    int g = 0, L = 0;
    double radius = T;
    bool direct = false;
#pragma unroll
    for (int k = 0; k < NPER; ++k) { const int e = lane + 32 * k; if (e < ld) xsm[e] = xr[k]; }
    __syncwarp();
    int lastmod = -1;
    // levels above K1's action level where nothing changed in this launch and
    // K1 descended (no merge) into an existing child group are stepped over
    unsigned cleanmask = 0u;
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
#ifdef PCY_TIMELINE
    tl_head += clock64() - tl_h0;
#endif
    for (;;) {
      if (!direct && ((cleanmask >> L) & 1u)) {   // unchanged level: K1's descent stands
        g = S.rb[cur][L].child;
        radius = rmul(radius, 0.25);
        ++L;
        continue;
      }
      int bj = -1, li = -1;
      double bp = INFINITY;
#ifdef PCY_TIMELINE
      ++tl_lev;
      const long long tl_s0 = clock64();
#endif
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
#ifdef PCY_TIMELINE
        ++tl_nd; tl_cd += clock64() - tl_s0;
#endif
      }
      int bt = -1;
#ifdef PCY_TIMELINE
      const long long tl_s1 = clock64();
      if ((gbits[g >> 5] >> (g & 31)) & 1u) ++tl_nn;
#endif
      if ((gbits[g >> 5] >> (g & 31)) & 1u) {
        // one new member per lane: sequential dot over the padded smem row
        double np_ = INFINITY; int nt = 0x7fffffff;
        if (gram) {
          // same-launch nodes are rows of this batch: (current, earlier) entry of the batch Gram
          const double* grow = growb + cur * PCY_PAR_MAXITEMS;
          for (int c0 = 0; c0 < nnew; c0 += 64) {   // two independent entries per lane and pass
            const int t0 = c0 + lane, t1 = t0 + 32;
            const bool v0 = t0 < nnew && S.tgrp[t0] == g, v1 = t1 < nnew && S.tgrp[t1] == g;
            const double p0 = v0 ? radd(S.trn[t0], rmul(grow[t0], -2.0)) : INFINITY;
            const double p1 = v1 ? radd(S.trn[t1], rmul(grow[t1], -2.0)) : INFINITY;
            if (p0 < np_) { np_ = p0; nt = t0; }
            if (p1 < np_) { np_ = p1; nt = t1; }
          }
        } else
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
      const long long tl_s2 = clock64();
      tl_scan += tl_s2 - tl_s0;
      tl_cn += tl_s2 - tl_s1;
#endif
      if (bj < 0 || radd(bp, rsq_c) > radius) {
        // group.add(node): u keeps its statistics (coreset.py:403-406)
        const int t = nnew++;
        if (!gram) {
          double* rr = tref + (long long)t * lds;
#pragma unroll
          for (int k = 0; k < NPER; ++k) { const int e = lane + 32 * k; if (e < ld) rr[e] = xr[k]; }
        }
        const bool had = ((gbits[g >> 5] >> (g & 31)) & 1u) != 0;
        int gs;
        if (had) gs = gmap_find(S, g);
        else {
          gs = (int)(((unsigned)g * 2654435761u) >> 24) & (PCY_GMAP_SLOTS - 1);
          while (S.gkey[gs] >= 0) gs = (gs + 1) & (PCY_GMAP_SLOTS - 1);
        }
        if (t < ts_cap) {
          double* hs = tsr + (long long)t * ld;
#pragma unroll
          for (int k = 0; k < NPER; ++k) { const int e = lane + 32 * k; if (e < ld) hs[e] = su[k]; }
        }
        if (lane == 0) {
          S.tdirty[t] = 0;
          S.tid[t] = u; S.tgrp[t] = g; S.tchild[t] = -1; S.tnext[t] = -1; S.titem[t] = (int)gq0;
          S.tw[t] = wu_c; S.tq[t] = qu_c; S.tsn[t] = snu_c; S.trn[t] = rsq_c;
          if (had) { S.tnext[S.gtail[gs]] = t; S.gtail[gs] = t; }
          else { S.gkey[gs] = g; S.ghead[gs] = t; S.gtail[gs] = t; gbits[g >> 5] |= 1u << (g & 31); }
        }
        ++F;
        __syncwarp();
        break;
      }
      // merge test with the host (coreset.py:407-417)
      const bool touched = bt < 0 && ((mbits[bj >> 5] >> (bj & 31)) & 1u);
      const bool shost = bt >= 0 && bt < ts_cap;   // the host's s row is in shared memory
      int ms = -1;
      bool merge;
      long long mw; double mq, mnorm;
      long long hw; double hq, hsn;
      if (bt < 0 && li >= 0 && !touched) {
        const ChainLvl& rc = S.rb[cur][li];
        hw = rc.w; hq = rc.q; hsn = rc.sn;
        merge = rc.take != 0; mw = rc.w + wu_c; mq = rc.nq; mnorm = rc.nsn;
#ifdef PCY_TIMELINE
        ++tl_nrec;
#endif
      } else {
#ifdef PCY_TIMELINE
        if (shost) ++tl_nsm; else if (bj != prnode) ++tl_nglob;
#endif
        if (bt >= 0) { hw = S.tw[bt]; hq = S.tq[bt]; hsn = S.tsn[bt]; }
        else if (touched) { ms = map_find(S, bj); hw = S.mw[ms]; hq = S.mq[ms]; hsn = S.msn[ms]; }
        else { hw = E.w[bj]; hq = E.q[bj]; hsn = E.sn[bj]; }
        double acc = 0.0;
        if (shost) {
          const double* hs = tsr + (long long)bt * ld;
#pragma unroll
          for (int k = 0; k < NPER; ++k) {
            const int e = lane + 32 * k;
            const double v = radd(e < ld ? hs[e] : 0.0, su[k]);
            acc = fma(v, v, acc);
          }
        } else {
          if (bj != prnode) { load_row<NPER>(pr, E.s + (long long)bj * ld, d, lane); prnode = bj; }
#pragma unroll
          for (int k = 0; k < NPER; ++k) { const double v = radd(pr[k], su[k]); acc = fma(v, v, acc); }
        }
        mnorm = warp_sum(acc);
        mw = hw + wu_c; mq = radd(hq, qu_c);
        merge = rsub(mq, rdiv(mnorm, (double)mw)) <= T;
      }
#ifdef PCY_TIMELINE
      const long long tl_s3 = clock64();
      tl_cm += tl_s3 - tl_s2;
#endif
      if (merge) {
        if (shost) {
          double* hs = tsr + (long long)bt * ld;
#pragma unroll
          for (int k = 0; k < NPER; ++k) { const int e = lane + 32 * k; if (e < d) hs[e] = radd(hs[e], su[k]); }
          if (lane == 0) S.tdirty[bt] = 1;
        } else {
          if (bj != prnode) { load_row<NPER>(pr, E.s + (long long)bj * ld, d, lane); prnode = bj; }
#pragma unroll
          for (int k = 0; k < NPER; ++k) pr[k] = radd(pr[k], su[k]);
          store_row<NPER>(E.s + (long long)bj * ld, pr, d, lane);
        }
        if (bt >= 0) {
          if (lane == 0) { S.tw[bt] = mw; S.tq[bt] = mq; S.tsn[bt] = mnorm; }
          __syncwarp();
        } else {
          int child_now;
          if (touched) { if (ms < 0) ms = map_find(S, bj); child_now = S.mchild[ms]; }
          else child_now = li >= 0 ? S.rb[cur][li].child : E.child[bj];
          ms = map_put(S, mbits, bj, mw, mq, mnorm, child_now, lane);
          if (lane == 0) { E.w[bj] = mw; E.q[bj] = mq; E.sn[bj] = mnorm; }
        }
        if constexpr (PAR) {
          if (lane == 0) {
            E.alive[u] = 0;
            const unsigned long long t = atomicAdd(&par->open_ticket, 1ULL);   // free-stack pushes
            E.free_ids[par->freen0 + (long long)t] = u;
          }
        } else {
          if (lane == 0) { E.alive[u] = 0; E.free_ids[freen] = u; }
          ++freen;
        }
        lastmod = shost ? -1 : bj;   // a shared-memory host is never a K1-predicted node
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
        if (tnow && ms < 0) ms = map_find(S, bj);
        c = tnow ? S.mchild[ms] : (li >= 0 ? S.rb[cur][li].child : E.child[bj]);
        if (c < 0) {
          c = new_group();
          if (lane == 0) { E.g_count[c] = 0; E.g_cap[c] = 0; E.g_base[c] = 0; E.child[bj] = c; }
          if (tnow) { if (lane == 0) S.mchild[ms] = c; __syncwarp(); }
          else ms = map_put(S, mbits, bj, hw, hq, hsn, c, lane);
        }
      }
      g = c;
      radius = rmul(radius, 0.25);
      ++L;
#ifdef PCY_TIMELINE
      tl_ctail += clock64() - tl_s3;
#endif
    }
    __syncwarp();
#ifdef PCY_TIMELINE
    const long long tl_w0 = clock64();
#endif
    if (has_next) {
      uint4* dst = reinterpret_cast<uint4*>(&S.rb[cur ^ 1][0]);
#pragma unroll
      for (int q = 0; q < (REC_CHUNKS + 31) / 32; ++q) { const int c = lane + 32 * q; if (c < REC_CHUNKS) dst[c] = rpf[q]; }
#pragma unroll
      for (int k = 0; k < NPER; ++k) { xr[k] = xn[k]; su[k] = sun[k]; }
      int nextnode = hn.predj;
      if (nextnode >= 0 && nextnode == lastmod) {
        if (prnode == lastmod) {
#pragma unroll
          for (int k = 0; k < NPER; ++k) pn[k] = pr[k];
        } else nextnode = -1;
      }
#pragma unroll
      for (int k = 0; k < NPER; ++k) pr[k] = pn[k];
      prnode = nextnode;
      hc = hn; hn = h2;
      u_c = u_n; u_n = u2;
      wu_c = wu_n; qu_c = qu_n; snu_c = snu_n; rsq_c = rsq_n;
      cp_async_wait_all();   // the next item's Gram row
      cur ^= 1;
    }
    gq0 = gq1; gq1 = gq2; gq2 = gq3;
    __syncwarp();
#ifdef PCY_TIMELINE
    if (__shfl_sync(PCY_FULL, xr[0] + su[0] + (double)wu_c, 0) == 1.2345e-300) ++tl_lev;   // wait for the prefetched rows
    tl_wait += clock64() - tl_w0;
#endif
  }
  cp_async_wait_all();

  // ---- cleanup: statistics of placed nodes, memberships in position order
  __syncwarp();
  for (int t = 0; t < nnew && t < ts_cap; ++t) {
    if (!S.tdirty[t]) continue;
    const double* hs = tsr + (long long)t * ld;
    double* dst = E.s + (long long)S.tid[t] * ld;
    for (int e = lane; e < d; e += 32) dst[e] = hs[e];
  }
  for (int t = lane; t < nnew; t += 32) {
    const int node = S.tid[t];
    E.w[node] = S.tw[t]; E.q[node] = S.tq[t]; E.sn[node] = S.tsn[t];
    E.child[node] = S.tchild[t];
    const int g = S.tgrp[t];
    S.tcnt[t] = E.g_count[g]; S.tcap[t] = E.g_cap[g]; S.tbase[t] = E.g_base[g];
  }
  // rank within the group and the group's first entry: walk each group's
  // list of new entries (linked in placement order through tnext)
  for (int gs = lane; gs < PCY_GMAP_SLOTS; gs += 32) {
    if (S.gkey[gs] < 0) continue;
    const int f = S.ghead[gs];
    int k = 0;
    for (int t = f; t >= 0; t = S.tnext[t]) { S.tk[t] = k++; S.tfirst[t] = f; }
    S.tgn[f] = k;
  }
  __syncwarp();
  bool arena_ok = true;
  for (int t = 0; t < nnew; ++t) {
    if (S.tfirst[t] != t) continue;
    const int g = S.tgrp[t];
    const int total = S.tgn[t];
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
  } else status = ST_ARENA;
  __syncwarp();
  if constexpr (PAR) {
    int lastf = 0;   // this CTA finished the window: its warp publishes
#ifdef PCY_TIMELINE
    if (lane == 0) { tl_rea(n, clock64() - tl_t0, tl_wait, nnew, tl_lev, tl_scan); tl_rea2(n, tl_nd, tl_head, tl_nn, tl_cn, tl_nrec, tl_nglob, tl_nsm, tl_cm, tl_ctail); }
#endif
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

template <int NPER, bool PAR = false>
__global__ void __launch_bounds__(32, 1) k_reattach2(EngDev E, const int* __restrict__ order, long long n,
                                                     int nnew_cap, const ChainHdr* __restrict__ H,
                                                     const ChainLvl* __restrict__ R, ParCtl* __restrict__ par = nullptr,
                                                     const double* __restrict__ gram = nullptr, long long gld = 0) {
  reattach2_body<NPER, PAR>(E, order, n, nnew_cap, H, R, par, gram, gld, nullptr, 0, 0);
}

// One launch for either choice of k_plan (as k_resolve2x).
template <int NPER>
__global__ void __launch_bounds__(32, 1) k_reattach2x(EngDev E, const int* __restrict__ order, long long n,
                                                      int nnew_cap, const ChainHdr* __restrict__ H,
                                                      const ChainLvl* __restrict__ R, ParCtl* __restrict__ par,
                                                      const double* __restrict__ gram, long long gld,
                                                      EngCtl* pub, long long pseq, int ts_cap) {
  pdl_wait();   // k_plan has finished (programmatic launch)
  if (par->mode == 0) reattach2_body<NPER, true>(E, order, n, nnew_cap, H, R, par, gram, gld, pub, pseq, ts_cap);
  else if (blockIdx.x == 0) reattach2_body<NPER, false>(E, order, n, nnew_cap, H, R, par, gram, gld, pub, pseq, ts_cap);
}
