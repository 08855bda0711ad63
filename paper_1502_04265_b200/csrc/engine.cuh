// Device-resident BICO clustering-feature engine: data layout shared by the
// kernels in engine.cu (see DESIGN.md §3 for the HBM layout).
#pragma once
#include "common.cuh"
#include <cstddef>

#define PCY_MAXL 24          // chain levels recorded per item by k_chain
#define PCY_GROUP_MIN_CAP 4  // first arena extent of a group

// Status codes written by the sequential kernels into EngCtl::status.
enum {
  ST_DONE = 0,
  ST_REBUILD = 1,   // open-one-copy at full budget: rebuild, then resume item `stop`
  ST_INVALID = 2,   // item `stop` failed validation (err holds the code)
  ST_BUILD = 3,     // bootstrap saw budget+1 distinct locations at item `stop`
  ST_GROW = 4,      // bootstrap pending buffer full before item `stop`
  ST_ARENA = 5,     // member arena exhausted (internal error)
  ST_FULL = 6,      // resolve tables full before item `stop`: relaunch from there
  ST_PAR_BROKEN = 7,  // a subtree-parallel resolve CTA met a stop k_plan excludes (internal error)
};

struct EngCtl {
  long long F;            // live features (_num_features)
  long long F_alloc;      // node slots ever handed out (<= NC)
  long long free_n;       // free-slot stack depth
  long long G_alloc;      // groups in use (group 0 = roots)
  long long A_alloc;      // member-arena bump pointer
  long long next_index;   // creation counter (_next_index)
  long long G_snap;       // groups that existed at the chain snapshot
  long long total_w;      // total weight consumed
  double T;               // threshold
  long long npend, ndist; // bootstrap pending entries / distinct keys
  int status, err;
  long long stop, remaining;
  long long max_depth;
  // instrumentation (k_resolve2): levels walked, direct scans, demand row
  // loads, full capacity evaluations, items resolved
  long long cnt_levels, cnt_direct, cnt_demand, cnt_slow, cnt_items, cnt_dem_fast, cnt_touch_child;
  long long root_count, root_base;   // group 0 (copied by k_publish for the host)
  // visited-groups K1 (d <= 256): members in the tensor-core panel (groups of
  // >= PCY_PANEL_MIN members, k_publish_panel) and the work counters --
  // member visits of the chain walks (the reference's own dgemv work,
  // coreset.py:172) and the visits served by direct fp64 scans
  long long panel_n, cnt_vis, cnt_vis_direct;
  // largest member count any group reached since the last tree reset: below
  // PCY_PANEL_MIN no group is in the K1 panel, so the resolve kernels publish
  // the counters themselves and the panel publication is skipped
  long long maxg;
  long long seq;          // publication sequence number (mapped host mirror)
  // k_plan's early publication (mirror only, written after `seq`'s words): the
  // window it chose for K1 batch `plan_seq`, so the host can enqueue the next
  // batch while the resolve kernel runs
  long long plan_mode, plan_nwin, plan_seq;
  // device only: publication number of the last window whose tree writes are
  // complete (set by the finishing resolve CTA before it copies the counters
  // to the host mirror); the run-ahead chain walk waits on it (flag_wait)
  long long win_done;
};

// groups of at least this many members are contracted on the tensor cores
// (the K1 panel, k_publish_panel); smaller groups are scanned directly
constexpr int PCY_PANEL_MIN = 128;



// Subtree-parallel resolve (k_plan + k_resolve2<NPER, true>, resolve_fast.cuh).
// Between two changes of the root group, an item's decisions read and write
// only the subtree of its root winner (coreset.py:318-372 descend from
// group.nodes[j] into its children), so the items of a window with no root
// open, no rebuild (F0 + window <= budget) and no invalid row are resolved by
// one CTA per root subtree, each in stream order.  k_plan writes the window
// and the per-CTA item lists; the resolve CTAs allocate slots, groups and
// arena extents through the tickets and the last CTA publishes the counters.
#define PCY_PAR_MAXCTA 148
#define PCY_PAR_MAXITEMS 1024
struct ParCtl {
  int mode;            // 0: parallel window, 1: sequential kernel
  int P;               // resolve CTAs with items
  long long n_win;     // items in the window (parallel) / for the sequential kernel
  long long n_total;   // items chained by K1 (the block)
  long long F0, Falloc0, freen0, Galloc0, Aalloc0, nidx0;   // control snapshot
  unsigned long long open_ticket, g_ticket, a_ticket, done, opens;
  int arena_fail, pad;
  long long ready;     // k_plan's launch number once every field above/below is written (flag_wait)
  int dbg_sets, dbg_maxset, dbg_maxcta, dbg_pad;   // PCY_TRACE builds: domain sets, largest set, longest CTA list
  int off[PCY_PAR_MAXCTA + 1];
  int list[PCY_PAR_MAXITEMS];
};

struct EngDev {
  int d, ld;
  long long m, NC, GC, AC;
  // nodes (slot-indexed)
  long long* w; double* q; double* sn; double* rn; long long* idx;
  int* child; int* alive; int* free_ids;
  double* s; double* r;            // NC x ld, row-major
  // groups: members live in arena[g_base .. g_base + g_count)
  int* g_base; int* g_count; int* g_cap; int* g_bs; int* g_bsbase;
  int* arena;
  EngCtl* ctl;
  // staged batch
  double* xb; double* xsq; long long* wb; unsigned long long* hsh; int* bad;
  int* ch_node; double* ch_part; int* ch_len;
  // bootstrap
  double* pend_x; long long* pend_w; double* pend_xsq; long long pend_cap;
  double* dist_x; int* htab; long long hcap;
  // full-set K1 on the tensor cores (tc_dots.cu): 3xTF32 dots of the block
  // against every slot, centred norms and the error factor; null when unused
  const float* tc_dots; long long tc_ldo; const double* tc_rnc; const double* tc_xn2; double tc_tau;
  // live columns of the full-set contraction: slot -> column (assigned when a
  // slot first holds a node, recompacted after every rebuild)
  const int* col_of;
  // column order of the full-set contraction: group g's members occupy the
  // contiguous columns [fs_gofs[g], fs_gofs[g] + g_count[g]) (fs_list = slots)
  int* fs_list; int* fs_gofs; int* fs_cnt;
  // visited-groups K1: panel column of group g's first member, -1 when the
  // group is scanned directly (null outside panel mode; = fs_gofs)
  const int* panel_gofs;
  // K1 winners per level (Bmax x PCY_FMAXL ints, -1 past the record): k_plan's compact view of the chains
  int* pathj;
  // rebuild / extraction scratch
  int* order; int* lvl; int* stk_g; int* stk_p;
  unsigned long long* minbits;
};

// One warp copies the device counters to the mapped host mirror (a word per
// lane: one L2 round trip, not one per word) and then writes the sequence
// number the host spins on (same protocol as k_publish).  Counters other CTAs
// updated with atomics are read at L2 (volatile).  Call with the whole warp.
__device__ __forceinline__ void ctl_publish_warp(const EngDev& E, EngCtl* dst, long long seq, int lane) {
  EngCtl* src = E.ctl;
  if (lane == 0) {
    src->root_count = *(volatile const int*)&E.g_count[0];
    src->root_base = *(volatile const int*)&E.g_base[0];
  }
  __syncwarp();
  const int words = (int)(offsetof(EngCtl, seq) / sizeof(long long));
  volatile const long long* s = reinterpret_cast<volatile const long long*>(src);
  volatile long long* t = reinterpret_cast<volatile long long*>(dst);
  for (int k = lane; k < words; k += 32) t[k] = s[k];
  __threadfence_system();
  __syncwarp();
  if (lane == 0) t[words] = seq;
}

// Build-time timeline (PCY_NVCC_EXTRA=-DPCY_TIMELINE): kernels stamp the
// global timer at entry / exit; the engine prints the mean phase durations and
// gaps of the insertion windows when it is destroyed.
#ifdef PCY_TIMELINE
#define PCY_TL_CAP (1 << 18)
__device__ unsigned long long g_tl[PCY_TL_CAP];
__device__ unsigned int g_tl_n;
__device__ __forceinline__ void tl_stamp(int tag) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const unsigned i = atomicAdd(&g_tl_n, 1u);
  if (i < PCY_TL_CAP) g_tl[i] = (t << 4) | (unsigned long long)tag;
}
#define PCY_TL(tag) tl_stamp(tag)
// per resolve CTA: items, new nodes, slow-path evaluations, cycles
__device__ unsigned long long g_tlc[PCY_TL_CAP];
__device__ unsigned int g_tlc_n;
__device__ __forceinline__ void tl_cta(long long items, int nnew, long long slow, long long cyc) {
  const unsigned i = atomicAdd(&g_tlc_n, 1u);
  if (i < PCY_TL_CAP)
    g_tlc[i] = ((unsigned long long)(cyc & 0xffffff) << 40) | ((unsigned long long)(slow & 0xfff) << 28) |
               ((unsigned long long)(nnew & 0xfff) << 16) | (unsigned long long)(items & 0xffff);
}
// decision-warp cycle split per list-length bucket: count, wait-for-staging,
// slow-path, start-up, clean-up, demand-load cycles
__device__ unsigned long long g_tls[8][8];
__device__ __forceinline__ void tl_split(long long items, long long wait, long long slow, long long start, long long clean, long long dem, long long fast) {
  const int b = items <= 2 ? 0 : items <= 4 ? 1 : items <= 8 ? 2 : items <= 12 ? 3 : items <= 16 ? 4 : items <= 24 ? 5 : items <= 48 ? 6 : 7;
  atomicAdd(&g_tls[b][0], 1ULL); atomicAdd(&g_tls[b][1], (unsigned long long)wait); atomicAdd(&g_tls[b][2], (unsigned long long)slow);
  atomicAdd(&g_tls[b][3], (unsigned long long)start); atomicAdd(&g_tls[b][4], (unsigned long long)clean); atomicAdd(&g_tls[b][5], (unsigned long long)dem);
  atomicAdd(&g_tls[b][6], (unsigned long long)fast);
}
__device__ unsigned long long g_tls2[8][8];
__device__ __forceinline__ void tl_split2(long long items, long long dir, long long nw, long long cap, long long ndir, long long nnew, long long nlev, long long ncl) {
  const int b = items <= 2 ? 0 : items <= 4 ? 1 : items <= 8 ? 2 : items <= 12 ? 3 : items <= 16 ? 4 : items <= 24 ? 5 : items <= 48 ? 6 : 7;
  atomicAdd(&g_tls2[b][1], (unsigned long long)dir); atomicAdd(&g_tls2[b][2], (unsigned long long)nw);
  atomicAdd(&g_tls2[b][3], (unsigned long long)cap); atomicAdd(&g_tls2[b][4], (unsigned long long)ndir); atomicAdd(&g_tls2[b][5], (unsigned long long)nnew);
  atomicAdd(&g_tls2[b][6], (unsigned long long)nlev); atomicAdd(&g_tls2[b][7], (unsigned long long)ncl);
}
// reattach CTAs by list length: count, cycles, items, stage-wait cycles, adds, levels, new-member scan cycles
__device__ unsigned long long g_tlr[8][8];
__device__ __forceinline__ void tl_rea(long long items, long long cyc, long long wait, long long adds, long long lev, long long scan) {
  const int b = items <= 8 ? 0 : items <= 16 ? 1 : items <= 32 ? 2 : items <= 64 ? 3 : items <= 128 ? 4 : items <= 256 ? 5 : items <= 512 ? 6 : 7;
  atomicAdd(&g_tlr[b][0], 1ULL); atomicAdd(&g_tlr[b][1], (unsigned long long)cyc); atomicAdd(&g_tlr[b][2], (unsigned long long)items);
  atomicAdd(&g_tlr[b][3], (unsigned long long)wait); atomicAdd(&g_tlr[b][4], (unsigned long long)adds); atomicAdd(&g_tlr[b][5], (unsigned long long)lev);
  atomicAdd(&g_tlr[b][6], (unsigned long long)scan);
}
__device__ unsigned long long g_tlp[10];   // k_plan phase cycles (thread 0)
__device__ unsigned long long g_tlr2[8][12];
__device__ __forceinline__ void tl_rea2(long long items, long long a0, long long a1, long long a2, long long a3, long long a4, long long a5, long long a6, long long a7, long long a8) {
  const int b = items <= 8 ? 0 : items <= 16 ? 1 : items <= 32 ? 2 : items <= 64 ? 3 : items <= 128 ? 4 : items <= 256 ? 5 : items <= 512 ? 6 : 7;
  const long long v[9] = {a0, a1, a2, a3, a4, a5, a6, a7, a8};
  for (int k = 0; k < 9; ++k) atomicAdd(&g_tlr2[b][k], (unsigned long long)v[k]);
}
#else
#define PCY_TL(tag) ((void)0)
#endif

// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may be scheduled while its predecessor
// in the stream still runs; pdl_wait() blocks until the predecessor has
// completed and its writes are visible (a no-op for ordinary launches), and
// pdl_launch_dependents() lets the successor's CTAs be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Flag hand-off between two kernels of one stream where the second was
// launched programmatically and is already resident: thread 0 of the CTA polls
// a device word the producer stores after a __threadfence() (relaxed loads at
// L2, then an acquire fence at GPU scope: later loads of this SM do not hit
// stale L1 lines), the CTA then
// meets at a barrier.  The wait for full grid completion (drain, flush, the
// producer's host-mirror writes) is skipped.  After `spins` unsuccessful polls
// the CTA falls back to griddepcontrol.wait, which is always sufficient.
__device__ __forceinline__ long long ld_relaxed_gpu(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void flag_wait(const long long* flag, long long want, int spins = 4096) {
  if (threadIdx.x == 0) {
    bool ok = false;
    for (int it = 0; it < spins; ++it) {
      if (ld_relaxed_gpu(flag) >= want) { ok = true; break; }   // polls at L2; the fence below acquires
      __nanosleep(40);
    }
    if (!ok) asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  __syncthreads();
}
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// cp.async helpers (global -> shared without registers)
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
