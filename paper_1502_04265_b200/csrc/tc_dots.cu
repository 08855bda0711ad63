// Approximate distance contraction on the 5th-generation tensor cores.
//
// The BICO nearest-reference search (coreset.py:318-330: argmin over a
// group's members of |r|^2 - 2 r.x) is a GEMM of the block's points against
// the allocated reference slots.  Here it runs as split-TF32 ("3xTF32") on
// tcgen05:
//   x = hi + lo with hi = tf32(x - c), lo = tf32((x - c) - hi)   (k_tc_split)
//   D = Ahi Bhi^T + Ahi Blo^T + Alo Bhi^T                          (k_tc_dots)
// accumulated in fp32 in TMEM, operands fed by TMA (SWIZZLE_128B, K-major),
// one elected thread issuing tcgen05.mma.kind::tf32.  c is a per-launch
// centre (parts are shift-covariant: |r-c|^2 - 2(r-c).(x-c) = part + f(x),
// so the argmin is unchanged and the error bound shrinks with |x-c||r-c|).
//
// The products are fp32-faithful, not exact: the chain walk (K1) takes the
// members whose approximate part lies within the rigorous error window of the
// minimum and re-decides them with exact fp64 dots (tc_error_tau below), so
// the decisions equal the fp64 ones -- the "near-tie recheck".
#include "common.cuh"
#include <cuda.h>
#include <mutex>

namespace {

constexpr int TBM = 128, TBN = 128, TBK = 32, TSTAGES = 3;
constexpr int TILE_BYTES = TBM * TBK * 4;            // 16 KB: one operand tile (hi or lo)
constexpr int STAGE_BYTES = 4 * TILE_BYTES;          // Ahi, Alo, Bhi, Blo
constexpr int TC_SMEM = TSTAGES * STAGE_BYTES + 1024 + 256;
// K is split into up to TC_NACC consecutive chunks, each accumulated in its own
// 128-column TMEM accumulator (4 x 128 = all 512 columns); the epilogue adds
// the chunk sums in fp64.  Fewer fp32 accumulation steps per sum tighten the
// rigorous error bound (pcy_tc_error_tau) and so the near-tie window.
constexpr int TC_NACC = 4;
__host__ __device__ inline int tc_nacc(int nk) { return nk < TC_NACC ? nk : TC_NACC; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "TC_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra TC_DONE;\n\t"
      "bra TC_WAIT;\n"
      "TC_DONE:\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"((uint64_t)map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// K-major operand tile, 128 B rows, SWIZZLE_128B: 8-row atoms of 1024 B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// D[m][n] ~= sum_k A[m][k] B[n][k] (3xTF32).  Grid: (ceil(N/128), ceil(M/128)).
// Out: fp32 dots, row-major with leading dim ldo.
__global__ void __launch_bounds__(128, 1) k_tc_dots(const __grid_constant__ CUtensorMap mAhi,
                                                    const __grid_constant__ CUtensorMap mAlo,
                                                    const __grid_constant__ CUtensorMap mBhi,
                                                    const __grid_constant__ CUtensorMap mBlo, int M, int N, int Kp,
                                                    float* __restrict__ out, long long ldo,
                                                    const int* __restrict__ n_dev) {
  extern __shared__ __align__(1024) uint8_t tc_smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)tc_smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* full = (uint64_t*)(smem + TSTAGES * STAGE_BYTES);
  uint64_t* empty = full + TSTAGES;
  uint64_t* accum_full = empty + TSTAGES;
  uint32_t* tmem_slot = (uint32_t*)(accum_full + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // row tiles fastest: the CTAs sharing a B panel run together (one HBM read of B)
  const int m0 = blockIdx.x * TBM, n0 = blockIdx.y * TBN;
  const int nk = Kp / TBK;
  if (n_dev) { N = min(N, *n_dev); if (n0 >= N) return; }

  if (threadIdx.x == 0) {
    for (int s = 0; s < TSTAGES; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, 1); }
    mbar_init(accum_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mAhi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&mBhi) : "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % TSTAGES;
      mbar_wait(empty + s, ((kb / TSTAGES) & 1) ^ 1);
      uint8_t* st = smem + s * STAGE_BYTES;
      mbar_expect_tx(full + s, STAGE_BYTES);
      const int k0 = kb * TBK;
      tma_load_2d(st, &mAhi, full + s, k0, m0);
      tma_load_2d(st + TILE_BYTES, &mAlo, full + s, k0, m0);
      tma_load_2d(st + 2 * TILE_BYTES, &mBhi, full + s, k0, n0);
      tma_load_2d(st + 3 * TILE_BYTES, &mBlo, full + s, k0, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer: M=128, N=128, K=8 per instruction, fp32 accumulate
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TBN >> 3) << 17) |
                           ((uint32_t)(TBM >> 4) << 24);
    const int nacc = tc_nacc(nk);
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % TSTAGES;
      mbar_wait(full + s, (kb / TSTAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a_hi = smem_u32(smem + s * STAGE_BYTES);
      const uint32_t a_lo = a_hi + TILE_BYTES, b_hi = a_hi + 2 * TILE_BYTES, b_lo = a_hi + 3 * TILE_BYTES;
      const int ac = (kb * nacc) / nk;                                  // this stage's K chunk
      const bool first = kb == 0 || ((kb - 1) * nacc) / nk != ac;      // first stage of the chunk
      const uint32_t dcol = tmem + (uint32_t)(ac * TBN);
#pragma unroll
      for (int ks = 0; ks < TBK / 8; ++ks) {
        const uint32_t off = ks * 32;   // 8 tf32 = 32 B along K inside the swizzle atom
        const uint32_t acc0 = (first && ks == 0) ? 0u : 1u;
        mma_tf32(dcol, sw128_desc(a_hi + off), sw128_desc(b_hi + off), idesc, acc0);
        mma_tf32(dcol, sw128_desc(a_hi + off), sw128_desc(b_lo + off), idesc, 1u);
        mma_tf32(dcol, sw128_desc(a_lo + off), sw128_desc(b_hi + off), idesc, 1u);
      }
      mma_commit(empty + s);   // frees the stage when these MMAs complete
    }
    mma_commit(accum_full);
  }
  __syncwarp();

  // epilogue: thread t <-> TMEM lane t <-> tile row t
  mbar_wait(accum_full, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;
  const long long gm = m0 + row;
  const int nacc = tc_nacc(nk);
  for (int c0 = 0; c0 < TBN; c0 += 32) {
    double acc[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = 0.0;
    for (int ac = 0; ac < nacc; ++ac) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(ac * TBN + c0);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 32; ++q) acc[q] += (double)__uint_as_float(v[q]);   // chunk order, fp64
    }
    if (gm < M) {
      float* o = out + gm * ldo + n0 + c0;
      if (n0 + c0 + 32 <= N && ((ldo & 3) == 0)) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          reinterpret_cast<float4*>(o)[q] = make_float4((float)acc[4 * q], (float)acc[4 * q + 1], (float)acc[4 * q + 2],
                                                        (float)acc[4 * q + 3]);
      } else {
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (n0 + c0 + q < N) o[q] = (float)acc[q];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// One warp per row: hi/lo TF32 split of (row - c), zero padded to Kp, and the
// centred squared norm |row - c|^2 (fp64, fixed lane-strided order).
__global__ void k_tc_split(const double* __restrict__ src, const int* __restrict__ idx, long long ld, int d,
                           long long rows, const int* __restrict__ rows_dev, const double* __restrict__ center,
                           int Kp, float* __restrict__ hi, float* __restrict__ lo, double* __restrict__ nrm2) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= rows || (rows_dev && i >= *rows_dev)) return;
  const double* x = src + (long long)(idx ? idx[i] : i) * ld;
  float* h = hi + i * Kp;
  float* l = lo + i * Kp;
  double acc = 0.0;
  for (int k = lane; k < Kp; k += 32) {
    const double v = k < d ? x[k] - center[k] : 0.0;
    const float vh = to_tf32((float)v);
    const float vl = to_tf32((float)(v - (double)vh));
    h[k] = vh;
    l[k] = vl;
    acc = fma(v, v, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0 && nrm2) nrm2[i] = acc;
}

// Reference slots, split in place (row = slot) once per reference: a slot is
// re-split when it is alive and its creation index differs from the one it
// was split for (references never change while a node lives, coreset.py:193).
__global__ void k_tc_split_slots(const double* __restrict__ src, long long ld, int d, long long nslots,
                                 const int* __restrict__ alive, const long long* __restrict__ cidx,
                                 long long* __restrict__ done_idx, const double* __restrict__ center, int Kp,
                                 float* __restrict__ hi, float* __restrict__ lo, double* __restrict__ nrm2,
                                 int* __restrict__ col_of, int* __restrict__ col_slot, int* __restrict__ ncol) {
  const int lane = threadIdx.x & 31;
  const long long i = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= nslots || !alive[i] || done_idx[i] == cidx[i]) return;
  int c = 0;
  if (lane == 0) c = atomicAdd(ncol, 1);   // column order is free: a dot does not depend on its column
  c = __shfl_sync(PCY_FULL, c, 0);
  const double* x = src + i * ld;
  float* h = hi + (long long)c * Kp;
  float* l = lo + (long long)c * Kp;
  double acc = 0.0;
  for (int k = lane; k < Kp; k += 32) {
    const double v = k < d ? x[k] - center[k] : 0.0;
    const float vh = to_tf32((float)v);
    const float vl = to_tf32((float)(v - (double)vh));
    h[k] = vh;
    l[k] = vl;
    acc = fma(v, v, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) { nrm2[i] = acc; done_idx[i] = cidx[i]; col_of[i] = c; col_slot[c] = (int)i; }
}

__global__ void k_copy_row(const double* __restrict__ src, const int* __restrict__ idx, long long ld, int d,
                           double* __restrict__ dst) {
  for (int k = threadIdx.x; k < d; k += blockDim.x) dst[k] = src[(long long)(idx ? idx[0] : 0) * ld + k];
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

int make_map(CUtensorMap* map, const float* base, long long rows, int Kp) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) { pcy_set_error("cuTensorMapEncodeTiled unavailable"); return PCY_ECUDA; }
  const cuuint64_t dims[2] = {(cuuint64_t)Kp, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)Kp * 4};
  const cuuint32_t box[2] = {(cuuint32_t)TBK, (cuuint32_t)TBM};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { pcy_set_error("cuTensorMapEncodeTiled failed (%d)", (int)r); return PCY_ECUDA; }
  return PCY_OK;
}

}  // namespace

// Rigorous bound on |approx - exact| of a 3xTF32 dot over Kp (padded) terms,
// relative to |a - c| |b - c|: split residues (<= 3 * 2^-22 per term); per K
// chunk one fp32 rounding (<= 2^-23 of the chunk's running magnitude, at most
// the chunk's sum of |terms|) per accumulation step: 3 products x Kc/8 MMAs
// and <= 4 steps inside each 8-term MMA.  The chunk sums are added in fp64 and
// their |terms| sums add up to <= |a-c||b-c| (1 + 2^-10) by Cauchy-Schwarz;
// the fp32 output adds 2^-24 of |dot| <= |a-c||b-c|.
double pcy_tc_error_tau(int Kp) {
  const int nk = Kp / TBK;
  const int nacc = tc_nacc(nk > 0 ? nk : 1);
  const int kc = ((nk + nacc - 1) / nacc) * TBK;   // longest chunk
  const double steps = 3.0 * (kc / 8.0) * 5.0 + 8.0;
  return (steps * 0x1p-23 + 3.0 * 0x1p-22 + 0x1p-24 + 8.0 * 0x1p-53) * (1.0 + 0x1p-9);
}

int pcy_tc_pad(int d) { return (d + TBK - 1) / TBK * TBK; }

// Split rows (optionally gathered through idx) into TF32 hi/lo operands.
// center (device, d): the launch centre.  nrm2 (device, nullable) receives
// |row - c|^2.
int pcy_tc_split(const double* src, const int* idx, long long ld, int d, long long rows, const int* rows_dev,
                 const double* center, float* hi, float* lo, double* nrm2, cudaStream_t st) {
  if (rows <= 0) return PCY_OK;
  const int Kp = pcy_tc_pad(d);
  k_tc_split<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(src, idx, ld, d, rows, rows_dev, center, Kp, hi, lo, nrm2);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

int pcy_tc_split_slots(const double* src, long long ld, int d, long long nslots, const int* alive,
                       const long long* cidx, long long* done_idx, const double* center, float* hi, float* lo,
                       double* nrm2, int* col_of, int* col_slot, int* ncol, cudaStream_t st) {
  if (nslots <= 0) return PCY_OK;
  const int Kp = pcy_tc_pad(d);
  k_tc_split_slots<<<(unsigned)((nslots + 7) / 8), 256, 0, st>>>(src, ld, d, nslots, alive, cidx, done_idx, center, Kp,
                                                                 hi, lo, nrm2, col_of, col_slot, ncol);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

int pcy_tc_center(const double* src, const int* idx, long long ld, int d, double* center, cudaStream_t st) {
  k_copy_row<<<1, 256, 0, st>>>(src, idx, ld, d, center);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

// out[m][n] ~= (A[m]-c).(B[n]-c) for the split operands (row capacities
// a_cap / b_cap rows of Kp floats, Kp a multiple of 32).
int pcy_tc_dots(const float* Ahi, const float* Alo, long long a_cap, int M, const float* Bhi, const float* Blo,
                long long b_cap, int N, const int* n_dev, int Kp, float* out, long long ldo, cudaStream_t st) {
  if (M <= 0 || N <= 0) return PCY_OK;
  static std::once_flag attr;
  std::call_once(attr, [] { cudaFuncSetAttribute(k_tc_dots, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM); });
  CUtensorMap ma, mal, mb, mbl;
  int rc;
  if ((rc = make_map(&ma, Ahi, a_cap, Kp)) || (rc = make_map(&mal, Alo, a_cap, Kp)) ||
      (rc = make_map(&mb, Bhi, b_cap, Kp)) || (rc = make_map(&mbl, Blo, b_cap, Kp)))
    return rc;
  dim3 grid((unsigned)((M + TBM - 1) / TBM), (unsigned)((N + TBN - 1) / TBN));
  k_tc_dots<<<grid, 128, TC_SMEM, st>>>(ma, mal, mb, mbl, M, N, Kp, out, ldo, n_dev);
  pcy_count_launch();
  PCY_LAUNCH_CHECK();
  return PCY_OK;
}

// Test entry: approximate dots of two fp64 row sets (centre = A's first row),
// for the parity test of the tensor-core contraction against fp64.
extern "C" int pcy_tc_dots_f64(const double* A, long long lda, int M, const double* B, long long ldb, int N, int d,
                               float* out, double* tau_out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int Kp = pcy_tc_pad(d);
  const long long ac = ((M + TBM - 1) / TBM) * TBM, bc = ((N + TBN - 1) / TBN) * TBN;
  float *ah, *al, *bh, *bl;
  double* c;
  PCY_CUDA(pcy_malloc_async(&ah, sizeof(float) * ac * Kp, st));
  PCY_CUDA(pcy_malloc_async(&al, sizeof(float) * ac * Kp, st));
  PCY_CUDA(pcy_malloc_async(&bh, sizeof(float) * bc * Kp, st));
  PCY_CUDA(pcy_malloc_async(&bl, sizeof(float) * bc * Kp, st));
  PCY_CUDA(pcy_malloc_async(&c, sizeof(double) * Kp, st));
  PCY_CUDA(cudaMemsetAsync(ah, 0, sizeof(float) * ac * Kp, st));
  PCY_CUDA(cudaMemsetAsync(al, 0, sizeof(float) * ac * Kp, st));
  PCY_CUDA(cudaMemsetAsync(bh, 0, sizeof(float) * bc * Kp, st));
  PCY_CUDA(cudaMemsetAsync(bl, 0, sizeof(float) * bc * Kp, st));
  int rc = pcy_tc_center(A, nullptr, lda, d, c, st);
  if (!rc) rc = pcy_tc_split(A, nullptr, lda, d, M, nullptr, c, ah, al, nullptr, st);
  if (!rc) rc = pcy_tc_split(B, nullptr, ldb, d, N, nullptr, c, bh, bl, nullptr, st);
  if (!rc) rc = pcy_tc_dots(ah, al, ac, M, bh, bl, bc, N, nullptr, Kp, out, N, st);
  cudaFreeAsync(ah, st); cudaFreeAsync(al, st); cudaFreeAsync(bh, st); cudaFreeAsync(bl, st); cudaFreeAsync(c, st);
  if (tau_out) *tau_out = pcy_tc_error_tau(Kp);
  return rc;
}
