/*
 * piecy_b200.h -- C ABI of the B200-native piecy / piecy-mr hot path.
 *
 * The reference (/root/reference/pkg/src/piecy, pure Python + numpy) has no
 * FFI; its "operator API" is the Python surface re-exported by
 * piecy/__init__.py:4-33.  Each entry point below replaces the reference
 * function named in its comment.  The Python package paper_1502_04265_b200
 * binds this header with ctypes (paper_1502_04265_b200/_native.py); any other
 * host language can bind it the same way.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Arrays marked (device) are CUDA device
 *     pointers owned by the caller; (host) are host pointers.
 *   - `stream` is a cudaStream_t passed as void*; every call enqueues on it.
 *   - Return 0 on success or a negative PCY_E* code; pcy_last_error() holds a
 *     thread-local message.  There is no CPU fallback: without a CUDA device
 *     every compute call fails.
 *   - Matrices are row-major, one point per row, fp64 unless stated.
 */
#ifndef PIECY_B200_H
#define PIECY_B200_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PCY_OK = 0, PCY_EINVAL = -1, PCY_ENONFINITE = -2, PCY_EOVERFLOW = -3, PCY_EWEIGHT = -4,
  PCY_ECUDA = -5, PCY_ENOMEM = -6, PCY_ENCCL = -7, PCY_ESTATE = -8
};

const char* pcy_last_error(void);

/* ------------------------------------------------------------ BICO engine */

/* BicoEngine(dim, budget, *, bootstrap_cap=1001) -- coreset.py:223-238.
 * block_rows: rows per device block (<= 0: default 4096). */
int pcy_engine_create(int device, int dim, long long budget, long long bootstrap_cap,
                      long long block_rows, void** engine_out);

/* Frees all device state of the engine. */
int pcy_engine_destroy(void* engine);

/* BicoEngine.insert(point, weight) for n rows in stream order -- coreset.py:264-281.
 * x (device): n rows, row stride `stride` elements, dtype 0 = float64, 1 = float32
 * (upcast exactly, as np.asarray(..., float64) does).  w (device, nullable):
 * int64 weights, NULL = unit.  Validation as the reference: weight < 1 -> code 3,
 * non-finite coordinates -> 1, finite coordinates whose |x|^2 overflows -> 2.
 * Stops at the first invalid row: *consumed = rows absorbed, *bad_code = its code
 * (0 if none); the engine then holds exactly the earlier rows. */
int pcy_engine_insert(void* engine, const void* x, int dtype, long long stride, const long long* w,
                      long long n, void* stream, long long* consumed, int* bad_code);

/* Properties num_features / threshold / total_weight -- coreset.py:240-260.
 * *built = 0 while the engine is still buffering (bootstrap, :283-295). */
int pcy_engine_stats(void* engine, long long* num_features, double* threshold,
                     long long* total_weight, int* built, void* stream);

/* features() -- coreset.py:425-441: DFS pre-order (level, weight, linear sum,
 * square sum, reference); bootstrap form :429-432.  Output arrays (device,
 * each nullable) sized for `cap` features; *count = feature count. */
int pcy_engine_features(void* engine, int* level, long long* weight, double* linear_sum,
                        double* square_sum, double* reference, long long cap, long long* count,
                        void* stream);

/* extract_coreset() -- coreset.py:443-451: points (device, cap x dim) = s / n,
 * weights (device, cap) = n, same order as features(). */
int pcy_engine_extract(void* engine, double* points, long long* weights, long long cap,
                       long long* count, void* stream);

/* Instrumentation of the in-order resolve: out6 (host) = [levels walked,
 * tensor-core near-tie rechecks, demand row loads, full capacity evaluations,
 * items, max depth]. */
int pcy_engine_counters(void* engine, long long* out6);
/* The same counters summed over every engine destroyed so far in the process. */
int pcy_engine_counters_total(long long* out6);

/* K1 work of the engine's chain walks (insertion and rebuild reattach), for
 * the useful-work fraction of SURVEY.md §8d: out4 (host) = [member visits --
 * the reference's own nearest-reference work, one d-length dot per member of
 * every visited group (coreset.py:158-180, :324-329) --, visits served by
 * direct fp64 scans, tensor-pipe flops of the panel contractions (3 TF32
 * products over padded 128x128 tiles), panel launches]. */
int pcy_engine_work(void* engine, double* out4);

/* --------------------------------------------------- clustering on coreset */

/* kmeanspp_seed for `reps` repetitions -- evaluation.py:56-82 with _draw :49-53.
 * P (device, n x d), w (device, n, fp64 > 0), U (device, reps x k): the exact
 * rng.random() draws of each repetition (k per repetition).  centers (device,
 * reps x k x d).  picks_out (host, nullable, reps x k) receives chosen rows. */
int pcy_kmeanspp(const double* P, const double* w, long long n, int d, int k, int reps,
                 const double* U, double* centers, long long* picks_out, void* stream);

/* lloyd_iterate for `reps` center sets in place -- evaluation.py:85-139.
 * cost_log (host, nullable, reps x max_iters) and iters_out (host, reps):
 * the per-iteration costs appended before each stop test. */
int pcy_lloyd(const double* P, const double* w, long long n, int d, int k, int reps, double* centers,
              int max_iters, double tol, double* cost_log, int* iters_out, void* stream);

/* weighted_cost for `reps` center sets -- evaluation.py:142-149; costs (host, reps). */
int pcy_weighted_cost(const double* P, const double* w, long long n, int d, int k, int reps,
                      const double* centers, double* costs, void* stream);

/* The same into device memory without a host sync: costs_dev (device, reps);
 * w (device, nullable = unit weights).  The streaming evaluation
 * (evaluate_cost_multi, evaluation.py:157-180) costs each chunk with it. */
int pcy_weighted_cost_dev(const double* P, const double* w, long long n, int d, int k, int reps,
                          const double* centers, double* costs_dev, void* stream);

/* evaluate_cost_multi block (evaluation.py:157-180): rows P (device, n x d) against
 * one centre set C (device, k x d); out (device) receives the unweighted sum of the
 * first-minimum GEMM-form distances of every `chunk` consecutive rows at
 * out[c * out_stride]. */
int pcy_cost_chunks(const double* P, long long n, int d, const double* C, int k, long long chunk,
                    double* out, long long out_stride, void* stream);

/* ------------------------------------------------------------- projection */

/* randomized_truncated_svd -- linalg.py:167-206, with _fix_signs/_clip_small :77-94.
 * A (device, rows x cols).  omega (device, cols x r) and omega2 (device, r x r,
 * used when rows > 4r) are the reference rng's standard_normal draws.
 * V (device, cols x ell), sigma_host (host, ell). */
int pcy_rsvd(const double* A, long long rows, int cols, int ell, int r, int power, const double* omega,
             const double* omega2, double* V, double* sigma_host, void* stream);

/* project -- linalg.py:209-221: out (device, rows x cols) = (A V) V^T. */
int pcy_project(const double* A, long long rows, int cols, const double* V, int ell, double* out,
                void* stream);

/* weighted_best_fit row scaling -- linalg.py:247: out = A * sqrt(w)[:, None]. */
int pcy_scale_rows_sqrtw(const double* A, const long long* w, long long rows, int cols, double* out,
                         void* stream);

/* Plain fp64 GEMM (cuBLAS): C = alpha op(A) op(B) + beta C (row-major). */
int pcy_dgemm(int M, int N, int K, double alpha, const double* A, long long lda, int ta,
              const double* B, long long ldb, int tb, double beta, double* C, long long ldc,
              void* stream);

/* Exact upcasts and the as_matrix finiteness check (linalg.py:26-35). */
int pcy_cast_f32_f64(const float* src, long long n, double* dst, void* stream);
int pcy_cast_i64_f64(const long long* src, long long n, double* dst, void* stream);
int pcy_all_finite(const void* p, long long n, int dtype, int* out_host, void* stream);

/* --------------------------------------------- distance contraction (test) */

/* Split-TF32 (3xTF32) dots on tcgen05: out (device, M x N fp32) ~= (A_m - c).(B_n - c)
 * with c = A_0, A/B (device) fp64 rows of dimension d.  *tau_out (host) = the
 * rigorous relative error factor: |out - exact| <= tau |A_m - c| |B_n - c|.
 * This is the contraction of the full-set nearest-reference search
 * (coreset.py:318-330) that the engine runs for d >= 256. */
int pcy_tc_dots_f64(const double* A, long long lda, int M, const double* B, long long ldb, int N, int d,
                    float* out, double* tau_out, void* stream);

/* -------------------------------------------------------- instrumentation */
long long pcy_launch_count(void);
int pcy_prof_enable(int on);
int pcy_prof_reset(void);
int pcy_prof_read(int slot, double* ms, long long* count, long long* units);

/* ------------------------------------------------------- paper generators */

/* structured_with_noise -- datagen.py:104-112.  Rows (device, out, clusters*ppc
 * x dim, leading dim ld) from numpy's Philox4x64-10 stream with key
 * (key_lo, key_hi): base (device, clusters) = global draw index of each
 * cluster's first point, inv (device, clusters x dim) = position of each dim
 * in the cluster's active list or -1 (the permutation stays on the host). */
int pcy_gen_swn(double* out, long long ld, int clusters, long long ppc, int dim, int active_dims,
                unsigned long long key_lo, unsigned long long key_hi, const unsigned long long* base,
                const int* inv, double noise, double spread, void* stream);

/* random_cube -- datagen.py:131-135: n x cols uniforms in [-spread, spread]
 * from draw `start` of the Philox stream. */
int pcy_gen_cube(double* out, long long ld, long long n, long long cols, unsigned long long key_lo,
                 unsigned long long key_hi, unsigned long long start, double spread, void* stream);

/* lower_bound -- datagen.py:115-128 (deterministic nested simplices). */
int pcy_gen_lower_bound(double* out, long long ld, int k, long long n, double spread, double noise, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PIECY_B200_H */
