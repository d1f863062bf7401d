/*
 * rbc.h -- C ABI of the B200-native randomized bilinear-computation (BC)
 * matrix-multiply engine (librbc.so).
 *
 * Drop-in boundary.  The reference (`randbc`, pure Python/numpy) funnels every
 * multiply through two engine functions that its L2 callers resolve by module
 * attribute at call time:
 *
 *   randbc._engine.apply_levels(levels, a, b, mode, stats=None)
 *       -- reference pkg/src/randbc/_engine.py:117-149
 *   randbc._engine.leaf_matmul(x, y, mode)
 *       -- reference pkg/src/randbc/_engine.py:42-61
 *
 * rbc_apply_levels / rbc_leaf_matmul are exactly those two calls over plain
 * pointers (host buffers, synchronous, GIL-free under ctypes).  The Python
 * binding paper_1905_07439_b200.engine exposes them with the reference's
 * signatures and installs them into randbc._engine.
 *
 * Everything else is an accelerator-side extension:
 *   - *_async twins take device pointers and a cudaStream_t and never
 *     synchronise (throughput path, CUDA-graph capturable);
 *   - the plan path (rbc_apply_plans*) evaluates exact +-1 formulas straight
 *     from the randomization plans (reference randomize.py:163-178 hatted
 *     tensors, folded into the kernels);
 *   - rbc_truth_async / rbc_rel_errors_async are the binary64 ground truth and
 *     relative Frobenius error of experiments.py:251-261.
 *
 * Layouts are the reference's, C-contiguous:
 *   operands a, b : (T0, N, N)        T0 in {1, T}
 *   level q u/v/w : (Tc_q, R_q, n_q, n_q)  Tc_q in {1, T}, levels[0] splits A
 *   result        : (T, N, N)
 * dtype codes: RBC_F64 (binary64), RBC_F32 (binary32), RBC_F16 (binary16).
 *
 * Arithmetic contract: every output element follows the reference's rounding
 * sequence (one IEEE RNE rounding per multiply and per add, fixed fold orders),
 * so results are bitwise equal in value to the reference's.
 *
 * Status codes map to the reference's exceptions:
 *   RBC_EVALUE       -> ValueError        (shapes, empty level list, ...)
 *   RBC_EOVERFLOW    -> OverflowError     (non-finite result, _engine.py:147-148)
 *   RBC_ERUNTIME     -> RuntimeError      (CUDA failure)
 *   RBC_EUNSUPPORTED -> NotImplementedError
 * rbc_last_error() returns the message of the calling thread's last failure.
 */
#ifndef RBC_H_
#define RBC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RBC_ABI_VERSION 1

#define RBC_F64 0
#define RBC_F32 1
#define RBC_F16 2

#define RBC_FORMULA_STRASSEN 1  /* reference formula.py:98-114           */
#define RBC_FORMULA_LADERMAN 2  /* formulas/laderman.txt    */
#define RBC_FORMULA_STANDARD2 3 /* reference formula.py:117-137, n = 2    */
#define RBC_FORMULA_STANDARD3 4 /* reference formula.py:117-137, n = 3    */

#define RBC_OK 0
#define RBC_EVALUE 1
#define RBC_EOVERFLOW 2
#define RBC_ERUNTIME 3
#define RBC_EUNSUPPORTED 4

/* Bytes of one packed plan level (see rbc_pack_plans). */
#define RBC_PLAN_BYTES 40

int rbc_abi_version(void);
const char* rbc_last_error(void);
int rbc_device_count(void);

/* Give back the device memory the host-buffer calls keep between calls (one
 * arena per process, grown to the largest call) and the unused part of the
 * stream-ordered scratch pool.  Synchronises the device.  The next host-buffer
 * call allocates again.  For processes that alternate host-buffer calls with
 * device-resident pipelines of their own (rbc_*_async) on a full GPU. */
int rbc_release_device_memory(void);

/* Stage profiler: when enabled, every engine launch is bracketed by CUDA
 * events on its own stream and tagged with its algorithmic bytes and flops.
 * rbc_profile_summary synchronises the recorded events and writes a JSON
 * object {stage: {count, ms, bytes, flops}}; returns the length needed. */
void rbc_profile_enable(int on);
int64_t rbc_profile_summary(char* buf, size_t len);

/* ---- reference engine boundary (host buffers, synchronous) --------------- */

/* randbc._engine.apply_levels  (_engine.py:117-149).
 * n[q], R[q], Tc[q]: level shapes; u[q], v[q], w[q]: host coefficient tables.
 * T must equal max(T0, Tc[*]).  leaf_multiplies (optional) += T * prod(R). */
int rbc_apply_levels(int dtype, int Q, const int32_t* n, const int32_t* R, const int64_t* Tc,
                     const void* const* u, const void* const* v, const void* const* w,
                     int64_t T0, int64_t N, const void* a, const void* b, int64_t T, void* out,
                     uint64_t* leaf_multiplies);

/* randbc._engine.leaf_matmul  (_engine.py:42-61), batched x (.., M, K) @ y (.., K, N);
 * x_bstride / y_bstride are 0 (broadcast) or M*K / K*N. */
int rbc_leaf_matmul(int dtype, int64_t batch, int64_t x_bstride, int64_t y_bstride, int64_t M,
                    int64_t K, int64_t N, const void* x, const void* y, void* out);

/* ---- plan path (exact +-1 formulas) -------------------------------------- */

/* Pack `count` plan levels (reference RandomizationPlan: perms (3, n) int64,
 * signs (3, n) binary64 in {-1, +1}) into RBC_PLAN_BYTES-byte device records.
 * Returns RBC_EVALUE for n > 4 or entries that are not a signed permutation. */
int rbc_pack_plans(int n, int64_t count, const int64_t* perms, const double* signs, void* packed);

/* Q-level evaluation of an exact formula under per-trial plans
 * packed_plans: (Tp, Q) packed levels, Tp in {1, T}, level 0 outermost.
 * nonfinite (optional, T bytes) receives per-trial overflow flags; the call
 * returns RBC_EOVERFLOW when any is set. */
int rbc_apply_plans(int dtype, int formula, int Q, int64_t Tp, const void* packed_plans,
                    int64_t T0, int64_t N, const void* a, const void* b, int64_t T, void* out,
                    uint8_t* nonfinite, uint64_t* leaf_multiplies);

/* ---- diagonal rescaling baseline (reference rescale.py:60-99) -----------
 * randbc.rescale.rescaled_multiply(A, B, Q, schedule, mode, formula) on the
 * device: steps[i] = 0 (outside) or 1 (inside); the abs-max, reciprocal,
 * square-root and diagonal-scaling steps run as kernels in the mode with the
 * reference's roundings, then the deterministic recursion (formula > 0: an
 * exact +-1 formula id; formula = 0: dense tables u/v/w[q] (R[q], n[q], n[q])
 * in the mode), then the restores.  Host buffers (N x N), synchronous.
 * RBC_EVALUE "degenerate input: zero row|column maximum" (rescale.py:36-41);
 * RBC_EOVERFLOW when the recursion's result is non-finite (_engine.py:146). */
int rbc_rescaled_multiply(int dtype, int formula, int Q, const int32_t* n, const int32_t* R,
                          const void* const* u, const void* const* v, const void* const* w,
                          int nsteps, const int32_t* steps, int64_t N, const void* a,
                          const void* b, void* out);

/* experiments._rel_errors (reference experiments.py:258-261) on host buffers:
 * err[t] = ||widen(c[t]) - ref[t or 0]||_F / ||ref[t or 0]||_F in binary64;
 * c: (T, N, N) in the mode, ref: (N, N) (ref_tstride 0) or (T, N, N) binary64.
 * Copies H2D, reduces on the device, copies the T errors back. */
int rbc_rel_errors(int dtype, int64_t T, int64_t N, const void* c, const double* ref,
                   int64_t ref_tstride, double* err);

/* ---- device-pointer twins (stream ordered, no synchronisation) ------------ */

size_t rbc_levels_workspace_bytes(int dtype, int Q, const int32_t* n, const int32_t* R,
                                  int64_t T, int64_t N);
int rbc_apply_levels_async(int dtype, int Q, const int32_t* n, const int32_t* R,
                           const int64_t* Tc, const void* const* u, const void* const* v,
                           const void* const* w, int64_t T0, int64_t N, const void* a,
                           const void* b, int64_t T, void* out, uint8_t* nonfinite,
                           void* workspace, size_t workspace_bytes, void* stream);

size_t rbc_plans_workspace_bytes(int dtype, int formula, int Q, int64_t T, int64_t N);
int rbc_apply_plans_async(int dtype, int formula, int Q, int64_t Tp, const void* packed_plans,
                          int64_t T0, int64_t N, const void* a, const void* b, int64_t T,
                          void* out, uint8_t* nonfinite, void* workspace, size_t workspace_bytes,
                          void* stream);

int rbc_leaf_matmul_async(int dtype_in, int dtype_out, int64_t batch, int64_t x_bstride,
                          int64_t y_bstride, int64_t M, int64_t K, int64_t N, const void* x,
                          const void* y, void* out, void* stream);

/* ---- error check (experiments.py:251-261) -------------------------------- */

/* ref[t] = standard_multiply(widen(a[t]), widen(b[t]), DOUBLE): the binary64
 * inner-product product of the mode-rounded operands, k ascending. */
int rbc_truth_async(int dtype_in, int64_t T, int64_t N, const void* a, const void* b,
                    double* ref, void* stream);

size_t rbc_rel_errors_scratch_bytes(int64_t T);
/* err[t] = ||widen(c[t]) - ref[t * ref_tstride/N^2]||_F / ||ref[..]||_F, ref_tstride in {0, N*N}. */
int rbc_rel_errors_async(int dtype, int64_t T, int64_t N, const void* c, const double* ref,
                         int64_t ref_tstride, double* err, void* scratch, void* stream);

/* total[e] = fl(...fl(total[e] + x[0][e]) ... + x[T-1][e]) in binary64, trials in
 * order: the sequential average accumulation of enumerate_expectation
 * (randomize.py:317-326) and the averaging experiments (experiments.py:382-383). */
int rbc_sum_trials_async(int dtype, int64_t T, int64_t N, const void* x, double* total,
                         void* stream);

/* nonfinite[t] = 1 if x[t] (N*N elements) holds a non-finite value. */
int rbc_nonfinite_async(int dtype, int64_t T, int64_t N, const void* x, uint8_t* nonfinite,
                        void* stream);

/* ---- seeded test matrices on the device -------------
 * Reference matgen.generate (pkg/src/randbc/matgen.py:55-97) over derive_rng
 * (rng.py:20-23): out[c] (n x n, dtype, device) is bit-identical to the
 * host draw of matrix `which[c]` (0 = A from derive_rng(mseed, 0), 1 = B from
 * derive_rng(mseed, 1)) rounded into the mode, given the Philox key of that
 * stream (keys[2c], keys[2c+1] = Philox(SeedSequence(..)).state key, host
 * array).  kind: RBC_MAT_* (reference MATRIX_KINDS order, then the builder
 * kinds).  nonfinite (device, optional, count bytes) gets 1 where the
 * rounding into the mode overflowed (ScalarMode.array raises OverflowError).
 * Synchronises `stream` (the ziggurat tail is evaluated on the host with the
 * C library's log1p, as numpy does).  count <= 65535. */
#define RBC_MAT_GAUSSIAN 0
#define RBC_MAT_UNIFORM 1
#define RBC_MAT_ADV1 2
#define RBC_MAT_ADV2 3
#define RBC_MAT_ADV3 4
#define RBC_MAT_HILBERT 5
#define RBC_MAT_UNIFORM_PM1 6
#define RBC_MAT_QUADRANT100 7
int rbc_matgen(int kind, int dtype, int64_t count, int64_t n, const uint64_t* keys,
               const int32_t* which, void* out, uint8_t* nonfinite, void* stream);

/* ---- host seed derivation and plan draws (reference rng.py:20-29,
 * randomize.py:118-127), numpy's SeedSequence / Philox4x64-10 / bounded-
 * integer / shuffle algorithms restated in C++ (csrc/hostrng.cu), bit for bit.
 * Stream i = derive_rng(seeds[i * seed_stride], *paths[i]) (seed_stride 0:
 * one seed for all), paths: (count, depth) u64 spawn keys.
 *   rbc_derive_seeds : out[i] = derive_seed(seed_i, *paths[i])
 *   rbc_philox_keys  : keys[2i], keys[2i+1] = that stream's Philox key
 *                      (the rbc_matgen input)
 *   rbc_draw_plans   : perms (count, 3, n) int64 and signs (count, 3, n) f64 of
 *                      draw_plan(n, derive_rng(seed_i, *paths[i]))
 * Host only (no device needed); multithreaded for large counts. */
int rbc_derive_seeds(const uint64_t* seeds, int64_t seed_stride, int depth,
                     const uint64_t* paths, int64_t count, uint64_t* out);
int rbc_philox_keys(const uint64_t* seeds, int64_t seed_stride, int depth, const uint64_t* paths,
                    int64_t count, uint64_t* keys);
int rbc_draw_plans(int n, const uint64_t* seeds, int64_t seed_stride, int depth,
                   const uint64_t* paths, int64_t count, int64_t* perms, double* signs);

/* ---- error trials: the per-pair work of the distribution experiments ----
 * (experiments.py:248-261, 327-379): for each trial t with operands
 * (a[t], b[t]) in the mode, ref_t = binary64 inner-product truth, then the
 * randomized product under rand_plans[t] (packed (T, Q)) and/or the
 * deterministic product (identity plans), each with its relative Frobenius
 * error against ref_t and a per-trial non-finite flag.
 * Host variant: host buffers in/out, H2D/D2H inside the call. */
int rbc_error_trials(int dtype, int formula, int Q, int64_t T, int64_t N, const void* a,
                     const void* b, const void* rand_plans, int with_det, double* err_rand,
                     double* err_det, uint8_t* nonfinite_rand, uint8_t* nonfinite_det);

/* The same call in two halves, so that consecutive calls overlap: _begin
 * enqueues the copies, kernels and result copies of one call and returns a
 * ticket; _end(ticket) waits for them and reports failures.  At most two
 * calls are in flight.  With a second call begun before the first is ended,
 * its operands are copied while the first call still computes (one call alone
 * leaves the GPU idle during its first copy).  All host buffers of a call
 * (operands, plans, results; pinned for the copies to be asynchronous) must
 * stay valid and untouched until its _end.  Calls of one shape share a device
 * layout; a call of another shape, and every other host-buffer entry point of
 * this library, first waits for the calls in flight.  rbc_error_trials is
 * _begin followed by _end. */
int rbc_error_trials_begin(int dtype, int formula, int Q, int64_t T, int64_t N, const void* a,
                           const void* b, const void* rand_plans, int with_det, double* err_rand,
                           double* err_det, uint8_t* nf_rand, uint8_t* nf_det, int64_t* ticket);
int rbc_error_trials_end(int64_t ticket);

size_t rbc_error_trials_workspace_bytes(int dtype, int formula, int Q, int64_t T, int64_t N);

/* ---- averaging trials (experiments.py:264-296; BASELINE config 3) --------
 * For each of P operand pairs (a[p], b[p]): the binary64 truth, optionally
 * the deterministic product from det_u/v/w (Tc = 1 tables per level), and G
 * randomized products from u/v/w (per level (P*G, R, n, n) hatted tables; pair
 * p owns trials p*G .. p*G+G-1).  Outputs: per-plan errors err_rand (P*G),
 * running binary64 mean errors err_mean (P * ncheck) at the ascending
 * checkpoints (1..G; total_i = fl(total_{i-1} + C_i), error of fl(total_i / i)),
 * deterministic errors err_det (P).  Device pointers, stream ordered. */
size_t rbc_average_trials_workspace_bytes(int dtype, int Q, const int32_t* n, const int32_t* R,
                                          int64_t G, int64_t N);
int rbc_average_trials_async(int dtype, int Q, const int32_t* n, const int32_t* R, int64_t P,
                             int64_t G, int64_t N, const void* a, const void* b,
                             const void* const* u, const void* const* v, const void* const* w,
                             const void* const* det_u, const void* const* det_v,
                             const void* const* det_w, int ncheck, const int32_t* checkpoints,
                             double* err_rand, double* err_mean, double* err_det,
                             uint8_t* nonfinite_rand, uint8_t* nonfinite_det, void* workspace,
                             size_t workspace_bytes, void* stream);
/* Device variant: det_plans is a device (1, Q) identity table or NULL. */
int rbc_error_trials_async(int dtype, int formula, int Q, int64_t T, int64_t N, const void* a,
                           const void* b, const void* rand_plans, const void* det_plans,
                           double* err_rand, double* err_det, uint8_t* nonfinite_rand,
                           uint8_t* nonfinite_det, void* workspace, size_t workspace_bytes,
                           void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RBC_H_ */
