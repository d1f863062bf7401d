// Internal host-side launch interface of the B200 BC engine (not part of the
// C-ABI; see include/rbc.h for that).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "common.cuh"
#include "rbc.h"

namespace rbc {

enum Dtype : int { kF64 = 0, kF32 = 1, kF16 = 2 };

inline size_t dtype_size(int dt) { return dt == kF64 ? 8 : dt == kF32 ? 4 : 2; }

// Records a CUDA failure as the thread's last error; returns RBC_ERUNTIME.
int fail_cuda(cudaError_t e, const char* expr, const char* file, int line);

#ifndef CUDA_TRY
#define CUDA_TRY(expr)                                                      \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) return fail_cuda(_e, #expr, __FILE__, __LINE__); \
  } while (0)
#endif

// ---- stage profiler (rbc_profile_enable) ------------------------------------
// When enabled, Stage records a CUDA event pair around a launch on its stream,
// tagged with the launch's algorithmic bytes and flops.
bool prof_on();
void prof_record(cudaStream_t st, const char* name, double bytes, double flops, bool start);
struct Stage {
  cudaStream_t st;
  const char* name;
  double bytes, flops;
  Stage(cudaStream_t s, const char* n, double b, double f) : st(s), name(n), bytes(b), flops(f) {
    if (prof_on()) prof_record(st, name, bytes, flops, true);
  }
  ~Stage() {
    if (prof_on()) prof_record(st, name, bytes, flops, false);
  }
};

// Largest vector width (elements per thread) that divides the block side.
int pick_width(int dtype, int64_t mb, int cap_elems);

// ---- plan path: exact +-1 formulas, per-trial signed permutations ---------
// Expansion of one level for operand A (which == 0: rows by perm 1, cols by
// perm 2) or B (which == 1: rows by perm 2, cols by perm 3).
//   x    : (T or 1, K, s, s)   x_tstride = K*s*s or 0 (broadcast)
//   out  : (T, K*R, s/n, s/n)
//   plans: PlanLevel[(t * plan_tstride) + level]; plan_tstride = Q or 0
cudaError_t launch_expand_plan(int dtype, int formula, int which, const void* x,
                               int64_t x_tstride, int64_t K, int64_t s, void* out,
                               const PlanLevel* plans, int64_t plan_tstride, int level,
                               int64_t T, cudaStream_t st);

// Contraction of one level: ch (T, K, R, mb, mb) -> out (T, K, n*mb, n*mb).
// nonfinite (optional, T bytes) gets 1 for trials with a non-finite output.
// Two contraction levels (level + 1 into level) in one pass; `ch` holds the
// level-(level + 2) blocks (K * R * R per trial, side mb2).  Same support as
// expand2 (expand2_supported); cudaErrorNotSupported otherwise.
cudaError_t launch_contract2_plan(int dtype, int formula, const void* ch, int64_t K, int64_t mb2,
                                  void* out, const PlanLevel* plans, int64_t plan_tstride,
                                  int level, int64_t ntr, uint8_t* nonfinite, cudaStream_t st);
cudaError_t launch_contract_plan(int dtype, int formula, const void* ch, int64_t K, int64_t mb,
                                 void* out, const PlanLevel* plans, int64_t plan_tstride,
                                 int level, int64_t T, uint8_t* nonfinite, cudaStream_t st);

// Expansion of levels `level` and `level + 1` in one pass (no level+1 array in
// HBM): x (T or 1, K, s, s) -> out (T, K*R*R, s/n^2, s/n^2).  Same values as
// two launch_expand_plan calls.  expand2_supported: an instantiation exists.
cudaError_t launch_expand2_plan(int dtype, int formula, int which, const void* x,
                                int64_t x_tstride, int64_t K, int64_t s, void* out,
                                const PlanLevel* plans, int64_t plan_tstride, int level,
                                int64_t ntr, cudaStream_t st);
bool expand2_supported(int dtype, int formula);

int formula_n(int formula);
int formula_R(int formula);

// Fused bottom subtree (kernels_fused.cu): L levels below q0 for every
// (trial, level-q0 block) in shared memory.  x, y: (T, K0, s0, s0) blocks
// (xy_tstride elements per trial, 0 = broadcast), out: (T, K0, s0, s0).
// subtree_smem_bytes returns 0 when no instantiation covers (formula, L, M).
size_t subtree_smem_bytes(int dtype, int formula, int L, int M);
cudaError_t launch_subtree(int dtype, int formula, int L, int M, const void* x, const void* y,
                           int64_t xy_tstride, int64_t K0, void* out, const PlanLevel* plans,
                           int64_t plan_tstride, int q0, int64_t ntr, uint8_t* nonfinite,
                           cudaStream_t st);

// ---- dense path: arbitrary coefficient tables (Tc, R, n, n) --------------
cudaError_t launch_expand_dense(int dtype, const void* x, int64_t x_tstride, int64_t K, int64_t s,
                                int n, int R, const void* coeff, int64_t c_tstride, void* out,
                                int64_t T, cudaStream_t st);
cudaError_t launch_contract_dense(int dtype, const void* ch, int64_t K, int64_t mb, int n, int R,
                                  const void* w, int64_t w_tstride, void* out, int64_t T,
                                  uint8_t* nonfinite, cudaStream_t st);

// ---- leaf: exact-order batched product ------------------------------------
// out[b] = x[b] @ y[b], k ascending, first term initialises, one rounding per
// multiply and per add.  dtype_out may be wider than dtype_in (f64 truth of
// f32/f16 operands: inputs are widened exactly).
cudaError_t launch_leaf(int dtype_in, int dtype_out, int64_t batch, int64_t M, int64_t K,
                        int64_t N, const void* x, int64_t x_bstride, const void* y,
                        int64_t y_bstride, void* out, cudaStream_t st);

// Binary64 product of binary64/32/16 operands on the DFMA pipe (truth.cu):
// same contract as launch_leaf with dtype_out = f64; cudaErrorNotSupported
// for empty shapes.
cudaError_t launch_truth(int dtype_in, int64_t batch, int64_t M, int64_t K, int64_t N,
                         const void* x, int64_t x_bstride, const void* y, int64_t y_bstride,
                         void* out, cudaStream_t st);

// The stream-ordered default pool of `device` retains up to 4 GiB of freed
// scratch (truth panels, generator words) instead of returning it at every
// synchronisation (truth.cu).
cudaError_t keep_pool(int device);

// ---- seeded test matrices (matgen.cu) -----------------------------------
// Matrix families, in the order of reference MATRIX_KINDS (matgen.py:21)
// followed by the builder kinds.
enum MatgenKind : int {
  kMatGaussian = 0, kMatUniform = 1, kMatAdv1 = 2, kMatAdv2 = 3, kMatAdv3 = 4, kMatHilbert = 5,
  kMatUniformPm1 = 6, kMatQuadrant100 = 7
};
// out[c] (n x n, dtype) = the family's matrix drawn from the Philox stream
// with key keys[2c], keys[2c+1] (host array), which[c] = 0 for A, 1 for B
// (host array); flags (device, optional) set to 1 for non-finite results.
// Synchronises the stream (the tail of the normal ziggurat runs on the host).
int matgen(int kind, int dtype, int64_t count, int64_t n, const uint64_t* keys, const int* which,
           void* out, uint8_t* flags, cudaStream_t st);

// ---- error check -----------------------------------------------------------
// err[t] = ||widen(c[t]) - ref[t or 0]||_F / ||ref[t or 0]||_F   (binary64)
// scratch: at least error_scratch_bytes(T) bytes of device memory.
size_t error_scratch_bytes(int64_t T);
cudaError_t launch_rel_errors(int dtype, int64_t T, int64_t N2, const void* c, const double* ref,
                              int64_t ref_tstride, double* err, void* scratch, cudaStream_t st);

// total[e] += x[0][e] + ... + x[ntr-1][e], sequentially in binary64.
cudaError_t launch_sum_trials(int dtype, int64_t ntr, int64_t N2, const void* x, double* total,
                              cudaStream_t st);

// Set nonfinite[t] = 1 when any element of x[t] (N2 elements) is non-finite.
cudaError_t launch_nonfinite(int dtype, int64_t T, int64_t N2, const void* x, uint8_t* flags,
                             cudaStream_t st);

// ---- diagonal rescaling (rescale.cu; reference rescale.py:36-99) ----------
// Maxima of |x| (N x N, mode dtype) along rows (axis 1) or columns (axis 0)
// into out (N, mode dtype); *zero set to 1 when one is 0.  scratch: at least
// absmax_scratch_bytes(N) bytes.
size_t absmax_scratch_bytes(int64_t N);
cudaError_t launch_absmax(int dtype, const void* x, int64_t N, int axis, void* out, uint8_t* zero,
                          void* scratch, cudaStream_t st);
// out = fl(1 / d)
cudaError_t launch_recip(int dtype, const void* d, int64_t N, void* out, cudaStream_t st);
// d = fl(sqrt(fl(bmax / amax))), rd = fl(1 / d)
cudaError_t launch_inside_factors(int dtype, const void* bmax, const void* amax, int64_t N,
                                  void* d, void* rd, cudaStream_t st);
// In place: for s in order, x[i][j] = fl(row_s[i] * x[i][j]), then
// x[i][j] = fl(x[i][j] * col_s[j]) (null vectors skipped).
struct ScaleList {
  const void* row[8];
  const void* col[8];
  int n;
};
cudaError_t launch_scale(int dtype, void* x, int64_t N, const ScaleList& sl, cudaStream_t st);

}  // namespace rbc
