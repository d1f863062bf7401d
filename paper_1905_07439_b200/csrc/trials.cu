// Error-trial pipeline: the per-pair work of the reference's distribution
// experiments (experiments.py:248-261, 327-379) on the device.
//
// For every trial t (one operand pair (A_t, B_t) in the mode, one plan):
//   ref_t  = standard_multiply(widen(A_t), widen(B_t), DOUBLE)   exact order
//   C_t    = BC product under plan t          (plan path, exact +-1 formula)
//   err_t  = ||widen(C_t) - ref_t||_F / ||ref_t||_F              binary64
// and, optionally, the deterministic product (identity plan) and its error
// against the same ref_t.  Non-finite products are flagged per trial (their
// error is still computed; it is inf/nan).
//
// Trials are processed in chunks sized by the workspace; per chunk the
// working set is ref (8 B/elt), one product buffer, and the engine workspace.

#include <algorithm>
#include <cstring>
#include <vector>

#include "../../include/rbc.h"
#include "kernels.h"

extern "C" int rbc_apply_plans_async(int, int, int, int64_t, const void*, int64_t, int64_t,
                                     const void*, const void*, int64_t, void*, uint8_t*, void*,
                                     size_t, void*);

namespace rbc {
int set_error_public(int code, const char* msg);
}

namespace {

size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
  size_t ref, prod, scratch, engine, total;
};

Layout layout_for(int dtype, int formula, int Q, int64_t chunk, int64_t N) {
  Layout L;
  const size_t N2 = (size_t)N * (size_t)N;
  L.ref = a256((size_t)chunk * N2 * 8);
  L.prod = a256((size_t)chunk * N2 * rbc::dtype_size(dtype));
  L.scratch = a256(rbc::error_scratch_bytes(chunk));
  L.engine = a256(rbc_plans_workspace_bytes(dtype, formula, Q, chunk, N));
  L.total = L.ref + L.prod + L.scratch + L.engine;
  return L;
}

}  // namespace

extern "C" {

size_t rbc_error_trials_workspace_bytes(int dtype, int formula, int Q, int64_t T, int64_t N) {
  if (T < 1) T = 1;
  return layout_for(dtype, formula, Q, T, N).total;
}

int rbc_error_trials_async(int dtype, int formula, int Q, int64_t T, int64_t N, const void* a,
                           const void* b, const void* rand_plans, const void* det_plans,
                           double* err_rand, double* err_det, uint8_t* nf_rand, uint8_t* nf_det,
                           void* workspace, size_t workspace_bytes, void* stream) {
  using namespace rbc;
  cudaStream_t st = (cudaStream_t)stream;
  if (T == 0 || N == 0) return RBC_OK;
  if (!rand_plans && !det_plans) return set_error_public(RBC_EVALUE, "no product requested");
  if (formula_n(formula) == 0) return set_error_public(RBC_EVALUE, "unknown formula id");
  // largest chunk that fits
  int64_t chunk = T;
  while (chunk > 1 && layout_for(dtype, formula, Q, chunk, N).total > workspace_bytes)
    chunk = (chunk + 1) / 2;
  const Layout L = layout_for(dtype, formula, Q, chunk, N);
  if (L.total > workspace_bytes)
    return set_error_public(RBC_EVALUE, "workspace too small for one trial");
  char* base = (char*)workspace;
  double* ref = (double*)base;
  void* prod = base + L.ref;
  void* scratch = base + L.ref + L.prod;
  void* eng = base + L.ref + L.prod + L.scratch;
  const size_t es = dtype_size(dtype);
  const int64_t N2 = N * N;
  for (int64_t t0 = 0; t0 < T; t0 += chunk) {
    const int64_t nt = std::min(chunk, T - t0);
    const char* at = (const char*)a + (size_t)t0 * N2 * es;
    const char* bt = (const char*)b + (size_t)t0 * N2 * es;
    cudaError_t e;
    {
      Stage stage(st, "truth_f64", (double)nt * N2 * (2.0 * es + 8.0), 2.0 * nt * (double)N2 * N);
      e = launch_leaf(dtype, kF64, nt, N, N, N, at, N2, bt, N2, ref, st);
    }
    if (e != cudaSuccess) return fail_cuda(e, "truth", __FILE__, __LINE__);
    for (int which = 0; which < 2; ++which) {
      const void* plans = which == 0 ? det_plans : rand_plans;
      if (!plans) continue;
      double* err = which == 0 ? err_det : err_rand;
      uint8_t* nf = which == 0 ? nf_det : nf_rand;
      const int64_t Tp = which == 0 ? 1 : nt;
      const void* pl = which == 0 ? plans : (const char*)plans + (size_t)t0 * Q * RBC_PLAN_BYTES;
      int rc = rbc_apply_plans_async(dtype, formula, Q, Tp, pl, nt, N, at, bt, nt, prod,
                                     nf ? nf + t0 : nullptr, eng, L.engine, stream);
      if (rc != RBC_OK) return rc;
      if (err) {
        Stage stage(st, "rel_errors", (double)nt * N2 * (es + 8.0), 3.0 * nt * (double)N2);
        e = launch_rel_errors(dtype, nt, N2, prod, ref, N2, err + t0, scratch, st);
        if (e != cudaSuccess) return fail_cuda(e, "rel_errors", __FILE__, __LINE__);
      }
    }
  }
  return RBC_OK;
}

}  // extern "C"
