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
#include <mutex>
#include <vector>

#include "../../include/rbc.h"
#include "kernels.h"


namespace rbc {
int set_error_public(int code, const char* msg);
}

#define CUDA_TRY(expr)                                                             \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) return ::rbc::fail_cuda(_e, #expr, __FILE__, __LINE__); \
  } while (0)

namespace {

size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

// Per chunk: the binary64 truth, then one "lane" per product (deterministic,
// randomized) with its own product buffer, error scratch and engine
// workspace, so the three can run concurrently on forked streams.
struct Layout {
  size_t ref, prod, scratch, engine, lane, total;
};

Layout layout_for(int dtype, int formula, int Q, int64_t chunk, int64_t N) {
  Layout L;
  const size_t N2 = (size_t)N * (size_t)N;
  L.ref = a256((size_t)chunk * N2 * 8);
  L.prod = a256((size_t)chunk * N2 * rbc::dtype_size(dtype));
  L.scratch = a256(rbc::error_scratch_bytes(chunk));
  L.engine = a256(rbc_plans_workspace_bytes(dtype, formula, Q, chunk, N));
  L.lane = L.prod + L.scratch + L.engine;
  L.total = L.ref + 2 * L.lane;
  return L;
}

// Auxiliary streams (truth, deterministic lane, randomized lane) of the
// current device, created once.  Work is forked from and joined back into
// the caller's stream with events, so the whole pass stays stream ordered
// (and graph capturable).
struct AuxStreams {
  cudaStream_t s[3];
  cudaEvent_t fork, join[3], truth_done, lane_done[2];
};

// One lane set per (device, caller stream): two passes issued on different
// caller streams (the host-buffer pipeline's two compute streams) must not
// queue behind each other on shared lanes.
AuxStreams* aux_streams(cudaStream_t caller) {
  struct Entry {
    int dev;
    cudaStream_t caller;
    AuxStreams* ax;
  };
  static std::mutex mu;
  static std::vector<Entry> sets;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (const Entry& e : sets)
    if (e.dev == dev && e.caller == caller) return e.ax;
  AuxStreams* a = new AuxStreams;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  for (int i = 0; i < 3; ++i) {
    // the truth lane (FP64 pipe) gets the highest priority so its CTAs
    // interleave with the shared-memory-bound product kernels (equal
    // priorities, or the product lanes high, measured within 0.03 ms on c2)
    cudaStreamCreateWithPriority(&a->s[i], cudaStreamNonBlocking, i == 0 ? hi : lo);
    cudaEventCreateWithFlags(&a->join[i], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&a->fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&a->truth_done, cudaEventDisableTiming);
  for (int i = 0; i < 2; ++i) cudaEventCreateWithFlags(&a->lane_done[i], cudaEventDisableTiming);
  sets.push_back({dev, caller, a});
  return a;
}

}  // namespace

// ---- running mean (reference experiments.py:279-289) ----------------------
// total_i = fl(total_{i-1} + C_i) in binary64 from total_0 = 0, plan order;
// at each checkpoint i: sum over elements of (fl(total_i / i) - ref)^2.
constexpr int kMaxCheckpoints = 32;
struct Checkpoints {
  int n;
  int at[kMaxCheckpoints];
};

constexpr int kMeanThreads = 256;
constexpr int kMeanBlocks = 148 * 4;  // enough CTAs to stream G*N^2 elements at HBM rate

template <class T>
__global__ void __launch_bounds__(kMeanThreads) running_mean_kernel(
    int G, int64_t N2, const T* __restrict__ C, const double* __restrict__ ref, Checkpoints cp,
    double* __restrict__ part /* (cp.n + 1) x gridDim.x */) {
  __shared__ double sh[kMeanThreads / 32];
  double s[kMaxCheckpoints + 1];
#pragma unroll
  for (int c = 0; c <= kMaxCheckpoints; ++c) s[c] = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * kMeanThreads + threadIdx.x; e < N2;
       e += (int64_t)gridDim.x * kMeanThreads) {
    const double r = ref[e];
    double total = 0.0;
    int c = 0;
    // the products of kBatch plans are loaded together (independent loads in
    // flight), then added in plan order
    constexpr int kBatch = 8;
    for (int t0 = 0; t0 < G; t0 += kBatch) {
      T v[kBatch];
#pragma unroll
      for (int q = 0; q < kBatch; ++q)
        v[q] = t0 + q < G ? C[(int64_t)(t0 + q) * N2 + e] : T(0);
#pragma unroll
      for (int q = 0; q < kBatch; ++q) {
        const int t = t0 + q;
        if (t >= G) break;
        total = __dadd_rn(total, rbc::Arith<T>::widen(v[q]));
        if (c < cp.n && t + 1 == cp.at[c]) {
          const double d = __dsub_rn(__ddiv_rn(total, (double)(t + 1)), r);
#pragma unroll
          for (int k = 0; k < kMaxCheckpoints; ++k)
            if (k == c) s[k] += d * d;
          ++c;
        }
      }
    }
    s[kMaxCheckpoints] += r * r;
  }
  for (int c = 0; c <= cp.n; ++c) {
    double v = c == cp.n ? s[kMaxCheckpoints] : 0.0;
#pragma unroll
    for (int k = 0; k < kMaxCheckpoints; ++k)
      if (k == c && c < cp.n) v = s[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < kMeanThreads / 32; ++w) tot += sh[w];
      part[c * gridDim.x + blockIdx.x] = tot;
    }
    __syncthreads();
  }
}

__global__ void running_mean_finish(int ncp, int nb, const double* __restrict__ part,
                                    double* __restrict__ err) {
  const int c = threadIdx.x;
  if (c >= ncp) return;
  double num = 0.0, den = 0.0;
  for (int b = 0; b < nb; ++b) {
    num += part[c * nb + b];
    den += part[ncp * nb + b];
  }
  err[c] = sqrt(num) / sqrt(den);
}

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
  const size_t es = dtype_size(dtype);
  const int64_t N2 = N * N;
  // Concurrent lanes unless the stage profiler is on (overlapping stages
  // would blur its per-kernel durations) or RBC_SERIAL_LANES=1.
  static const bool serial_env = [] {
    const char* v = getenv("RBC_SERIAL_LANES");
    return v && v[0] == '1';
  }();
  const bool conc = !prof_on() && !serial_env;
  AuxStreams* ax = aux_streams(st);
  cudaStream_t lanes[3] = {st, st, st};
  if (conc) {
    for (int i = 0; i < 3; ++i) lanes[i] = ax->s[i];
    CUDA_TRY(cudaEventRecord(ax->fork, st));
    for (int i = 0; i < 3; ++i) CUDA_TRY(cudaStreamWaitEvent(ax->s[i], ax->fork, 0));
  }
  cudaStream_t s_truth = lanes[0];
  for (int64_t t0 = 0; t0 < T; t0 += chunk) {
    const int64_t nt = std::min(chunk, T - t0);
    const char* at = (const char*)a + (size_t)t0 * N2 * es;
    const char* bt = (const char*)b + (size_t)t0 * N2 * es;
    cudaError_t e;
    if (t0 > 0)  // ref is reused: the previous chunk's error kernels must be done
      for (int w = 0; w < 2; ++w) CUDA_TRY(cudaStreamWaitEvent(s_truth, ax->lane_done[w], 0));
    {
      Stage stage(s_truth, "truth_f64", (double)nt * N2 * (2.0 * es + 8.0), 2.0 * nt * (double)N2 * N);
      e = launch_leaf(dtype, kF64, nt, N, N, N, at, N2, bt, N2, ref, s_truth);
    }
    if (e != cudaSuccess) return fail_cuda(e, "truth", __FILE__, __LINE__);
    CUDA_TRY(cudaEventRecord(ax->truth_done, s_truth));
    for (int which = 0; which < 2; ++which) {
      cudaStream_t ls = lanes[1 + which];
      char* lane = base + L.ref + (size_t)which * L.lane;
      void* prod = lane;
      void* scratch = lane + L.prod;
      void* eng = lane + L.prod + L.scratch;
      const void* plans = which == 0 ? det_plans : rand_plans;
      if (!plans) {
        CUDA_TRY(cudaEventRecord(ax->lane_done[which], ls));
        continue;
      }
      double* err = which == 0 ? err_det : err_rand;
      uint8_t* nf = which == 0 ? nf_det : nf_rand;
      const int64_t Tp = which == 0 ? 1 : nt;
      const void* pl = which == 0 ? plans : (const char*)plans + (size_t)t0 * Q * RBC_PLAN_BYTES;
      // The lanes start together.  Starting the randomized lane's (HBM-bound)
      // expansions after the deterministic lane's, to run them beside its
      // (issue-bound) leaves, measured slower (c2 9.05 vs 8.90 ms, c4 21.94
      // vs 21.85): the leaf CTAs leave too little of an SM for a streaming
      // kernel beside them.
      int rc = rbc_apply_plans_async(dtype, formula, Q, Tp, pl, nt, N, at, bt, nt, prod,
                                     nf ? nf + t0 : nullptr, eng, L.engine, ls);
      if (rc != RBC_OK) return rc;
      CUDA_TRY(cudaStreamWaitEvent(ls, ax->truth_done, 0));
      if (err) {
        Stage stage(ls, "rel_errors", (double)nt * N2 * (es + 8.0), 3.0 * nt * (double)N2);
        e = launch_rel_errors(dtype, nt, N2, prod, ref, N2, err + t0, scratch, ls);
        if (e != cudaSuccess) return fail_cuda(e, "rel_errors", __FILE__, __LINE__);
      }
      CUDA_TRY(cudaEventRecord(ax->lane_done[which], ls));
    }
  }
  if (conc) {
    for (int i = 0; i < 3; ++i) {
      CUDA_TRY(cudaEventRecord(ax->join[i], ax->s[i]));
      CUDA_TRY(cudaStreamWaitEvent(st, ax->join[i], 0));
    }
  }
  return RBC_OK;
}

// ---- averaging trials (config 3; reference _run_average, experiments.py:264-296)
// For each of P pairs: binary64 truth, optional deterministic product
// (coefficient tables det_u/v/w, Tc = 1), G randomized products (tables
// u/v/w with P*G trials, pair p owning trials p*G .. p*G+G-1), their
// per-plan errors, and the running-mean error at each checkpoint.
size_t rbc_average_trials_workspace_bytes(int dtype, int Q, const int32_t* n, const int32_t* R,
                                          int64_t G, int64_t N) {
  using namespace rbc;
  const size_t N2 = (size_t)N * N;
  return a256(N2 * 8) + a256((size_t)G * N2 * dtype_size(dtype)) +
         a256(error_scratch_bytes(G)) + a256((size_t)(kMaxCheckpoints + 1) * kMeanBlocks * 8) +
         a256(rbc_levels_workspace_bytes(dtype, Q, n, R, G, N));
}

int rbc_average_trials_async(int dtype, int Q, const int32_t* n, const int32_t* R, int64_t P,
                             int64_t G, int64_t N, const void* a, const void* b,
                             const void* const* u, const void* const* v, const void* const* w,
                             const void* const* det_u, const void* const* det_v,
                             const void* const* det_w, int ncheck, const int32_t* checkpoints,
                             double* err_rand, double* err_mean, double* err_det,
                             uint8_t* nf_rand, uint8_t* nf_det, void* workspace,
                             size_t workspace_bytes, void* stream) {
  using namespace rbc;
  cudaStream_t st = (cudaStream_t)stream;
  if (P == 0 || G == 0 || N == 0) return RBC_OK;
  if (ncheck < 0 || ncheck > kMaxCheckpoints)
    return set_error_public(RBC_EVALUE, "at most 32 checkpoints");
  Checkpoints cp;
  cp.n = ncheck;
  for (int c = 0; c < ncheck; ++c) {
    cp.at[c] = checkpoints[c];
    if (cp.at[c] < 1 || cp.at[c] > G || (c && cp.at[c] <= cp.at[c - 1]))
      return set_error_public(RBC_EVALUE, "checkpoints must ascend within 1..G");
  }
  const size_t need = rbc_average_trials_workspace_bytes(dtype, Q, n, R, G, N);
  if (workspace_bytes < need) return set_error_public(RBC_EVALUE, "workspace too small");
  const size_t es = dtype_size(dtype);
  const int64_t N2 = N * N;
  char* base = (char*)workspace;
  double* ref = (double*)base;
  base += a256(N2 * 8);
  void* prod = base;
  base += a256((size_t)G * N2 * es);
  void* scratch = base;
  base += a256(error_scratch_bytes(G));
  double* part = (double*)base;
  base += a256((size_t)(kMaxCheckpoints + 1) * kMeanBlocks * 8);
  void* eng = base;
  const size_t eng_bytes = rbc_levels_workspace_bytes(dtype, Q, n, R, G, N);
  std::vector<const void*> pu(Q), pv(Q), pw(Q);
  std::vector<int64_t> tcG(Q, G), tc1(Q, 1);
  // The pair's truth (one product: a fraction of the GPU's CTAs at config
  // 3's size) runs on the truth lane beside the deterministic product and
  // the start of the randomized one; the first error kernel joins it.  The
  // fork is recorded after the previous pair's running mean, the last
  // reader of `ref`.  Serial while the stage profiler runs.
  static const bool serial_env = [] {
    const char* v = getenv("RBC_SERIAL_LANES");
    return v && v[0] == '1';
  }();
  const bool conc = !prof_on() && !serial_env;
  AuxStreams* ax = conc ? aux_streams(st) : nullptr;
  for (int64_t p = 0; p < P; ++p) {
    const char* ap = (const char*)a + (size_t)p * N2 * es;
    const char* bp = (const char*)b + (size_t)p * N2 * es;
    cudaError_t e;
    cudaStream_t s_truth = st;
    if (conc) {
      s_truth = ax->s[0];
      CUDA_TRY(cudaEventRecord(ax->fork, st));
      CUDA_TRY(cudaStreamWaitEvent(s_truth, ax->fork, 0));
    }
    {
      Stage stage(s_truth, "truth_f64", (double)N2 * (2.0 * es + 8.0), 2.0 * (double)N2 * N);
      e = launch_leaf(dtype, kF64, 1, N, N, N, ap, N2, bp, N2, ref, s_truth);
    }
    if (e != cudaSuccess) return fail_cuda(e, "truth", __FILE__, __LINE__);
    bool joined = !conc;
    auto join_truth = [&]() -> int {
      if (!joined) {
        CUDA_TRY(cudaEventRecord(ax->truth_done, s_truth));
        CUDA_TRY(cudaStreamWaitEvent(st, ax->truth_done, 0));
        joined = true;
      }
      return RBC_OK;
    };
    if (det_u && err_det) {
      int rc = rbc_apply_levels_async(dtype, Q, n, R, tc1.data(), det_u, det_v, det_w, 1, N, ap,
                                      bp, 1, prod, nf_det ? nf_det + p : nullptr, eng, eng_bytes,
                                      stream);
      if (rc != RBC_OK) return rc;
      {
        const int jr = join_truth();
        if (jr != RBC_OK) return jr;
      }
      Stage stage(st, "rel_errors", (double)N2 * (es + 8.0), 3.0 * (double)N2);
      e = launch_rel_errors(dtype, 1, N2, prod, ref, 0, err_det + p, scratch, st);
      if (e != cudaSuccess) return fail_cuda(e, "rel_errors", __FILE__, __LINE__);
    }
    for (int q = 0; q < Q; ++q) {
      const size_t off = (size_t)p * G * R[q] * n[q] * n[q] * es;
      pu[q] = (const char*)u[q] + off;
      pv[q] = (const char*)v[q] + off;
      pw[q] = (const char*)w[q] + off;
    }
    int rc = rbc_apply_levels_async(dtype, Q, n, R, tcG.data(), pu.data(), pv.data(), pw.data(), 1,
                                    N, ap, bp, G, prod, nf_rand ? nf_rand + p * G : nullptr, eng,
                                    eng_bytes, stream);
    if (rc != RBC_OK) return rc;
    {
      const int jr = join_truth();
      if (jr != RBC_OK) return jr;
    }
    {
      Stage stage(st, "rel_errors", (double)G * N2 * (es + 8.0), 3.0 * (double)G * N2);
      e = launch_rel_errors(dtype, G, N2, prod, ref, 0, err_rand + p * G, scratch, st);
    }
    if (e != cudaSuccess) return fail_cuda(e, "rel_errors", __FILE__, __LINE__);
    if (ncheck && err_mean) {
      Stage stage(st, "running_mean", (double)G * N2 * es + N2 * 8.0, 2.0 * (double)G * N2);
      switch (dtype) {
        case kF64:
          running_mean_kernel<double><<<kMeanBlocks, kMeanThreads, 0, st>>>(
              (int)G, N2, (const double*)prod, ref, cp, part);
          break;
        case kF32:
          running_mean_kernel<float><<<kMeanBlocks, kMeanThreads, 0, st>>>(
              (int)G, N2, (const float*)prod, ref, cp, part);
          break;
        default:
          running_mean_kernel<__half><<<kMeanBlocks, kMeanThreads, 0, st>>>(
              (int)G, N2, (const __half*)prod, ref, cp, part);
      }
      running_mean_finish<<<1, 32, 0, st>>>(ncheck, kMeanBlocks, part, err_mean + p * ncheck);
      e = cudaGetLastError();
      if (e != cudaSuccess) return fail_cuda(e, "running_mean", __FILE__, __LINE__);
    }
  }
  return RBC_OK;
}

}  // extern "C"
