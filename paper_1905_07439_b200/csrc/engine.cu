// Orchestration and C ABI of the B200 BC engine (declared in include/rbc.h).
//
// Breadth-first evaluation, as in the reference apply_levels
// (pkg/src/randbc/_engine.py:117-149): Q level-wide expansions of A, Q of B,
// one batched exact-order leaf product, Q contractions in reverse, then the
// non-finite check.  Intermediate levels live in a caller-provided (async
// API) or pooled (host API) workspace of four equal buffers:
//
//   bufX, bufY : deepest expansions of A and B          (L_Q elements/trial)
//   ping, pong : intermediate levels, leaf product, contractions
//
// each sized max_q L_q per trial, L_q = prod_{j<q} R_j * (N / prod_{j<q} n_j)^2.
// Trials are processed in chunks that fit the workspace; chunking never
// changes values (every output element's operation chain is per trial).

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/rbc.h"
#include "kernels.h"

namespace rbc {

static thread_local std::string g_last_error;

static int set_error(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int set_error_public(int code, const char* msg) { return set_error(code, "%s", msg); }

int fail_cuda(cudaError_t e, const char* expr, const char* file, int line) {
  return set_error(RBC_ERUNTIME, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
                   cudaGetErrorString(e), file, line, expr);
}


#define RBC_TRY(expr)          \
  do {                         \
    int _rc = (expr);          \
    if (_rc != RBC_OK) return _rc; \
  } while (0)

// ------------------------------------------------------------- level plan --
struct LevelShape {
  int n;
  int R;
};

struct Geometry {
  int Q = 0;
  int64_t N = 0;
  std::vector<LevelShape> lv;
  int64_t maxL = 0;   // elements per trial of the largest level (q >= 1)
  int64_t leaves = 1; // prod R
  int64_t leaf_m = 0; // leaf block side
};

static int make_geometry(int Q, const int32_t* n, const int32_t* R, int64_t N, Geometry* g) {
  if (Q < 1) return set_error(RBC_EVALUE, "need at least one level");
  if (N < 0) return set_error(RBC_EVALUE, "operand size must be >= 0");
  g->Q = Q;
  g->N = N;
  g->lv.resize(Q);
  int64_t s = N, K = 1;
  g->maxL = 0;
  for (int q = 0; q < Q; ++q) {
    if (n[q] < 1 || R[q] < 1) return set_error(RBC_EVALUE, "level %d: need n >= 1 and R >= 1", q);
    if (s % n[q]) return set_error(RBC_EVALUE, "operand size not divisible by block grid");
    g->lv[q] = {n[q], R[q]};
    s /= n[q];
    K *= R[q];
    g->maxL = std::max(g->maxL, K * s * s);
  }
  g->leaves = K;
  g->leaf_m = s;
  return RBC_OK;
}

static size_t per_trial_ws(const Geometry& g, int dtype) {
  return (size_t)4 * (size_t)g.maxL * dtype_size(dtype);
}

// Workspace the async entry points need for `T` trials in one chunk
// (4 sub-buffers, each rounded up to 256 bytes).
static size_t ws_for(const Geometry& g, int dtype, int64_t T) {
  const size_t sub = (((size_t)T * (size_t)g.maxL * dtype_size(dtype)) + 255) & ~(size_t)255;
  return 4 * sub;
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// ---------------------------------------------------------- stage profiler --
struct ProfRec {
  std::string name;
  cudaEvent_t ev0, ev1;
  double bytes, flops;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_prof_pool;

bool prof_on() { return g_prof_on; }

static cudaEvent_t prof_event() {
  if (!g_prof_pool.empty()) {
    cudaEvent_t e = g_prof_pool.back();
    g_prof_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

void prof_record(cudaStream_t st, const char* name, double bytes, double flops, bool start) {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  if (start) {
    ProfRec r{name, prof_event(), nullptr, bytes, flops};
    cudaEventRecord(r.ev0, st);
    g_prof.push_back(r);
  } else {
    for (auto it = g_prof.rbegin(); it != g_prof.rend(); ++it)
      if (!it->ev1 && it->name == name) {
        it->ev1 = prof_event();
        cudaEventRecord(it->ev1, st);
        break;
      }
  }
}

static void prof_clear() {
  for (auto& r : g_prof) {
    if (r.ev0) g_prof_pool.push_back(r.ev0);
    if (r.ev1) g_prof_pool.push_back(r.ev1);
  }
  g_prof.clear();
}

// RBC_DEBUG_SYNC=1: synchronise after every launch so a fault is attributed
// to the stage that caused it.
static bool debug_sync() {
  static const bool on = [] {
    const char* v = getenv("RBC_DEBUG_SYNC");
    return v && v[0] == '1';
  }();
  return on;
}

// RBC_NO_FUSION=1 forces the plain breadth-first schedule (tests compare both).
static bool fusion_enabled() {
  const char* v = getenv("RBC_NO_FUSION");
  return !(v && v[0] == '1');
}

// RBC_NO_EXPAND2=1 evaluates every expansion level in its own pass.
static bool expand2_enabled() {
  const char* v = getenv("RBC_NO_EXPAND2");
  return !(v && v[0] == '1');
}

static constexpr size_t kMaxSubtreeSmem = 200 * 1024;

static cudaError_t stage_done(cudaError_t e, cudaStream_t st) {
  if (e != cudaSuccess || !debug_sync()) return e;
  return cudaStreamSynchronize(st);
}

// One chunked breadth-first pass.  `kind` selects the combination kernels.
struct PassArgs {
  int dtype;
  bool plan;        // plan path (formula kernels) vs dense coefficient tables
  int formula;      // plan path
  const PlanLevel* plans;
  int64_t Tp;
  std::vector<const void*> u, v, w;  // dense path, device pointers
  std::vector<int64_t> Tc;           // dense path
  int64_t T0, T;
  const void* a;
  const void* b;
  void* out;
  uint8_t* nonfinite;
};

static int run_pass(const Geometry& g, const PassArgs& p, void* ws, size_t ws_bytes,
                    cudaStream_t st) {
  const int dt = p.dtype;
  const size_t es = dtype_size(dt);
  const int64_t N2 = g.N * g.N;
  const size_t ptw = per_trial_ws(g, dt);
  if (p.T == 0 || g.N == 0) {
    // empty operands: no product, no overflow (the flags may sit on stale
    // arena bytes of an earlier call)
    if (p.nonfinite && p.T) CUDA_TRY(cudaMemsetAsync(p.nonfinite, 0, (size_t)p.T, st));
    return RBC_OK;
  }
  int64_t chunk = ptw ? (int64_t)(ws_bytes / ptw) : p.T;
  chunk = std::min(chunk, p.T);
  while (chunk > 0 && ws_for(g, dt, chunk) > ws_bytes) --chunk;
  if (chunk < 1)
    return set_error(RBC_EVALUE, "workspace too small: need %zu bytes per trial", ws_for(g, dt, 1));
  // 4 sub-buffers of chunk * maxL elements each
  const size_t buf_elems = align_up((size_t)chunk * (size_t)g.maxL * es) / es;
  char* base = (char*)ws;
  void* bufX = base;
  void* bufY = base + buf_elems * es;
  void* ping = base + 2 * buf_elems * es;
  void* pong = base + 3 * buf_elems * es;
  if (p.nonfinite) CUDA_TRY(cudaMemsetAsync(p.nonfinite, 0, (size_t)p.T, st));

  // Fuse the bottom levels into one shared-memory subtree kernel when an
  // instantiation exists for (formula, depth, leaf side) and fits on chip.
  int fuseL = 0;
  if (p.plan && fusion_enabled()) {
    for (int L = std::min(2, g.Q); L >= 1 && !fuseL; --L) {
      const size_t sm = subtree_smem_bytes(dt, p.formula, L, (int)g.leaf_m);
      if (sm && sm <= kMaxSubtreeSmem) fuseL = L;
    }
  }
  const int q0 = g.Q - fuseL;  // levels evaluated breadth-first over HBM
  int64_t K_q0 = 1, s_q0 = g.N;
  for (int q = 0; q < q0; ++q) {
    K_q0 *= g.lv[q].R;
    s_q0 /= g.lv[q].n;
  }

  for (int64_t t0 = 0; t0 < p.T; t0 += chunk) {
    const int64_t nt = std::min(chunk, p.T - t0);
    // --- expansions of A and B
    for (int which = 0; which < 2; ++which) {
      const void* cur = which == 0 ? p.a : p.b;
      int64_t cur_ts = p.T0 == 1 ? 0 : N2;
      if (p.T0 != 1) cur = (const char*)cur + (size_t)t0 * N2 * es;
      int64_t K = 1, s = g.N;
      for (int q = 0; q < q0;) {
        const int n = g.lv[q].n, R = g.lv[q].R;
        // plan path: two levels per pass where an instantiation exists
        int step = (p.plan && expand2_enabled() && q + 1 < q0 &&
                    expand2_supported(dt, p.formula)) ? 2 : 1;
        const int qlast = q + step - 1;
        void* dst = (qlast == q0 - 1) ? (which == 0 ? bufX : bufY) : (cur == ping ? pong : ping);
        cudaError_t e = cudaErrorNotSupported;
        const int64_t pts = p.Tp == 1 ? 0 : g.Q;
        const PlanLevel* pl = p.plans + (p.Tp == 1 ? 0 : t0 * g.Q);
        if (step == 2) {
          const double mb2 = (double)(s / (n * n));
          Stage stage(st, "expand2_plan",
                      ((cur_ts ? (double)nt : 1.0) * K * s * s + (double)nt * K * R * R * mb2 * mb2) * es,
                      (double)nt * K * R * (R + 1) * mb2 * mb2 * n * n * 2.0);
          e = launch_expand2_plan(dt, p.formula, which, cur, cur_ts, K, s, dst, pl, pts, q, nt, st);
          if (e == cudaErrorNotSupported) {
            step = 1;
            dst = (q == q0 - 1) ? (which == 0 ? bufX : bufY) : (cur == ping ? pong : ping);
          }
        }
        if (step == 1) {
          const double mbq = (double)(s / n);
          Stage stage(st, p.plan ? "expand_plan" : "expand_dense",
                      ((cur_ts ? (double)nt : 1.0) * K * s * s + (double)nt * K * R * mbq * mbq) * es,
                      (double)nt * K * R * mbq * mbq * n * n * 2.0);
          if (p.plan) {
            e = launch_expand_plan(dt, p.formula, which, cur, cur_ts, K, s, dst, pl, pts, q, nt, st);
          } else {
            const void* c = which == 0 ? p.u[q] : p.v[q];
            const int64_t cts = p.Tc[q] == 1 ? 0 : (int64_t)R * n * n;
            c = (const char*)c + (size_t)(p.Tc[q] == 1 ? 0 : t0 * cts) * es;
            e = launch_expand_dense(dt, cur, cur_ts, K, s, n, R, c, cts, dst, nt, st);
          }
        }
        e = stage_done(e, st);
        if (e != cudaSuccess) return fail_cuda(e, "expand", __FILE__, __LINE__);
        for (int k = 0; k < step; ++k) {
          s /= n;
          K *= R;
        }
        cur = dst;
        cur_ts = K * s * s;
        q += step;
      }
    }
    // --- leaves (or the fused bottom subtree)
    const int64_t m = g.leaf_m;
    if (fuseL) {
      const bool top = q0 == 0;
      const char* xs = top ? (const char*)p.a + (p.T0 == 1 ? 0 : (size_t)t0 * N2 * es) : (const char*)bufX;
      const char* ys = top ? (const char*)p.b + (p.T0 == 1 ? 0 : (size_t)t0 * N2 * es) : (const char*)bufY;
      const int64_t xy_ts = top ? (p.T0 == 1 ? 0 : N2) : K_q0 * s_q0 * s_q0;
      void* dst = top ? (char*)p.out + (size_t)t0 * N2 * es : ping;
      const int64_t pts = p.Tp == 1 ? 0 : g.Q;
      const PlanLevel* pl = p.plans + (p.Tp == 1 ? 0 : t0 * g.Q);
      Stage stage(st, "subtree_fused",
                  ((top && p.T0 == 1 ? 2.0 : 2.0 * nt) + nt) * (double)K_q0 * s_q0 * s_q0 * es,
                  2.0 * nt * g.leaves * (double)m * m * m);
      cudaError_t e = launch_subtree(dt, p.formula, fuseL, (int)m, xs, ys, xy_ts, K_q0, dst, pl,
                                     pts, q0, nt, (top && p.nonfinite) ? p.nonfinite + t0 : nullptr,
                                     st);
      e = stage_done(e, st);
      if (e != cudaSuccess) return fail_cuda(e, "subtree", __FILE__, __LINE__);
    } else {
      Stage stage(st, dt == kF64 ? "leaf_f64" : dt == kF32 ? "leaf_f32" : "leaf_f16",
                  3.0 * nt * g.leaves * m * m * es, 2.0 * nt * g.leaves * (double)m * m * m);
      cudaError_t e = launch_leaf(dt, dt, nt * g.leaves, m, m, m, bufX, m * m, bufY, m * m, ping, st);
      e = stage_done(e, st);
      if (e != cudaSuccess) return fail_cuda(e, "leaf", __FILE__, __LINE__);
    }
    // --- contractions, innermost level first (plan path: two levels per pass
    // where an instantiation exists, the mirror of the expansions)
    const void* cur = ping;
    int64_t K = K_q0, mb = s_q0;
    for (int q = q0 - 1; q >= 0;) {
      const int n = g.lv[q].n, R = g.lv[q].R;
      const int64_t pts = p.Tp == 1 ? 0 : g.Q;
      const PlanLevel* pl = p.plans + (p.Tp == 1 ? 0 : t0 * g.Q);
      cudaError_t e = cudaErrorNotSupported;
      if (p.plan && expand2_enabled() && q >= 1 && expand2_supported(dt, p.formula)) {
        const int64_t K2 = K / R / g.lv[q - 1].R;  // level-(q-1) parents per trial
        void* dst = q == 1 ? (char*)p.out + (size_t)t0 * N2 * es : (cur == ping ? pong : ping);
        uint8_t* nf = (q == 1 && p.nonfinite) ? p.nonfinite + t0 : nullptr;
        const double sq = (double)(mb * n * n);
        Stage stage(st, "contract2_plan",
                    ((double)nt * K * mb * mb + (double)nt * K2 * sq * sq) * es,
                    (double)nt * K * mb * mb * (R + 1) * n * n * 2.0);
        e = launch_contract2_plan(dt, p.formula, cur, K2, mb, dst, pl, pts, q - 1, nt, nf, st);
        if (e != cudaErrorNotSupported) {
          e = stage_done(e, st);
          if (e != cudaSuccess) return fail_cuda(e, "contract2", __FILE__, __LINE__);
          K = K2;
          cur = dst;
          mb *= n * n;
          q -= 2;
          continue;
        }
      }
      K /= R;
      void* dst = q == 0 ? (char*)p.out + (size_t)t0 * N2 * es : (cur == ping ? pong : ping);
      uint8_t* nf = (q == 0 && p.nonfinite) ? p.nonfinite + t0 : nullptr;
      const double sq = (double)(mb * n);
      Stage stage(st, p.plan ? "contract_plan" : "contract_dense",
                  ((double)nt * K * R * mb * mb + (double)nt * K * sq * sq) * es,
                  (double)nt * K * sq * sq * R * 2.0);
      if (p.plan) {
        e = launch_contract_plan(dt, p.formula, cur, K, mb, dst, pl, pts, q, nt, nf, st);
      } else {
        const int64_t cts = p.Tc[q] == 1 ? 0 : (int64_t)R * n * n;
        const void* c = (const char*)p.w[q] + (size_t)(p.Tc[q] == 1 ? 0 : t0 * cts) * es;
        e = launch_contract_dense(dt, cur, K, mb, n, R, c, cts, dst, nt, nf, st);
      }
      e = stage_done(e, st);
      if (e != cudaSuccess) return fail_cuda(e, "contract", __FILE__, __LINE__);
      cur = dst;
      mb *= n;
      --q;
    }
  }
  return RBC_OK;
}

// ------------------------------------------------------------ device pool --
// Host-API calls are synchronous; one growing device arena per process is
// reused across calls (guarded by a mutex, calls are serialised).
struct Arena {
  std::mutex mu;
  char* ptr = nullptr;
  size_t cap = 0;
  size_t off = 0;
  unsigned gen = 0;  // bumped whenever the allocation moves
  unsigned epoch = 0;  // bumped by every reserve(): a layout made earlier is stale
  void (*drain)() = nullptr;  // waits for host-buffer calls still in flight (begin/end)
  int reserve(size_t bytes) {
    if (drain) drain();
    ++epoch;
    if (bytes <= cap) {
      off = 0;
      return RBC_OK;
    }
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    cap = 0;
    ++gen;
    cudaError_t e = cudaMalloc((void**)&ptr, bytes);
    if (e != cudaSuccess) return fail_cuda(e, "cudaMalloc(arena)", __FILE__, __LINE__);
    cap = bytes;
    off = 0;
    return RBC_OK;
  }
  void* take(size_t bytes) {
    void* r = ptr + off;
    off += align_up(bytes);
    return r;
  }
};

static Arena& arena() {
  static Arena a;
  return a;
}

static int check_device() {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0)
    return set_error(RBC_ERUNTIME, "no CUDA device available (%s)", cudaGetErrorString(e));
  return RBC_OK;
}

// Workspace for a synchronous call: everything not already accounted for,
// bounded by the free device memory.
static size_t host_ws_budget(size_t fixed, size_t want) {
  // no device query when the arena already holds the request (see
  // rbc_error_trials: cudaMemGetInfo can stall behind driver queries)
  if (fixed + want + 256 <= arena().cap) return want;
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return want;
  const size_t usable = (size_t)((double)(free_b + arena().cap) * 0.85);
  if (usable <= fixed) return 0;
  return std::min(want, usable - fixed);
}

static int validate_trials(int64_t T, int64_t T0) {
  if (T < 0 || T0 < 0) return set_error(RBC_EVALUE, "negative trial count");
  if (!(T0 == 1 || T0 == T)) return set_error(RBC_EVALUE, "operand trials %lld do not broadcast to %lld",
                                              (long long)T0, (long long)T);
  return RBC_OK;
}

}  // namespace rbc

using namespace rbc;

extern "C" {

int rbc_abi_version(void) { return RBC_ABI_VERSION; }

void rbc_profile_enable(int on) {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  prof_clear();
  g_prof_on = on != 0;
}

int64_t rbc_profile_summary(char* buf, size_t len) {
  std::lock_guard<std::mutex> lock(g_prof_mu);
  struct Agg {
    int64_t count = 0;
    double ms = 0, bytes = 0, flops = 0;
  };
  std::vector<std::pair<std::string, Agg>> aggs;
  for (auto& r : g_prof) {
    if (!r.ev1) continue;
    if (cudaEventSynchronize(r.ev1) != cudaSuccess) continue;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.ev0, r.ev1);
    auto it = std::find_if(aggs.begin(), aggs.end(), [&](auto& p) { return p.first == r.name; });
    if (it == aggs.end()) {
      aggs.push_back({r.name, Agg{}});
      it = aggs.end() - 1;
    }
    it->second.count += 1;
    it->second.ms += ms;
    it->second.bytes += r.bytes;
    it->second.flops += r.flops;
  }
  std::string js = "{";
  char tmp[512];
  for (size_t i = 0; i < aggs.size(); ++i) {
    const Agg& a = aggs[i].second;
    snprintf(tmp, sizeof tmp, "%s\"%s\": {\"count\": %lld, \"ms\": %.6f, \"bytes\": %.6e, \"flops\": %.6e}",
             i ? ", " : "", aggs[i].first.c_str(), (long long)a.count, a.ms, a.bytes, a.flops);
    js += tmp;
  }
  js += "}";
  if (buf && len > 0) {
    const size_t n = std::min(len - 1, js.size());
    memcpy(buf, js.data(), n);
    buf[n] = 0;
  }
  return (int64_t)js.size() + 1;
}

const char* rbc_last_error(void) { return g_last_error.c_str(); }

int rbc_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

int rbc_release_device_memory(void) {
  std::lock_guard<std::mutex> lock(arena().mu);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail_cuda(e, "cudaDeviceSynchronize", __FILE__, __LINE__);
  Arena& A = arena();
  if (A.ptr) cudaFree(A.ptr);
  A.ptr = nullptr;
  A.cap = A.off = 0;
  ++A.gen;
  ++A.epoch;
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
    cudaMemPoolTrimTo(pool, 0);
  return RBC_OK;
}

size_t rbc_levels_workspace_bytes(int dtype, int Q, const int32_t* n, const int32_t* R, int64_t T,
                                  int64_t N) {
  Geometry g;
  if (make_geometry(Q, n, R, N, &g) != RBC_OK) return 0;
  return ws_for(g, dtype, T);
}

size_t rbc_plans_workspace_bytes(int dtype, int formula, int Q, int64_t T, int64_t N) {
  const int n = formula_n(formula), R = formula_R(formula);
  if (!n || Q < 1) return 0;
  std::vector<int32_t> nv(Q, n), Rv(Q, R);
  return rbc_levels_workspace_bytes(dtype, Q, nv.data(), Rv.data(), T, N);
}

int rbc_apply_levels_async(int dtype, int Q, const int32_t* n, const int32_t* R, const int64_t* Tc,
                           const void* const* u, const void* const* v, const void* const* w,
                           int64_t T0, int64_t N, const void* a, const void* b, int64_t T, void* out,
                           uint8_t* nonfinite, void* workspace, size_t workspace_bytes,
                           void* stream) {
  if (dtype < 0 || dtype > 2) return set_error(RBC_EVALUE, "bad dtype %d", dtype);
  Geometry g;
  RBC_TRY(make_geometry(Q, n, R, N, &g));
  RBC_TRY(validate_trials(T, T0));
  PassArgs p;
  p.dtype = dtype;
  p.plan = false;
  p.formula = 0;
  p.plans = nullptr;
  p.Tp = 1;
  for (int q = 0; q < Q; ++q) {
    if (n[q] > 8) return set_error(RBC_EUNSUPPORTED, "block grids above 8x8 are not supported");
    if (!(Tc[q] == 1 || Tc[q] == T)) return set_error(RBC_EVALUE, "coefficient trials do not broadcast");
    p.u.push_back(u[q]);
    p.v.push_back(v[q]);
    p.w.push_back(w[q]);
    p.Tc.push_back(Tc[q]);
  }
  p.T0 = T0;
  p.T = T;
  p.a = a;
  p.b = b;
  p.out = out;
  p.nonfinite = nonfinite;
  return run_pass(g, p, workspace, workspace_bytes, (cudaStream_t)stream);
}

int rbc_apply_plans_async(int dtype, int formula, int Q, int64_t Tp, const void* packed_plans,
                          int64_t T0, int64_t N, const void* a, const void* b, int64_t T, void* out,
                          uint8_t* nonfinite, void* workspace, size_t workspace_bytes,
                          void* stream) {
  if (dtype < 0 || dtype > 2) return set_error(RBC_EVALUE, "bad dtype %d", dtype);
  const int n = formula_n(formula), R = formula_R(formula);
  if (!n) return set_error(RBC_EVALUE, "unknown formula id %d", formula);
  if (Q < 1) return set_error(RBC_EVALUE, "need at least one level");
  std::vector<int32_t> nv(Q, n), Rv(Q, R);
  Geometry g;
  RBC_TRY(make_geometry(Q, nv.data(), Rv.data(), N, &g));
  RBC_TRY(validate_trials(T, T0));
  if (!(Tp == 1 || Tp == T)) return set_error(RBC_EVALUE, "plan trials do not broadcast");
  PassArgs p;
  p.dtype = dtype;
  p.plan = true;
  p.formula = formula;
  p.plans = (const PlanLevel*)packed_plans;
  p.Tp = Tp;
  p.T0 = T0;
  p.T = T;
  p.a = a;
  p.b = b;
  p.out = out;
  p.nonfinite = nonfinite;
  return run_pass(g, p, workspace, workspace_bytes, (cudaStream_t)stream);
}

int rbc_pack_plans(int n, int64_t count, const int64_t* perms, const double* signs, void* packed) {
  if (n < 1 || n > kMaxPlanN) return set_error(RBC_EVALUE, "plan grid n=%d unsupported (max %d)", n, kMaxPlanN);
  PlanLevel* out = (PlanLevel*)packed;
  for (int64_t c = 0; c < count; ++c) {
    PlanLevel pl;
    memset(&pl, 0, sizeof pl);
    for (int i = 0; i < 3; ++i) {
      int seen = 0;
      for (int j = 0; j < n; ++j) {
        const int64_t pj = perms[(c * 3 + i) * n + j];
        const double sj = signs[(c * 3 + i) * n + j];
        if (pj < 0 || pj >= n || (seen >> pj) & 1)
          return set_error(RBC_EVALUE, "each perms row must be a permutation of 0..n-1");
        if (!(sj == 1.0 || sj == -1.0)) return set_error(RBC_EVALUE, "signs must be +1 or -1");
        seen |= 1 << pj;
        pl.perm[i][j] = (int8_t)pj;
        pl.inv[i][pj] = (int8_t)j;
        pl.neg[i][j] = sj < 0 ? 1 : 0;
      }
    }
    out[c] = pl;
  }
  return RBC_OK;
}

int rbc_leaf_matmul_async(int dtype_in, int dtype_out, int64_t batch, int64_t xs, int64_t ys,
                          int64_t M, int64_t K, int64_t N, const void* x, const void* y, void* out,
                          void* stream) {
  if (K == 0) return set_error(RBC_EVALUE, "empty shared dimension is handled by the caller");
  cudaError_t e = launch_leaf(dtype_in, dtype_out, batch, M, K, N, x, xs, y, ys, out,
                              (cudaStream_t)stream);
  if (e != cudaSuccess) return fail_cuda(e, "leaf", __FILE__, __LINE__);
  return RBC_OK;
}

int rbc_truth_async(int dtype_in, int64_t T, int64_t N, const void* a, const void* b, double* ref,
                    void* stream) {
  if (N == 0 || T == 0) return RBC_OK;
  cudaError_t e = launch_leaf(dtype_in, kF64, T, N, N, N, a, N * N, b, N * N, ref,
                              (cudaStream_t)stream);
  if (e != cudaSuccess) return fail_cuda(e, "truth", __FILE__, __LINE__);
  return RBC_OK;
}

int rbc_matgen(int kind, int dtype, int64_t count, int64_t n, const uint64_t* keys,
               const int32_t* which, void* out, uint8_t* nonfinite, void* stream) {
  if (kind < kMatGaussian || kind > kMatQuadrant100)
    return set_error(RBC_EVALUE, "unknown matrix kind %d", kind);
  if (dtype != kF64 && dtype != kF32 && dtype != kF16)
    return set_error(RBC_EVALUE, "unknown dtype %d", dtype);
  if (count < 0 || n < 0 || count > 65535)
    return set_error(RBC_EVALUE, "matrix count %lld / size %lld out of range", (long long)count,
                     (long long)n);
  if (count == 0 || n == 0) return RBC_OK;
  if (n > (int64_t)1 << 24) return set_error(RBC_EVALUE, "matrix size %lld too large", (long long)n);
  for (int64_t c = 0; c < count; ++c)
    if (which[c] != 0 && which[c] != 1) return set_error(RBC_EVALUE, "which must be 0 (A) or 1 (B)");
  return matgen(kind, dtype, count, n, keys, which, out, nonfinite, (cudaStream_t)stream);
}

size_t rbc_rel_errors_scratch_bytes(int64_t T) { return error_scratch_bytes(T); }

int rbc_rel_errors_async(int dtype, int64_t T, int64_t N, const void* c, const double* ref,
                         int64_t ref_tstride, double* err, void* scratch, void* stream) {
  if (T == 0) return RBC_OK;
  cudaError_t e = launch_rel_errors(dtype, T, N * N, c, ref, ref_tstride, err, scratch,
                                    (cudaStream_t)stream);
  if (e != cudaSuccess) return fail_cuda(e, "rel_errors", __FILE__, __LINE__);
  return RBC_OK;
}

int rbc_sum_trials_async(int dtype, int64_t T, int64_t N, const void* x, double* total,
                         void* stream) {
  if (T == 0 || N == 0) return RBC_OK;
  cudaError_t e = launch_sum_trials(dtype, T, N * N, x, total, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail_cuda(e, "sum_trials", __FILE__, __LINE__);
  return RBC_OK;
}

int rbc_nonfinite_async(int dtype, int64_t T, int64_t N, const void* x, uint8_t* nonfinite,
                        void* stream) {
  if (T == 0) return RBC_OK;
  cudaError_t e = cudaMemsetAsync(nonfinite, 0, (size_t)T, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail_cuda(e, "memset", __FILE__, __LINE__);
  if (N == 0) return RBC_OK;
  e = launch_nonfinite(dtype, T, N * N, x, nonfinite, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail_cuda(e, "nonfinite", __FILE__, __LINE__);
  return RBC_OK;
}

// ------------------------------------------------------- host-buffer API --

static int finish_sync(int rc) {
  if (rc != RBC_OK) return rc;
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail_cuda(e, "cudaDeviceSynchronize", __FILE__, __LINE__);
  return RBC_OK;
}

int rbc_apply_levels(int dtype, int Q, const int32_t* n, const int32_t* R, const int64_t* Tc,
                     const void* const* u, const void* const* v, const void* const* w, int64_t T0,
                     int64_t N, const void* a, const void* b, int64_t T, void* out,
                     uint64_t* leaf_multiplies) {
  if (dtype < 0 || dtype > 2) return set_error(RBC_EVALUE, "bad dtype %d", dtype);
  Geometry g;
  RBC_TRY(make_geometry(Q, n, R, N, &g));
  RBC_TRY(validate_trials(T, T0));
  for (int q = 0; q < Q; ++q) {
    if (!(Tc[q] == 1 || Tc[q] == T)) return set_error(RBC_EVALUE, "coefficient trials do not broadcast");
    if (n[q] > 8) return set_error(RBC_EUNSUPPORTED, "block grids above 8x8 are not supported");
  }
  RBC_TRY(check_device());
  const size_t es = dtype_size(dtype);
  const int64_t N2 = N * N;
  std::lock_guard<std::mutex> lock(arena().mu);
  size_t fixed = align_up(T0 * N2 * es) * 2 + align_up(T * N2 * es) + align_up(T) + 4096;
  std::vector<size_t> cbytes(Q);
  for (int q = 0; q < Q; ++q) {
    cbytes[q] = (size_t)Tc[q] * R[q] * n[q] * n[q] * es;
    fixed += 3 * align_up(cbytes[q]);
  }
  const size_t ptw = per_trial_ws(g, dtype);
  size_t ws_bytes = host_ws_budget(fixed, ws_for(g, dtype, std::max<int64_t>(T, 1)));
  if (ptw && ws_bytes < ws_for(g, dtype, 1)) return set_error(RBC_ERUNTIME, "not enough device memory for one trial");
  RBC_TRY(arena().reserve(fixed + ws_bytes + 256));
  Arena& A = arena();
  void* da = A.take(T0 * N2 * es);
  void* db = A.take(T0 * N2 * es);
  void* dout = A.take(T * N2 * es);
  uint8_t* dnf = (uint8_t*)A.take((size_t)std::max<int64_t>(T, 1));
  std::vector<const void*> du(Q), dv(Q), dw(Q);
  for (int q = 0; q < Q; ++q) {
    void* pu = A.take(cbytes[q]);
    void* pv = A.take(cbytes[q]);
    void* pw = A.take(cbytes[q]);
    CUDA_TRY(cudaMemcpy(pu, u[q], cbytes[q], cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(pv, v[q], cbytes[q], cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(pw, w[q], cbytes[q], cudaMemcpyHostToDevice));
    du[q] = pu;
    dv[q] = pv;
    dw[q] = pw;
  }
  void* dws = A.take(ws_bytes);
  CUDA_TRY(cudaMemcpy(da, a, T0 * N2 * es, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(db, b, T0 * N2 * es, cudaMemcpyHostToDevice));
  RBC_TRY(finish_sync(rbc_apply_levels_async(dtype, Q, n, R, Tc, du.data(), dv.data(), dw.data(),
                                             T0, N, da, db, T, dout, dnf, dws, ws_bytes, nullptr)));
  if (leaf_multiplies) *leaf_multiplies += (uint64_t)T * (uint64_t)g.leaves;
  std::vector<uint8_t> nf((size_t)T);
  if (T) CUDA_TRY(cudaMemcpy(nf.data(), dnf, (size_t)T, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(out, dout, T * N2 * es, cudaMemcpyDeviceToHost));
  for (int64_t t = 0; t < T; ++t)
    if (nf[t]) return set_error(RBC_EOVERFLOW, "non-finite result in trial %lld", (long long)t);
  return RBC_OK;
}

int rbc_apply_plans(int dtype, int formula, int Q, int64_t Tp, const void* packed_plans,
                    int64_t T0, int64_t N, const void* a, const void* b, int64_t T, void* out,
                    uint8_t* nonfinite, uint64_t* leaf_multiplies) {
  const int n = formula_n(formula), R = formula_R(formula);
  if (!n) return set_error(RBC_EVALUE, "unknown formula id %d", formula);
  if (Q < 1) return set_error(RBC_EVALUE, "need at least one level");
  std::vector<int32_t> nv(Q, n), Rv(Q, R);
  Geometry g;
  RBC_TRY(make_geometry(Q, nv.data(), Rv.data(), N, &g));
  RBC_TRY(validate_trials(T, T0));
  if (!(Tp == 1 || Tp == T)) return set_error(RBC_EVALUE, "plan trials do not broadcast");
  RBC_TRY(check_device());
  const size_t es = dtype_size(dtype);
  const int64_t N2 = N * N;
  std::lock_guard<std::mutex> lock(arena().mu);
  const size_t pbytes = (size_t)Tp * Q * sizeof(PlanLevel);
  size_t fixed = align_up(T0 * N2 * es) * 2 + align_up(T * N2 * es) + align_up(T) +
                 align_up(pbytes) + 4096;
  const size_t ptw = per_trial_ws(g, dtype);
  size_t ws_bytes = host_ws_budget(fixed, ws_for(g, dtype, std::max<int64_t>(T, 1)));
  if (ptw && ws_bytes < ws_for(g, dtype, 1)) return set_error(RBC_ERUNTIME, "not enough device memory for one trial");
  RBC_TRY(arena().reserve(fixed + ws_bytes + 256));
  Arena& A = arena();
  void* da = A.take(T0 * N2 * es);
  void* db = A.take(T0 * N2 * es);
  void* dout = A.take(T * N2 * es);
  uint8_t* dnf = (uint8_t*)A.take((size_t)std::max<int64_t>(T, 1));
  void* dpl = A.take(pbytes);
  void* dws = A.take(ws_bytes);
  CUDA_TRY(cudaMemcpy(dpl, packed_plans, pbytes, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(da, a, T0 * N2 * es, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(db, b, T0 * N2 * es, cudaMemcpyHostToDevice));
  RBC_TRY(finish_sync(rbc_apply_plans_async(dtype, formula, Q, Tp, dpl, T0, N, da, db, T, dout,
                                            dnf, dws, ws_bytes, nullptr)));
  if (leaf_multiplies) *leaf_multiplies += (uint64_t)T * (uint64_t)g.leaves;
  std::vector<uint8_t> nf((size_t)T);
  if (T) CUDA_TRY(cudaMemcpy(nf.data(), dnf, (size_t)T, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(out, dout, T * N2 * es, cudaMemcpyDeviceToHost));
  bool any = false;
  for (int64_t t = 0; t < T; ++t) {
    if (nonfinite) nonfinite[t] = nf[t];
    any = any || nf[t];
  }
  if (any) return set_error(RBC_EOVERFLOW, "non-finite result");
  return RBC_OK;
}

// Diagonal rescaling baseline (reference rescale.py:60-99), device-resident:
// one H2D per operand, the scaling steps (rescale.cu), the deterministic
// recursion (plan path with identity plans for the exact +-1 formulas, dense
// tables otherwise; Q = 0 is the standard product), the restores, one D2H.
int rbc_rescaled_multiply(int dtype, int formula, int Q, const int32_t* n, const int32_t* R,
                          const void* const* u, const void* const* v, const void* const* w,
                          int nsteps, const int32_t* steps, int64_t N, const void* a,
                          const void* b, void* out) {
  if (dtype < 0 || dtype > 2) return set_error(RBC_EVALUE, "bad dtype %d", dtype);
  if (Q < 0 || N < 0 || nsteps < 0) return set_error(RBC_EVALUE, "negative size");
  for (int i = 0; i < nsteps; ++i)
    if (steps[i] != 0 && steps[i] != 1) return set_error(RBC_EVALUE, "unknown schedule step");
  std::vector<int32_t> nv, Rv;
  if (formula > 0) {
    if (!formula_n(formula)) return set_error(RBC_EVALUE, "unknown formula id %d", formula);
    nv.assign(Q, formula_n(formula));
    Rv.assign(Q, formula_R(formula));
  } else {
    nv.assign(n, n + Q);
    Rv.assign(R, R + Q);
  }
  Geometry g;
  if (Q > 0) {
    RBC_TRY(make_geometry(Q, nv.data(), Rv.data(), N, &g));
    for (int q = 0; q < Q; ++q)
      if (nv[q] > 8) return set_error(RBC_EUNSUPPORTED, "block grids above 8x8 are not supported");
  }
  RBC_TRY(check_device());
  if (N == 0) return RBC_OK;
  const size_t es = dtype_size(dtype);
  const size_t N2b = (size_t)N * N * es, vb = (size_t)N * es;
  std::lock_guard<std::mutex> lock(arena().mu);
  std::vector<size_t> cbytes(Q, 0);
  size_t fixed = 3 * align_up(N2b) + (size_t)4 * nsteps * align_up(vb) + align_up(2 * nsteps + 1) +
                 align_up(absmax_scratch_bytes(N)) + align_up((size_t)Q * RBC_PLAN_BYTES + 1) + 4096;
  if (formula <= 0)
    for (int q = 0; q < Q; ++q) {
      cbytes[q] = (size_t)Rv[q] * nv[q] * nv[q] * es;
      fixed += 3 * align_up(cbytes[q]);
    }
  const size_t ws_want = Q > 0 ? ws_for(g, dtype, 1) : 0;
  const size_t ws_bytes = host_ws_budget(fixed, ws_want);
  if (ws_bytes < ws_want) return set_error(RBC_ERUNTIME, "not enough device memory for one trial");
  RBC_TRY(arena().reserve(fixed + ws_bytes + 256));
  Arena& A = arena();
  void* dA = A.take(N2b);
  void* dB = A.take(N2b);
  void* dC = A.take(N2b);
  std::vector<void*> vec((size_t)4 * nsteps);
  for (auto& p : vec) p = A.take(vb);
  uint8_t* flags = (uint8_t*)A.take(2 * nsteps + 1);  // [2 s], [2 s + 1]: zero maxima; [2n]: overflow
  void* scratch = A.take(absmax_scratch_bytes(N));
  void* dplans = A.take((size_t)Q * RBC_PLAN_BYTES + 1);
  std::vector<const void*> du(Q), dv(Q), dw(Q);
  if (formula <= 0)
    for (int q = 0; q < Q; ++q) {
      void* pu = A.take(cbytes[q]);
      void* pv = A.take(cbytes[q]);
      void* pw = A.take(cbytes[q]);
      CUDA_TRY(cudaMemcpy(pu, u[q], cbytes[q], cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(pv, v[q], cbytes[q], cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(pw, w[q], cbytes[q], cudaMemcpyHostToDevice));
      du[q] = pu;
      dv[q] = pv;
      dw[q] = pw;
    }
  void* dws = A.take(ws_bytes);
  cudaStream_t st = nullptr;
  CUDA_TRY(cudaMemcpy(dA, a, N2b, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dB, b, N2b, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemsetAsync(flags, 0, 2 * nsteps + 1, st));
  // schedule (rescale.py:84-97)
  std::vector<std::pair<const void*, const void*>> restore;
  for (int i = 0; i < nsteps; ++i) {
    void** vv = vec.data() + 4 * i;
    if (steps[i] == 0) {  // outside: da = rowmax|A|, db = colmax|B|; A = diag(1/da) A, B = B diag(1/db)
      CUDA_TRY(launch_absmax(dtype, dA, N, 1, vv[0], flags + 2 * i, scratch, st));
      CUDA_TRY(launch_absmax(dtype, dB, N, 0, vv[1], flags + 2 * i + 1, scratch, st));
      CUDA_TRY(launch_recip(dtype, vv[0], N, vv[2], st));
      CUDA_TRY(launch_recip(dtype, vv[1], N, vv[3], st));
      ScaleList ra{{vv[2]}, {nullptr}, 1}, cb{{nullptr}, {vv[3]}, 1};
      CUDA_TRY(launch_scale(dtype, dA, N, ra, st));
      CUDA_TRY(launch_scale(dtype, dB, N, cb, st));
      restore.emplace_back(vv[0], vv[1]);
    } else {  // inside: d = sqrt(rowmax|B| / colmax|A|); A = A diag(d), B = diag(1/d) B
      CUDA_TRY(launch_absmax(dtype, dB, N, 1, vv[0], flags + 2 * i, scratch, st));
      CUDA_TRY(launch_absmax(dtype, dA, N, 0, vv[1], flags + 2 * i + 1, scratch, st));
      CUDA_TRY(launch_inside_factors(dtype, vv[0], vv[1], N, vv[2], vv[3], st));
      ScaleList ca{{nullptr}, {vv[2]}, 1}, rb{{vv[3]}, {nullptr}, 1};
      CUDA_TRY(launch_scale(dtype, dA, N, ca, st));
      CUDA_TRY(launch_scale(dtype, dB, N, rb, st));
    }
  }
  std::vector<uint8_t> hf(2 * nsteps + 1, 0);
  if (nsteps) {
    CUDA_TRY(cudaMemcpy(hf.data(), flags, 2 * nsteps, cudaMemcpyDeviceToHost));
    // the reference's check order: within a step the row maxima (of A for
    // outside, of B for inside) are checked before the column maxima
    for (int i = 0; i < nsteps; ++i) {
      if (hf[2 * i]) return set_error(RBC_EVALUE, "degenerate input: zero row maximum");
      if (hf[2 * i + 1]) return set_error(RBC_EVALUE, "degenerate input: zero column maximum");
    }
  }
  // the deterministic recursion (rescale.py:95, multiply.py:72-99)
  uint8_t* nf = flags + 2 * nsteps;
  if (Q == 0) {  // standard_multiply: no finiteness check (multiply.py:44-51)
    CUDA_TRY(launch_leaf(dtype, dtype, 1, N, N, N, dA, 0, dB, 0, dC, st));
  } else if (formula > 0) {
    std::vector<PlanLevel> ident(Q);
    const int nn = nv[0];
    for (int q = 0; q < Q; ++q) {
      memset(&ident[q], 0, sizeof(PlanLevel));
      for (int r = 0; r < 3; ++r)
        for (int j = 0; j < nn; ++j) ident[q].perm[r][j] = ident[q].inv[r][j] = (int8_t)j;
    }
    CUDA_TRY(cudaMemcpy(dplans, ident.data(), (size_t)Q * sizeof(PlanLevel), cudaMemcpyHostToDevice));
    RBC_TRY(rbc_apply_plans_async(dtype, formula, Q, 1, dplans, 1, N, dA, dB, 1, dC, nf, dws,
                                  ws_bytes, st));
  } else {
    std::vector<int64_t> Tc(Q, 1);
    RBC_TRY(rbc_apply_levels_async(dtype, Q, nv.data(), Rv.data(), Tc.data(), du.data(), dv.data(),
                                   dw.data(), 1, N, dA, dB, 1, dC, nf, dws, ws_bytes, st));
  }
  CUDA_TRY(cudaMemcpy(&hf[2 * nsteps], nf, 1, cudaMemcpyDeviceToHost));
  if (hf[2 * nsteps]) return set_error(RBC_EOVERFLOW, "non-finite result");
  // restores in reverse schedule order (rescale.py:96-98), one pass
  for (size_t k0 = 0; k0 < restore.size(); k0 += 8) {
    ScaleList sl{};
    for (size_t k = k0; k < restore.size() && k < k0 + 8; ++k) {
      const auto& rv = restore[restore.size() - 1 - k];
      sl.row[sl.n] = rv.first;
      sl.col[sl.n] = rv.second;
      ++sl.n;
    }
    CUDA_TRY(launch_scale(dtype, dC, N, sl, st));
  }
  CUDA_TRY(cudaMemcpy(out, dC, N2b, cudaMemcpyDeviceToHost));
  return RBC_OK;
}

int rbc_rel_errors(int dtype, int64_t T, int64_t N, const void* c, const double* ref,
                   int64_t ref_tstride, double* err) {
  if (dtype < 0 || dtype > 2) return set_error(RBC_EVALUE, "bad dtype %d", dtype);
  if (ref_tstride != 0 && ref_tstride != N * N)
    return set_error(RBC_EVALUE, "ref_tstride must be 0 or N*N");
  if (T == 0) return RBC_OK;
  RBC_TRY(check_device());
  const size_t N2 = (size_t)N * N;
  const size_t cb = (size_t)T * N2 * dtype_size(dtype);
  const size_t rb = (ref_tstride ? (size_t)T : 1) * N2 * sizeof(double);
  const size_t eb = (size_t)T * sizeof(double);
  const size_t sb = error_scratch_bytes(T);
  std::lock_guard<std::mutex> lock(arena().mu);
  RBC_TRY(arena().reserve(align_up(cb) + align_up(rb) + align_up(eb) + align_up(sb) + 1024));
  Arena& A = arena();
  void* dc = A.take(cb);
  double* dref = (double*)A.take(rb);
  double* derr = (double*)A.take(eb);
  void* dscratch = A.take(sb);
  CUDA_TRY(cudaMemcpy(dc, c, cb, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dref, ref, rb, cudaMemcpyHostToDevice));
  RBC_TRY(finish_sync(rbc_rel_errors_async(dtype, T, N, dc, dref, ref_tstride, derr, dscratch, nullptr)));
  CUDA_TRY(cudaMemcpy(err, derr, eb, cudaMemcpyDeviceToHost));
  return RBC_OK;
}

int rbc_leaf_matmul(int dtype, int64_t batch, int64_t xs, int64_t ys, int64_t M, int64_t K,
                    int64_t N, const void* x, const void* y, void* out) {
  if (dtype < 0 || dtype > 2) return set_error(RBC_EVALUE, "bad dtype %d", dtype);
  if (K == 0) return set_error(RBC_EVALUE, "empty shared dimension is handled by the caller");
  RBC_TRY(check_device());
  const size_t es = dtype_size(dtype);
  const size_t xb = (size_t)(xs ? batch : 1) * M * K * es;
  const size_t yb = (size_t)(ys ? batch : 1) * K * N * es;
  const size_t ob = (size_t)batch * M * N * es;
  std::lock_guard<std::mutex> lock(arena().mu);
  RBC_TRY(arena().reserve(align_up(xb) + align_up(yb) + align_up(ob) + 1024));
  Arena& A = arena();
  void* dx = A.take(xb);
  void* dy = A.take(yb);
  void* dout = A.take(ob);
  CUDA_TRY(cudaMemcpy(dx, x, xb, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaMemcpy(dy, y, yb, cudaMemcpyHostToDevice));
  RBC_TRY(finish_sync(rbc_leaf_matmul_async(dtype, dtype, batch, xs, ys, M, K, N, dx, dy, dout, nullptr)));
  CUDA_TRY(cudaMemcpy(out, dout, ob, cudaMemcpyDeviceToHost));
  return RBC_OK;
}

static cudaStream_t make_stream() {
  cudaStream_t x = nullptr;
  cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
  return x;
}

static cudaStream_t host_stream(int i = 0) {
  static cudaStream_t s[2] = {make_stream(), make_stream()};
  return s[i];
}

static cudaStream_t copy_stream(int i = 0) {
  static cudaStream_t s[2] = {make_stream(), make_stream()};
  return s[i];
}

constexpr int kSlots = 3;  // input slots of the host-buffer pipeline

static cudaEvent_t pipe_event(int i) {
  static cudaEvent_t ev[2 * kSlots + 1] = {nullptr};
  if (!ev[i]) cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
  return ev[i];
}

// Host-buffer error trials, pipelined: trials are cut into chunks; chunk k+1
// is copied host->device on a copy stream (into a ring of three input slots)
// while chunks k and k-1 compute on two alternating compute streams with
// their own workspaces, so the small per-chunk grids of consecutive chunks
// share the GPU.  With pinned host buffers the PCIe transfer hides behind the
// kernels.  (Measured and dropped in round 1: more slots, a second copy
// stream, ramped chunk sizes and per-chunk CUDA graphs -- all equal or
// slower.)
//
// The call comes in two halves so that the ring runs ACROSS calls:
// rbc_error_trials_begin enqueues a call's copies, kernels and result copies
// and returns; rbc_error_trials_end waits for them.  With a second call begun
// before the first is ended, its first chunks are copied while the first
// call's last chunks compute (a single call leaves the GPU idle for its first
// copy: 9.8 ms of config 5's 176 ms).  Two calls may be in flight; calls of
// one shape share the arena layout, a call of another shape -- or any other
// host-buffer API that takes the arena -- first waits for the calls in flight.
struct HostPipe {
  bool valid = false;
  unsigned epoch = 0;  // arena epoch of the layout
  int dtype = 0, formula = 0, Q = 0, with_det = 0, has_plans = 0;
  int64_t T = 0, N = 0, C = 0;
  int64_t k = 0;       // chunks enqueued on this layout (ring position)
  int64_t serial = 0;  // tickets handed out
  bool busy[2] = {false, false};
  int64_t ticket[2] = {-1, -1};
  void* da[kSlots];
  void* dbb[kSlots];
  void* dpl[kSlots];
  void* ddet = nullptr;
  void* dws[2] = {nullptr, nullptr};
  size_t ws = 0;
  double* derr_r[2];
  double* derr_d[2];
  uint8_t* dnf_r[2];
  uint8_t* dnf_d[2];
};

static HostPipe& host_pipe() {
  static HostPipe p;
  return p;
}

static cudaEvent_t done_event(int i) {
  static cudaEvent_t ev[2] = {nullptr, nullptr};
  if (!ev[i]) cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
  return ev[i];
}

// everything a begun call queued has run (arena lock held by the caller)
static void drain_host_pipe() {
  HostPipe& P = host_pipe();
  if (!P.busy[0] && !P.busy[1] && !P.valid) return;
  cudaStreamSynchronize(copy_stream(0));
  cudaStreamSynchronize(host_stream(0));
  cudaStreamSynchronize(host_stream(1));
  cudaStreamSynchronize(copy_stream(1));
}

int rbc_error_trials_begin(int dtype, int formula, int Q, int64_t T, int64_t N, const void* a,
                           const void* b, const void* rand_plans, int with_det, double* err_rand,
                           double* err_det, uint8_t* nf_rand, uint8_t* nf_det, int64_t* ticket) {
  if (!ticket) return set_error(RBC_EVALUE, "ticket pointer is null");
  *ticket = -1;
  if (dtype < 0 || dtype > 2) return set_error(RBC_EVALUE, "bad dtype %d", dtype);
  const int n = formula_n(formula);
  if (!n) return set_error(RBC_EVALUE, "unknown formula id %d", formula);
  if (Q < 1) return set_error(RBC_EVALUE, "need at least one level");
  if (T < 0 || N < 0) return set_error(RBC_EVALUE, "negative size");
  {
    int64_t s = N;
    for (int q = 0; q < Q; ++q) {
      if (s % n) return set_error(RBC_EVALUE, "operand size not divisible by block grid");
      s /= n;
    }
  }
  if (!rand_plans && !with_det) return set_error(RBC_EVALUE, "no product requested");
  RBC_TRY(check_device());
  std::lock_guard<std::mutex> lock(arena().mu);
  HostPipe& P = host_pipe();
  if (P.busy[0] && P.busy[1]) return set_error(RBC_EVALUE, "two host-buffer calls already in flight");
  const int slotp = P.busy[(int)(P.serial & 1)] ? (int)((P.serial + 1) & 1) : (int)(P.serial & 1);
  if (T == 0 || N == 0) {  // nothing to do: a ticket that is already complete
    P.busy[slotp] = true;
    P.ticket[slotp] = P.serial;
    *ticket = P.serial++;
    cudaEventRecord(done_event(slotp), copy_stream(1));
    return RBC_OK;
  }
  const size_t es = dtype_size(dtype);
  const size_t N2 = (size_t)N * N;
  const size_t db = (size_t)Q * RBC_PLAN_BYTES;
  // pipeline chunks: about 8 MB of operands per chunk, at most 16 (config 2
  // with two compute streams: 12 chunks 11.21 ms per call, 16: 11.20, 32:
  // 11.4)
  int64_t nchunks =
      std::min<int64_t>(16, std::max<int64_t>(1, (int64_t)(2 * T * N2 * es >> 23)));
  int64_t C = std::max<int64_t>(1, (T + nchunks - 1) / nchunks);
  if (C > 8) C = (C + 7) / 8 * 8;  // whole multiples of 8 trials keep grids regular
  // Two compute streams pay off for many small chunks (config 2: 1000 pairs
  // of 243); products of 512 and up are whole-GPU jobs per chunk, and their
  // truth scratch comes from the stream-ordered pool, which two streams
  // fragment (config 4 calls went from 24 to 24-80 ms): one stream there.
  const bool two = N < 512;
  if (!two) {
    // whole-GPU jobs per chunk: a chunk should fill about four waves of
    // 128 x 128 truth / leaf tiles, or its last wave runs half empty (config
    // 4, 256 tiles per product: chunks of 1 / 2 / 4 pairs 23.40 / 22.69 /
    // 22.18 ms per streamed call), while at least two chunks keep the copies
    // of a single call behind its kernels
    const int64_t tiles = ((N + 127) / 128) * ((N + 127) / 128);
    int64_t cmin = 1;
    while (cmin * tiles < 4 * 148) cmin *= 2;
    C = std::max(C, std::min(cmin, std::max<int64_t>(1, (T + 1) / 2)));
  }
  auto need = [&](int64_t c) {
    const size_t slot = 2 * align_up(c * N2 * es) + align_up(c * Q * RBC_PLAN_BYTES);
    return kSlots * slot + align_up(db) + 2 * (2 * align_up(T * 8) + 2 * align_up(T)) + 4096 +
           (two ? 2 : 1) * align_up(rbc_error_trials_workspace_bytes(dtype, formula, Q, c, N));
  };
  Arena& A = arena();
  cudaStream_t scs[2] = {host_stream(0), host_stream(1)};
  cudaStream_t sc = scs[0];
  cudaStream_t sx = copy_stream(0);
  cudaStream_t sr = copy_stream(1);  // result copies
  const bool same = P.valid && P.epoch == A.epoch && P.dtype == dtype && P.formula == formula &&
                    P.Q == Q && P.T == T && P.N == N && P.with_det == with_det &&
                    P.has_plans == (rand_plans != nullptr);
  if (!same) {
    // The device memory query runs only when the arena must grow: in steady
    // state an earlier call's arena already holds this chunking, and
    // cudaMemGetInfo can stall the host for tens of ms behind concurrent
    // driver queries (NVML polling; a host phase trace showed 31 and 97 ms
    // "setup" phases in 30 calls).
    if (need(C) > A.cap) {
      drain_host_pipe();
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      const size_t budget = (size_t)((double)(free_b + A.cap) * 0.85);
      while (C > 1 && need(C) > budget) C = (C + 1) / 2;
      if (need(C) > budget) return set_error(RBC_ERUNTIME, "not enough device memory for one trial");
    }
    P.valid = false;
    RBC_TRY(A.reserve(need(C) + 256));  // waits for calls in flight (Arena::drain)
    for (int k = 0; k < kSlots; ++k) {
      P.da[k] = A.take(C * N2 * es);
      P.dbb[k] = A.take(C * N2 * es);
      P.dpl[k] = A.take(C * Q * RBC_PLAN_BYTES);
    }
    P.ddet = A.take(db);
    for (int h = 0; h < 2; ++h) {
      P.derr_r[h] = (double*)A.take(T * 8);
      P.derr_d[h] = (double*)A.take(T * 8);
      P.dnf_r[h] = (uint8_t*)A.take(T);
      P.dnf_d[h] = (uint8_t*)A.take(T);
    }
    P.ws = rbc_error_trials_workspace_bytes(dtype, formula, Q, C, N);
    P.dws[0] = A.take(P.ws);
    P.dws[1] = two ? A.take(P.ws) : nullptr;
    std::vector<PlanLevel> ident(Q);
    for (int q = 0; q < Q; ++q) {
      memset(&ident[q], 0, sizeof(PlanLevel));
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < n; ++j) ident[q].perm[i][j] = ident[q].inv[i][j] = (int8_t)j;
    }
    // the identity plans of the deterministic product: uploaded once per layout
    CUDA_TRY(cudaMemcpyAsync(P.ddet, ident.data(), db, cudaMemcpyHostToDevice, sc));
    CUDA_TRY(cudaStreamSynchronize(sc));  // ident is a local
    P.dtype = dtype, P.formula = formula, P.Q = Q, P.with_det = with_det;
    P.has_plans = rand_plans != nullptr;
    P.T = T, P.N = N, P.C = C, P.k = 0;
    P.epoch = A.epoch;
    P.valid = true;
    A.drain = drain_host_pipe;
  }
  C = P.C;
  // Chunk sizes: C, ..., C, then the remainder cut in halves (multiples of
  // 8): the copies are the critical path (PCIe), so after the last copy only
  // a small chunk is left to compute.
  std::vector<int64_t> sizes;
  {
    int64_t rem = T;
    while (rem > C) {
      sizes.push_back(C);
      rem -= C;
    }
    while (rem > 8) {
      const int64_t c = ((rem + 1) / 2 + 7) / 8 * 8;
      sizes.push_back(std::min(c, rem));
      rem -= std::min(c, rem);
    }
    if (rem > 0) sizes.push_back(rem);
  }
  double* derr_r = P.derr_r[slotp];
  double* derr_d = P.derr_d[slotp];
  uint8_t* dnf_r = P.dnf_r[slotp];
  uint8_t* dnf_d = P.dnf_d[slotp];
  auto enqueue = [&]() -> int {
    int64_t t0 = 0;
    for (int64_t i = 0; i < (int64_t)sizes.size(); t0 += sizes[i], ++i, ++P.k) {
      const int64_t nt = sizes[i];
      const int64_t k = P.k;  // ring position, continuing across calls
      const int slot = (int)(k % kSlots);
      const int lane = two ? (int)(k & 1) : 0;
      cudaStream_t sk = scs[lane];
      cudaEvent_t copied = pipe_event(slot), computed = pipe_event(kSlots + slot);
      if (k >= kSlots) CUDA_TRY(cudaStreamWaitEvent(sx, computed, 0));  // slot free again
      CUDA_TRY(cudaMemcpyAsync(P.da[slot], (const char*)a + t0 * N2 * es, nt * N2 * es,
                               cudaMemcpyHostToDevice, sx));
      CUDA_TRY(cudaMemcpyAsync(P.dbb[slot], (const char*)b + t0 * N2 * es, nt * N2 * es,
                               cudaMemcpyHostToDevice, sx));
      if (rand_plans)
        CUDA_TRY(cudaMemcpyAsync(P.dpl[slot], (const char*)rand_plans + t0 * Q * RBC_PLAN_BYTES,
                                 nt * Q * RBC_PLAN_BYTES, cudaMemcpyHostToDevice, sx));
      CUDA_TRY(cudaEventRecord(copied, sx));
      CUDA_TRY(cudaStreamWaitEvent(sk, copied, 0));
      RBC_TRY(rbc_error_trials_async(dtype, formula, Q, nt, N, P.da[slot], P.dbb[slot],
                                     rand_plans ? P.dpl[slot] : nullptr,
                                     with_det ? P.ddet : nullptr, derr_r + t0, derr_d + t0,
                                     dnf_r + t0, dnf_d + t0, P.dws[lane], P.ws, sk));
      CUDA_TRY(cudaEventRecord(computed, sk));
    }
    // results: copied back on their own stream once both compute streams have
    // passed this call's chunks, so the next call's chunks queue right behind
    for (int l = 0; l < (two ? 2 : 1); ++l) {
      CUDA_TRY(cudaEventRecord(pipe_event(2 * kSlots), scs[l]));
      CUDA_TRY(cudaStreamWaitEvent(sr, pipe_event(2 * kSlots), 0));
    }
    if (rand_plans) {
      CUDA_TRY(cudaMemcpyAsync(err_rand, derr_r, T * 8, cudaMemcpyDeviceToHost, sr));
      if (nf_rand) CUDA_TRY(cudaMemcpyAsync(nf_rand, dnf_r, T, cudaMemcpyDeviceToHost, sr));
    }
    if (with_det) {
      CUDA_TRY(cudaMemcpyAsync(err_det, derr_d, T * 8, cudaMemcpyDeviceToHost, sr));
      if (nf_det) CUDA_TRY(cudaMemcpyAsync(nf_det, dnf_d, T, cudaMemcpyDeviceToHost, sr));
    }
    CUDA_TRY(cudaEventRecord(done_event(slotp), sr));
    return RBC_OK;
  };
  const int rc = enqueue();
  if (rc != RBC_OK) {
    // nothing that reads the caller's host buffers or the arena may stay
    // queued behind a failed call
    drain_host_pipe();
    P.valid = false;
    return rc;
  }
  P.busy[slotp] = true;
  P.ticket[slotp] = P.serial;
  *ticket = P.serial++;
  return RBC_OK;
}

int rbc_error_trials_end(int64_t ticket) {
  int slotp = -1;
  {
    std::lock_guard<std::mutex> lock(arena().mu);
    HostPipe& P = host_pipe();
    for (int h = 0; h < 2; ++h)
      if (P.busy[h] && P.ticket[h] == ticket) slotp = h;
  }
  if (slotp < 0) return set_error(RBC_EVALUE, "no host-buffer call in flight with that ticket");
  const cudaError_t e = cudaEventSynchronize(done_event(slotp));
  {
    std::lock_guard<std::mutex> lock(arena().mu);
    HostPipe& P = host_pipe();
    P.busy[slotp] = false;
    P.ticket[slotp] = -1;
    if (e != cudaSuccess) P.valid = false;
  }
  if (e != cudaSuccess) return fail_cuda(e, "host-buffer error trials", __FILE__, __LINE__);
  return RBC_OK;
}

int rbc_error_trials(int dtype, int formula, int Q, int64_t T, int64_t N, const void* a,
                     const void* b, const void* rand_plans, int with_det, double* err_rand,
                     double* err_det, uint8_t* nf_rand, uint8_t* nf_det) {
  int64_t ticket = -1;
  RBC_TRY(rbc_error_trials_begin(dtype, formula, Q, T, N, a, b, rand_plans, with_det, err_rand,
                                 err_det, nf_rand, nf_det, &ticket));
  return rbc_error_trials_end(ticket);
}

}  // extern "C"
