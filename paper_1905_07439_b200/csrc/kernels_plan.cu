// Plan-path combination kernels for exact +-1 formulas.
//
// Reference semantics (pkg/src/randbc/_engine.py:64-114 applied to the
// hatted tensors of randomize.py:163-178):
//   child_r(pos)      = sum_kl uh[r,k,l] X[k][l](pos),
//   uh[r,k,l]         = u[r, p1(k), p2(l)] s1(k) s2(l)
//   out[i][j](pos)    = sum_r wh[r,i,j] P_r(pos),
//   wh[r,i,j]         = w[r, p1(i), p3(j)] s1(i) s3(j)      (1/(1-kappa) == 1)
//
// Instead of multiplying by hatted coefficients, the expansion gathers the
// parent grid through the plan (G[k'][l'] = s1(k) s2(l) X[k][l] with
// k = p1^-1(k'), l = p2^-1(l'): a sign flip is exact) and runs the formula's
// generated base-coordinate network (formulas_gen.cuh); the contraction runs
// the base network and scatters base block (I, J) to hatted block
// (p1^-1(I), p3^-1(J)) with sign s1 s3.  Both are bitwise equal in value to
// the reference (see tools/gen_formulas.py for the fold-order argument).
//
// One thread handles W consecutive columns of one position of one parent
// block; memory traffic per thread is n*n loads + R stores (expand) or
// R loads + n*n stores (contract), all coalesced along block rows.

#include "formulas_gen.cuh"
#include "kernels.h"

#include <cstdlib>

namespace rbc {

namespace {

constexpr int kThreads = 256;
// CTA size of the lockstep (SYNC) two-level kernels (compile-time tuning knob;
// c2 expand2 at 128 threads: 0.415 vs 0.332 ms -- a bigger lockstep group
// writes longer runs of each output block)
#ifndef RBC_SYNC_THREADS
#define RBC_SYNC_THREADS 256
#endif
constexpr int kSyncThreads = RBC_SYNC_THREADS;

template <class F, class T, int W, int WHICH>
__global__ void __launch_bounds__(kThreads) expand_plan_kernel(
    const T* __restrict__ x, int64_t x_tstride, int K, int s, T* __restrict__ out,
    const PlanLevel* __restrict__ plans, int64_t plan_tstride, int level, int64_t ntr) {
  constexpr int n = F::n;
  constexpr int R = F::R;
  const int mb = s / n;
  const int P = (mb * mb) / W;             // packs per parent block
  const int64_t items = (int64_t)K * P;    // packs per trial
  const int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (e >= items) return;
  const int Kp = (int)(e / P);
  const int p = (int)(e - (int64_t)Kp * P);
  const int pos = p * W;
  const int i = pos / mb;
  const int j = pos - i * mb;
  constexpr int ri = WHICH == 0 ? 0 : 1;  // plan index permuting block rows
  constexpr int ci = WHICH == 0 ? 1 : 2;  // plan index permuting block cols
  using O = PackOps<T, W>;
  for (int64_t t = blockIdx.y; t < ntr; t += gridDim.y) {
    const PlanLevel& pl = plans[t * plan_tstride + level];
    const T* xb = x + t * x_tstride + (int64_t)Kp * s * s + (int64_t)i * s + j;
    Pack<T, W> g[n * n];
#pragma unroll
    for (int kb = 0; kb < n; ++kb) {
      const int hk = pl.inv[ri][kb];
#pragma unroll
      for (int lb = 0; lb < n; ++lb) {
        const int hl = pl.inv[ci][lb];
        const uint32_t m = sign_mask(pl.neg[ri][hk] ^ pl.neg[ci][hl]);
        g[kb * n + lb] = O::flip(pload<T, W>(xb + (int64_t)hk * mb * s + hl * mb), m);
      }
    }
    Pack<T, W> o[R];
    if (WHICH == 0)
      F::template expand_u<T, W>(g, o, pl.perm[ri][n - 1], pl.perm[ci][n - 1]);
    else
      F::template expand_v<T, W>(g, o, pl.perm[ri][n - 1], pl.perm[ci][n - 1]);
    T* ob = out + (t * K + Kp) * (int64_t)R * mb * mb + pos;
#pragma unroll
    for (int r = 0; r < R; ++r) pstore<T, W>(ob + (int64_t)r * mb * mb, o[r]);
  }
}

// Two expansion levels (q, q+1) in one pass: a thread owns one position of
// the level-(q+2) blocks under one level-q parent, loads the n^4 parent
// elements that feed it (read exactly once per trial, coalesced along rows),
// forms each level-(q+1) child r1 at its n*n sub-positions with the
// single-output network (expand_u1 / expand_v1: the same per-element fold as
// the full network), and expands those into the R grandchildren with the full
// network.  Both plans' gathers are folded into the load addresses (level
// q+1's permutation picks which sub-position feeds which network input; its
// sign is applied to the child value), so every register index is static.
// Values equal two expand_plan_kernel launches; the level-(q+1) array never
// goes through HBM.
// resident lockstep CTAs per SM the registers aim at (2: 128 registers,
// 0.357 vs 0.332 ms on c2 -- more CTAs per SM interleave more output blocks)
#ifndef RBC_EXPAND2_MINB
#define RBC_EXPAND2_MINB 1
#endif
template <class F, class T, int W, int WHICH, bool SYNC>
__global__ void __launch_bounds__(SYNC ? kSyncThreads : kThreads, SYNC ? RBC_EXPAND2_MINB : 1) expand2_plan_kernel(
    const T* __restrict__ x, int64_t x_tstride, int K, int s, T* __restrict__ out,
    const PlanLevel* __restrict__ plans, int64_t plan_tstride, int level, int64_t ntr) {
  constexpr int n = F::n;
  constexpr int R = F::R;
  constexpr int NN = n * n;
  const int mb1 = s / n, mb2 = mb1 / n;
  const int P = (mb2 * mb2) / W;
  const int64_t items = (int64_t)K * P;
  int64_t e = (int64_t)blockIdx.x * (SYNC ? kSyncThreads : kThreads) + threadIdx.x;
  const bool live = e < items;
  if (!SYNC && !live) return;
  if (!live) e = items - 1;  // SYNC: idle lanes mirror the last item, stores masked
  const int Kp = (int)(e / P);
  const int p = (int)(e - (int64_t)Kp * P);
  const int pos = p * W;
  const int i = pos / mb2;
  const int j = pos - i * mb2;
  constexpr int ri = WHICH == 0 ? 0 : 1;
  constexpr int ci = WHICH == 0 ? 1 : 2;
  using O = PackOps<T, W>;
  for (int64_t t = blockIdx.y; t < ntr; t += gridDim.y) {
    const PlanLevel& p0 = plans[t * plan_tstride + level];
    const PlanLevel& p1 = plans[t * plan_tstride + level + 1];
    const T* xb = x + t * x_tstride + (int64_t)Kp * s * s + (int64_t)i * s + j;
    Pack<T, W> g0[NN][NN];
    uint32_t m1[NN];
#pragma unroll
    for (int kb1 = 0; kb1 < n; ++kb1) {
      const int a = p1.inv[ri][kb1];
#pragma unroll
      for (int lb1 = 0; lb1 < n; ++lb1) {
        const int b = p1.inv[ci][lb1];
        m1[kb1 * n + lb1] = sign_mask(p1.neg[ri][a] ^ p1.neg[ci][b]);
        const T* xs = xb + (int64_t)a * mb2 * s + b * mb2;
#pragma unroll
        for (int kb0 = 0; kb0 < n; ++kb0) {
          const int hk = p0.inv[ri][kb0];
#pragma unroll
          for (int lb0 = 0; lb0 < n; ++lb0) {
            const int hl = p0.inv[ci][lb0];
            const uint32_t m0 = sign_mask(p0.neg[ri][hk] ^ p0.neg[ci][hl]);
            g0[kb1 * n + lb1][kb0 * n + lb0] =
                O::flip(pload<T, W>(xs + (int64_t)hk * mb1 * s + hl * mb1), m0);
          }
        }
      }
    }
    const int l0r = p0.perm[ri][n - 1], l0c = p0.perm[ci][n - 1];
    const int l1r = p1.perm[ri][n - 1], l1c = p1.perm[ci][n - 1];
    T* ob = out + (t * K + Kp) * (int64_t)R * R * mb2 * mb2 + pos;
#pragma unroll
    for (int r1 = 0; r1 < R; ++r1) {
      Pack<T, W> g1[NN];
#pragma unroll
      for (int q = 0; q < NN; ++q) {
        const Pack<T, W> v = WHICH == 0 ? F::template expand_u1<T, W>(g0[q], r1, l0r, l0c)
                                        : F::template expand_v1<T, W>(g0[q], r1, l0r, l0c);
        g1[q] = O::flip(v, m1[q]);
      }
      Pack<T, W> o[R];
      if (WHICH == 0)
        F::template expand_u<T, W>(g1, o, l1r, l1c);
      else
        F::template expand_v<T, W>(g1, o, l1r, l1c);
      if (live) {
#pragma unroll
        for (int r2 = 0; r2 < R; ++r2) pstore<T, W>(ob + (int64_t)(r1 * R + r2) * mb2 * mb2, o[r2]);
      }
      // SYNC: the CTA writes the grandchildren of r1 together, so each output
      // block's lines are completed in one short window (write locality)
      if (SYNC) __syncthreads();
    }
  }
}

template <class F, class T, int W>
__global__ void __launch_bounds__(kThreads) contract_plan_kernel(
    const T* __restrict__ ch, int K, int mb, T* __restrict__ out,
    const PlanLevel* __restrict__ plans, int64_t plan_tstride, int level, int64_t ntr,
    uint8_t* __restrict__ nonfinite) {
  constexpr int n = F::n;
  constexpr int R = F::R;
  const int s = n * mb;
  const int P = (mb * mb) / W;
  const int64_t items = (int64_t)K * P;
  const int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (e >= items) return;
  const int Kp = (int)(e / P);
  const int p = (int)(e - (int64_t)Kp * P);
  const int pos = p * W;
  const int i = pos / mb;
  const int j = pos - i * mb;
  using O = PackOps<T, W>;
  for (int64_t t = blockIdx.y; t < ntr; t += gridDim.y) {
    const PlanLevel& pl = plans[t * plan_tstride + level];
    const T* cb = ch + (t * K + Kp) * (int64_t)R * mb * mb + pos;
    Pack<T, W> pr[R];
#pragma unroll
    for (int r = 0; r < R; ++r) pr[r] = pload<T, W>(cb + (int64_t)r * mb * mb);
    Pack<T, W> o[n * n];
    F::template contract_w<T, W>(pr, o);
    T* obase = out + (t * K + Kp) * (int64_t)s * s + (int64_t)i * s + j;
    bool ok = true;
#pragma unroll
    for (int I = 0; I < n; ++I) {
      const int hi = pl.inv[0][I];
#pragma unroll
      for (int J = 0; J < n; ++J) {
        const int hj = pl.inv[2][J];
        const Pack<T, W> val = O::flip(o[I * n + J], sign_mask(pl.neg[0][hi] ^ pl.neg[2][hj]));
        if (nonfinite) ok = ok && O::all_finite(val);
        pstore<T, W>(obase + (int64_t)hi * mb * s + hj * mb, val);
      }
    }
    if (!ok) nonfinite[t] = 1;
  }
}

// Two contraction levels (q+1, q) in one pass, the mirror of
// expand2_plan_kernel: a thread owns one position of the level-(q+2) product
// blocks under one level-q parent.  For each level-(q+1) block r1 (ascending)
// it loads the R grandchildren at its position, contracts them with the
// network (contract_w: the level-(q+1) value at the n*n sub-positions, base
// coordinates), applies the level-(q+1) plan's sign, and folds that value into
// the level-q accumulators of those sub-positions with contract_w_step (the
// reference's r-ascending fold, _engine.py:104-112, streamed over r1).  The
// level-(q+1) array never goes through HBM; values equal two
// contract_plan_kernel launches.
template <class F, class T, int W, bool SYNC>
__global__ void __launch_bounds__(SYNC ? kSyncThreads : kThreads) contract2_plan_kernel(
    const T* __restrict__ ch, int K, int mb2, T* __restrict__ out,
    const PlanLevel* __restrict__ plans, int64_t plan_tstride, int level, int64_t ntr,
    uint8_t* __restrict__ nonfinite) {
  constexpr int n = F::n;
  constexpr int R = F::R;
  constexpr int NN = n * n;
  const int mb1 = n * mb2, s = n * mb1;
  const int P = (mb2 * mb2) / W;
  const int64_t items = (int64_t)K * P;
  int64_t e = (int64_t)blockIdx.x * (SYNC ? kSyncThreads : kThreads) + threadIdx.x;
  const bool live = e < items;
  if (!SYNC && !live) return;
  if (!live) e = items - 1;  // SYNC: idle lanes mirror the last item, stores masked
  const int Kp = (int)(e / P);
  const int p = (int)(e - (int64_t)Kp * P);
  const int pos = p * W;
  const int i = pos / mb2;
  const int j = pos - i * mb2;
  const int64_t blk2 = (int64_t)mb2 * mb2;
  using O = PackOps<T, W>;
  for (int64_t t = blockIdx.y; t < ntr; t += gridDim.y) {
    const PlanLevel& p0 = plans[t * plan_tstride + level];
    const PlanLevel& p1 = plans[t * plan_tstride + level + 1];
    // level-(q+1) base sub-block q1 = (I1, J1) sits at hatted (inv0, inv2), signed
    uint32_t m1[NN];
#pragma unroll
    for (int I = 0; I < n; ++I)
#pragma unroll
      for (int J = 0; J < n; ++J)
        m1[I * n + J] = sign_mask(p1.neg[0][p1.inv[0][I]] ^ p1.neg[2][p1.inv[2][J]]);
    const T* cb = ch + (t * K + Kp) * (int64_t)R * R * blk2 + pos;
    Pack<T, W> acc[NN][NN];  // [level-(q+1) sub-position q1][level-q base block]
#pragma unroll
    for (int r1 = 0; r1 < R; ++r1) {
      Pack<T, W> pr[R];
#pragma unroll
      for (int r2 = 0; r2 < R; ++r2) pr[r2] = pload<T, W>(cb + (int64_t)(r1 * R + r2) * blk2);
      Pack<T, W> o1[NN];
      F::template contract_w<T, W>(pr, o1);
#pragma unroll
      for (int q = 0; q < NN; ++q) F::template contract_w_step<T, W>(acc[q], O::flip(o1[q], m1[q]), r1);
      // SYNC: the CTA reads the grandchildren of r1 together (read locality of
      // small blocks, as in expand2_plan_kernel)
      if (SYNC) __syncthreads();
    }
    bool ok = true;
#pragma unroll
    for (int q = 0; q < NN; ++q) {
      F::template contract_w_finish<T, W>(acc[q]);
      const int hi1 = p1.inv[0][q / n], hj1 = p1.inv[2][q % n];
      T* ob = out + (t * K + Kp) * (int64_t)s * s + (int64_t)(hi1 * mb2 + i) * s + hj1 * mb2 + j;
#pragma unroll
      for (int I = 0; I < n; ++I) {
        const int hi = p0.inv[0][I];
#pragma unroll
        for (int J = 0; J < n; ++J) {
          const int hj = p0.inv[2][J];
          const Pack<T, W> val = O::flip(acc[q][I * n + J], sign_mask(p0.neg[0][hi] ^ p0.neg[2][hj]));
          if (nonfinite) ok = ok && O::all_finite(val);
          if (live) pstore<T, W>(ob + (int64_t)hi * mb1 * s + hj * mb1, val);
        }
      }
    }
    if (nonfinite && live && !ok) nonfinite[t] = 1;
  }
}

inline dim3 grid_for(int64_t items, int64_t ntr, int nt = kThreads) {
  const int64_t bx = (items + nt - 1) / nt;
  return dim3((unsigned)bx, (unsigned)(ntr < 65535 ? ntr : 65535), 1);
}

template <class F, class T, int W>
cudaError_t expand_plan_w(int which, const void* x, int64_t xs, int64_t K, int64_t s, void* out,
                          const PlanLevel* plans, int64_t pts, int level, int64_t ntr,
                          cudaStream_t st) {
  const int64_t mb = s / F::n;
  const dim3 grid = grid_for(K * (mb * mb / W), ntr);
  if (which == 0)
    expand_plan_kernel<F, T, W, 0><<<grid, kThreads, 0, st>>>(
        (const T*)x, xs, (int)K, (int)s, (T*)out, plans, pts, level, ntr);
  else
    expand_plan_kernel<F, T, W, 1><<<grid, kThreads, 0, st>>>(
        (const T*)x, xs, (int)K, (int)s, (T*)out, plans, pts, level, ntr);
  return cudaGetLastError();
}

template <class F, class T, int W>
cudaError_t expand2_plan_w(int which, const void* x, int64_t xs, int64_t K, int64_t s, void* out,
                           const PlanLevel* plans, int64_t pts, int level, int64_t ntr,
                           cudaStream_t st) {
  const int64_t mb2 = s / (F::n * F::n);
  const dim3 grid = grid_for(K * (mb2 * mb2 / W), ntr);
  // Lockstep (a CTA barrier after each r1) when the grandchild blocks are
  // small: a thread writes R^2 blocks, so without it each output line
  // collects its pieces from drifting warps over the whole launch and L2
  // evicts to scattered DRAM pages (config 2, 27x27 binary32 blocks: 0.534 ->
  // 0.332 ms/launch).  Large blocks have whole lines per warp store, where the
  // barrier only costs (config 5: 0.68 vs 0.73).
  const bool sync = mb2 * mb2 * (int64_t)sizeof(T) < (64 << 10);
  const dim3 gs = grid_for(K * (mb2 * mb2 / W), ntr, kSyncThreads);
  if (which == 0 && sync)
    expand2_plan_kernel<F, T, W, 0, true><<<gs, kSyncThreads, 0, st>>>(
        (const T*)x, xs, (int)K, (int)s, (T*)out, plans, pts, level, ntr);
  else if (which == 0)
    expand2_plan_kernel<F, T, W, 0, false><<<grid, kThreads, 0, st>>>(
        (const T*)x, xs, (int)K, (int)s, (T*)out, plans, pts, level, ntr);
  else if (sync)
    expand2_plan_kernel<F, T, W, 1, true><<<gs, kSyncThreads, 0, st>>>(
        (const T*)x, xs, (int)K, (int)s, (T*)out, plans, pts, level, ntr);
  else
    expand2_plan_kernel<F, T, W, 1, false><<<grid, kThreads, 0, st>>>(
        (const T*)x, xs, (int)K, (int)s, (T*)out, plans, pts, level, ntr);
  return cudaGetLastError();
}

// n^4 live input packs per thread: binary64 Laderman (81 doubles) and wide
// packs would spill, so those keep the two single-level launches.
template <class F, class T>
constexpr int expand2_max_width() {
  constexpr int bytes = F::n * F::n * F::n * F::n * (int)sizeof(T);
  if (F::n >= 3 && sizeof(T) != 4) return 0;  // binary16 n = 3 spills (half pack ops)
  return bytes > 384 ? 0 : (bytes * 4 <= 384 ? 4 : bytes * 2 <= 384 ? 2 : 1);
}

template <class F, class T>
cudaError_t expand2_plan_t(int dtype, int which, const void* x, int64_t xs, int64_t K, int64_t s,
                           void* out, const PlanLevel* plans, int64_t pts, int level, int64_t ntr,
                           cudaStream_t st) {
  constexpr int cap = expand2_max_width<F, T>();
  if constexpr (cap == 0) {
    return cudaErrorNotSupported;
  } else {
    const int W = pick_width(dtype, s / (F::n * F::n), cap);
    switch (W) {
      case 4: return expand2_plan_w<F, T, (cap >= 4 ? 4 : 1)>(which, x, xs, K, s, out, plans, pts, level, ntr, st);
      case 2: return expand2_plan_w<F, T, (cap >= 2 ? 2 : 1)>(which, x, xs, K, s, out, plans, pts, level, ntr, st);
      default: return expand2_plan_w<F, T, 1>(which, x, xs, K, s, out, plans, pts, level, ntr, st);
    }
  }
}

template <class T>
cudaError_t expand2_plan_f(int dtype, int formula, int which, const void* x, int64_t xs, int64_t K,
                           int64_t s, void* out, const PlanLevel* plans, int64_t pts, int level,
                           int64_t ntr, cudaStream_t st) {
  switch (formula) {
    case FStrassen::kId: return expand2_plan_t<FStrassen, T>(dtype, which, x, xs, K, s, out, plans, pts, level, ntr, st);
    case FLaderman::kId: return expand2_plan_t<FLaderman, T>(dtype, which, x, xs, K, s, out, plans, pts, level, ntr, st);
    case FStandard2::kId: return expand2_plan_t<FStandard2, T>(dtype, which, x, xs, K, s, out, plans, pts, level, ntr, st);
    case FStandard3::kId: return expand2_plan_t<FStandard3, T>(dtype, which, x, xs, K, s, out, plans, pts, level, ntr, st);
  }
  return cudaErrorInvalidValue;
}

template <class F, class T, int W>
cudaError_t contract_plan_w(const void* ch, int64_t K, int64_t mb, void* out,
                            const PlanLevel* plans, int64_t pts, int level, int64_t ntr,
                            uint8_t* nonfinite, cudaStream_t st) {
  const dim3 grid = grid_for(K * (mb * mb / W), ntr);
  contract_plan_kernel<F, T, W><<<grid, kThreads, 0, st>>>(
      (const T*)ch, (int)K, (int)mb, (T*)out, plans, pts, level, ntr, nonfinite);
  return cudaGetLastError();
}

template <class F, class T, int W>
cudaError_t contract2_plan_w(const void* ch, int64_t K, int64_t mb2, void* out,
                             const PlanLevel* plans, int64_t pts, int level, int64_t ntr,
                             uint8_t* nonfinite, cudaStream_t st) {
  const dim3 grid = grid_for(K * (mb2 * mb2 / W), ntr);
  // lockstep for small blocks, as in expand2_plan_w
  const bool sync = mb2 * mb2 * (int64_t)sizeof(T) < (64 << 10);
  const dim3 gs = grid_for(K * (mb2 * mb2 / W), ntr, kSyncThreads);
  // (n = 2 formulas read R^2 = 49 blocks per thread: no lockstep variant,
  // its unrolled barrier loop costs 255 registers)
  if constexpr (F::R > 8) {
    if (sync) {
      contract2_plan_kernel<F, T, W, true><<<gs, kSyncThreads, 0, st>>>(
          (const T*)ch, (int)K, (int)mb2, (T*)out, plans, pts, level, ntr, nonfinite);
      return cudaGetLastError();
    }
  }
    contract2_plan_kernel<F, T, W, false><<<grid, kThreads, 0, st>>>(
        (const T*)ch, (int)K, (int)mb2, (T*)out, plans, pts, level, ntr, nonfinite);
  return cudaGetLastError();
}

template <class F, class T>
cudaError_t contract2_plan_t(int dtype, const void* ch, int64_t K, int64_t mb2, void* out,
                             const PlanLevel* plans, int64_t pts, int level, int64_t ntr,
                             uint8_t* nonfinite, cudaStream_t st) {
  constexpr int cap = expand2_max_width<F, T>();  // n^4 live accumulator packs, as expand2
  if constexpr (cap == 0) {
    return cudaErrorNotSupported;
  } else {
    const int W = pick_width(dtype, mb2, cap);
    switch (W) {
      case 4: return contract2_plan_w<F, T, (cap >= 4 ? 4 : 1)>(ch, K, mb2, out, plans, pts, level, ntr, nonfinite, st);
      case 2: return contract2_plan_w<F, T, (cap >= 2 ? 2 : 1)>(ch, K, mb2, out, plans, pts, level, ntr, nonfinite, st);
      default: return contract2_plan_w<F, T, 1>(ch, K, mb2, out, plans, pts, level, ntr, nonfinite, st);
    }
  }
}

template <class T>
cudaError_t contract2_plan_f(int dtype, int formula, const void* ch, int64_t K, int64_t mb2,
                             void* out, const PlanLevel* plans, int64_t pts, int level,
                             int64_t ntr, uint8_t* nonfinite, cudaStream_t st) {
  switch (formula) {
    case FStrassen::kId: return contract2_plan_t<FStrassen, T>(dtype, ch, K, mb2, out, plans, pts, level, ntr, nonfinite, st);
    case FLaderman::kId: return contract2_plan_t<FLaderman, T>(dtype, ch, K, mb2, out, plans, pts, level, ntr, nonfinite, st);
    case FStandard2::kId: return contract2_plan_t<FStandard2, T>(dtype, ch, K, mb2, out, plans, pts, level, ntr, nonfinite, st);
    case FStandard3::kId: return contract2_plan_t<FStandard3, T>(dtype, ch, K, mb2, out, plans, pts, level, ntr, nonfinite, st);
  }
  return cudaErrorInvalidValue;
}

// Width dispatch.  Large-R formulas (Laderman: 23 live packs) cap the width
// so the children stay in registers.
template <class F, class T>
cudaError_t expand_plan_t(int dtype, int which, const void* x, int64_t xs, int64_t K, int64_t s,
                          void* out, const PlanLevel* plans, int64_t pts, int level, int64_t ntr,
                          cudaStream_t st) {
  const int cap = (F::R > 8 ? 8 : 16) / (int)sizeof(T);
  const int W = pick_width(dtype, s / F::n, cap);
  switch (W) {
    case 8: return expand_plan_w<F, T, (sizeof(T) == 2 ? 8 : 1)>(which, x, xs, K, s, out, plans, pts, level, ntr, st);
    case 4: return expand_plan_w<F, T, (sizeof(T) <= 4 ? 4 : 1)>(which, x, xs, K, s, out, plans, pts, level, ntr, st);
    case 2: return expand_plan_w<F, T, 2>(which, x, xs, K, s, out, plans, pts, level, ntr, st);
    default: return expand_plan_w<F, T, 1>(which, x, xs, K, s, out, plans, pts, level, ntr, st);
  }
}

template <class F, class T>
cudaError_t contract_plan_t(int dtype, const void* ch, int64_t K, int64_t mb, void* out,
                            const PlanLevel* plans, int64_t pts, int level, int64_t ntr,
                            uint8_t* nonfinite, cudaStream_t st) {
  const int cap = (F::R > 8 ? 8 : 16) / (int)sizeof(T);
  const int W = pick_width(dtype, mb, cap);
  switch (W) {
    case 8: return contract_plan_w<F, T, (sizeof(T) == 2 ? 8 : 1)>(ch, K, mb, out, plans, pts, level, ntr, nonfinite, st);
    case 4: return contract_plan_w<F, T, (sizeof(T) <= 4 ? 4 : 1)>(ch, K, mb, out, plans, pts, level, ntr, nonfinite, st);
    case 2: return contract_plan_w<F, T, 2>(ch, K, mb, out, plans, pts, level, ntr, nonfinite, st);
    default: return contract_plan_w<F, T, 1>(ch, K, mb, out, plans, pts, level, ntr, nonfinite, st);
  }
}

template <class T>
cudaError_t expand_plan_f(int dtype, int formula, int which, const void* x, int64_t xs, int64_t K,
                          int64_t s, void* out, const PlanLevel* plans, int64_t pts, int level,
                          int64_t ntr, cudaStream_t st) {
  switch (formula) {
    case FStrassen::kId: return expand_plan_t<FStrassen, T>(dtype, which, x, xs, K, s, out, plans, pts, level, ntr, st);
    case FLaderman::kId: return expand_plan_t<FLaderman, T>(dtype, which, x, xs, K, s, out, plans, pts, level, ntr, st);
    case FStandard2::kId: return expand_plan_t<FStandard2, T>(dtype, which, x, xs, K, s, out, plans, pts, level, ntr, st);
    case FStandard3::kId: return expand_plan_t<FStandard3, T>(dtype, which, x, xs, K, s, out, plans, pts, level, ntr, st);
  }
  return cudaErrorInvalidValue;
}

template <class T>
cudaError_t contract_plan_f(int dtype, int formula, const void* ch, int64_t K, int64_t mb,
                            void* out, const PlanLevel* plans, int64_t pts, int level, int64_t ntr,
                            uint8_t* nonfinite, cudaStream_t st) {
  switch (formula) {
    case FStrassen::kId: return contract_plan_t<FStrassen, T>(dtype, ch, K, mb, out, plans, pts, level, ntr, nonfinite, st);
    case FLaderman::kId: return contract_plan_t<FLaderman, T>(dtype, ch, K, mb, out, plans, pts, level, ntr, nonfinite, st);
    case FStandard2::kId: return contract_plan_t<FStandard2, T>(dtype, ch, K, mb, out, plans, pts, level, ntr, nonfinite, st);
    case FStandard3::kId: return contract_plan_t<FStandard3, T>(dtype, ch, K, mb, out, plans, pts, level, ntr, nonfinite, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

int formula_n(int formula) {
  switch (formula) {
    case FStrassen::kId: return FStrassen::n;
    case FLaderman::kId: return FLaderman::n;
    case FStandard2::kId: return FStandard2::n;
    case FStandard3::kId: return FStandard3::n;
  }
  return 0;
}

int formula_R(int formula) {
  switch (formula) {
    case FStrassen::kId: return FStrassen::R;
    case FLaderman::kId: return FLaderman::R;
    case FStandard2::kId: return FStandard2::R;
    case FStandard3::kId: return FStandard3::R;
  }
  return 0;
}

cudaError_t launch_expand_plan(int dtype, int formula, int which, const void* x, int64_t x_tstride,
                               int64_t K, int64_t s, void* out, const PlanLevel* plans,
                               int64_t plan_tstride, int level, int64_t ntr, cudaStream_t st) {
  switch (dtype) {
    case kF64: return expand_plan_f<double>(dtype, formula, which, x, x_tstride, K, s, out, plans, plan_tstride, level, ntr, st);
    case kF32: return expand_plan_f<float>(dtype, formula, which, x, x_tstride, K, s, out, plans, plan_tstride, level, ntr, st);
    case kF16: return expand_plan_f<__half>(dtype, formula, which, x, x_tstride, K, s, out, plans, plan_tstride, level, ntr, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_expand2_plan(int dtype, int formula, int which, const void* x,
                                int64_t x_tstride, int64_t K, int64_t s, void* out,
                                const PlanLevel* plans, int64_t plan_tstride, int level,
                                int64_t ntr, cudaStream_t st) {
  switch (dtype) {
    case kF64: return expand2_plan_f<double>(dtype, formula, which, x, x_tstride, K, s, out, plans, plan_tstride, level, ntr, st);
    case kF32: return expand2_plan_f<float>(dtype, formula, which, x, x_tstride, K, s, out, plans, plan_tstride, level, ntr, st);
    case kF16: return expand2_plan_f<__half>(dtype, formula, which, x, x_tstride, K, s, out, plans, plan_tstride, level, ntr, st);
  }
  return cudaErrorInvalidValue;
}

bool expand2_supported(int dtype, int formula) {
  auto ok = [&](auto f) {
    using F = decltype(f);
    switch (dtype) {
      case kF64: return expand2_max_width<F, double>() > 0;
      case kF32: return expand2_max_width<F, float>() > 0;
      case kF16: return expand2_max_width<F, __half>() > 0;
    }
    return false;
  };
  switch (formula) {
    case FStrassen::kId: return ok(FStrassen{});
    case FLaderman::kId: return ok(FLaderman{});
    case FStandard2::kId: return ok(FStandard2{});
    case FStandard3::kId: return ok(FStandard3{});
  }
  return false;
}

cudaError_t launch_contract2_plan(int dtype, int formula, const void* ch, int64_t K, int64_t mb2,
                                  void* out, const PlanLevel* plans, int64_t plan_tstride,
                                  int level, int64_t ntr, uint8_t* nonfinite, cudaStream_t st) {
  switch (dtype) {
    case kF64: return contract2_plan_f<double>(dtype, formula, ch, K, mb2, out, plans, plan_tstride, level, ntr, nonfinite, st);
    case kF32: return contract2_plan_f<float>(dtype, formula, ch, K, mb2, out, plans, plan_tstride, level, ntr, nonfinite, st);
    case kF16: return contract2_plan_f<__half>(dtype, formula, ch, K, mb2, out, plans, plan_tstride, level, ntr, nonfinite, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_contract_plan(int dtype, int formula, const void* ch, int64_t K, int64_t mb,
                                 void* out, const PlanLevel* plans, int64_t plan_tstride,
                                 int level, int64_t ntr, uint8_t* nonfinite, cudaStream_t st) {
  switch (dtype) {
    case kF64: return contract_plan_f<double>(dtype, formula, ch, K, mb, out, plans, plan_tstride, level, ntr, nonfinite, st);
    case kF32: return contract_plan_f<float>(dtype, formula, ch, K, mb, out, plans, plan_tstride, level, ntr, nonfinite, st);
    case kF16: return contract_plan_f<__half>(dtype, formula, ch, K, mb, out, plans, plan_tstride, level, ntr, nonfinite, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace rbc
