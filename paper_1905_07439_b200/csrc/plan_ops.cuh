// Per-position plan-path operations shared by the breadth-first kernels
// (kernels_plan.cu) and the fused subtree kernel (kernels_fused.cu).
//
// expand_at  : W consecutive columns at position (i, j) of one parent block
//              -> the R children at the same position (reference _expand,
//              _engine.py:64-90, on hatted tensors, randomize.py:163-178)
// contract_at: the R children at one position -> the n*n parent blocks
//              at that position (reference _contract, _engine.py:93-114)
// Pointers may address global or shared memory.
#pragma once

#include "formulas_gen.cuh"

namespace rbc {

// WHICH = 0: operand A (rows permuted by plan 1, cols by plan 2, network U)
// WHICH = 1: operand B (rows by plan 2, cols by plan 3, network V)
template <class F, class T, int W, int WHICH>
__device__ __forceinline__ void expand_at(const T* __restrict__ parent, int s,
                                          T* __restrict__ kids, int kid_stride,
                                          const PlanLevel& pl, int i, int j) {
  constexpr int n = F::n;
  constexpr int R = F::R;
  constexpr int ri = WHICH == 0 ? 0 : 1;
  constexpr int ci = WHICH == 0 ? 1 : 2;
  using O = PackOps<T, W>;
  const int mb = s / n;
  const T* base = parent + i * s + j;
  Pack<T, W> g[n * n];
#pragma unroll
  for (int kb = 0; kb < n; ++kb) {
    const int hk = pl.inv[ri][kb];
#pragma unroll
    for (int lb = 0; lb < n; ++lb) {
      const int hl = pl.inv[ci][lb];
      const uint32_t m = sign_mask(pl.neg[ri][hk] ^ pl.neg[ci][hl]);
      g[kb * n + lb] = O::flip(pload<T, W>(base + (hk * mb) * s + hl * mb), m);
    }
  }
  Pack<T, W> o[R];
  if (WHICH == 0)
    F::template expand_u<T, W>(g, o, pl.perm[ri][n - 1], pl.perm[ci][n - 1]);
  else
    F::template expand_v<T, W>(g, o, pl.perm[ri][n - 1], pl.perm[ci][n - 1]);
  T* kb0 = kids + i * mb + j;
#pragma unroll
  for (int r = 0; r < R; ++r) pstore<T, W>(kb0 + r * kid_stride, o[r]);
}

// Returns false when any written value is non-finite (only checked if asked).
template <class F, class T, int W, bool CHECK>
__device__ __forceinline__ bool contract_at(const T* __restrict__ kids, int kid_stride, int mb,
                                            T* __restrict__ parent, const PlanLevel& pl, int i,
                                            int j) {
  constexpr int n = F::n;
  constexpr int R = F::R;
  using O = PackOps<T, W>;
  const int s = n * mb;
  const T* kb0 = kids + i * mb + j;
  Pack<T, W> pr[R];
#pragma unroll
  for (int r = 0; r < R; ++r) pr[r] = pload<T, W>(kb0 + r * kid_stride);
  Pack<T, W> o[n * n];
  F::template contract_w<T, W>(pr, o);
  T* base = parent + i * s + j;
  bool ok = true;
#pragma unroll
  for (int I = 0; I < n; ++I) {
    const int hi = pl.inv[0][I];
#pragma unroll
    for (int J = 0; J < n; ++J) {
      const int hj = pl.inv[2][J];
      const Pack<T, W> val = O::flip(o[I * n + J], sign_mask(pl.neg[0][hi] ^ pl.neg[2][hj]));
      if (CHECK) ok = ok && O::all_finite(val);
      pstore<T, W>(base + (hi * mb) * s + hj * mb, val);
    }
  }
  return ok;
}

// ---- precomputed variants: the plan-dependent gather/scatter offsets of one
// (level, operand) are computed once per thread and reused for every position.
template <int n>
struct alignas(16) GatherTab {
  int off[n * n];        // element offset of base block (kb, lb) in the parent
  uint32_t msk[n * n];   // sign flip of that block
  int lastrow, lastcol;  // base index added last in 3-term folds
};

template <int n, int WHICH>
__device__ __forceinline__ void make_gather(const PlanLevel& pl, int s, GatherTab<n>& gt) {
  constexpr int ri = WHICH == 0 ? 0 : 1;
  constexpr int ci = WHICH == 0 ? 1 : 2;
  const int mb = s / n;
#pragma unroll
  for (int kb = 0; kb < n; ++kb) {
    const int hk = pl.inv[ri][kb];
#pragma unroll
    for (int lb = 0; lb < n; ++lb) {
      const int hl = pl.inv[ci][lb];
      gt.off[kb * n + lb] = hk * mb * s + hl * mb;
      gt.msk[kb * n + lb] = sign_mask(pl.neg[ri][hk] ^ pl.neg[ci][hl]);
    }
  }
  gt.lastrow = pl.perm[ri][n - 1];
  gt.lastcol = pl.perm[ci][n - 1];
}

// Scatter table of a contraction: base block (I, J) -> hatted position.
template <int n>
__device__ __forceinline__ void make_scatter(const PlanLevel& pl, int mb, GatherTab<n>& gt) {
  const int s = n * mb;
#pragma unroll
  for (int I = 0; I < n; ++I) {
    const int hi = pl.inv[0][I];
#pragma unroll
    for (int J = 0; J < n; ++J) {
      const int hj = pl.inv[2][J];
      gt.off[I * n + J] = hi * mb * s + hj * mb;
      gt.msk[I * n + J] = sign_mask(pl.neg[0][hi] ^ pl.neg[2][hj]);
    }
  }
  gt.lastrow = gt.lastcol = 0;
}

// Position-major ("SoA") shared-memory layouts of the fused subtree: element
// (block beta, position pi) of a level lives at pi * NB + beta, and a level-1
// block stores its n x n sub-blocks contiguously (blocked order).  Gather and
// scatter offsets then only depend on the hatted sub-block index:
// off = (hk * n + hl) * sub_stride.
template <int n, int WHICH>
__device__ __forceinline__ void make_gather_soa(const PlanLevel& pl, int sub_stride,
                                                GatherTab<n>& gt) {
  constexpr int ri = WHICH == 0 ? 0 : 1;
  constexpr int ci = WHICH == 0 ? 1 : 2;
#pragma unroll
  for (int kb = 0; kb < n; ++kb) {
    const int hk = pl.inv[ri][kb];
#pragma unroll
    for (int lb = 0; lb < n; ++lb) {
      const int hl = pl.inv[ci][lb];
      gt.off[kb * n + lb] = (hk * n + hl) * sub_stride;
      gt.msk[kb * n + lb] = sign_mask(pl.neg[ri][hk] ^ pl.neg[ci][hl]);
    }
  }
  gt.lastrow = pl.perm[ri][n - 1];
  gt.lastcol = pl.perm[ci][n - 1];
}

template <int n>
__device__ __forceinline__ void make_scatter_soa(const PlanLevel& pl, int sub_stride,
                                                 GatherTab<n>& gt) {
#pragma unroll
  for (int I = 0; I < n; ++I) {
    const int hi = pl.inv[0][I];
#pragma unroll
    for (int J = 0; J < n; ++J) {
      const int hj = pl.inv[2][J];
      gt.off[I * n + J] = (hi * n + hj) * sub_stride;
      gt.msk[I * n + J] = sign_mask(pl.neg[0][hi] ^ pl.neg[2][hj]);
    }
  }
  gt.lastrow = gt.lastcol = 0;
}

template <class F, class T, int W, int WHICH>
__device__ __forceinline__ void expand_tab(const T* __restrict__ base, const GatherTab<F::n>& gt,
                                           T* __restrict__ kid0, int kid_stride) {
  constexpr int n = F::n;
  constexpr int R = F::R;
  using O = PackOps<T, W>;
  Pack<T, W> g[n * n];
#pragma unroll
  for (int k = 0; k < n * n; ++k) g[k] = O::flip(pload<T, W>(base + gt.off[k]), gt.msk[k]);
  Pack<T, W> o[R];
  if (WHICH == 0)
    F::template expand_u<T, W>(g, o, gt.lastrow, gt.lastcol);
  else
    F::template expand_v<T, W>(g, o, gt.lastrow, gt.lastcol);
#pragma unroll
  for (int r = 0; r < R; ++r) pstore<T, W>(kid0 + r * kid_stride, o[r]);
}

template <class F, class T, int W, bool CHECK>
__device__ __forceinline__ bool contract_tab(const T* __restrict__ kid0, int kid_stride,
                                             T* __restrict__ base, const GatherTab<F::n>& st) {
  constexpr int n = F::n;
  constexpr int R = F::R;
  using O = PackOps<T, W>;
  Pack<T, W> pr[R];
#pragma unroll
  for (int r = 0; r < R; ++r) pr[r] = pload<T, W>(kid0 + r * kid_stride);
  Pack<T, W> o[n * n];
  F::template contract_w<T, W>(pr, o);
  bool ok = true;
#pragma unroll
  for (int k = 0; k < n * n; ++k) {
    const Pack<T, W> val = O::flip(o[k], st.msk[k]);
    if (CHECK) ok = ok && O::all_finite(val);
    pstore<T, W>(base + st.off[k], val);
  }
  return ok;
}

}  // namespace rbc
