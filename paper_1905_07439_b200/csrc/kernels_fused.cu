// Fused subtree kernel: the bottom L levels of the recursion for one
// (trial, level-q0 block) pair, entirely in shared memory.
//
// The reference evaluates every level breadth-first over the whole batch
// (_engine.py:117-149).  With small leaves (config 2: 3x3, the golden
// artifact at Q=5: 10x10) the deepest levels are the largest arrays but each
// subtree is tiny, so breadth-first HBM round trips dominate.  Here one CTA
// takes the level-q0 operand blocks X, Y (s0 x s0, s0 = M * n^L) of one
// trial, expands them L levels into shared memory, forms the R^L leaf
// products there, contracts back to the s0 x s0 product block and writes
// only that to HBM.  Every output element sees exactly the same operation
// sequence as in the breadth-first evaluation (the per-element chains are
// independent of the evaluation schedule), so values are
// identical.
//
// Shared memory: for l = 1..L, X_l and Y_l (R^l blocks of (s0/n^l)^2), plus
// the leaf products P_L (R^L M^2).  Contractions reuse the dead X_l buffers.

#include <cstdlib>
#include <type_traits>

#include "kernels.h"
#include "plan_ops.cuh"
#include "bulk.cuh"

namespace rbc {

namespace {

constexpr int kThreads = 256;

template <int B, int E>
struct Pow {
  static constexpr int v = B * Pow<B, E - 1>::v;
};
template <int B>
struct Pow<B, 0> {
  static constexpr int v = 1;
};

template <class F, class T, int L, int M>
struct Subtree {
  static constexpr int n = F::n;
  static constexpr int R = F::R;
  static constexpr int s0 = M * Pow<n, L>::v;
  // side of the blocks at depth l below q0
  static constexpr __host__ __device__ int side(int l) {
    int s = s0;
    for (int k = 0; k < l; ++k) s /= n;
    return s;
  }
  static constexpr __host__ __device__ int count(int l) {
    int c = 1;
    for (int k = 0; k < l; ++k) c *= R;
    return c;
  }
  static constexpr __host__ __device__ int elems(int l) { return count(l) * side(l) * side(l); }
  // offsets (elements) of X_l, Y_l (l = 1..L) and P_L in shared memory
  static constexpr __host__ __device__ int x_off(int l) {
    int o = 0;
    for (int k = 1; k < l; ++k) o += 2 * elems(k);
    return o;
  }
  static constexpr __host__ __device__ int y_off(int l) { return x_off(l) + elems(l); }
  // leaves of side <= 4 are multiplied by one thread each, in place over X_L
  static constexpr bool kInPlace = M <= 4;
  static constexpr __host__ __device__ int p_off() { return kInPlace ? x_off(L) : x_off(L + 1); }
  static constexpr __host__ __device__ int total() {
    return kInPlace ? x_off(L + 1) : x_off(L + 1) + elems(L);
  }
  // header: L plan records, then 3 gather/scatter tables per level
  static constexpr size_t kTabBytes = sizeof(GatherTab<n>);
  static constexpr size_t header() {
    return ((sizeof(PlanLevel) * L + 15) / 16) * 16 + 3 * L * kTabBytes;
  }
  static constexpr size_t smem_bytes() { return (size_t)total() * sizeof(T) + header(); }
};

// Expansion of one (level, operand) over all positions of the stage, the
// plan's gather table hoisted out of the position loop.
template <class F, class T, int WHICH>
__device__ __forceinline__ void expand_stage(const GatherTab<F::n>& gt_sm, const T* par0, int sp,
                                             T* dst0, int parents, int lt, int nthreads) {
  constexpr int n = F::n;
  constexpr int R = F::R;
  const int mb = sp / n;
  const int kids = mb * mb;
  const GatherTab<n> gt = gt_sm;  // registers
  const int items = parents * kids;
  // parent-minor order: neighbouring threads take the same position in
  // neighbouring parents, whose odd strides (R * kids, sp * sp) spread over
  // all shared-memory banks
  for (int e = lt; e < items; e += nthreads) {
    const int pos = e / parents;
    const int Kp = e - pos * parents;
    const int i = pos / mb;
    const int j = pos - i * mb;
    expand_tab<F, T, 1, WHICH>(par0 + Kp * sp * sp + i * sp + j, gt,
                               dst0 + Kp * R * kids + i * mb + j, kids);
  }
}

template <class F, class T, int L, int M, int NT>
__global__ void __launch_bounds__(NT) subtree_kernel(
    const T* __restrict__ x, const T* __restrict__ y, int64_t xy_tstride, int K0,
    T* __restrict__ out, const PlanLevel* __restrict__ plans, int64_t plan_tstride, int q0,
    int64_t ntr, uint8_t* __restrict__ nonfinite) {
  using S = Subtree<F, T, L, M>;
  constexpr int n = F::n;
  constexpr int R = F::R;
  constexpr int s0 = S::s0;
  constexpr int kThreads = NT;
  constexpr int kHalf = kThreads / 2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PlanLevel* spl = reinterpret_cast<PlanLevel*>(smem_raw);
  GatherTab<n>* tabs = reinterpret_cast<GatherTab<n>*>(
      smem_raw + ((sizeof(PlanLevel) * L + 15) / 16) * 16);
  T* sm = reinterpret_cast<T*>(smem_raw + S::header());
  const int k0 = blockIdx.x;
  using A = Arith<T>;
  // operand A on the first half of the warps, B on the second (warp-uniform)
  const int which = threadIdx.x >= kHalf;
  const int lt = threadIdx.x - which * kHalf;

  for (int64_t t = blockIdx.y; t < ntr; t += gridDim.y) {
    __syncthreads();  // previous trial's readers of spl / sm are done
    {
      // the L plan records q0 .. q0+L-1 are contiguous: copy them as words
      constexpr int kWords = (int)(sizeof(PlanLevel) / 4) * L;
      const int* src = reinterpret_cast<const int*>(plans + t * plan_tstride + q0);
      if (threadIdx.x < kWords) reinterpret_cast<int*>(spl)[threadIdx.x] = src[threadIdx.x];
    }
    __syncthreads();
    // one thread per (level, table): X gather, Y gather, contraction scatter
    if (threadIdx.x < 3 * L) {
      const int l = threadIdx.x / 3, kind = threadIdx.x - 3 * (threadIdx.x / 3);
      int sp = s0;
      for (int k = 0; k < l; ++k) sp /= n;
      GatherTab<n> tab;
      if (kind == 0)
        make_gather<n, 0>(spl[l], sp, tab);
      else if (kind == 1)
        make_gather<n, 1>(spl[l], sp, tab);
      else
        make_scatter<n>(spl[l], sp / n, tab);
      tabs[threadIdx.x] = tab;
    }
    __syncthreads();
    const T* src = (which ? y : x) + t * xy_tstride + (int64_t)k0 * s0 * s0;

    // ---- expansions: level l -> l + 1
#pragma unroll
    for (int l = 0; l < L; ++l) {
      const int sp = S::side(l);
      const T* par0 = l == 0 ? src : sm + (which ? S::y_off(l) : S::x_off(l));
      T* dst0 = sm + (which ? S::y_off(l + 1) : S::x_off(l + 1));
      if (which)
        expand_stage<F, T, 1>(tabs[3 * l + 1], par0, sp, dst0, S::count(l), lt, kHalf);
      else
        expand_stage<F, T, 0>(tabs[3 * l + 0], par0, sp, dst0, S::count(l), lt, kHalf);
      __syncthreads();
    }

    // ---- leaves: k ascending, first term initialises
    {
      constexpr int leaves = S::count(L);
      const T* XL = sm + S::x_off(L);
      const T* YL = sm + S::y_off(L);
      T* PL = sm + S::p_off();
      if (S::kInPlace) {
        // one thread per leaf product, operands in registers, result written
        // over the thread's own X leaf (PL == XL)
        for (int leaf = threadIdx.x; leaf < leaves; leaf += kThreads) {
          T xa[M * M], yb[M * M];
#pragma unroll
          for (int q = 0; q < M * M; ++q) {
            xa[q] = XL[leaf * M * M + q];
            yb[q] = YL[leaf * M * M + q];
          }
#pragma unroll
          for (int i = 0; i < M; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j) {
              T acc = A::mul(xa[i * M], yb[j]);
#pragma unroll
              for (int k = 1; k < M; ++k) acc = A::add(acc, A::mul(xa[i * M + k], yb[k * M + j]));
              PL[leaf * M * M + i * M + j] = acc;
            }
        }
      } else {
        // one thread per (leaf, row)
        for (int it = threadIdx.x; it < leaves * M; it += kThreads) {
          const int leaf = it / M;
          const int i = it - leaf * M;
          const T* xr = XL + leaf * M * M + i * M;
          const T* yl = YL + leaf * M * M;
          T acc[M];
#pragma unroll
          for (int j = 0; j < M; ++j) acc[j] = A::mul(xr[0], yl[j]);
#pragma unroll
          for (int k = 1; k < M; ++k) {
            const T xv = xr[k];
#pragma unroll
            for (int j = 0; j < M; ++j) acc[j] = A::add(acc[j], A::mul(xv, yl[k * M + j]));
          }
          T* pr = PL + leaf * M * M + i * M;
#pragma unroll
          for (int j = 0; j < M; ++j) pr[j] = acc[j];
        }
      }
      __syncthreads();
    }

    // ---- contractions: level l + 1 -> l (into the dead X_l, or HBM at l = 0)
    bool ok = true;
#pragma unroll
    for (int l = L - 1; l >= 0; --l) {
      const int mb = S::side(l + 1);
      const int sp = S::side(l);
      const int kids = mb * mb;
      const int items = S::count(l) * kids;
      const GatherTab<n> st = tabs[3 * l + 2];
      const T* ksrc = sm + (l == L - 1 ? S::p_off() : S::x_off(l + 1));
      T* dbase = l == 0 ? out + (t * K0 + k0) * (int64_t)s0 * s0 : sm + S::x_off(l);
      const int parents = S::count(l);
      for (int e = threadIdx.x; e < items; e += kThreads) {
        const int pos = e / parents;
        const int Kp = e - pos * parents;
        const int i = pos / mb;
        const int j = pos - i * mb;
        const T* ks = ksrc + Kp * R * kids + i * mb + j;
        T* dst = dbase + Kp * sp * sp + i * sp + j;
        if (l == 0 && nonfinite)
          ok = contract_tab<F, T, 1, true>(ks, kids, dst, st) && ok;
        else
          contract_tab<F, T, 1, false>(ks, kids, dst, st);
      }
      __syncthreads();
    }
    if (nonfinite && !ok) nonfinite[t] = 1;
  }
}

// ---- position-major (SoA) two-level subtree ---------------------------------
// Same arithmetic and stages as subtree_kernel<F, T, 2, M>, different shared
// memory layout.  Element (block beta, position pi) of a level is stored at
// pi * NB + beta (NB = blocks of that level in the subtree), level-1 blocks in
// blocked order (their n x n sub-blocks contiguous).  With the parent-minor
// item order e = Kp + R * pi, every access of every stage is bank-conflict
// free for odd R: parents read at e + off, children written at R * e + r, leaves
// read at consecutive addresses (simulated 1338 vs 1956 wavefronts per CTA for
// config 2 with the row-major layout).
template <class F, class T, int M, int H>
struct SubtreeSoA {
  static constexpr int n = F::n;
  static constexpr int R = F::R;
  static constexpr int s1 = M * n;
  static constexpr int s0 = s1 * n;
  static constexpr int kids1 = s1 * s1;
  static constexpr int leafE = M * M;
  // level-1 parents are processed in H groups of at most G (smaller leaf
  // buffers -> more CTAs per SM, which this latency-bound kernel needs)
  static constexpr int G = (R + H - 1) / H;
  static constexpr int NB2 = G * R;  // leaves held at a time
  static constexpr bool kInPlace = M <= 4;
  static constexpr int x1_off = 0;
  static constexpr int y1_off = kids1 * R;
  static constexpr int x2_off = 2 * kids1 * R;
  static constexpr int y2_off = x2_off + leafE * NB2;
  static constexpr int p2_off = kInPlace ? x2_off : y2_off + leafE * NB2;
  static constexpr int total = kInPlace ? y2_off + leafE * NB2 : p2_off + leafE * NB2;
  static constexpr size_t header() {
    return ((sizeof(PlanLevel) * 2 + 15) / 16) * 16 + 6 * sizeof(GatherTab<n>);
  }
  static constexpr size_t smem_bytes() { return header() + sizeof(T) * (size_t)total; }
};

template <class F, class T, int M, int H, int NT>
__global__ void __launch_bounds__(NT) subtree_soa_kernel(
    const T* __restrict__ x, const T* __restrict__ y, int64_t xy_tstride, int K0,
    T* __restrict__ out, const PlanLevel* __restrict__ plans, int64_t plan_tstride, int q0,
    int64_t ntr, uint8_t* __restrict__ nonfinite) {
  using S = SubtreeSoA<F, T, M, H>;
  constexpr int n = F::n;
  constexpr int R = F::R;
  constexpr int s0 = S::s0, s1 = S::s1, kids1 = S::kids1, leafE = S::leafE;
  constexpr int G = S::G;
  constexpr int kHalf = NT / 2;
  using A = Arith<T>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PlanLevel* spl = reinterpret_cast<PlanLevel*>(smem_raw);
  GatherTab<n>* tabs =
      reinterpret_cast<GatherTab<n>*>(smem_raw + ((sizeof(PlanLevel) * 2 + 15) / 16) * 16);
  T* sm = reinterpret_cast<T*>(smem_raw + S::header());
  T* X1 = sm + S::x1_off;
  T* Y1 = sm + S::y1_off;
  T* X2 = sm + S::x2_off;
  T* Y2 = sm + S::y2_off;
  T* P2 = sm + S::p2_off;
  const int k0 = blockIdx.x;
  const int which = threadIdx.x >= kHalf;
  const int lt = threadIdx.x - which * kHalf;

  for (int64_t t = blockIdx.y; t < ntr; t += gridDim.y) {
    __syncthreads();
    {
      constexpr int kWords = (int)(sizeof(PlanLevel) / 4) * 2;
      const int* src = reinterpret_cast<const int*>(plans + t * plan_tstride + q0);
      if (threadIdx.x < kWords) reinterpret_cast<int*>(spl)[threadIdx.x] = src[threadIdx.x];
    }
    __syncthreads();
    if (threadIdx.x < 6) {
      GatherTab<n> tab;
      switch (threadIdx.x) {
        case 0: make_gather<n, 0>(spl[0], s0, tab); break;  // level q0, row-major in HBM
        case 1: make_gather<n, 1>(spl[0], s0, tab); break;
        case 2: make_scatter<n>(spl[0], s1, tab); break;
        case 3: make_gather_soa<n, 0>(spl[1], leafE * R, tab); break;  // level q0+1, SoA
        case 4: make_gather_soa<n, 1>(spl[1], leafE * R, tab); break;
        default: make_scatter_soa<n>(spl[1], leafE * R, tab); break;
      }
      tabs[threadIdx.x] = tab;
    }
    __syncthreads();

    // ---- expansion q0 -> q0+1: HBM (row-major) -> X1/Y1 (SoA, blocked)
    {
      const T* src = (which ? y : x) + t * xy_tstride + (int64_t)k0 * s0 * s0;
      T* dst = which ? Y1 : X1;
      const GatherTab<n> gt = tabs[which];
      for (int b = lt; b < kids1; b += kHalf) {
        const int sb = b / leafE, ip = b - (b / leafE) * leafE;
        const int i = (sb / n) * M + ip / M, j = (sb - (sb / n) * n) * M + (ip - (ip / M) * M);
        if (which)
          expand_tab<F, T, 1, 1>(src + i * s0 + j, gt, dst + b * R, 1);
        else
          expand_tab<F, T, 1, 0>(src + i * s0 + j, gt, dst + b * R, 1);
      }
    }
    __syncthreads();

#pragma unroll 1
    for (int kp0 = 0; kp0 < R; kp0 += G) {
      const int ng = R - kp0 < G ? R - kp0 : G;  // parents in this group
      const int nb2 = ng * R;                    // leaves in this group
      // ---- expansion q0+1 -> q0+2 of the group, item e = Kl + ng * pi
      {
        const GatherTab<n> gt = tabs[3 + which];
        const T* par = (which ? Y1 : X1) + kp0;
        T* kid = which ? Y2 : X2;
        for (int e = lt; e < ng * leafE; e += kHalf) {
          const int pi = e / ng, kl = e - (e / ng) * ng;
          if (which)
            expand_tab<F, T, 1, 1>(par + pi * R + kl, gt, kid + e * R, 1);
          else
            expand_tab<F, T, 1, 0>(par + pi * R + kl, gt, kid + e * R, 1);
        }
      }
      __syncthreads();

      // ---- leaf products, k ascending; element q of leaf l at q * nb2 + l
      if (S::kInPlace) {
        for (int l = threadIdx.x; l < nb2; l += NT) {
          T xa[leafE], yb[leafE];
#pragma unroll
          for (int q = 0; q < leafE; ++q) {
            xa[q] = X2[q * nb2 + l];
            yb[q] = Y2[q * nb2 + l];
          }
#pragma unroll
          for (int i = 0; i < M; ++i)
#pragma unroll
            for (int j = 0; j < M; ++j) {
              T acc = A::mul(xa[i * M], yb[j]);
#pragma unroll
              for (int k = 1; k < M; ++k) acc = A::add(acc, A::mul(xa[i * M + k], yb[k * M + j]));
              P2[(i * M + j) * nb2 + l] = acc;
            }
        }
      } else {
        for (int it = threadIdx.x; it < nb2 * M; it += NT) {
          const int i = it / nb2, l = it - (it / nb2) * nb2;
          T acc[M];
#pragma unroll
          for (int j = 0; j < M; ++j) acc[j] = A::mul(X2[(i * M) * nb2 + l], Y2[j * nb2 + l]);
#pragma unroll
          for (int k = 1; k < M; ++k) {
            const T xv = X2[(i * M + k) * nb2 + l];
#pragma unroll
            for (int j = 0; j < M; ++j) acc[j] = A::add(acc[j], A::mul(xv, Y2[(k * M + j) * nb2 + l]));
          }
#pragma unroll
          for (int j = 0; j < M; ++j) P2[(i * M + j) * nb2 + l] = acc[j];
        }
      }
      __syncthreads();

      // ---- contraction q0+2 -> q0+1 of the group into the dead X1 slots
      {
        const GatherTab<n> st = tabs[5];
        for (int e = threadIdx.x; e < ng * leafE; e += NT) {
          const int pi = e / ng, kl = e - (e / ng) * ng;
          contract_tab<F, T, 1, false>(P2 + e * R, 1, X1 + pi * R + kp0 + kl, st);
        }
      }
      __syncthreads();
    }

    // ---- contraction q0+1 -> q0: X1 -> HBM (row-major)
    bool ok = true;
    {
      const GatherTab<n> st = tabs[2];
      T* dbase = out + (t * K0 + k0) * (int64_t)s0 * s0;
      for (int b = threadIdx.x; b < kids1; b += NT) {
        const int sb = b / leafE, ip = b - (b / leafE) * leafE;
        const int i = (sb / n) * M + ip / M, j = (sb - (sb / n) * n) * M + (ip - (ip / M) * M);
        if (nonfinite)
          ok = contract_tab<F, T, 1, true>(X1 + b * R, 1, dbase + i * s0 + j, st) && ok;
        else
          contract_tab<F, T, 1, false>(X1 + b * R, 1, dbase + i * s0 + j, st);
      }
    }
    if (nonfinite && !ok) nonfinite[t] = 1;
  }
}

template <class F, class T, int M>
cudaError_t launch_subtree_soa(const void* x, const void* y, int64_t xy_tstride, int64_t K0,
                               void* out, const PlanLevel* plans, int64_t pts, int q0,
                               int64_t ntr, uint8_t* nonfinite, cudaStream_t st) {
  constexpr int NT = 256;
  // one parent group per subtree (two halve the leaf buffers -- 6 instead of 4
  // CTAs per SM on config 2 -- but the extra barrier rounds cost more: 5.3 vs
  // 5.0 ms per launch)
  using S = SubtreeSoA<F, T, M, 1>;
  const size_t smem = S::smem_bytes();
  auto kern = subtree_soa_kernel<F, T, M, 1, NT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)K0, (unsigned)(ntr < 65535 ? ntr : 65535));
  kern<<<grid, NT, smem, st>>>((const T*)x, (const T*)y, xy_tstride, (int)K0, (T*)out, plans, pts,
                               q0, ntr, nonfinite);
  return cudaGetLastError();
}

// ---- register-resident two-level subtree (small leaves) ----------------------
// Same arithmetic as subtree_kernel<F, T, 2, M>, with the level-(q0+1) stage
// moved out of shared memory.  Lane (r1, i) of a group of M lanes owns leaf
// row i of every sub-block of level-(q0+1) block r1: its X, Y and Z "fibers"
// (n*n sub-blocks x M columns) sit in registers.  Both folds of that level
// run element-wise down the fibers:
//   expansion  child r2 = fold over the n*n sub-blocks (formula networks,
//              one output r2 at a time: expand_u1 / expand_v1);
//   contraction Z(I,J)  = fold over r2 ascending (contract_w_step), i.e. the
//              reference's order (_engine.py:104-112) streamed over r2.
// Only the M x M leaf needs other lanes' data: the Y rows of the group,
// exchanged with warp shuffles.  The leaf keeps the reference's k-ascending
// order (_engine.py:42-61).
//
// Shared memory holds the level-(q0+1) blocks X1, Y1 position-major
// (element (block r, position p) at p * RP + r; RP pads R so the M rows a
// warp loads at once fall in disjoint banks, and keeps 2-element alignment).
// Positions are in the level-(q0+1) plan's BASE coordinates with the plan's
// sign already applied: stage A writes each child element where stage B's
// gather would read it, so stage B addresses are compile-time constants and
// Z goes back unpermuted; stage C reads Z through the plan's scatter and
// flips each child before contracting -- the same values the breadth-first
// kernels produce.  Z overwrites X1 in place: a lane writes exactly the rows
// {k*M + i} of block r1 it read.
// 4-byte elements: the next step's level-q0 blocks are prefetched by TMA bulk
// copies into two staging buffers (3.01 vs 3.28 ms per config-2 launch for
// operands read straight from HBM in stage A, which 2-byte elements do).
template <class F, class T, int M>
struct SubtreeReg {
  static constexpr int SUB = 1;  // subtrees per CTA step (2: 3.02 -> 3.16 ms, 3: 3.57)
  static constexpr int n = F::n;
  static constexpr int R = F::R;
  static constexpr int s1 = M * n;
  static constexpr int s0 = s1 * n;
  static constexpr int kids1 = s1 * s1;
  static constexpr int GPW = 32 / M;                      // leaf-row groups per warp
  static constexpr int NW = (SUB * R + GPW - 1) / GPW;    // one group per level-1 block
  static constexpr int NT = NW * 32;
  static constexpr int IA = (SUB * 2 * kids1 + NT - 1) / NT;  // stage-A items per thread
  static constexpr int IC = (SUB * kids1 + NT - 1) / NT;      // stage-C items per thread
  // child stride: (s1 * RP) mod 32 spreads the M rows of a warp over disjoint banks
  static constexpr int RP = (F::R == 23 && M == 3) ? 26 : R + (R & 1);
  static constexpr int slot = 2 * kids1 * RP;             // X1 + Y1 of one subtree
  // resident CTAs per SM the register budget aims at (about 128 registers a thread)
  // the two-row leaf holds a third 27-register fiber: one resident CTA fewer
  // keeps it spill-free
  static constexpr int kMinBlocks = 65536 / (128 * NT) > 1 ? 65536 / (128 * NT) - 1 : 1;
  static constexpr size_t header() {
    return ((sizeof(PlanLevel) * 2 + 15) / 16) * 16 + 3 * sizeof(GatherTab<n>);
  }
  // level-q0 blocks of a step's SUB subtrees (consecutive in HBM), prefetched
  // by TMA bulk copies into [buffers][X, Y][span] (4-byte elements): each
  // operand's blocks are copied as the 16-byte-aligned span that encloses them
  static constexpr bool kStage = sizeof(T) == 4;
  static constexpr int kBufs = 2;   // staging buffers
  static constexpr int kBanks = 1;  // X1/Y1 slot sets
  static constexpr int spanE = ((SUB * s0 * s0 + 4) + 3) / 4 * 4;  // SUB consecutive blocks
  static constexpr int stage_elems = kStage ? kBufs * 2 * spanE : 0;
  static constexpr int bank = SUB * slot;
  static constexpr size_t smem_bytes() {
    return header() + sizeof(T) * ((size_t)kBanks * bank + stage_elems) + (kStage ? 16 : 0);
  }
};

template <class T>
__device__ __forceinline__ T shfl_val(T v, int src) {
  return __shfl_sync(0xffffffffu, v, src);
}

template <int n>
__device__ __forceinline__ GatherTab<n> load_tab(const GatherTab<n>& src) {
  static_assert(sizeof(GatherTab<n>) % 16 == 0, "GatherTab is copied as int4");
  GatherTab<n> t;
  const int4* s = reinterpret_cast<const int4*>(&src);
  int4* d = reinterpret_cast<int4*>(&t);
#pragma unroll
  for (int k = 0; k < (int)(sizeof(GatherTab<n>) / 16); ++k) d[k] = s[k];
  return t;
}

// Stage-A item: one level-q0 position -> the R children, stored pairwise at
// dst + r (dst 2-element aligned) with the level-(q0+1) sign m applied.
// The ±1 network is odd (RN is symmetric under negation), so m is folded
// into the n*n gather flips instead of flipping the R outputs: same values,
// only the sign of an exact-zero child may differ (the plan path's
// np.array_equal contract).
template <class F, class T, int WHICH>
__device__ __forceinline__ void expand_to_children(const T* __restrict__ src,
                                                   const GatherTab<F::n>& gt, T* dst, uint32_t m) {
  constexpr int n = F::n;
  constexpr int R = F::R;
  using O = PackOps<T, 1>;
  Pack<T, 1> g[n * n];
#pragma unroll
  for (int k = 0; k < n * n; ++k) g[k] = O::flip(pload<T, 1>(src + gt.off[k]), gt.msk[k] ^ m);
  Pack<T, 1> o[R];
  if (WHICH == 0)
    F::template expand_u<T, 1>(g, o, gt.lastrow, gt.lastcol);
  else
    F::template expand_v<T, 1>(g, o, gt.lastrow, gt.lastcol);
#pragma unroll
  for (int r = 0; r + 1 < R; r += 2) {
    Pack<T, 2> v;
    v.v[0] = o[r].v[0];
    v.v[1] = o[r + 1].v[0];
    pstore<T, 2>(dst + r, v);
  }
  if (R & 1) dst[R - 1] = o[R - 1].v[0];
}

template <class F, class T, int M>
__global__ void __launch_bounds__(SubtreeReg<F, T, M>::NT, SubtreeReg<F, T, M>::kMinBlocks)
subtree_reg_kernel(
    const T* __restrict__ x, const T* __restrict__ y, int64_t xy_tstride, int K0, int kchunk,
    T* __restrict__ out, const PlanLevel* __restrict__ plans, int64_t plan_tstride, int q0,
    int64_t ntr, uint8_t* __restrict__ nonfinite) {
  using S = SubtreeReg<F, T, M>;
  using P = Pack<T, M>;
  constexpr int SUB = S::SUB;
  constexpr int n = F::n;
  constexpr int R = F::R;
  constexpr int s0 = S::s0, s1 = S::s1, kids1 = S::kids1, RP = S::RP, NT = S::NT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PlanLevel* spl = reinterpret_cast<PlanLevel*>(smem_raw);
  GatherTab<n>* tabs =
      reinterpret_cast<GatherTab<n>*>(smem_raw + ((sizeof(PlanLevel) * 2 + 15) / 16) * 16);
  T* sm = reinterpret_cast<T*>(smem_raw + S::header());
  // staged copies of the level-q0 blocks: [buf][X, Y][spanE]
  T* stg = sm + S::kBanks * S::bank;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(stg + S::stage_elems);

  // stage-B role of this lane: group -> (subtree slot u, level-1 block r1)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = lane / M;
  const int gwc = gw < S::GPW ? gw : S::GPW - 1;  // lanes past the last group mirror it
  const int gbase = gwc * M;
  const int li = gw < S::GPW ? lane - gw * M : (lane - gbase) % M;
  int grp = warp * S::GPW + gwc;
  const bool in_range = gw < S::GPW && grp < SUB * R;
  if (grp >= SUB * R) grp = SUB * R - 1;
  const int bu = grp / R, r1 = grp - (grp / R) * R;
  const int fib = bu * S::slot + li * s1 * RP + r1;  // lane's fiber origin

  const int kbeg = blockIdx.x * kchunk;
  const int kend = kbeg + kchunk < K0 ? kbeg + kchunk : K0;
  unsigned ctr = 0;  // staged copies consumed (buffer ctr % kBufs, phase (ctr / kBufs) & 1)
  if (S::kStage && threadIdx.x == 0) {
    for (int b = 0; b < S::kBufs; ++b) mbar_init(&mbar[b], 1);
    mbar_init_fence();
  }
  constexpr int blkE = s0 * s0;

  for (int64_t t = blockIdx.y; t < ntr; t += gridDim.y) {
    __syncthreads();
    {
      constexpr int kWords = (int)(sizeof(PlanLevel) / 4) * 2;
      const int* src = reinterpret_cast<const int*>(plans + t * plan_tstride + q0);
      if (threadIdx.x < kWords) reinterpret_cast<int*>(spl)[threadIdx.x] = src[threadIdx.x];
    }
    __syncthreads();
    if (threadIdx.x < 3) {
      GatherTab<n> tab;
      switch (threadIdx.x) {
        case 0: make_gather<n, 0>(spl[0], s0, tab); break;  // level q0 (HBM, row-major)
        case 1: make_gather<n, 1>(spl[0], s0, tab); break;
        default: make_scatter<n>(spl[0], s1, tab); break;
      }
      tabs[threadIdx.x] = tab;
    }
    // per-thread item maps of this trial (level q0+1 plan: hatted -> base)
    const PlanLevel& pl1 = spl[1];
    int a_src[S::IA], a_dst[S::IA];
    uint32_t a_msk[S::IA];
#pragma unroll
    for (int it = 0; it < S::IA; ++it) {
      const int e0 = threadIdx.x + it * NT;
      const int e = e0 < SUB * 2 * kids1 ? e0 : 0;
      const int u = e / (2 * kids1);
      const int eu = e - u * 2 * kids1;
      const int which = eu >= kids1;
      const int pos = eu - which * kids1;
      const int row = pos / s1, col = pos - (pos / s1) * s1;
      const int hk = row / M, hl = col / M;
      const int ri = which ? 1 : 0, ci = which ? 2 : 1;
      a_src[it] = u * s0 * s0 + row * s0 + col;
      a_dst[it] = u * S::slot + which * kids1 * RP +
                  ((pl1.perm[ri][hk] * M + (row - hk * M)) * s1 + pl1.perm[ci][hl] * M +
                   (col - hl * M)) * RP;
      a_msk[it] = sign_mask(pl1.neg[ri][hk] ^ pl1.neg[ci][hl]);
    }
    int c_src[S::IC];
    uint32_t c_msk[S::IC];
#pragma unroll
    for (int it = 0; it < S::IC; ++it) {
      const int e0 = threadIdx.x + it * NT;
      const int e = e0 < SUB * kids1 ? e0 : 0;
      const int u = e / kids1;
      const int pos = e - u * kids1;
      const int row = pos / s1, col = pos - (pos / s1) * s1;
      const int hi = row / M, hj = col / M;
      c_src[it] = u * S::slot +
                  ((pl1.perm[0][hi] * M + (row - hi * M)) * s1 + pl1.perm[2][hj] * M +
                   (col - hj * M)) * RP;
      c_msk[it] = sign_mask(pl1.neg[0][hi] ^ pl1.neg[2][hj]);
    }
    bool ok = true;
    auto issue = [&](int kp, unsigned bsel) {  // one thread
      const T* gx = x + t * xy_tstride + (int64_t)kp * blkE;
      const T* gy = y + t * xy_tstride + (int64_t)kp * blkE;
      const unsigned nb = (unsigned)(kend - kp < SUB ? kend - kp : SUB) * blkE * sizeof(T);
      const unsigned nx = span_bytes(gx, nb), ny = span_bytes(gy, nb);
      T* d = stg + bsel * 2 * S::spanE;
      fence_proxy_async();
      mbar_expect_tx(&mbar[bsel], nx + ny);
      bulk_g2s(d, span_start(gx), nx, &mbar[bsel]);
      bulk_g2s(d + S::spanE, span_start(gy), ny, &mbar[bsel]);
    };
    // ---- stage A: level q0 -> q0+1, level-q0 blocks -> X1 / Y1 (base order, signed)
    auto stage_a = [&](int k0, const T* buf, T* dst) {
      const int nsub = kend - k0 < SUB ? kend - k0 : SUB;
      const T* gx = x + t * xy_tstride + (int64_t)k0 * blkE;
      const T* gy = y + t * xy_tstride + (int64_t)k0 * blkE;
      const T* xsrc = gx;
      const T* ysrc = gy;
      if (S::kStage) {
        xsrc = buf + ((reinterpret_cast<uintptr_t>(gx) & 15) / sizeof(T));
        ysrc = buf + S::spanE + ((reinterpret_cast<uintptr_t>(gy) & 15) / sizeof(T));
      }
#pragma unroll
      for (int it = 0; it < S::IA; ++it) {
        const int e = threadIdx.x + it * NT;
        if (e < nsub * 2 * kids1) {
          const int which = (e - (e / (2 * kids1)) * 2 * kids1) >= kids1;
          if (which)
            expand_to_children<F, T, 1>(ysrc + a_src[it], load_tab(tabs[1]), dst + a_dst[it], a_msk[it]);
          else
            expand_to_children<F, T, 0>(xsrc + a_src[it], load_tab(tabs[0]), dst + a_dst[it], a_msk[it]);
        }
      }
    };
    // ---- stage B: level q0+1 -> leaves -> level q0+1, in registers
    auto stage_b = [&](int k0, T* base) {
      const int nsub = kend - k0 < SUB ? kend - k0 : SUB;
      const T* X1 = base;
      const T* Y1 = base + kids1 * RP;
      const int xlr = pl1.perm[0][n - 1], xlc = pl1.perm[1][n - 1];
      const int ylr = pl1.perm[1][n - 1], ylc = pl1.perm[2][n - 1];
      P z[n * n];
      {
        // Two Y rows per lane, one by shuffles: slot A = row ra (the lane's
        // own row, row 0 for lane 2), slot B = row rb from the lane whose
        // slot A holds it, slot C = row 2 on every lane.  The leaf fold
        // ((A + B) + C) then keeps k = 2 last with no selects (the first two
        // terms commute); the X fiber is loaded with its columns in slot
        // order.  3 shuffles instead of 9 for one more Y network per r2.
        static_assert(M == 3, "two-row leaf is for 3x3 leaves");
        const int ra = li == 2 ? 0 : li;
        const int rb = li == 1 ? 0 : 1;
        const int xcol[3] = {ra, rb, 2};
        const int fa = bu * S::slot + ra * s1 * RP + r1;
        const int fc = bu * S::slot + 2 * s1 * RP + r1;
        P xf[n * n], ya[n * n], yc[n * n];
#pragma unroll
        for (int k = 0; k < n * n; ++k) {
          const int o = ((k / n) * M * s1 + (k % n) * M) * RP;
#pragma unroll
          for (int j = 0; j < M; ++j) {
            xf[k].v[j] = X1[o + fib + xcol[j] * RP];
            ya[k].v[j] = Y1[o + fa + j * RP];
            yc[k].v[j] = Y1[o + fc + j * RP];
          }
        }
        using A = Arith<T>;
#pragma unroll
        for (int r2 = 0; r2 < R; ++r2) {
          const P xg = F::template expand_u1<T, M>(xf, r2, xlr, xlc);
          const P yag = F::template expand_v1<T, M>(ya, r2, ylr, ylc);
          const P ycg = F::template expand_v1<T, M>(yc, r2, ylr, ylc);
          P m, ybg;
#pragma unroll
          for (int j = 0; j < M; ++j) ybg.v[j] = shfl_val(yag.v[j], gbase + rb);
          if constexpr (std::is_same<T, float>::value && M == 3) {
            // columns 0 and 1 as one f32x2 pair (each lane rounds like the
            // scalar FMUL / FADD), column 2 scalar
            using O3 = PackOps<float, 3>;
            const uint64_t p01 = f2_add(
                f2_add(f2_mul_bcast(xg.v[0], O3::pr(yag), kcF2NegZero),
                       f2_mul_bcast(xg.v[1], O3::pr(ybg), kcF2NegZero)),
                f2_mul_bcast(xg.v[2], O3::pr(ycg), kcF2NegZero));
            m = O3::un(p01, A::add(A::add(A::mul(xg.v[0], yag.v[2]), A::mul(xg.v[1], ybg.v[2])),
                                   A::mul(xg.v[2], ycg.v[2])));
          } else {
#pragma unroll
            for (int j = 0; j < M; ++j)
              m.v[j] = A::add(A::add(A::mul(xg.v[0], yag.v[j]), A::mul(xg.v[1], ybg.v[j])),
                              A::mul(xg.v[2], ycg.v[j]));
          }
          F::template contract_w_step<T, M>(z, m, r2);
        }
      }
      F::template contract_w_finish<T, M>(z);
      if (in_range && bu < nsub) {
        T* Z1 = base;
#pragma unroll
        for (int k = 0; k < n * n; ++k) {
          const int o = ((k / n) * M * s1 + (k % n) * M) * RP + fib;
#pragma unroll
          for (int j = 0; j < M; ++j) Z1[o + j * RP] = z[k].v[j];
        }
      }
    };
    // ---- stage C: level q0+1 -> q0, Z1 -> HBM (row-major)
    auto stage_c = [&](int k0, const T* base) {
      const int nsub = kend - k0 < SUB ? kend - k0 : SUB;
      const GatherTab<n> sc = load_tab(tabs[2]);
#pragma unroll
      for (int it = 0; it < S::IC; ++it) {
        const int e = threadIdx.x + it * NT;
        if (e < nsub * kids1) {
          using O = PackOps<T, 1>;
          const int u = e / kids1, pos = e - (e / kids1) * kids1;
          // the child flip c_msk is folded into the n*n output flips (the
          // contraction network is odd too; see expand_to_children)
          const T* zc = base + c_src[it];
          Pack<T, 1> pr[R];
#pragma unroll
          for (int r = 0; r + 1 < R; r += 2) {
            const Pack<T, 2> v = pload<T, 2>(zc + r);
            pr[r].v[0] = v.v[0];
            pr[r + 1].v[0] = v.v[1];
          }
          if (R & 1) pr[R - 1].v[0] = zc[R - 1];
          Pack<T, 1> o[n * n];
          F::template contract_w<T, 1>(pr, o);
          const int row = pos / s1, col = pos - (pos / s1) * s1;
          T* d = out + (t * K0 + k0 + u) * (int64_t)s0 * s0 + row * s0 + col;
#pragma unroll
          for (int k = 0; k < n * n; ++k) {
            const Pack<T, 1> val = O::flip(o[k], sc.msk[k] ^ c_msk[it]);
            if (nonfinite) ok = ok && O::all_finite(val);
            pstore<T, 1>(d + sc.off[k], val);
          }
        }
      }
    };

    if (S::kStage && threadIdx.x == 0 && kbeg < kend) issue(kbeg, ctr & 1);
    for (int k0 = kbeg; k0 < kend; k0 += SUB, ++ctr) {
      if (S::kStage) mbar_wait(&mbar[ctr & 1], (ctr >> 1) & 1);
      __syncthreads();
      stage_a(k0, stg + (ctr & 1) * 2 * S::spanE, sm);
      __syncthreads();
      if (S::kStage && threadIdx.x == 0 && k0 + SUB < kend) issue(k0 + SUB, (ctr + 1) & 1);
      stage_b(k0, sm);
      __syncthreads();
      stage_c(k0, sm);
    }
    if (nonfinite && !ok) nonfinite[t] = 1;
  }
}

// Measured and not kept on config 2 (ms per launch; default 2.74): two or
// three subtrees per CTA step 3.16 / 3.57; the leaf's Y rows by 9 shuffles
// 2.96, a rotated 6-shuffle leaf 3.38; a shuffle-free leaf where every lane
// expands the whole Y fiber 8.5; one lane per leaf element 3.9; a
// warp-specialised schedule 8.4; the runtime fold order specialised by a
// CTA-uniform switch instead of fold3 selects 3.20; a pipelined two-barrier
// schedule 3.01; 8 or 48 subtrees per CTA 3.44 / 3.46; one THREAD per
// level-(q0+1) block, everything below it in registers 5.09 (255 registers,
// 8 warps per SM: latency-bound; profiles/r02/experiments).
template <class F, class T, int M>
cudaError_t launch_subtree_reg(const void* x, const void* y, int64_t xy_tstride, int64_t K0,
                               void* out, const PlanLevel* plans, int64_t pts, int q0,
                               int64_t ntr, uint8_t* nonfinite, cudaStream_t st) {
  using S = SubtreeReg<F, T, M>;
  const size_t smem = S::smem_bytes();
  auto kern = subtree_reg_kernel<F, T, M>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // about 24 subtrees per CTA, balanced so no CTA gets a short tail chunk
  // (config 2: 529 blocks -> 23 x 23 instead of 22 x 24 + 1: 3.02 -> 2.98 ms)
  const int64_t nchunks = (K0 + 23) / 24;
  int kchunk = (int)((K0 + nchunks - 1) / nchunks);
  kchunk = ((kchunk + S::SUB - 1) / S::SUB) * S::SUB;
  if (kchunk > K0) kchunk = (int)K0;
  const int64_t nkc = (K0 + kchunk - 1) / kchunk;
  dim3 grid((unsigned)nkc, (unsigned)(ntr < 65535 ? ntr : 65535));
  kern<<<grid, S::NT, smem, st>>>((const T*)x, (const T*)y, xy_tstride, (int)K0, kchunk, (T*)out,
                                  plans, pts, q0, ntr, nonfinite);
  return cudaGetLastError();
}

template <class F, class T, int L, int M>
cudaError_t launch_subtree_t(const void* x, const void* y, int64_t xy_tstride, int64_t K0,
                             void* out, const PlanLevel* plans, int64_t pts, int q0, int64_t ntr,
                             uint8_t* nonfinite, cudaStream_t st) {
  if constexpr (L == 2) {
    // 3 x 3 Laderman leaves: level q0+1 in registers
    if constexpr (F::kId == FLaderman::kId && M == 3 && !std::is_same<T, double>::value)
      return launch_subtree_reg<F, T, M>(x, y, xy_tstride, K0, out, plans, pts, q0, ntr, nonfinite, st);
    // other two-level shapes: position-major shared-memory layout
    return launch_subtree_soa<F, T, M>(x, y, xy_tstride, K0, out, plans, pts, q0, ntr, nonfinite, st);
  } else {
    using S = Subtree<F, T, L, M>;
    const size_t smem = S::smem_bytes();
    auto kern = subtree_kernel<F, T, L, M, kThreads>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid((unsigned)K0, (unsigned)(ntr < 65535 ? ntr : 65535));
    kern<<<grid, kThreads, smem, st>>>((const T*)x, (const T*)y, xy_tstride, (int)K0, (T*)out, plans,
                                       pts, q0, ntr, nonfinite);
    return cudaGetLastError();
  }
}

// Table of instantiated (formula, L, M) shapes.
template <class T>
cudaError_t dispatch(int formula, int L, int M, const void* x, const void* y, int64_t xs,
                     int64_t K0, void* out, const PlanLevel* plans, int64_t pts, int q0,
                     int64_t ntr, uint8_t* nf, cudaStream_t st) {
#define RBC_SUBTREE(FT, LL, MM)                                                               \
  if (formula == FT::kId && L == LL && M == MM)                                               \
    return launch_subtree_t<FT, T, LL, MM>(x, y, xs, K0, out, plans, pts, q0, ntr, nf, st);
  RBC_SUBTREE(FLaderman, 2, 3)
  RBC_SUBTREE(FLaderman, 2, 1)
  RBC_SUBTREE(FLaderman, 1, 3)
  RBC_SUBTREE(FLaderman, 1, 9)
  RBC_SUBTREE(FStrassen, 2, 10)
  RBC_SUBTREE(FStrassen, 2, 5)
  RBC_SUBTREE(FStrassen, 2, 8)
  RBC_SUBTREE(FStrassen, 2, 4)
  RBC_SUBTREE(FStrassen, 2, 2)
  RBC_SUBTREE(FStrassen, 2, 1)
  RBC_SUBTREE(FStrassen, 1, 16)
#undef RBC_SUBTREE
  return cudaErrorNotSupported;
}

template <class T>
size_t smem_of(int formula, int L, int M) {
#define RBC_SMEM(FT, LL, MM) \
  if (formula == FT::kId && L == LL && M == MM) return Subtree<FT, T, LL, MM>::smem_bytes();
  RBC_SMEM(FLaderman, 2, 3)
  RBC_SMEM(FLaderman, 2, 1)
  RBC_SMEM(FLaderman, 1, 3)
  RBC_SMEM(FLaderman, 1, 9)
  RBC_SMEM(FStrassen, 2, 10)
  RBC_SMEM(FStrassen, 2, 5)
  RBC_SMEM(FStrassen, 2, 8)
  RBC_SMEM(FStrassen, 2, 4)
  RBC_SMEM(FStrassen, 2, 2)
  RBC_SMEM(FStrassen, 2, 1)
  RBC_SMEM(FStrassen, 1, 16)
#undef RBC_SMEM
  return 0;
}

}  // namespace

size_t subtree_smem_bytes(int dtype, int formula, int L, int M) {
  switch (dtype) {
    case kF64: return smem_of<double>(formula, L, M);
    case kF32: return smem_of<float>(formula, L, M);
    case kF16: return smem_of<__half>(formula, L, M);
  }
  return 0;
}

cudaError_t launch_subtree(int dtype, int formula, int L, int M, const void* x, const void* y,
                           int64_t xy_tstride, int64_t K0, void* out, const PlanLevel* plans,
                           int64_t plan_tstride, int q0, int64_t ntr, uint8_t* nonfinite,
                           cudaStream_t st) {
  switch (dtype) {
    case kF64: return dispatch<double>(formula, L, M, x, y, xy_tstride, K0, out, plans, plan_tstride, q0, ntr, nonfinite, st);
    case kF32: return dispatch<float>(formula, L, M, x, y, xy_tstride, K0, out, plans, plan_tstride, q0, ntr, nonfinite, st);
    case kF16: return dispatch<__half>(formula, L, M, x, y, xy_tstride, K0, out, plans, plan_tstride, q0, ntr, nonfinite, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace rbc
