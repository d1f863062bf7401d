// Exact-order batched leaf products (reference leaf_matmul,
// pkg/src/randbc/_engine.py:42-61):
//
//   P[i,j] = fl(...fl(fl(x_i0*y_0j) + fl(x_i1*y_1j)) + ...),  k ascending,
//
// one rounding per multiply and per add, first term initialising, no FMA and
// no split-K.  This pins the rounding of every output element to the
// reference's, so per-trial errors match.  Consequently the
// kernels run on the CUDA-core FP pipes (FMUL + FADD per multiply-add), not
// on the tensor cores, whose internal accumulation would change the very
// rounding error the paper measures.
//
// Two kernels:
//  * leaf_small  -- one thread per output element, for leaves narrower than a
//                   tile (3x3, 10x10, 27x27 ...).
//  * leaf_tiled  -- BM x BN x BK register-tiled SGEMM/DGEMM structure:
//                   operand tiles double-buffered in shared memory (A stored
//                   k-major), each thread owns TM x TN outputs in VW-wide
//                   groups so fragments are read with 16-byte LDS, and every
//                   output keeps its own sequential k chain.
// Both also serve the binary64 ground truth of binary32/binary16 operands
// (TIn narrower than TAcc: operands are widened exactly on load).

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "bulk.cuh"
#include "kernels.h"

namespace rbc {

namespace {

template <class TIn, class TAcc>
__device__ __forceinline__ TAcc widen_to(TIn v);
template <> __device__ __forceinline__ float widen_to<float, float>(float v) { return v; }
template <> __device__ __forceinline__ double widen_to<double, double>(double v) { return v; }
template <> __device__ __forceinline__ double widen_to<float, double>(float v) { return (double)v; }
template <> __device__ __forceinline__ __half widen_to<__half, __half>(__half v) { return v; }
template <> __device__ __forceinline__ double widen_to<__half, double>(__half v) {
  return (double)__half2float(v);
}
template <> __device__ __forceinline__ float widen_to<__half, float>(__half v) {
  return __half2float(v);
}

// Multiply-add step acc <- fl(acc + fl(a*b)).  When the operands were widened
// from a narrower type into binary64 (f32 or f16 -> f64: the binary64 truth),
// a*b has at most 48 significant bits and is exact in binary64, so
// fl(acc + fl(a*b)) == fl(acc + a*b) == fma(a, b, acc) bit for bit: one DFMA
// replaces DMUL + DADD with identical results.  Same-type products are not
// exact and keep the separately rounded multiply and add.
template <class TIn, class TAcc>
struct Mac {
  static __device__ __forceinline__ TAcc step(TAcc acc, TAcc a, TAcc b) {
    return Arith<TAcc>::add(acc, Arith<TAcc>::mul(a, b));
  }
};
template <>
struct Mac<float, double> {
  static __device__ __forceinline__ double step(double acc, double a, double b) {
    return __fma_rn(a, b, acc);
  }
};
template <>
struct Mac<__half, double> {
  static __device__ __forceinline__ double step(double acc, double a, double b) {
    return __fma_rn(a, b, acc);
  }
};

// Test hook (tests/test_trials_gpu.py): RBC_LEAF_TILE=999 skips the
// specialised kernels so the generic tiles run at every size, 303 runs the
// bulk-copy binary64 kernel from 128 up, 205 the single-shot small-leaf kernel.
inline int tile_override() {
  const char* v = getenv("RBC_LEAF_TILE");
  return v ? atoi(v) : 0;
}

template <class TIn, class TAcc>
__global__ void __launch_bounds__(256) leaf_small_kernel(int64_t batch, int M, int K, int N,
                                                         const TIn* __restrict__ x, int64_t xs,
                                                         const TIn* __restrict__ y, int64_t ys,
                                                         TAcc* __restrict__ out) {
  using A = Arith<TAcc>;
  const int64_t per = (int64_t)M * N;
  const int64_t total = batch * per;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / per;
    const int rem = (int)(idx - b * per);
    const int i = rem / N;
    const int j = rem - i * N;
    const TIn* xr = x + b * xs + (int64_t)i * K;
    const TIn* yc = y + b * ys + j;
    TAcc acc = A::mul(widen_to<TIn, TAcc>(xr[0]), widen_to<TIn, TAcc>(yc[0]));
    for (int k = 1; k < K; ++k)
      acc = Mac<TIn, TAcc>::step(acc, widen_to<TIn, TAcc>(xr[k]), widen_to<TIn, TAcc>(yc[(int64_t)k * N]));
    out[idx] = acc;
  }
}

// VW = elements per 16-byte fragment read.
template <class TIn, class TAcc, int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), (BM / TM) * (BN / TN) >= 256 ? 2 : 4)
    leaf_tiled_kernel(int M, int K, int N, const TIn* __restrict__ x, int64_t xs,
                      const TIn* __restrict__ y, int64_t ys, TAcc* __restrict__ out,
                      int tiles_n) {
  constexpr int VW = 16 / (int)sizeof(TAcc) < TM ? 16 / (int)sizeof(TAcc) : TM;
  constexpr int DY = BM / TM;  // threads along M
  constexpr int DX = BN / TN;  // threads along N
  constexpr int NT = DY * DX;
  constexpr int GM = TM / VW;  // fragment groups along M
  constexpr int GN = TN / VW;
  constexpr int A_PER = BM * BK / NT;  // A elements loaded per thread per tile
  constexpr int B_PER = BK * BN / NT;
  static_assert(BM * BK % NT == 0 && BK * BN % NT == 0, "tile/threads");
  static_assert(TM % VW == 0 && TN % VW == 0, "fragment width");
  using A = Arith<TAcc>;

  // A is stored transposed (k-major).  A row of BM elements is a multiple of
  // 32 banks, so the 16-byte pad spreads the k rows a warp stores at once
  // over the banks (8-way -> conflict-free for f32, <= 3-way for f64) and
  // keeps the 16-byte fragment loads aligned.
  constexpr int APAD = 16 / (int)sizeof(TAcc);
  extern __shared__ __align__(16) unsigned char leaf_smem[];
  auto As = reinterpret_cast<TAcc(*)[BK][BM + APAD]>(leaf_smem);
  auto Bs = reinterpret_cast<TAcc(*)[BK][BN]>(leaf_smem + sizeof(TAcc) * 2 * BK * (BM + APAD));

  const int tid = threadIdx.x;
  const int tx = tid % DX;
  const int ty = tid / DX;
  const int64_t b = blockIdx.y + (int64_t)blockIdx.z * 65535;
  const int tm = blockIdx.x / tiles_n;
  const int tn = blockIdx.x - tm * tiles_n;
  const int m0 = tm * BM;
  const int n0 = tn * BN;
  const TIn* xb = x + b * xs;
  const TIn* yb = y + b * ys;

  // staged in the input type (narrow operands are widened at the smem store)
  TIn ra[A_PER];
  TIn rb[B_PER];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int q = 0; q < A_PER; ++q) {
      const int e = tid + q * NT;
      const int mm = e / BK, kk = e % BK;
      const int gm = m0 + mm, gk = k0 + kk;
      ra[q] = (gm < M && gk < K) ? xb[(int64_t)gm * K + gk] : TIn(0.0f);
    }
#pragma unroll
    for (int q = 0; q < B_PER; ++q) {
      const int e = tid + q * NT;
      const int kk = e / BN, nn = e % BN;
      const int gk = k0 + kk, gn = n0 + nn;
      rb[q] = (gk < K && gn < N) ? yb[(int64_t)gk * N + gn] : TIn(0.0f);
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int q = 0; q < A_PER; ++q) {
      const int e = tid + q * NT;
      As[buf][e % BK][e / BK] = widen_to<TIn, TAcc>(ra[q]);
    }
#pragma unroll
    for (int q = 0; q < B_PER; ++q) {
      const int e = tid + q * NT;
      Bs[buf][e / BN][e % BN] = widen_to<TIn, TAcc>(rb[q]);
    }
  };

  TAcc acc[TM][TN];
  // register fragments; for binary64 accumulation double-buffered over k so
  // the shared-memory loads of step k+1 are in flight during the DFMAs of
  // step k (f32: the extra registers cost more occupancy than they hide)
  constexpr bool kPipeFrag = sizeof(TAcc) == 8;
  TAcc fa[2][TM], fb[2][TN];
  auto load_frag = [&](int buf, int kk, int s) {
#pragma unroll
    for (int g = 0; g < GM; ++g)
#pragma unroll
      for (int v = 0; v < VW; ++v) fa[s][g * VW + v] = As[buf][kk][g * DY * VW + ty * VW + v];
#pragma unroll
    for (int g = 0; g < GN; ++g)
#pragma unroll
      for (int v = 0; v < VW; ++v) fb[s][g * VW + v] = Bs[buf][kk][g * DX * VW + tx * VW + v];
  };
  // one k step of the register tile (the very first k initialises)
  auto kstep = [&](int s, bool first) {
    if (first) {
#pragma unroll
      for (int ii = 0; ii < TM; ++ii)
#pragma unroll
        for (int jj = 0; jj < TN; ++jj) acc[ii][jj] = A::mul(fa[s][ii], fb[s][jj]);
    } else {
#pragma unroll
      for (int ii = 0; ii < TM; ++ii)
#pragma unroll
        for (int jj = 0; jj < TN; ++jj) acc[ii][jj] = Mac<TIn, TAcc>::step(acc[ii][jj], fa[s][ii], fb[s][jj]);
    }
  };
  const int ktiles = (K + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  for (int kt = 0; kt < ktiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ktiles) load_tile((kt + 1) * BK);
    const int kmax = min(BK, K - kt * BK);
    if constexpr (kPipeFrag) {
      load_frag(buf, 0, 0);
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        if (kk + 1 < BK) load_frag(buf, kk + 1, (kk + 1) & 1);
        if (kk < kmax) kstep(kk & 1, kt == 0 && kk == 0);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        if (kk < kmax) {
          load_frag(buf, kk, 0);
          kstep(0, kt == 0 && kk == 0);
        }
      }
    }
    if (kt + 1 < ktiles) {
      store_tile(buf ^ 1);
      __syncthreads();
    }
  }

  TAcc* ob = out + b * (int64_t)M * N;
#pragma unroll
  for (int gi = 0; gi < GM; ++gi)
#pragma unroll
    for (int v = 0; v < VW; ++v) {
      const int gm = m0 + gi * DY * VW + ty * VW + v;
      if (gm >= M) continue;
#pragma unroll
      for (int gj = 0; gj < GN; ++gj)
#pragma unroll
        for (int w = 0; w < VW; ++w) {
          const int gn = n0 + gj * DX * VW + tx * VW + w;
          if (gn < N) ob[(int64_t)gm * N + gn] = acc[gi * VW + v][gj * VW + w];
        }
    }
}

// Binary64 accumulation (the truth, and binary64 leaves of 128 and up):
// 128 x 128 x 16 tiles, 8 x 8 outputs per thread (64 independent chains),
// one CTA of 256 threads per SM.  Warps are 4 (M) x 8 (N) threads, so every
// 16-byte fragment load of a k step is one shared-memory wavefront (4 or 8
// distinct 16-byte spans), i.e. 8 wavefronts per 64 DFMA warp instructions;
// fragments are double-buffered over k.  Operands are widened to binary64 at
// the shared-memory store (once per element per CTA), never in the k loop.
// Every output keeps its own sequential k chain: the first product
// initialises (a multiply, not an FMA into +0, which would lose the sign of
// a -0 product) and K tails are skipped, not zero-padded (fl(-0 + 0*0) = +0).
template <class TIn, int BM, int BN, int BK, int TM, int TN, bool PIPE, int MINB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
    truth_tiled_kernel(int M, int K, int N, const TIn* __restrict__ x, int64_t xs,
                       const TIn* __restrict__ y, int64_t ys, double* __restrict__ out,
                       int tiles_n) {
  constexpr int VW = 2;           // doubles per 16-byte fragment load
  constexpr int DY = BM / TM;     // thread rows
  constexpr int DX = BN / TN;     // thread columns
  constexpr int NT = DY * DX;
  constexpr int GM = TM / VW, GN = TN / VW;
  constexpr int A_PER = BM * BK / NT, B_PER = BK * BN / NT;
  constexpr int WX = 8, WY = 4;   // warp shape (threads along N, M)
  static_assert(NT % 32 == 0 && DX % WX == 0 && DY % WY == 0, "warp tiling");
  static_assert(BM * BK % NT == 0 && BK * BN % NT == 0, "tile/threads");
  constexpr int APAD = 2, BPAD = 2;
  using Acc = Arith<double>;
  extern __shared__ __align__(16) unsigned char leaf_smem[];
  auto As = reinterpret_cast<double(*)[BK][BM + APAD]>(leaf_smem);
  auto Bs = reinterpret_cast<double(*)[BK][BN + BPAD]>(leaf_smem + sizeof(double) * 2 * BK * (BM + APAD));

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int WPX = DX / WX;  // warps along N
  const int tx = (warp % WPX) * WX + (lane % WX);
  const int ty = (warp / WPX) * WY + (lane / WX);
  const int64_t b = blockIdx.y + (int64_t)blockIdx.z * 65535;
  const int tm = blockIdx.x / tiles_n;
  const int tn = blockIdx.x - tm * tiles_n;
  const int m0 = tm * BM, n0 = tn * BN;
  const TIn* xb = x + b * xs;
  const TIn* yb = y + b * ys;

  // Per-thread load geometry, fixed across k tiles (NT divides BK * BN and
  // BM * BK): A element (m0 + a_m + q * AR, k0 + a_k), B element
  // (k0 + b_k + q * BR, n0 + b_n).  Interior k tiles skip the K checks, rows
  // and columns past M / N are masked once per thread.
  static_assert(NT % BK == 0 && NT % BN == 0, "load geometry");
  constexpr int AR = NT / BK, BR = NT / BN;
  static_assert(A_PER <= 32, "row mask");
  const int a_k = tid % BK, a_m = tid / BK;
  const int b_n = tid % BN, b_k = tid / BN;
  const TIn* pa = xb + (int64_t)(m0 + a_m) * K + a_k;
  const TIn* pb = yb + (int64_t)b_k * N + n0 + b_n;
  const int64_t sa = (int64_t)AR * K, sb = (int64_t)BR * N;
  uint32_t a_rows = 0;
#pragma unroll
  for (int q = 0; q < A_PER; ++q) a_rows |= (m0 + a_m + q * AR < M ? 1u : 0u) << q;
  const bool b_col = n0 + b_n < N;
  TIn ra[A_PER], rb[B_PER];
  auto load_tile = [&](int k0) {
    const TIn* p = pa + k0;
    const TIn* r = pb + (int64_t)k0 * N;
    if (k0 + BK <= K) {
#pragma unroll
      for (int q = 0; q < A_PER; ++q) ra[q] = ((a_rows >> q) & 1) ? p[q * sa] : TIn(0.0f);
#pragma unroll
      for (int q = 0; q < B_PER; ++q) rb[q] = b_col ? r[q * sb] : TIn(0.0f);
    } else {
      const bool ak = k0 + a_k < K;
#pragma unroll
      for (int q = 0; q < A_PER; ++q) ra[q] = (ak && ((a_rows >> q) & 1)) ? p[q * sa] : TIn(0.0f);
#pragma unroll
      for (int q = 0; q < B_PER; ++q)
        rb[q] = (b_col && k0 + b_k + q * BR < K) ? r[q * sb] : TIn(0.0f);
    }
  };
  auto store_tile = [&](int buf) {
    double* da = &As[buf][a_k][a_m];
    double* db = &Bs[buf][b_k][b_n];
#pragma unroll
    for (int q = 0; q < A_PER; ++q) da[q * AR] = widen_to<TIn, double>(ra[q]);
#pragma unroll
    for (int q = 0; q < B_PER; ++q) db[q * BR * (BN + BPAD)] = widen_to<TIn, double>(rb[q]);
  };

  double acc[TM][TN];
  double fa[PIPE ? 2 : 1][TM], fb[PIPE ? 2 : 1][TN];
  auto load_frag = [&](int buf, int kk, int s) {
#pragma unroll
    for (int g = 0; g < GM; ++g) {
      const double2 v = *reinterpret_cast<const double2*>(&As[buf][kk][g * DY * VW + ty * VW]);
      fa[s][g * VW] = v.x;
      fa[s][g * VW + 1] = v.y;
    }
#pragma unroll
    for (int g = 0; g < GN; ++g) {
      const double2 v = *reinterpret_cast<const double2*>(&Bs[buf][kk][g * DX * VW + tx * VW]);
      fb[s][g * VW] = v.x;
      fb[s][g * VW + 1] = v.y;
    }
  };
  auto kstep = [&](int s) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = Mac<TIn, double>::step(acc[i][j], fa[s][i], fb[s][j]);
  };

  const int ktiles = (K + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  for (int kt = 0; kt < ktiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ktiles) load_tile((kt + 1) * BK);
    const int kmax = min(BK, K - kt * BK);
    load_frag(buf, 0, 0);
    if (kt == 0) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = Acc::mul(fa[0][i], fb[0][j]);
    }
    if (kmax == BK) {
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        if constexpr (PIPE) {
          if (kk + 1 < BK) load_frag(buf, kk + 1, (kk + 1) & 1);
          if (kk > 0 || kt > 0) kstep(kk & 1);
        } else {
          if (kk > 0) load_frag(buf, kk, 0);
          if (kk > 0 || kt > 0) kstep(0);
        }
      }
    } else {
      // K tail: same chain, fewer steps
#pragma unroll 1
      for (int kk = 0; kk < kmax; ++kk) {
        load_frag(buf, kk, 0);
        if (kk > 0 || kt > 0) kstep(0);
      }
    }
    if (kt + 1 < ktiles) {
      store_tile(buf ^ 1);
      __syncthreads();
    }
  }

  double* ob = out + b * (int64_t)M * N;
#pragma unroll
  for (int gi = 0; gi < GM; ++gi)
#pragma unroll
    for (int v = 0; v < VW; ++v) {
      const int gm = m0 + gi * DY * VW + ty * VW + v;
      if (gm >= M) continue;
#pragma unroll
      for (int gj = 0; gj < GN; ++gj) {
        const int gn = n0 + gj * DX * VW + tx * VW;
        double* o = ob + (int64_t)gm * N + gn;
        if (gn + 1 < N && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
          *reinterpret_cast<double2*>(o) = make_double2(acc[gi * VW + v][gj * VW], acc[gi * VW + v][gj * VW + 1]);
        } else {
          if (gn < N) o[0] = acc[gi * VW + v][gj * VW];
          if (gn + 1 < N) o[1] = acc[gi * VW + v][gj * VW + 1];
        }
      }
    }
}

template <class TIn, int BM, int BN, int BK, int TM, int TN, bool PIPE = true, int MINB = 1>
cudaError_t run_truth(int64_t batch, int64_t M, int64_t K, int64_t N, const void* x, int64_t xs,
                      const void* y, int64_t ys, void* out, cudaStream_t st) {
  const int tiles_m = (int)((M + BM - 1) / BM);
  const int tiles_n = (int)((N + BN - 1) / BN);
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr size_t smem = sizeof(double) * 2 * BK * ((BM + 2) + (BN + 2));
  static const cudaError_t attr = cudaFuncSetAttribute(
      truth_tiled_kernel<TIn, BM, BN, BK, TM, TN, PIPE, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)smem);
  if (attr != cudaSuccess) return attr;
  for (int64_t b0 = 0; b0 < batch;) {
    const int64_t nb = std::min<int64_t>(batch - b0, (int64_t)65535 * 65535);
    const int64_t full = (nb / 65535) * 65535;
    if (full > 0) {
      dim3 grid(tiles_m * tiles_n, 65535, (unsigned)(full / 65535));
      truth_tiled_kernel<TIn, BM, BN, BK, TM, TN, PIPE, MINB><<<grid, NT, smem, st>>>(
          (int)M, (int)K, (int)N, (const TIn*)x + b0 * xs, xs, (const TIn*)y + b0 * ys, ys,
          (double*)out + b0 * M * N, tiles_n);
    }
    if (nb > full) {
      dim3 grid(tiles_m * tiles_n, (unsigned)(nb - full), 1);
      const int64_t bb = b0 + full;
      truth_tiled_kernel<TIn, BM, BN, BK, TM, TN, PIPE, MINB><<<grid, NT, smem, st>>>(
          (int)M, (int)K, (int)N, (const TIn*)x + bb * xs, xs, (const TIn*)y + bb * ys, ys,
          (double*)out + bb * M * N, tiles_n);
    }
    b0 += nb;
  }
  return cudaGetLastError();
}

// Small square leaves (M x M, M below a tile): one CTA stages LPB whole
// leaves of X and Y in shared memory with coalesced loads (leaves are
// contiguous), then each thread computes a TR x TR register tile of one leaf
// with the sequential k chain.  Serves config 3's 27x27 binary64 leaves.
template <class TIn, class TAcc, int M, int TR>
__global__ void __launch_bounds__(256) leaf_smem_kernel(int64_t batch, const TIn* __restrict__ x,
                                                        int64_t xs, const TIn* __restrict__ y,
                                                        int64_t ys, TAcc* __restrict__ out) {
  constexpr int TPL = (M / TR) * (M / TR);  // threads per leaf
  constexpr int LPB = 256 / TPL;            // leaves per block
  static_assert(M % TR == 0 && LPB >= 1, "leaf tiling");
  using A = Arith<TAcc>;
  __shared__ TAcc Xs[LPB][M * M];
  __shared__ TAcc Ys[LPB][M * M];
  const int64_t b0 = (int64_t)blockIdx.x * LPB;
  const int nl = batch - b0 < LPB ? (int)(batch - b0) : LPB;
  for (int e = threadIdx.x; e < nl * M * M; e += blockDim.x) {
    const int l = e / (M * M), q = e - l * (M * M);
    Xs[l][q] = widen_to<TIn, TAcc>(x[(b0 + l) * xs + q]);
    Ys[l][q] = widen_to<TIn, TAcc>(y[(b0 + l) * ys + q]);
  }
  __syncthreads();
  const int l = threadIdx.x / TPL;
  if (l >= nl) return;
  const int r = threadIdx.x - l * TPL;
  const int ti = (r / (M / TR)) * TR, tj = (r % (M / TR)) * TR;
  TAcc acc[TR][TR];
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < TR; ++j) acc[i][j] = A::mul(Xs[l][(ti + i) * M], Ys[l][tj + j]);
#pragma unroll 3
  for (int k = 1; k < M; ++k) {
    TAcc a[TR], bb[TR];
#pragma unroll
    for (int i = 0; i < TR; ++i) a[i] = Xs[l][(ti + i) * M + k];
#pragma unroll
    for (int j = 0; j < TR; ++j) bb[j] = Ys[l][k * M + tj + j];
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < TR; ++j) acc[i][j] = Mac<TIn, TAcc>::step(acc[i][j], a[i], bb[j]);
  }
  TAcc* o = out + (b0 + l) * (int64_t)M * M;
#pragma unroll
  for (int i = 0; i < TR; ++i)
#pragma unroll
    for (int j = 0; j < TR; ++j) o[(ti + i) * M + tj + j] = acc[i][j];
}

template <class TIn, class TAcc, int M, int TR>
cudaError_t run_smem(int64_t batch, const void* x, int64_t xs, const void* y, int64_t ys,
                     void* out, cudaStream_t st) {
  constexpr int LPB = 256 / ((M / TR) * (M / TR));
  const int64_t blocks = (batch + LPB - 1) / LPB;
  leaf_smem_kernel<TIn, TAcc, M, TR><<<(unsigned)blocks, 256, 0, st>>>(
      batch, (const TIn*)x, xs, (const TIn*)y, ys, (TAcc*)out);
  return cudaGetLastError();
}

// Long batches of small square leaves whose operand type equals the
// accumulation type (config 3's 27 x 27 binary64 leaves): one warp per leaf,
// TM x TN outputs per lane, leaves streamed through a CTA-wide ring of NSLOT
// bulk-copy slots (the TMA engine; each leaf's X and Y are copied as the
// 16-byte aligned spans enclosing them).  A producer lane fills the slots in
// order behind per-slot "empty" mbarriers; consumer warp w takes leaves
// w, w + NW, ... of the CTA's chunk behind the "full" mbarriers.  There is
// no CTA barrier in the steady state and no load instruction from global
// memory in the consumers.
//
// Why this shape: an 8-byte shared-memory load moves 256 bytes per warp, two
// cycles of the 128 B/clk crossbar, whatever the broadcast; with 3 x 3
// outputs per thread (6 loads per 9 multiply-adds) the crossbar was 93% busy
// with the FP64 pipe at 56% (9.5 TFLOP/s, round-1/2 kernel, three leaves per
// 243-thread CTA and a CTA barrier per group).  9 x 3 outputs need 12 loads
// per 27 multiply-adds; 27 of a warp's 32 lanes then hold one whole leaf, so
// a warp needs no partner and the ring replaces the barriers: 12.1 TFLOP/s
// = 66% of DMUL+DADD at 5.4 TB/s = 83% of HBM, which is this leaf's tighter
// roofline (2.25 flop per byte).  3 x 9 measured 10.1; k loops unrolled by 2
// and 6 instead of fully: 8.2 and 9.2; 8 to 16 consumer warps equal.
//
// Slot release: the consumers read the slot through the generic proxy and
// the refill writes it through the async proxy, so the arrive on "empty" is
// preceded by fence.proxy.async.  Without it the compiler placed the arrive
// right after the last LDS issue and the refill overtook loads still in
// flight: about one wrong output row per 10^5 leaves (found with the
// 3 x 9 variant, tools/experiments/leaf27_warp.cu).
template <class T, int M, int NSLOT>
struct LeafRing {
  static constexpr int E = M * M;
  static constexpr int SPAN = ((E * (int)sizeof(T) + 16) + 15) / 16 * 16;
  static constexpr size_t smem = (size_t)NSLOT * 2 * SPAN + 2 * NSLOT * sizeof(uint64_t);
};

template <class T, int M, int TM, int TN, int NW, int NSLOT>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    leaf_ring_kernel(int64_t batch, const T* __restrict__ x, int64_t xs, const T* __restrict__ y,
                     int64_t ys, T* __restrict__ out) {
  using S = LeafRing<T, M, NSLOT>;
  using A = Arith<T>;
  constexpr int E = S::E, SPAN = S::SPAN;
  constexpr int CJ = M / TN;  // lanes along N; a lane's columns are jt + CJ * j
  constexpr int TPL = (M / TM) * CJ;
  static_assert(M % TM == 0 && M % TN == 0 && TPL <= 32, "one warp per leaf");
  static_assert(M % 2 == 1, "the k loop below is written for odd M");
  extern __shared__ __align__(128) unsigned char ring_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(ring_smem + (size_t)NSLOT * 2 * SPAN);
  uint64_t* empty = full + NSLOT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init_fence();
  }
  __syncthreads();
  // this CTA's leaves: one contiguous chunk
  const int64_t per = (batch + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per;
  const int64_t hi = lo + per < batch ? lo + per : batch;
  const int n = hi > lo ? (int)(hi - lo) : 0;
  if (warp == NW) {  // producer
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        const int s = i % NSLOT, round = i / NSLOT;
        if (round > 0) mbar_wait_parked(&empty[s], (unsigned)((round - 1) & 1), 2000);
        const T* gx = x + (lo + i) * xs;
        const T* gy = y + (lo + i) * ys;
        const unsigned bx = span_bytes(gx, E * sizeof(T)), by = span_bytes(gy, E * sizeof(T));
        mbar_expect_tx(&full[s], bx + by);
        unsigned char* slot = ring_smem + (size_t)s * 2 * SPAN;
        bulk_g2s(slot, span_start(gx), bx, &full[s]);
        bulk_g2s(slot + SPAN, span_start(gy), by, &full[s]);
      }
    }
    return;
  }
  const int r = lane < TPL ? lane : 0;  // spare lanes shadow lane 0 and do not store
  const int it = r / CJ, jt = r % CJ;
  for (int i = warp; i < n; i += NW) {
    const int s = i % NSLOT;
    mbar_wait_parked(&full[s], (unsigned)((i / NSLOT) & 1), 1000);
    const T* gx = x + (lo + i) * xs;
    const T* gy = y + (lo + i) * ys;
    unsigned char* slot = ring_smem + (size_t)s * 2 * SPAN;
    const T* Xr = reinterpret_cast<const T*>(slot + (reinterpret_cast<uintptr_t>(gx) & 15)) + TM * it * M;
    const T* Yc = reinterpret_cast<const T*>(slot + SPAN + (reinterpret_cast<uintptr_t>(gy) & 15)) + jt;
    // operands of step k + 1 load while step k multiplies (two register
    // sets, k fully unrolled); every output keeps its sequential k chain
    T acc[TM][TN], a[2][TM], b[2][TN];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int ii = 0; ii < TM; ++ii) a[h][ii] = Xr[ii * M + h];
#pragma unroll
      for (int j = 0; j < TN; ++j) b[h][j] = Yc[h * M + CJ * j];
    }
#pragma unroll
    for (int ii = 0; ii < TM; ++ii)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[ii][j] = A::mul(a[0][ii], b[0][j]);
#pragma unroll
    for (int k = 1; k < M; ++k) {
      const int c = k & 1, nx = c ^ 1;
      if (k + 1 < M) {
#pragma unroll
        for (int ii = 0; ii < TM; ++ii) a[nx][ii] = Xr[ii * M + k + 1];
#pragma unroll
        for (int j = 0; j < TN; ++j) b[nx][j] = Yc[(k + 1) * M + CJ * j];
      }
#pragma unroll
      for (int ii = 0; ii < TM; ++ii)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[ii][j] = A::add(acc[ii][j], A::mul(a[c][ii], b[c][j]));
    }
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (lane < TPL) {
      T* o = out + (lo + i) * (int64_t)E + TM * it * M + jt;
#pragma unroll
      for (int ii = 0; ii < TM; ++ii)
#pragma unroll
        for (int j = 0; j < TN; ++j) o[ii * M + CJ * j] = acc[ii][j];
    }
  }
}

template <class T, int M, int TM, int TN>
cudaError_t run_leaf_ring(int64_t batch, const void* x, int64_t xs, const void* y, int64_t ys,
                          void* out, cudaStream_t st) {
  constexpr int NW = 12, NSLOT = 16;
  using S = LeafRing<T, M, NSLOT>;
  auto kern = leaf_ring_kernel<T, M, TM, TN, NW, NSLOT>;
  static const cudaError_t attr =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::smem);
  if (attr != cudaSuccess) return attr;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t blocks = std::min<int64_t>((batch + NW - 1) / NW, sms);
  kern<<<(unsigned)blocks, (NW + 1) * 32, S::smem, st>>>(batch, (const T*)x, xs, (const T*)y, ys,
                                                          (T*)out);
  return cudaGetLastError();
}

// Square small leaves with a shared-memory kernel instantiation; returns
// cudaErrorNotSupported when none applies.
template <class TIn, class TAcc>
cudaError_t small_square(int64_t batch, int64_t M, const void* x, int64_t xs, const void* y,
                         int64_t ys, void* out, cudaStream_t st) {
  if constexpr (std::is_same<TIn, TAcc>::value && sizeof(TIn) >= 4) {
    // one warp per leaf, 9 x 3 outputs per lane (leaf_ring_kernel above)
    if (M == 27 && batch >= 2048 && tile_override() == 0)
      return run_leaf_ring<TIn, 27, 9, 3>(batch, x, xs, y, ys, out, st);
  }
  switch (M) {
    case 27: return run_smem<TIn, TAcc, 27, 3>(batch, x, xs, y, ys, out, st);
    case 24: return run_smem<TIn, TAcc, 24, 3>(batch, x, xs, y, ys, out, st);
    case 18: return run_smem<TIn, TAcc, 18, 3>(batch, x, xs, y, ys, out, st);
    case 16: return run_smem<TIn, TAcc, 16, 2>(batch, x, xs, y, ys, out, st);
    case 12: return run_smem<TIn, TAcc, 12, 2>(batch, x, xs, y, ys, out, st);
    case 10: return run_smem<TIn, TAcc, 10, 2>(batch, x, xs, y, ys, out, st);
    case 9: return run_smem<TIn, TAcc, 9, 3>(batch, x, xs, y, ys, out, st);
    case 8: return run_smem<TIn, TAcc, 8, 2>(batch, x, xs, y, ys, out, st);
  }
  return cudaErrorNotSupported;
}

// binary16 leaves: the same tiling with half2 SIMD along N.  Each HMUL2 /
// HADD2 lane rounds exactly like the scalar __hmul_rn / __hadd_rn, so every
// output keeps its own sequential k chain (two adjacent outputs per op).
template <int BM, int BN, int BK, int TM, int TN>
__global__ void __launch_bounds__((BM / TM) * (BN / TN))
    leaf_tiled_h2_kernel(int M, int K, int N, const __half* __restrict__ x, int64_t xs,
                         const __half* __restrict__ y, int64_t ys, __half* __restrict__ out,
                         int tiles_n) {
  constexpr int DY = BM / TM;
  constexpr int DX = BN / TN;
  constexpr int NT = DY * DX;
  constexpr int A_PER = BM * BK / NT;
  constexpr int B_PER = BK * BN / NT;
  constexpr int TN2 = TN / 2;
  static_assert(TN % 2 == 0 && BM * BK % NT == 0 && BK * BN % NT == 0, "tile/threads");
  __shared__ __align__(16) __half As[2][BK][BM];
  __shared__ __align__(16) __half Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid % DX;
  const int ty = tid / DX;
  const int64_t b = blockIdx.y + (int64_t)blockIdx.z * 65535;
  const int tm = blockIdx.x / tiles_n;
  const int tn = blockIdx.x - tm * tiles_n;
  const int m0 = tm * BM, n0 = tn * BN;
  const __half* xb = x + b * xs;
  const __half* yb = y + b * ys;
  const __half zero = __float2half(0.f);
  __half ra[A_PER], rb[B_PER];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int q = 0; q < A_PER; ++q) {
      const int e = tid + q * NT;
      const int mm = e / BK, kk = e % BK;
      const int gm = m0 + mm, gk = k0 + kk;
      ra[q] = (gm < M && gk < K) ? xb[(int64_t)gm * K + gk] : zero;
    }
#pragma unroll
    for (int q = 0; q < B_PER; ++q) {
      const int e = tid + q * NT;
      const int kk = e / BN, nn = e % BN;
      const int gk = k0 + kk, gn = n0 + nn;
      rb[q] = (gk < K && gn < N) ? yb[(int64_t)gk * N + gn] : zero;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int q = 0; q < A_PER; ++q) {
      const int e = tid + q * NT;
      As[buf][e % BK][e / BK] = ra[q];
    }
#pragma unroll
    for (int q = 0; q < B_PER; ++q) {
      const int e = tid + q * NT;
      Bs[buf][e / BN][e % BN] = rb[q];
    }
  };
  // thread owns rows ty*TM .. +TM and column pairs tx*TN .. +TN
  __half2 acc[TM][TN2];
  const int ktiles = (K + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  // fragments are read with one vector LDS each (TM and TN contiguous halves)
  auto kstep = [&](int buf, int kk, bool first) {
    const Pack<__half, TM> pa = pload<__half, TM>(&As[buf][kk][ty * TM]);
    const Pack<__half, TN> pb = pload<__half, TN>(&Bs[buf][kk][tx * TN]);
    const __half2* b2 = reinterpret_cast<const __half2*>(pb.v);
    __half2 a2[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) a2[i] = __half2half2(pa.v[i]);
    if (first) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN2; ++j) acc[i][j] = __hmul2_rn(a2[i], b2[j]);
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN2; ++j) acc[i][j] = __hadd2_rn(acc[i][j], __hmul2_rn(a2[i], b2[j]));
    }
  };
  for (int kt = 0; kt < ktiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ktiles) load_tile((kt + 1) * BK);
    if ((kt + 1) * BK <= K) {
      if (kt == 0) {
        kstep(buf, 0, true);
#pragma unroll
        for (int kk = 1; kk < BK; ++kk) kstep(buf, kk, false);
      } else {
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) kstep(buf, kk, false);
      }
    } else {
      const int kmax = K - kt * BK;
      for (int kk = 0; kk < kmax; ++kk) kstep(buf, kk, kt == 0 && kk == 0);
    }
    if (kt + 1 < ktiles) {
      store_tile(buf ^ 1);
      __syncthreads();
    }
  }
  __half* ob = out + b * (int64_t)M * N;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN2; ++j) {
      const int gn = n0 + tx * TN + 2 * j;
      __half* o = &ob[(int64_t)gm * N + gn];
      // one 4-byte store where the pair is aligned (odd N puts every other
      // row, and odd M * N every other leaf, on a 2-byte boundary)
      if (gn + 1 < N && (reinterpret_cast<uintptr_t>(o) & 3) == 0) {
        *reinterpret_cast<__half2*>(o) = acc[i][j];
      } else {
        if (gn < N) o[0] = __low2half(acc[i][j]);
        if (gn + 1 < N) o[1] = __high2half(acc[i][j]);
      }
    }
  }
}

// binary16 leaves, issue-bound variant: exact-order HMUL2/HADD2 run at one
// instruction per clock per SM sub-partition, so every non-FP instruction in
// the k loop costs throughput.  A is stored in shared memory transposed and
// pre-broadcast as (a, a) half2 pairs, so the row fragment is two 16-byte
// loads with no per-k shuffles; each thread owns TM rows x TN columns
// (TN/2 half2 accumulators per row) for 2*TM*TN/2 FP instructions per four
// fragment loads.  Operand tiles move as 16-byte vectors (K, N multiples of
// 8), double-buffered through registers.  Same per-element chains as
// leaf_tiled_h2_kernel: k ascending, first product initialises.
template <int BM, int BN, int BK, int TM, int TN, int MINB>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
    leaf_h2dup_kernel(int M, int K, int N, const __half* __restrict__ x, int64_t xs,
                      const __half* __restrict__ y, int64_t ys, __half* __restrict__ out,
                      int tiles_n) {
  constexpr int DY = BM / TM, DX = BN / TN;
  constexpr int NT = DY * DX;
  constexpr int TN2 = TN / 2;
  constexpr int AV = BM * BK / 8 / NT;  // 16-byte A vectors per thread per tile
  constexpr int BV = BK * BN / 8 / NT;
  static_assert(AV >= 1 && BV >= 1 && BM * BK % (8 * NT) == 0 && BK * BN % (8 * NT) == 0, "tiles");
  static_assert(TM % 4 == 0 && TN2 % 4 == 0, "16-byte fragments");
  constexpr int APAD = 4;  // half2 pad per k row (bank spread of the transposed stores)
  __shared__ __align__(16) __half2 As[2][BK][BM + APAD];
  __shared__ __align__(16) __half Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid % DX, ty = tid / DX;
  const int64_t b = blockIdx.y + (int64_t)blockIdx.z * 65535;
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x - tm * tiles_n;
  const int m0 = tm * BM, n0 = tn * BN;
  const __half* xb = x + b * xs;
  const __half* yb = y + b * ys;
  uint4 ra[AV], rb[BV];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int q = 0; q < AV; ++q) {
      const int v = tid + q * NT;
      const int mm = v / (BK / 8), kk = (v % (BK / 8)) * 8;
      const int gm = m0 + mm, gk = k0 + kk;
      ra[q] = (gm < M && gk < K) ? *reinterpret_cast<const uint4*>(xb + (int64_t)gm * K + gk)
                                 : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < BV; ++q) {
      const int v = tid + q * NT;
      const int kk = v / (BN / 8), nn = (v % (BN / 8)) * 8;
      const int gk = k0 + kk, gn = n0 + nn;
      rb[q] = (gk < K && gn < N) ? *reinterpret_cast<const uint4*>(yb + (int64_t)gk * N + gn)
                                 : make_uint4(0, 0, 0, 0);
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int q = 0; q < AV; ++q) {
      const int v = tid + q * NT;
      const int mm = v / (BK / 8), kk = (v % (BK / 8)) * 8;
      const __half* h = reinterpret_cast<const __half*>(&ra[q]);
#pragma unroll
      for (int e = 0; e < 8; ++e) As[buf][kk + e][mm] = __half2half2(h[e]);
    }
#pragma unroll
    for (int q = 0; q < BV; ++q) {
      const int v = tid + q * NT;
      const int kk = v / (BN / 8), nn = (v % (BN / 8)) * 8;
      *reinterpret_cast<uint4*>(&Bs[buf][kk][nn]) = rb[q];
    }
  };
  __half2 acc[TM][TN2];
  auto kstep = [&](int buf, int kk, bool first) {
    __half2 a2[TM], b2[TN2];
#pragma unroll
    for (int g = 0; g < TM / 4; ++g) {
      const uint4 v = *reinterpret_cast<const uint4*>(&As[buf][kk][ty * TM + 4 * g]);
      const __half2* p = reinterpret_cast<const __half2*>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) a2[4 * g + e] = p[e];
    }
#pragma unroll
    for (int g = 0; g < TN2 / 4; ++g) {
      const uint4 v = *reinterpret_cast<const uint4*>(&Bs[buf][kk][tx * TN + 8 * g]);
      const __half2* p = reinterpret_cast<const __half2*>(&v);
#pragma unroll
      for (int e = 0; e < 4; ++e) b2[4 * g + e] = p[e];
    }
    if (first) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN2; ++j) acc[i][j] = __hmul2_rn(a2[i], b2[j]);
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN2; ++j) acc[i][j] = __hadd2_rn(acc[i][j], __hmul2_rn(a2[i], b2[j]));
    }
  };
  const int ktiles = (K + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  for (int kt = 0; kt < ktiles; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < ktiles) load_tile((kt + 1) * BK);
    if ((kt + 1) * BK <= K) {
      if (kt == 0) {
        kstep(buf, 0, true);
#pragma unroll
        for (int kk = 1; kk < BK; ++kk) kstep(buf, kk, false);
      } else {
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) kstep(buf, kk, false);
      }
    } else {
      const int kmax = K - kt * BK;
      for (int kk = 0; kk < kmax; ++kk) kstep(buf, kk, kt == 0 && kk == 0);
    }
    if (kt + 1 < ktiles) {
      store_tile(buf ^ 1);
      __syncthreads();
    }
  }
  __half* ob = out + b * (int64_t)M * N;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty * TM + i;
    if (gm >= M) continue;
#pragma unroll
    for (int g = 0; g < TN2 / 4; ++g) {
      const int gn = n0 + tx * TN + 8 * g;
      if (gn + 8 <= N) {
        *reinterpret_cast<uint4*>(&ob[(int64_t)gm * N + gn]) = *reinterpret_cast<const uint4*>(&acc[i][4 * g]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (gn + 2 * e < N) ob[(int64_t)gm * N + gn + 2 * e] = __low2half(acc[i][4 * g + e]);
          if (gn + 2 * e + 1 < N) ob[(int64_t)gm * N + gn + 2 * e + 1] = __high2half(acc[i][4 * g + e]);
        }
      }
    }
  }
}

// binary32 leaves, issue-bound (the exact-order chain needs a separately
// rounded multiply and add per step): 16-byte operand vectors (K, N
// multiples of 4), transposed A tile, float4 fragments, a k loop with no
// per-step guards -- the K tail of the last tile runs a separate loop -- and
// packed accumulators: each FFMA2 (rounded multiply, common.cuh) and FADD2
// covers two outputs of a row, the A element broadcast, so a k step of an
// 8 x 8 fragment issues 64 FP instructions instead of 128.  Same chains as
// leaf_tiled_kernel.
template <int BM, int BN, int BK, int TM, int TN, int MINB, bool PEEL>
__global__ void __launch_bounds__((BM / TM) * (BN / TN), MINB)
    leaf_f32v_kernel(int M, int K, int N, const float* __restrict__ x, int64_t xs,
                     const float* __restrict__ y, int64_t ys, float* __restrict__ out,
                     int tiles_n, uint64_t negz) {
  constexpr int DY = BM / TM, DX = BN / TN;
  constexpr int NT = DY * DX;
  constexpr int AV = BM * BK / 4 / NT;  // float4 vectors per thread per tile
  constexpr int BV = BK * BN / 4 / NT;
  static_assert(AV >= 1 && BV >= 1 && BM * BK % (4 * NT) == 0 && BK * BN % (4 * NT) == 0, "tiles");
  static_assert(TM % 4 == 0 && TN % 4 == 0, "float4 fragments");
  constexpr int APAD = 4;
  __shared__ __align__(16) float As[2][BK][BM + APAD];
  __shared__ __align__(16) float Bs[2][BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid % DX, ty = tid / DX;
  const int64_t b = blockIdx.y + (int64_t)blockIdx.z * 65535;
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x - tm * tiles_n;
  const int m0 = tm * BM, n0 = tn * BN;
  const float* xb = x + b * xs;
  const float* yb = y + b * ys;
  float4 ra[AV], rb[BV];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int q = 0; q < AV; ++q) {
      const int v = tid + q * NT;
      const int mm = v / (BK / 4), kk = (v % (BK / 4)) * 4;
      const int gm = m0 + mm, gk = k0 + kk;
      ra[q] = (gm < M && gk < K) ? *reinterpret_cast<const float4*>(xb + (int64_t)gm * K + gk)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < BV; ++q) {
      const int v = tid + q * NT;
      const int kk = v / (BN / 4), nn = (v % (BN / 4)) * 4;
      const int gk = k0 + kk, gn = n0 + nn;
      rb[q] = (gk < K && gn < N) ? *reinterpret_cast<const float4*>(yb + (int64_t)gk * N + gn)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int q = 0; q < AV; ++q) {
      const int v = tid + q * NT;
      const int mm = v / (BK / 4), kk = (v % (BK / 4)) * 4;
      As[buf][kk][mm] = ra[q].x;
      As[buf][kk + 1][mm] = ra[q].y;
      As[buf][kk + 2][mm] = ra[q].z;
      As[buf][kk + 3][mm] = ra[q].w;
    }
#pragma unroll
    for (int q = 0; q < BV; ++q) {
      const int v = tid + q * NT;
      const int kk = v / (BN / 4), nn = (v % (BN / 4)) * 4;
      *reinterpret_cast<float4*>(&Bs[buf][kk][nn]) = rb[q];
    }
  };
  uint64_t acc[TM][TN / 2];  // (acc[i][2j], acc[i][2j+1]) packed
  auto kstep = [&](const float* arow, const float* brow, bool first) {
    float a[TM];
    uint64_t bb[TN / 2];
#pragma unroll
    for (int g = 0; g < TM / 4; ++g) {
      const float4 v = *reinterpret_cast<const float4*>(arow + g * DY * 4);
      a[4 * g] = v.x; a[4 * g + 1] = v.y; a[4 * g + 2] = v.z; a[4 * g + 3] = v.w;
    }
#pragma unroll
    for (int g = 0; g < TN / 4; ++g) {
      const float4 v = *reinterpret_cast<const float4*>(brow + g * DX * 4);
      bb[2 * g] = f2_pack(v.x, v.y);
      bb[2 * g + 1] = f2_pack(v.z, v.w);
    }
    if (first) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN / 2; ++j) acc[i][j] = f2_mul_bcast(a[i], bb[j], negz);
    } else {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN / 2; ++j)
          acc[i][j] = f2_add(acc[i][j], f2_mul_bcast(a[i], bb[j], negz));
    }
  };
  const int ktiles = (K + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();
  // One k tile.  ptxas leaves a tile's loop-carried accumulators in other
  // registers than it found them and restores them with about 44 MOVs at the
  // end of the tile body (7.5% of all instructions with tiles of 8 steps),
  // and a non-FP instruction costs the FMA pipe a dispatch cycle.  Tiles of
  // 16 steps halve that share; PEEL takes the first tile (whose first step
  // initialises the chains) out of the loop.  Config 5 leaves (128 x 128):
  // 8 steps 31.9 TFLOP/s, peeled 32.6, 16 steps 33.6, 16 steps peeled 32.8
  // (spills at the 128-register bound); 32 steps (dynamic shared memory) 32.9
  // fetched at once and 31.8 fetched in two slices, both spilling.  Config 1
  // leaves (64 x 64): 28.4, 29.0, 29.8, 30.0.  Neither compiling the
  // partial-tile path out nor two tiles per loop trip changes the MOV count
  // per tile.
  auto ktile = [&](int kt, auto first_tag) {
    constexpr bool kFirst = decltype(first_tag)::value;
    const int buf = kt & 1;
    if (kt + 1 < ktiles) load_tile((kt + 1) * BK);
    const float* a0 = &As[buf][0][ty * 4];
    const float* b0 = &Bs[buf][0][tx * 4];
    if ((kt + 1) * BK <= K) {
      if (kFirst) kstep(a0, b0, true);
#pragma unroll
      for (int kk = kFirst ? 1 : 0; kk < BK; ++kk)
        kstep(a0 + kk * (BM + APAD), b0 + kk * BN, false);
    } else {
      const int kmax = K - kt * BK;
#pragma unroll 1
      for (int kk = 0; kk < kmax; ++kk)
        kstep(a0 + kk * (BM + APAD), b0 + kk * BN, kFirst && kk == 0);
    }
    if (kt + 1 < ktiles) {
      store_tile(buf ^ 1);
      __syncthreads();
    }
  };
  if constexpr (PEEL) {
    ktile(0, std::true_type{});
    for (int kt = 1; kt < ktiles; ++kt) ktile(kt, std::false_type{});
  } else {
    for (int kt = 0; kt < ktiles; ++kt) {
      if (kt == 0) ktile(kt, std::true_type{});
      else ktile(kt, std::false_type{});
    }
  }
  float* ob = out + b * (int64_t)M * N;
#pragma unroll
  for (int gi = 0; gi < TM / 4; ++gi)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int gm = m0 + gi * DY * 4 + ty * 4 + v;
      if (gm >= M) continue;
#pragma unroll
      for (int gj = 0; gj < TN / 4; ++gj) {
        const int gn = n0 + gj * DX * 4 + tx * 4;
        const int i = gi * 4 + v, j = gj * 2;
        const float o4[4] = {f2_lo(acc[i][j]), f2_hi(acc[i][j]), f2_lo(acc[i][j + 1]),
                             f2_hi(acc[i][j + 1])};
        if (gn + 4 <= N) {
          *reinterpret_cast<float4*>(&ob[(int64_t)gm * N + gn]) =
              make_float4(o4[0], o4[1], o4[2], o4[3]);
        } else {
#pragma unroll
          for (int w = 0; w < 4; ++w)
            if (gn + w < N) ob[(int64_t)gm * N + gn + w] = o4[w];
        }
      }
    }
}

template <int BM, int BN, int BK, int TM, int TN, int MINB, bool PEEL>
cudaError_t run_f32v(int64_t batch, int64_t M, int64_t K, int64_t N, const void* x, int64_t xs,
                     const void* y, int64_t ys, void* out, cudaStream_t st) {
  const int tiles_m = (int)((M + BM - 1) / BM);
  const int tiles_n = (int)((N + BN - 1) / BN);
  constexpr int NT = (BM / TM) * (BN / TN);
  for (int64_t b0 = 0; b0 < batch;) {
    const int64_t nb = std::min<int64_t>(batch - b0, (int64_t)65535 * 65535);
    const int64_t full = (nb / 65535) * 65535;
    if (full > 0) {
      dim3 grid(tiles_m * tiles_n, 65535, (unsigned)(full / 65535));
      leaf_f32v_kernel<BM, BN, BK, TM, TN, MINB, PEEL><<<grid, NT, 0, st>>>(
          (int)M, (int)K, (int)N, (const float*)x + b0 * xs, xs, (const float*)y + b0 * ys, ys,
          (float*)out + b0 * M * N, tiles_n, kF2NegZero);
    }
    if (nb > full) {
      dim3 grid(tiles_m * tiles_n, (unsigned)(nb - full), 1);
      const int64_t bb = b0 + full;
      leaf_f32v_kernel<BM, BN, BK, TM, TN, MINB, PEEL><<<grid, NT, 0, st>>>(
          (int)M, (int)K, (int)N, (const float*)x + bb * xs, xs, (const float*)y + bb * ys, ys,
          (float*)out + bb * M * N, tiles_n, kF2NegZero);
    }
    b0 += nb;
  }
  return cudaGetLastError();
}

template <int BM, int BN, int BK, int TM, int TN, int MINB>
cudaError_t run_h2dup(int64_t batch, int64_t M, int64_t K, int64_t N, const void* x, int64_t xs,
                      const void* y, int64_t ys, void* out, cudaStream_t st) {
  const int tiles_m = (int)((M + BM - 1) / BM);
  const int tiles_n = (int)((N + BN - 1) / BN);
  constexpr int NT = (BM / TM) * (BN / TN);
  for (int64_t b0 = 0; b0 < batch;) {
    const int64_t nb = std::min<int64_t>(batch - b0, (int64_t)65535 * 65535);
    const int64_t full = (nb / 65535) * 65535;
    if (full > 0) {
      dim3 grid(tiles_m * tiles_n, 65535, (unsigned)(full / 65535));
      leaf_h2dup_kernel<BM, BN, BK, TM, TN, MINB><<<grid, NT, 0, st>>>(
          (int)M, (int)K, (int)N, (const __half*)x + b0 * xs, xs, (const __half*)y + b0 * ys, ys,
          (__half*)out + b0 * M * N, tiles_n);
    }
    if (nb > full) {
      dim3 grid(tiles_m * tiles_n, (unsigned)(nb - full), 1);
      const int64_t bb = b0 + full;
      leaf_h2dup_kernel<BM, BN, BK, TM, TN, MINB><<<grid, NT, 0, st>>>(
          (int)M, (int)K, (int)N, (const __half*)x + bb * xs, xs, (const __half*)y + bb * ys, ys,
          (__half*)out + bb * M * N, tiles_n);
    }
    b0 += nb;
  }
  return cudaGetLastError();
}

template <int BM, int BN, int BK, int TM, int TN>
cudaError_t run_tiled_h2(int64_t batch, int64_t M, int64_t K, int64_t N, const void* x, int64_t xs,
                         const void* y, int64_t ys, void* out, cudaStream_t st) {
  const int tiles_m = (int)((M + BM - 1) / BM);
  const int tiles_n = (int)((N + BN - 1) / BN);
  constexpr int NT = (BM / TM) * (BN / TN);
  for (int64_t b0 = 0; b0 < batch;) {
    const int64_t nb = std::min<int64_t>(batch - b0, (int64_t)65535 * 65535);
    const int64_t full = (nb / 65535) * 65535;
    if (full > 0) {
      dim3 grid(tiles_m * tiles_n, 65535, (unsigned)(full / 65535));
      leaf_tiled_h2_kernel<BM, BN, BK, TM, TN><<<grid, NT, 0, st>>>(
          (int)M, (int)K, (int)N, (const __half*)x + b0 * xs, xs, (const __half*)y + b0 * ys, ys,
          (__half*)out + b0 * M * N, tiles_n);
    }
    if (nb > full) {
      dim3 grid(tiles_m * tiles_n, (unsigned)(nb - full), 1);
      const int64_t bb = b0 + full;
      leaf_tiled_h2_kernel<BM, BN, BK, TM, TN><<<grid, NT, 0, st>>>(
          (int)M, (int)K, (int)N, (const __half*)x + bb * xs, xs, (const __half*)y + bb * ys, ys,
          (__half*)out + bb * M * N, tiles_n);
    }
    b0 += nb;
  }
  return cudaGetLastError();
}

template <class TIn, class TAcc, int BM, int BN, int BK, int TM, int TN>
cudaError_t run_tiled(int64_t batch, int64_t M, int64_t K, int64_t N, const void* x, int64_t xs,
                      const void* y, int64_t ys, void* out, cudaStream_t st) {
  const int tiles_m = (int)((M + BM - 1) / BM);
  const int tiles_n = (int)((N + BN - 1) / BN);
  constexpr int NT = (BM / TM) * (BN / TN);
  constexpr size_t smem = sizeof(TAcc) * 2 * BK * ((BM + 16 / sizeof(TAcc)) + BN);
  if (smem > 48 * 1024) {
    static const cudaError_t attr = cudaFuncSetAttribute(
        leaf_tiled_kernel<TIn, TAcc, BM, BN, BK, TM, TN>,
        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (attr != cudaSuccess) return attr;
  }
  for (int64_t b0 = 0; b0 < batch; b0 += (int64_t)65535 * 65535) {
    const int64_t nb = batch - b0 < (int64_t)65535 * 65535 ? batch - b0 : (int64_t)65535 * 65535;
    const unsigned gy = (unsigned)(nb < 65535 ? nb : 65535);
    const unsigned gz = (unsigned)((nb + 65534) / 65535);
    // blocks with b >= nb in the last z slice are harmless only if we guard;
    // split instead into a full-z part and a remainder part.
    const int64_t full = (nb / 65535) * 65535;
    if (full > 0) {
      dim3 grid(tiles_m * tiles_n, 65535, (unsigned)(full / 65535));
      leaf_tiled_kernel<TIn, TAcc, BM, BN, BK, TM, TN><<<grid, NT, smem, st>>>(
          (int)M, (int)K, (int)N, (const TIn*)x + b0 * xs, xs, (const TIn*)y + b0 * ys, ys,
          (TAcc*)out + b0 * M * N, tiles_n);
    }
    if (nb > full) {
      dim3 grid(tiles_m * tiles_n, (unsigned)(nb - full), 1);
      const int64_t bb = b0 + full;
      leaf_tiled_kernel<TIn, TAcc, BM, BN, BK, TM, TN><<<grid, NT, smem, st>>>(
          (int)M, (int)K, (int)N, (const TIn*)x + bb * xs, xs, (const TIn*)y + bb * ys, ys,
          (TAcc*)out + bb * M * N, tiles_n);
    }
    (void)gy;
    (void)gz;
  }
  return cudaGetLastError();
}

template <class TIn, class TAcc>
cudaError_t run_small(int64_t batch, int64_t M, int64_t K, int64_t N, const void* x, int64_t xs,
                      const void* y, int64_t ys, void* out, cudaStream_t st) {
  const int64_t total = batch * M * N;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  leaf_small_kernel<TIn, TAcc><<<(unsigned)blocks, 256, 0, st>>>(
      batch, (int)M, (int)K, (int)N, (const TIn*)x, xs, (const TIn*)y, ys, (TAcc*)out);
  return cudaGetLastError();
}


template <class TIn, class TAcc>
cudaError_t leaf_dispatch(int64_t batch, int64_t M, int64_t K, int64_t N, const void* x,
                          int64_t xs, const void* y, int64_t ys, void* out, cudaStream_t st) {
  const int forced = tile_override();
  if constexpr (sizeof(TAcc) == 8) {
    // binary64 accumulation: from 512 up the widen pass + bulk-copy pipeline
    // (truth.cu; 8192: 28.8 vs 24.9 TFLOP/s); below it the widen pass costs
    // more than it saves (243 x 200: 15.8 vs 17.6) and the register-staged
    // tile runs (tools/leaf_bench.py)
    // binary64 operands of ragged sizes below 1024 (config 3: 729) skip the
    // panel pass too: 128 x 64 register-staged tiles, 0.194 vs 0.233 ms per
    // launch (config 4's 2048 binary16 truth stays on the bulk pipeline:
    // 10.2 vs 11.8 ms)
    if (forced == 0 && std::is_same<TIn, double>::value && M >= 512 && N >= 512 && K >= 1 &&
        M < 1024 && N < 1024 && (M % 128 || N % 128))
      return run_truth<TIn, 128, 64, 16, 8, 8, false>(batch, M, K, N, x, xs, y, ys, out, st);
    if (forced == 0 && M >= 512 && N >= 512 && K >= 1) {
      const cudaError_t e = launch_truth(std::is_same<TIn, double>::value ? kF64
                                         : std::is_same<TIn, float>::value ? kF32 : kF16,
                                         batch, M, K, N, x, xs, y, ys, out, st);
      if (e != cudaErrorNotSupported) return e;
      return run_truth<TIn, 128, 128, 16, 8, 8, false>(batch, M, K, N, x, xs, y, ys, out, st);
    }
    // ragged sizes (config 2: 243) do better with 128 x 64 tiles and 128-thread
    // CTAs (19.5 vs 18.0 TFLOP/s); whole 128-multiples with 128 x 128
    if (forced == 0 && M >= 128 && N >= 128 && K >= 1 && (M % 128 || N % 128))
      return run_truth<TIn, 128, 64, 16, 8, 8, false>(batch, M, K, N, x, xs, y, ys, out, st);
    if (forced == 0 && M >= 128 && N >= 128 && K >= 1)
      return run_truth<TIn, 128, 128, 16, 8, 8, false>(batch, M, K, N, x, xs, y, ys, out, st);
    if (forced == 303 && M >= 128 && N >= 128 && K >= 1)  // bulk kernel at any size
      return launch_truth(std::is_same<TIn, double>::value ? kF64
                          : std::is_same<TIn, float>::value ? kF32 : kF16,
                          batch, M, K, N, x, xs, y, ys, out, st);
  }
  // binary64: 128x64 tiles of 8x4 outputs per thread (truth 243: 15.3 vs
  // 14.5 TFLOP/s for 64x128, 13.9 for 64x64; tools/leaf_bench.py)
  if (sizeof(TAcc) == 8 && M >= 128 && N >= 64)
    return run_tiled<TIn, TAcc, 128, 64, 8, 8, 4>(batch, M, K, N, x, xs, y, ys, out, st);
  if (sizeof(TAcc) == 8 && M >= 64 && N >= 128)
    return run_tiled<TIn, TAcc, 64, 128, 8, 4, 8>(batch, M, K, N, x, xs, y, ys, out, st);
  if (M >= 128 && N >= 128 && sizeof(TAcc) <= 4)
    return run_tiled<TIn, TAcc, 128, 128, 8, 8, 8>(batch, M, K, N, x, xs, y, ys, out, st);
  if (M >= 64 && N >= 64)
    return run_tiled<TIn, TAcc, 64, 64, 8, 4, 4>(batch, M, K, N, x, xs, y, ys, out, st);
  if (M >= 32 && N >= 32)
    return run_tiled<TIn, TAcc, 32, 32, 8, 2, 2>(batch, M, K, N, x, xs, y, ys, out, st);
  if (M == N && M == K) {
    cudaError_t e = small_square<TIn, TAcc>(batch, M, x, xs, y, ys, out, st);
    if (e != cudaErrorNotSupported) return e;
  }
  return run_small<TIn, TAcc>(batch, M, K, N, x, xs, y, ys, out, st);
}

}  // namespace

cudaError_t launch_leaf(int dtype_in, int dtype_out, int64_t batch, int64_t M, int64_t K,
                        int64_t N, const void* x, int64_t xs, const void* y, int64_t ys, void* out,
                        cudaStream_t st) {
  if (batch == 0 || M == 0 || N == 0) return cudaSuccess;
  if (dtype_out == kF64) {
    if (dtype_in == kF64) return leaf_dispatch<double, double>(batch, M, K, N, x, xs, y, ys, out, st);
    if (dtype_in == kF32) return leaf_dispatch<float, double>(batch, M, K, N, x, xs, y, ys, out, st);
    if (dtype_in == kF16) return leaf_dispatch<__half, double>(batch, M, K, N, x, xs, y, ys, out, st);
  }
  if (dtype_out == kF32 && dtype_in == kF32) {
    const bool vec = K % 4 == 0 && N % 4 == 0 && (xs % 4 == 0 || batch == 1) &&
                     (ys % 4 == 0 || batch == 1) && ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) &&
                     ((uintptr_t)out % 16 == 0);
    const int forced = tile_override();
    // 128 x 128 x 16 tiles, 8 x 8 per thread
    if (vec && M >= 128 && N >= 128 && forced == 0)
      return run_f32v<128, 128, 16, 8, 8, 2, false>(batch, M, K, N, x, xs, y, ys, out, st);
    // 64-wide leaves (config 1): 4 x 8 per thread, 128 threads (26.2 vs
    // 20.5 TFLOP/s for 8 x 8 per thread)
    if (vec && M >= 64 && N >= 64 && forced == 0)
      return run_f32v<64, 64, 16, 4, 8, 4, true>(batch, M, K, N, x, xs, y, ys, out, st);
    return leaf_dispatch<float, float>(batch, M, K, N, x, xs, y, ys, out, st);
  }
  if (dtype_out == kF16 && dtype_in == kF16) {
    // 16-byte operand vectors need K, N multiples of 8 and aligned strides
    const bool vec = K % 8 == 0 && N % 8 == 0 && (xs % 8 == 0 || batch == 1) &&
                     (ys % 8 == 0 || batch == 1) && ((uintptr_t)x % 16 == 0) && ((uintptr_t)y % 16 == 0) &&
                     ((uintptr_t)out % 16 == 0);
    const int forced = tile_override();
    if (vec && M >= 128 && N >= 128 && forced == 0)
      return run_h2dup<128, 128, 16, 8, 16, 3>(batch, M, K, N, x, xs, y, ys, out, st);
    if (M >= 128 && N >= 128)
      return run_tiled_h2<128, 128, 8, 8, 8>(batch, M, K, N, x, xs, y, ys, out, st);
    if (M >= 64 && N >= 64)
      return run_tiled_h2<64, 64, 8, 4, 4>(batch, M, K, N, x, xs, y, ys, out, st);
    if (M >= 32 && N >= 32)
      return run_tiled_h2<32, 32, 8, 2, 2>(batch, M, K, N, x, xs, y, ys, out, st);
    return run_small<__half, __half>(batch, M, K, N, x, xs, y, ys, out, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace rbc
