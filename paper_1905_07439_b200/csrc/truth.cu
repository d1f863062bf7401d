// Binary64 ground truth and binary64 leaves on the DFMA pipe (reference
// standard_multiply, pkg/src/randbc/multiply.py:44-51, over leaf_matmul,
// pkg/src/randbc/_engine.py:42-61; the truth of experiments.py:251-254).
//
//   P[i,j] = fl(...fl(fl(x_i0*y_0j) + fl(x_i1*y_1j)) + ...),  k ascending.
//
// Two passes:
//  1. widen: X and Y to binary64 in 128-wide k-major panels, zero-padded to
//     whole tiles (HBM-bound, ~1% of a large product).  One k tile of one
//     operand is then a single contiguous span.
//  2. truth_bulk_kernel: 128 x 128 x 32 tiles, 8 x 8 outputs per thread,
//     one CTA of 256 threads per SM.  Operand tiles arrive by two bulk copies
//     per stage (cp.async.bulk, the TMA engine, issued by one lane) into a
//     3-stage shared-memory ring completed on mbarriers, so the threads issue
//     nothing but 16-byte fragment loads and the multiply-adds.  (A DFMA
//     holds the pipe's dispatch for two cycles and every other instruction
//     costs it one, so the per-stage waits, arrives and loop control are
//     worth amortising: k tiles of 16 x 4 stages 38.3 ms per 8192^3 product,
//     24 x 4: 37.4, 32 x 3: 37.2, 48 x 2: 42.5.)
//
// Rounding: for binary32/binary16 operands the widened products carry at most
// 48 significant bits and are exact in binary64, so fl(acc + fl(a*b)) ==
// fma(a, b, acc) and one DFMA per term is bit-identical to the reference's
// separate multiply and add.  Binary64 operands keep DMUL + DADD.  The first
// product initialises the chain (a multiply, not an FMA into +0, which would
// lose the sign of a -0 product) and K tails are skipped, never zero-padded.
// Pad rows/columns of the tile only feed outputs that are not stored.

#include <algorithm>
#include <cstdlib>

#include "bulk.cuh"
#include "kernels.h"

namespace rbc {

namespace {

constexpr int kBM = 128, kBN = 128, kBK = 32, kTM = 8, kTN = 8, kStages = 3;
constexpr int kThreads = (kBM / kTM) * (kBN / kTN);  // 256

template <class TIn>
__device__ __forceinline__ double widen(TIn v);
template <> __device__ __forceinline__ double widen<double>(double v) { return v; }
template <> __device__ __forceinline__ double widen<float>(float v) { return (double)v; }
template <> __device__ __forceinline__ double widen<__half>(__half v) {
  return (double)__half2float(v);
}

// Panel layouts of the widened operands (tile-contiguous, so one k tile of
// one operand is a single contiguous span and one bulk copy):
//   xt[b][tm][k][m'] = widen(x[b][tm*128 + m'][k])   (0 for rows >= M)
//   yw[b][tn][k][n'] = widen(y[b][k][tn*128 + n'])   (0 for cols >= N)
// 32 x 32 tiles through shared memory for the transpose; blockIdx.z = b.
template <class TIn>
__global__ void __launch_bounds__(256) widen_x_kernel(int M, int K, int tiles_m,
                                                      const TIn* __restrict__ x, int64_t xs,
                                                      double* __restrict__ xt) {
  __shared__ double tile[32][33];
  const int64_t b = blockIdx.z;
  const int m0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  const TIn* xb = x + b * xs;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int m = m0 + r, k = k0 + tx;
    tile[r][tx] = (m < M && k < K) ? widen<TIn>(xb[(int64_t)m * K + k]) : 0.0;
  }
  __syncthreads();
  const int tm = m0 / kBM, mo = m0 % kBM;
  double* ob = xt + (b * tiles_m + tm) * (int64_t)K * kBM + mo;
#pragma unroll
  for (int r = ty; r < 32; r += 8) {
    const int k = k0 + r;
    if (k < K) ob[(int64_t)k * kBM + tx] = tile[tx][r];
  }
}

// one (b, k) row of y per blockIdx.y, 128 columns per blockIdx.x
template <class TIn>
__global__ void __launch_bounds__(128) widen_y_kernel(int K, int N, int tiles_n,
                                                      const TIn* __restrict__ y, int64_t ys,
                                                      double* __restrict__ yw) {
  const int64_t row = blockIdx.y;
  const int64_t b = row / K;
  const int k = (int)(row - b * K);
  const int tn = blockIdx.x;
  const int n = tn * kBN + threadIdx.x;
  const double v = n < N ? widen<TIn>(y[b * ys + (int64_t)k * N + n]) : 0.0;
  yw[((b * tiles_n + tn) * (int64_t)K + k) * kBN + threadIdx.x] = v;
}

template <bool FMA>
__device__ __forceinline__ double mac(double acc, double a, double b) {
  if constexpr (FMA) return __fma_rn(a, b, acc);
  else return __dadd_rn(acc, __dmul_rn(a, b));
}

// FMA: operands were widened from binary32/binary16 (exact products).
// Stage reuse is tracked by per-stage "empty" mbarriers (one arrival per
// warp): only the issuing lane (warp 0, lane 0) waits for a stage to drain,
// the other warps run free between their "full" waits -- no CTA barrier in
// the k loop.
template <bool FMA>
__global__ void __launch_bounds__(kThreads, 1)
    truth_bulk_kernel(int M, int K, int N, int tiles_m_arg, const double* __restrict__ xt,
                      const double* __restrict__ yw, double* __restrict__ out, int tiles_n) {
  constexpr int VW = 2;  // doubles per 16-byte fragment load
  constexpr int DY = kBM / kTM, DX = kBN / kTN;
  constexpr int GM = kTM / VW, GN = kTN / VW;
  constexpr int WX = 8, WY = 4;  // warp shape: 4 (M) x 8 (N) threads
  constexpr int WPX = DX / WX;
  extern __shared__ __align__(128) unsigned char smem[];
  auto As = reinterpret_cast<double(*)[kBK][kBM]>(smem);
  auto Bs = reinterpret_cast<double(*)[kBK][kBN]>(smem + sizeof(double) * kStages * kBK * kBM);
  uint64_t* full =
      reinterpret_cast<uint64_t*>(smem + sizeof(double) * kStages * kBK * (kBM + kBN));
  uint64_t* empty = full + kStages;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int tx = (warp % WPX) * WX + (lane % WX);
  const int ty = (warp / WPX) * WY + (lane / WX);
  const int64_t b = blockIdx.y;
  // Tiles in row order.  (A grouped raster -- 8 consecutive tile rows swept
  // column by column, sharing their X panels in L2 -- cuts DRAM reads at 8192
  // from 32.8 to 10.3 GB per product but runs 3% slower: the kernel is
  // DFMA-bound either way.)
  const int tiles_m = tiles_m_arg;
  const int tm = blockIdx.x / tiles_n;
  const int tn = blockIdx.x - tm * tiles_n;
  const int m0 = tm * kBM, n0 = tn * kBN;
  const double* xa = xt + (b * tiles_m + tm) * (int64_t)K * kBM;  // panel: row k at xa + k*128
  const double* yb = yw + (b * (int64_t)tiles_n + tn) * (int64_t)K * kBN;
  const int ktiles = (K + kBK - 1) / kBK;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kThreads / 32);
    }
    mbar_init_fence();
  }
  __syncthreads();

  // one lane fills stage kt % kStages with k tile kt: two contiguous spans
  auto issue = [&](int kt) {
    const int s = kt % kStages;
    const int k0 = kt * kBK;
    const unsigned rows = (unsigned)min(kBK, K - k0);
    fence_proxy_async();
    mbar_expect_tx(&full[s], rows * (kBM + kBN) * (unsigned)sizeof(double));
    bulk_g2s(&As[s][0][0], xa + (int64_t)k0 * kBM, rows * kBM * (unsigned)sizeof(double), &full[s]);
    bulk_g2s(&Bs[s][0][0], yb + (int64_t)k0 * kBN, rows * kBN * (unsigned)sizeof(double), &full[s]);
  };
  if (tid == 0)
    for (int kt = 0; kt < kStages && kt < ktiles; ++kt) issue(kt);

  double acc[kTM][kTN];
  double fa[kTM], fb[kTN];
  auto load_frag = [&](int s, int kk) {
#pragma unroll
    for (int g = 0; g < GM; ++g) {
      const double2 v = *reinterpret_cast<const double2*>(&As[s][kk][g * DY * VW + ty * VW]);
      fa[g * VW] = v.x;
      fa[g * VW + 1] = v.y;
    }
#pragma unroll
    for (int g = 0; g < GN; ++g) {
      const double2 v = *reinterpret_cast<const double2*>(&Bs[s][kk][g * DX * VW + tx * VW]);
      fb[g * VW] = v.x;
      fb[g * VW + 1] = v.y;
    }
  };
  auto kstep = [&]() {
#pragma unroll
    for (int i = 0; i < kTM; ++i)
#pragma unroll
      for (int j = 0; j < kTN; ++j) acc[i][j] = mac<FMA>(acc[i][j], fa[i], fb[j]);
  };

  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % kStages;
    mbar_wait(&full[s], (unsigned)((kt / kStages) & 1));
    const int kmax = min(kBK, K - kt * kBK);
    load_frag(s, 0);
    if (kt == 0) {
#pragma unroll
      for (int i = 0; i < kTM; ++i)
#pragma unroll
        for (int j = 0; j < kTN; ++j) acc[i][j] = __dmul_rn(fa[i], fb[j]);
    } else {
      kstep();
    }
    if (kmax == kBK) {
#pragma unroll
      for (int kk = 1; kk < kBK; ++kk) {
        load_frag(s, kk);
        kstep();
      }
    } else {
#pragma unroll 1
      for (int kk = 1; kk < kmax; ++kk) {
        load_frag(s, kk);
        kstep();
      }
    }
    // The warp read stage s through the generic proxy and the refill writes
    // it through the async proxy: order the two before the release (the
    // compiler is free to place the arrive right after the last LDS issue,
    // ahead of the DFMAs that wait for those loads; see leaf_ring_kernel).
    fence_proxy_async();
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    if (tid == 0 && kt + kStages < ktiles) {
      mbar_wait(&empty[s], (unsigned)((kt / kStages) & 1));
      issue(kt + kStages);
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
        const double e0 = acc[gi * VW + v][gj * VW], e1 = acc[gi * VW + v][gj * VW + 1];
        if (gn + 1 < N && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
          *reinterpret_cast<double2*>(o) = make_double2(e0, e1);
        } else {
          if (gn < N) o[0] = e0;
          if (gn + 1 < N) o[1] = e1;
        }
      }
    }
}

constexpr size_t kSmem = sizeof(double) * kStages * kBK * (kBM + kBN) + 2 * sizeof(uint64_t) * kStages;

// The stream-ordered pool keeps freed scratch for reuse instead of returning
// it to the driver at every synchronisation -- up to 4 GiB (two launches'
// worth of the <= 2 GiB scratch below; anything above is released at the
// next synchronisation).  The host-buffer calls size their arenas to 85% of
// free + arena memory (engine.cu host_ws_budget / rbc_error_trials), so the
// retained scratch always fits in the remaining 15% (27 GB on a B200).
}  // namespace

cudaError_t keep_pool(int device) {
  static int done = -1;
  if (done == device) return cudaSuccess;
  cudaMemPool_t pool;
  cudaError_t e = cudaDeviceGetDefaultMemPool(&pool, device);
  if (e != cudaSuccess) return e;
  uint64_t keep = (uint64_t)4 << 30;
  e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  if (e == cudaSuccess) done = device;
  return e;
}

namespace {

template <class TIn>
cudaError_t run_truth_bulk(int64_t batch, int64_t M, int64_t K, int64_t N, const void* x,
                           int64_t xs, const void* y, int64_t ys, void* out, cudaStream_t st) {
  constexpr bool kFma = sizeof(TIn) < sizeof(double);
  static const cudaError_t attr = cudaFuncSetAttribute(
      truth_bulk_kernel<kFma>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
  if (attr != cudaSuccess) return attr;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = keep_pool(dev);
  if (e != cudaSuccess) return e;
  const int64_t Mp = (M + kBM - 1) / kBM * kBM;
  const int64_t Np = (N + kBN - 1) / kBN * kBN;
  const int64_t per = K * (Mp + Np);  // scratch doubles per product
  const int64_t cap = std::max<int64_t>(1, ((int64_t)2 << 30) / (int64_t)(per * sizeof(double)));
  const int64_t chunk = std::min<int64_t>({batch, cap, (int64_t)65535});
  double* scratch = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&scratch), (size_t)(chunk * per * sizeof(double)), st);
  if (e != cudaSuccess) return e;
  const int tiles_m = (int)(Mp / kBM), tiles_n = (int)(Np / kBN);
  for (int64_t b0 = 0; b0 < batch && e == cudaSuccess; b0 += chunk) {
    const int64_t nb = std::min(chunk, batch - b0);
    double* xt = scratch;
    double* yw = scratch + nb * K * Mp;
    const TIn* xb = static_cast<const TIn*>(x) + b0 * xs;
    const TIn* yb = static_cast<const TIn*>(y) + b0 * ys;
    dim3 tg((unsigned)(Mp / 32), (unsigned)((K + 31) / 32), (unsigned)nb);
    widen_x_kernel<TIn><<<tg, 256, 0, st>>>((int)M, (int)K, tiles_m, xb, xs, xt);
    const int64_t pp = std::max<int64_t>(1, 65535 / K);  // whole products per launch
    for (int64_t p0 = 0; p0 < nb; p0 += pp) {
      const int64_t np = std::min(pp, nb - p0);
      dim3 pg((unsigned)tiles_n, (unsigned)(np * K), 1);
      widen_y_kernel<TIn><<<pg, kBN, 0, st>>>((int)K, (int)N, tiles_n, yb + p0 * ys, ys,
                                              yw + p0 * K * Np);
    }
    dim3 grid((unsigned)(tiles_m * tiles_n), (unsigned)nb, 1);
    truth_bulk_kernel<kFma><<<grid, kThreads, kSmem, st>>>(
        (int)M, (int)K, (int)N, tiles_m, xt, yw, static_cast<double*>(out) + b0 * M * N,
        tiles_n);
    e = cudaGetLastError();
  }
  const cudaError_t f = cudaFreeAsync(scratch, st);
  return e != cudaSuccess ? e : f;
}

}  // namespace

cudaError_t launch_truth(int dtype_in, int64_t batch, int64_t M, int64_t K, int64_t N,
                         const void* x, int64_t xs, const void* y, int64_t ys, void* out,
                         cudaStream_t st) {
  if (K < 1 || M < 1 || N < 1 || K > 65535) return cudaErrorNotSupported;
  if (dtype_in == kF32) return run_truth_bulk<float>(batch, M, K, N, x, xs, y, ys, out, st);
  if (dtype_in == kF16) return run_truth_bulk<__half>(batch, M, K, N, x, xs, y, ys, out, st);
  if (dtype_in == kF64) return run_truth_bulk<double>(batch, M, K, N, x, xs, y, ys, out, st);
  return cudaErrorNotSupported;
}

}  // namespace rbc
