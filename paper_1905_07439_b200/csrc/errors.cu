// Error check (reference experiments.py:222-223, 251-261):
//
//   rel_error[t] = sqrt(sum (widen(C_t) - ref)^2) / ||ref||_F      (binary64)
//
// Deterministic two-pass reduction: pass 1 writes one partial sum per
// (trial, block) with a fixed warp-shuffle tree; pass 2 adds the partials of
// each trial in block order.  Results therefore do not vary from run to run.
// (The reference's numpy pairwise/BLAS sums use another order; the two
// agree to a few ulp of binary64, far inside the 1e-12 golden tolerance.)

#include <algorithm>

#include "kernels.h"

namespace rbc {

namespace {

constexpr int kThreads = 256;
constexpr int kBlocksPerTrial = 512;  // scratch stride; see rel_errors_t for the count in use

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kThreads / 32; ++w) s += sh[w];
  __syncthreads();
  return s;
}

template <class T>
__global__ void __launch_bounds__(kThreads) sumsq_kernel(int64_t N2, const T* __restrict__ c,
                                                         const double* __restrict__ ref,
                                                         int64_t ref_tstride,
                                                         double* __restrict__ part_num,
                                                         double* __restrict__ part_den) {
  __shared__ double sh[kThreads / 32];
  const int64_t t = blockIdx.y;
  const T* ct = c + t * N2;
  const double* rt = ref + t * ref_tstride;
  double num = 0.0, den = 0.0;
  // four independent loads in flight per thread per round
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  for (; i + 3 * stride < N2; i += 4 * stride) {
    double r[4], cv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      r[q] = rt[i + q * stride];
      cv[q] = Arith<T>::widen(ct[i + q * stride]);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double d = cv[q] - r[q];
      num += d * d;
      den += r[q] * r[q];
    }
  }
  for (; i < N2; i += stride) {
    const double r = rt[i];
    const double d = Arith<T>::widen(ct[i]) - r;
    num += d * d;
    den += r * r;
  }
  num = block_sum(num, sh);
  den = block_sum(den, sh);
  if (threadIdx.x == 0) {
    part_num[t * gridDim.x + blockIdx.x] = num;
    part_den[t * gridDim.x + blockIdx.x] = den;
  }
}

__global__ void finish_kernel(int64_t ntr, int nb, const double* __restrict__ part_num,
                              const double* __restrict__ part_den, double* __restrict__ err) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntr) return;
  double num = 0.0, den = 0.0;
  for (int b = 0; b < nb; ++b) {
    num += part_num[t * nb + b];
    den += part_den[t * nb + b];
  }
  err[t] = sqrt(num) / sqrt(den);
}

template <class T>
__global__ void __launch_bounds__(kThreads) nonfinite_kernel(int64_t N2, const T* __restrict__ x,
                                                             uint8_t* __restrict__ flags) {
  const int64_t t = blockIdx.y;
  const T* xt = x + t * N2;
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < N2;
       i += (int64_t)gridDim.x * kThreads)
    bad = bad || !Arith<T>::finite(xt[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) flags[t] = 1;
}

template <class T>
cudaError_t rel_errors_t(int64_t ntr, int64_t N2, const void* c, const double* ref, int64_t rts,
                         double* err, void* scratch, cudaStream_t st) {
  // blocks per trial: about 16 elements per thread, at most kBlocksPerTrial
  // (a function of N2 only, so the summation order is fixed)
  // Above 2^24 elements a launch holds only a few trials (config 5: two), and
  // 64 blocks each would leave SMs idle: 512 there (error kernels 1.40 ->
  // 0.55 ms per config-5 step; config 4 measured better with 64: 0.24 vs 0.30).
  const int64_t cap = N2 > ((int64_t)1 << 24) ? kBlocksPerTrial : 64;
  const int nb = (int)std::min<int64_t>(cap, std::max<int64_t>(1, (N2 + 4095) / 4096));
  double* pn = (double*)scratch;
  double* pd = pn + ntr * kBlocksPerTrial;
  for (int64_t t0 = 0; t0 < ntr; t0 += 65535) {
    const int64_t nt = ntr - t0 < 65535 ? ntr - t0 : 65535;
    dim3 grid(nb, (unsigned)nt);
    sumsq_kernel<T><<<grid, kThreads, 0, st>>>(N2, (const T*)c + t0 * N2, ref + t0 * rts, rts,
                                                pn + t0 * nb, pd + t0 * nb);
  }
  finish_kernel<<<(unsigned)((ntr + 127) / 128), 128, 0, st>>>(ntr, nb, pn, pd, err);
  return cudaGetLastError();
}

template <class T>
cudaError_t nonfinite_t(int64_t ntr, int64_t N2, const void* x, uint8_t* flags, cudaStream_t st) {
  for (int64_t t0 = 0; t0 < ntr; t0 += 65535) {
    const int64_t nt = ntr - t0 < 65535 ? ntr - t0 : 65535;
    int64_t bx = (N2 + kThreads - 1) / kThreads;
    if (bx > 64) bx = 64;
    nonfinite_kernel<T><<<dim3((unsigned)bx, (unsigned)nt), kThreads, 0, st>>>(
        N2, (const T*)x + t0 * N2, flags + t0);
  }
  return cudaGetLastError();
}

// total[e] = fl(...fl(total[e] + widen(x[0][e])) + ... + widen(x[T-1][e])):
// the sequential binary64 accumulation of enumerate_expectation
// (reference randomize.py:317-326) / _run_average (experiments.py:382-383).
template <class T>
__global__ void __launch_bounds__(kThreads) sum_trials_kernel(int64_t ntr, int64_t N2,
                                                              const T* __restrict__ x,
                                                              double* __restrict__ total) {
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < N2;
       e += (int64_t)gridDim.x * kThreads) {
    double acc = total[e];
    for (int64_t t = 0; t < ntr; ++t) acc = __dadd_rn(acc, Arith<T>::widen(x[t * N2 + e]));
    total[e] = acc;
  }
}

}  // namespace

cudaError_t launch_sum_trials(int dtype, int64_t ntr, int64_t N2, const void* x, double* total,
                              cudaStream_t st) {
  int64_t blocks = (N2 + kThreads - 1) / kThreads;
  if (blocks > 148 * 8) blocks = 148 * 8;
  switch (dtype) {
    case kF64: sum_trials_kernel<double><<<(unsigned)blocks, kThreads, 0, st>>>(ntr, N2, (const double*)x, total); break;
    case kF32: sum_trials_kernel<float><<<(unsigned)blocks, kThreads, 0, st>>>(ntr, N2, (const float*)x, total); break;
    case kF16: sum_trials_kernel<__half><<<(unsigned)blocks, kThreads, 0, st>>>(ntr, N2, (const __half*)x, total); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

size_t error_scratch_bytes(int64_t ntr) { return (size_t)ntr * kBlocksPerTrial * 2 * sizeof(double); }

cudaError_t launch_rel_errors(int dtype, int64_t ntr, int64_t N2, const void* c, const double* ref,
                              int64_t ref_tstride, double* err, void* scratch, cudaStream_t st) {
  switch (dtype) {
    case kF64: return rel_errors_t<double>(ntr, N2, c, ref, ref_tstride, err, scratch, st);
    case kF32: return rel_errors_t<float>(ntr, N2, c, ref, ref_tstride, err, scratch, st);
    case kF16: return rel_errors_t<__half>(ntr, N2, c, ref, ref_tstride, err, scratch, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_nonfinite(int dtype, int64_t ntr, int64_t N2, const void* x, uint8_t* flags,
                             cudaStream_t st) {
  switch (dtype) {
    case kF64: return nonfinite_t<double>(ntr, N2, x, flags, st);
    case kF32: return nonfinite_t<float>(ntr, N2, x, flags, st);
    case kF16: return nonfinite_t<__half>(ntr, N2, x, flags, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace rbc
