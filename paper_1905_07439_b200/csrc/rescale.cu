// Diagonal rescaling around the deterministic recursion, on the device
// (reference pkg/src/randbc/rescale.py:36-99).
//
// The O(N^2) steps of the "2x O-I" baseline, in the measured mode with the
// reference's rounding sequence:
//   abs-max along rows / columns : exact (comparisons);
//   reciprocal                   : fl(1 / d), one rounding (rescale.py:44-47);
//   inside factor                : d = fl(sqrt(fl(bmax / amax))) (rescale.py:88-90);
//   row / column scaling         : fl(d_i * x_ij), one rounding per entry
//                                  (rescale.py:50-57), a row and a column
//                                  factor applied in that order when both.
// binary16 divides and square roots run in binary32 and round once more to
// binary16: double rounding is innocuous for +, -, *, / and sqrt when the
// wider format has >= 2p + 2 bits (24 >= 2 * 11 + 2), which is also how
// numpy's float16 ufuncs compute, so the values are the reference's.
// The orchestration (rbc_rescaled_multiply) lives in engine.cu.

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.h"

namespace rbc {

namespace {

// Per-column partial maxima over a chunk of rows: part[chunk][col].  The
// maximum of |x| is exact in any order; binary16 values compare exactly in
// binary32.
template <class T, class M>
__global__ void absmax_cols_part_kernel(const T* __restrict__ x, int64_t N, int64_t rows_per,
                                        M* __restrict__ part) {
  const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (col >= N) return;
  const int64_t r0 = blockIdx.y * rows_per, r1 = min(N, r0 + rows_per);
  M m = 0;
  for (int64_t r = r0; r < r1; ++r) {
    const T e = x[r * N + col];
    M a;
    if constexpr (sizeof(T) == 2) a = (M)fabsf(__half2float(e));
    else a = (M)fabs(e);
    m = a > m ? a : m;
  }
  part[blockIdx.y * N + col] = m;
}

// Per-row maxima: one warp per row.
template <class T, class M>
__global__ void absmax_rows_kernel(const T* __restrict__ x, int64_t N, M* __restrict__ out) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (row >= N) return;
  const T* xr = x + row * N;
  M m = 0;
  for (int64_t c = lane; c < N; c += 32) {
    const T e = xr[c];
    M a;
    if constexpr (sizeof(T) == 2) a = (M)fabsf(__half2float(e));
    else a = (M)fabs(e);
    m = a > m ? a : m;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const M t = __shfl_xor_sync(0xffffffffu, m, o);
    m = t > m ? t : m;
  }
  if (lane == 0) out[row] = m;
}

// Column maxima from the partials; writes the mode-typed maxima and raises
// *zero when one of them is 0 (rescale.py:36-41: degenerate input).
template <class T, class M>
__global__ void absmax_finish_kernel(const M* __restrict__ part, int chunks, int64_t N,
                                     T* __restrict__ out, uint8_t* __restrict__ zero) {
  const int64_t col = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (col >= N) return;
  M m = 0;
  for (int c = 0; c < chunks; ++c) {
    const M a = part[c * N + col];
    m = a > m ? a : m;
  }
  if (m == (M)0) *zero = 1;
  if constexpr (sizeof(T) == 2) out[col] = __float2half_rn((float)m);  // exact: m is a binary16 value
  else out[col] = (T)m;
}

template <class T, class M>
__global__ void rows_to_mode_kernel(const M* __restrict__ m, int64_t N, T* __restrict__ out,
                                    uint8_t* __restrict__ zero) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  if (m[i] == (M)0) *zero = 1;
  if constexpr (sizeof(T) == 2) out[i] = __float2half_rn((float)m[i]);
  else out[i] = (T)m[i];
}

// fl(1 / d) (rescale.py:44-47)
template <class T>
__device__ __forceinline__ T recip(T d);
template <> __device__ __forceinline__ float recip<float>(float d) { return __frcp_rn(d); }
template <> __device__ __forceinline__ double recip<double>(double d) { return __drcp_rn(d); }
template <> __device__ __forceinline__ __half recip<__half>(__half d) {
  return __float2half_rn(__frcp_rn(__half2float(d)));
}

template <class T>
__device__ __forceinline__ T div_rn(T a, T b);
template <> __device__ __forceinline__ float div_rn<float>(float a, float b) { return __fdiv_rn(a, b); }
template <> __device__ __forceinline__ double div_rn<double>(double a, double b) { return __ddiv_rn(a, b); }
template <> __device__ __forceinline__ __half div_rn<__half>(__half a, __half b) {
  return __float2half_rn(__fdiv_rn(__half2float(a), __half2float(b)));
}

template <class T>
__device__ __forceinline__ T sqrt_rn(T a);
template <> __device__ __forceinline__ float sqrt_rn<float>(float a) { return __fsqrt_rn(a); }
template <> __device__ __forceinline__ double sqrt_rn<double>(double a) { return __dsqrt_rn(a); }
template <> __device__ __forceinline__ __half sqrt_rn<__half>(__half a) {
  return __float2half_rn(__fsqrt_rn(__half2float(a)));
}

template <class T>
__global__ void recip_kernel(const T* __restrict__ d, int64_t N, T* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < N) out[i] = recip(d[i]);
}

// inside step: d = fl(sqrt(fl(bmax / amax))), rd = fl(1 / d)
template <class T>
__global__ void inside_factors_kernel(const T* __restrict__ bmax, const T* __restrict__ amax,
                                      int64_t N, T* __restrict__ d, T* __restrict__ rd) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  const T v = sqrt_rn(div_rn(bmax[i], amax[i]));
  d[i] = v;
  rd[i] = recip(v);
}

// x[i][j] = fl(fl(row[i] * x[i][j]) * col[j]) for each (row, col) pair in
// order (either may be null); in place, one rounding per multiply.
template <class T>
__global__ void scale_kernel(T* __restrict__ x, int64_t N, ScaleList sl) {
  const int64_t total = N * N;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / N, j = e - i * N;
    T v = x[e];
    for (int s = 0; s < sl.n; ++s) {
      if (sl.row[s]) v = Arith<T>::mul(static_cast<const T*>(sl.row[s])[i], v);
      if (sl.col[s]) v = Arith<T>::mul(v, static_cast<const T*>(sl.col[s])[j]);
    }
    x[e] = v;
  }
}

constexpr int kChunkRows = 128;

template <class T, class M>
cudaError_t absmax_impl(const void* x, int64_t N, int axis, void* out, uint8_t* zero,
                        void* scratch, cudaStream_t st) {
  M* m = static_cast<M*>(scratch);
  if (axis == 1) {  // row maxima
    absmax_rows_kernel<T, M><<<(unsigned)((N + 7) / 8), 256, 0, st>>>(static_cast<const T*>(x), N, m);
    rows_to_mode_kernel<T, M><<<(unsigned)((N + 255) / 256), 256, 0, st>>>(m, N, static_cast<T*>(out), zero);
  } else {  // column maxima
    const int chunks = (int)((N + kChunkRows - 1) / kChunkRows);
    dim3 grid((unsigned)((N + 255) / 256), (unsigned)chunks);
    absmax_cols_part_kernel<T, M><<<grid, 256, 0, st>>>(static_cast<const T*>(x), N, kChunkRows, m);
    absmax_finish_kernel<T, M><<<(unsigned)((N + 255) / 256), 256, 0, st>>>(
        m, chunks, N, static_cast<T*>(out), zero);
  }
  return cudaGetLastError();
}

}  // namespace

size_t absmax_scratch_bytes(int64_t N) {
  return (size_t)8 * (size_t)((N + kChunkRows - 1) / kChunkRows + 1) * (size_t)N;
}

cudaError_t launch_absmax(int dtype, const void* x, int64_t N, int axis, void* out, uint8_t* zero,
                          void* scratch, cudaStream_t st) {
  if (N == 0) return cudaSuccess;
  if (dtype == kF64) return absmax_impl<double, double>(x, N, axis, out, zero, scratch, st);
  if (dtype == kF32) return absmax_impl<float, float>(x, N, axis, out, zero, scratch, st);
  if (dtype == kF16) return absmax_impl<__half, float>(x, N, axis, out, zero, scratch, st);
  return cudaErrorInvalidValue;
}

cudaError_t launch_recip(int dtype, const void* d, int64_t N, void* out, cudaStream_t st) {
  if (N == 0) return cudaSuccess;
  const unsigned g = (unsigned)((N + 255) / 256);
  if (dtype == kF64) recip_kernel<double><<<g, 256, 0, st>>>((const double*)d, N, (double*)out);
  else if (dtype == kF32) recip_kernel<float><<<g, 256, 0, st>>>((const float*)d, N, (float*)out);
  else recip_kernel<__half><<<g, 256, 0, st>>>((const __half*)d, N, (__half*)out);
  return cudaGetLastError();
}

cudaError_t launch_inside_factors(int dtype, const void* bmax, const void* amax, int64_t N,
                                  void* d, void* rd, cudaStream_t st) {
  if (N == 0) return cudaSuccess;
  const unsigned g = (unsigned)((N + 255) / 256);
  if (dtype == kF64)
    inside_factors_kernel<double><<<g, 256, 0, st>>>((const double*)bmax, (const double*)amax, N,
                                                     (double*)d, (double*)rd);
  else if (dtype == kF32)
    inside_factors_kernel<float><<<g, 256, 0, st>>>((const float*)bmax, (const float*)amax, N,
                                                    (float*)d, (float*)rd);
  else
    inside_factors_kernel<__half><<<g, 256, 0, st>>>((const __half*)bmax, (const __half*)amax, N,
                                                     (__half*)d, (__half*)rd);
  return cudaGetLastError();
}

cudaError_t launch_scale(int dtype, void* x, int64_t N, const ScaleList& sl, cudaStream_t st) {
  if (N == 0 || sl.n == 0) return cudaSuccess;
  const int64_t total = N * N;
  const unsigned g = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (dtype == kF64) scale_kernel<double><<<g, 256, 0, st>>>((double*)x, N, sl);
  else if (dtype == kF32) scale_kernel<float><<<g, 256, 0, st>>>((float*)x, N, sl);
  else scale_kernel<__half><<<g, 256, 0, st>>>((__half*)x, N, sl);
  return cudaGetLastError();
}

}  // namespace rbc
