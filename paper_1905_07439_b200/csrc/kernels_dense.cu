// Dense-coefficient combination kernels: the general engine path for any
// coefficient tables (approximate / perturbed formulas, arbitrary n and R).
//
// Exactly the reference's arithmetic (pkg/src/randbc/_engine.py:64-114):
// every coefficient -- zeros included -- is multiplied and added, the
// expansion folds l inside each row k and then folds the row sums over k,
// the contraction folds r ascending, first term initialising.  The result is
// therefore bit-identical to the reference, signed zeros and non-finite
// propagation included.
//
// Coefficients are per trial ((Tc, R, n, n), Tc in {1, T}); every thread of a
// block row reads the same coefficient, so the loads are broadcasts.

#include <cstdlib>

#include "kernels.h"

namespace rbc {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxDenseN = 8;

template <class T, int W, int NMAX>
__global__ void __launch_bounds__(kThreads) expand_dense_kernel(
    const T* __restrict__ x, int64_t x_tstride, int K, int s, int n, int R,
    const T* __restrict__ coeff, int64_t c_tstride, T* __restrict__ out, int64_t ntr) {
  const int mb = s / n;
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
    const T* xb = x + t * x_tstride + (int64_t)Kp * s * s + (int64_t)i * s + j;
    Pack<T, W> g[NMAX * NMAX];
#pragma unroll
    for (int k = 0; k < NMAX; ++k)
#pragma unroll
      for (int l = 0; l < NMAX; ++l)
        if (k < n && l < n) g[k * NMAX + l] = pload<T, W>(xb + (int64_t)k * mb * s + l * mb);
    const T* ct = coeff + t * c_tstride;
    T* ob = out + (t * K + Kp) * (int64_t)R * mb * mb + pos;
    for (int r = 0; r < R; ++r) {
      const T* cr = ct + (int64_t)r * n * n;
      Pack<T, W> acc;
#pragma unroll
      for (int k = 0; k < NMAX; ++k) {
        if (k < n) {
          Pack<T, W> row = O::mul_scalar(cr[k * n], g[k * NMAX]);
#pragma unroll
          for (int l = 1; l < NMAX; ++l)
            if (l < n) row = O::add(row, O::mul_scalar(cr[k * n + l], g[k * NMAX + l]));
          acc = (k == 0) ? row : O::add(acc, row);
        }
      }
      pstore<T, W>(ob + (int64_t)r * mb * mb, acc);
    }
  }
}

template <class T, int W>
__global__ void __launch_bounds__(kThreads) contract_dense_kernel(
    const T* __restrict__ ch, int K, int mb, int n, int R, const T* __restrict__ w,
    int64_t w_tstride, T* __restrict__ out, int64_t ntr, uint8_t* __restrict__ nonfinite) {
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
    const T* cb = ch + (t * K + Kp) * (int64_t)R * mb * mb + pos;
    const T* wt = w + t * w_tstride;
    T* obase = out + (t * K + Kp) * (int64_t)s * s + (int64_t)i * s + j;
    bool ok = true;
    for (int I = 0; I < n; ++I) {
      for (int J = 0; J < n; ++J) {
        Pack<T, W> acc = O::mul_scalar(wt[I * n + J], pload<T, W>(cb));
        for (int r = 1; r < R; ++r)
          acc = O::add(acc, O::mul_scalar(wt[((int64_t)r * n + I) * n + J],
                                          pload<T, W>(cb + (int64_t)r * mb * mb)));
        if (nonfinite) ok = ok && O::all_finite(acc);
        pstore<T, W>(obase + (int64_t)I * mb * s + J * mb, acc);
      }
    }
    if (!ok) nonfinite[t] = 1;
  }
}

// ---- staged variants: one CTA per (trial, 256*PPT positions); the trial's
// coefficient table lives in shared memory (broadcast reads) and each thread
// carries PPT positions so one coefficient read feeds PPT multiply-adds.
constexpr int kPPT = 4;

template <class T, int N>
__global__ void __launch_bounds__(kThreads) expand_dense_staged(
    const T* __restrict__ x, int64_t x_tstride, int K, int s, int R, const T* __restrict__ coeff,
    int64_t c_tstride, T* __restrict__ out, int64_t ntr) {
  extern __shared__ __align__(16) unsigned char sraw[];
  T* sc = reinterpret_cast<T*>(sraw);
  using A = Arith<T>;
  const int mb = s / N;
  const int P = mb * mb;
  const int64_t items = (int64_t)K * P;
  for (int64_t t = blockIdx.y; t < ntr; t += gridDim.y) {
    __syncthreads();
    for (int q = threadIdx.x; q < R * N * N; q += kThreads) sc[q] = coeff[t * c_tstride + q];
    __syncthreads();
    const T* xt = x + t * x_tstride;
    T g[kPPT][N * N];
    int64_t obase[kPPT];
    bool live[kPPT];
#pragma unroll
    for (int p = 0; p < kPPT; ++p) {
      const int64_t e = ((int64_t)blockIdx.x * kPPT + p) * kThreads + threadIdx.x;
      live[p] = e < items;
      const int64_t ee = live[p] ? e : 0;
      const int Kp = (int)(ee / P);
      const int pos = (int)(ee - (int64_t)Kp * P);
      const int i = pos / mb, j = pos - (pos / mb) * mb;
      const T* xb = xt + (int64_t)Kp * s * s + (int64_t)i * s + j;
#pragma unroll
      for (int k = 0; k < N; ++k)
#pragma unroll
        for (int l = 0; l < N; ++l) g[p][k * N + l] = live[p] ? xb[(int64_t)k * mb * s + l * mb] : T(0);
      obase[p] = (t * K + Kp) * (int64_t)R * P + pos;
    }
    for (int r = 0; r < R; ++r) {
      const T* cr = sc + r * N * N;
      T acc[kPPT];
#pragma unroll
      for (int k = 0; k < N; ++k) {
        T row[kPPT];
#pragma unroll
        for (int p = 0; p < kPPT; ++p) row[p] = A::mul(cr[k * N], g[p][k * N]);
#pragma unroll
        for (int l = 1; l < N; ++l) {
          const T c = cr[k * N + l];
#pragma unroll
          for (int p = 0; p < kPPT; ++p) row[p] = A::add(row[p], A::mul(c, g[p][k * N + l]));
        }
#pragma unroll
        for (int p = 0; p < kPPT; ++p) acc[p] = (k == 0) ? row[p] : A::add(acc[p], row[p]);
      }
#pragma unroll
      for (int p = 0; p < kPPT; ++p)
        if (live[p]) out[obase[p] + (int64_t)r * P] = acc[p];
    }
  }
}

// binary64 tables of n = 3 carry fewer positions per thread: the n*n*PPT
// accumulators plus the batched child loads must leave room for more than
// one resident CTA per SM
template <class T, int N>
constexpr int contract_ppt() {
  return sizeof(T) == 8 && N >= 3 ? 2 : kPPT;
}

template <class T, int N, int CP = contract_ppt<T, N>(), int kRB = 4>
__global__ void __launch_bounds__(kThreads) contract_dense_staged(
    const T* __restrict__ ch, int K, int mb, int R, const T* __restrict__ w, int64_t w_tstride,
    T* __restrict__ out, int64_t ntr, uint8_t* __restrict__ nonfinite) {
  extern __shared__ __align__(16) unsigned char sraw[];
  T* sw = reinterpret_cast<T*>(sraw);
  using A = Arith<T>;
  const int s = N * mb;
  const int P = mb * mb;
  const int64_t items = (int64_t)K * P;
  for (int64_t t = blockIdx.y; t < ntr; t += gridDim.y) {
    __syncthreads();
    for (int q = threadIdx.x; q < R * N * N; q += kThreads) sw[q] = w[t * w_tstride + q];
    __syncthreads();
    int64_t cbase[CP], obase[CP];
    bool live[CP];
#pragma unroll
    for (int p = 0; p < CP; ++p) {
      const int64_t e = ((int64_t)blockIdx.x * CP + p) * kThreads + threadIdx.x;
      live[p] = e < items;
      const int64_t ee = live[p] ? e : 0;
      const int Kp = (int)(ee / P);
      const int pos = (int)(ee - (int64_t)Kp * P);
      const int i = pos / mb, j = pos - (pos / mb) * mb;
      cbase[p] = (t * K + Kp) * (int64_t)R * P + pos;
      obase[p] = (t * K + Kp) * (int64_t)s * s + (int64_t)i * s + j;
    }
    T acc[N * N][CP];
    // the children of kRB consecutive terms are loaded together (kRB * CP
    // independent loads in flight), then folded in ascending r
    for (int r0 = 0; r0 < R; r0 += kRB) {
      T pr[kRB][CP];
#pragma unroll
      for (int q = 0; q < kRB; ++q)
#pragma unroll
        for (int p = 0; p < CP; ++p)
          pr[q][p] = (live[p] && r0 + q < R) ? ch[cbase[p] + (int64_t)(r0 + q) * P] : T(0);
#pragma unroll
      for (int q = 0; q < kRB; ++q) {
        const int r = r0 + q;
        if (r >= R) break;
        const T* wr = sw + r * N * N;
#pragma unroll
        for (int ij = 0; ij < N * N; ++ij) {
          const T c = wr[ij];
#pragma unroll
          for (int p = 0; p < CP; ++p)
            acc[ij][p] = (r == 0) ? A::mul(c, pr[q][p]) : A::add(acc[ij][p], A::mul(c, pr[q][p]));
        }
      }
    }
    bool ok = true;
#pragma unroll
    for (int p = 0; p < CP; ++p) {
      if (!live[p]) continue;
#pragma unroll
      for (int I = 0; I < N; ++I)
#pragma unroll
        for (int J = 0; J < N; ++J) {
          const T v = acc[I * N + J][p];
          if (nonfinite) ok = ok && Arith<T>::finite(v);
          out[obase[p] + (int64_t)I * mb * s + J * mb] = v;
        }
    }
    if (!ok) nonfinite[t] = 1;
  }
}

template <class T, int N>
cudaError_t staged_expand_n(const void* x, int64_t xs, int64_t K, int64_t s, int R, const void* c,
                            int64_t cs, void* out, int64_t ntr, cudaStream_t st) {
  const int64_t items = K * (s / N) * (s / N);
  const size_t smem = (size_t)R * N * N * sizeof(T);
  auto kern = expand_dense_staged<T, N>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((unsigned)((items + kThreads * kPPT - 1) / (kThreads * kPPT)),
            (unsigned)(ntr < 65535 ? ntr : 65535));
  kern<<<grid, kThreads, smem, st>>>((const T*)x, xs, (int)K, (int)s, R, (const T*)c, cs, (T*)out, ntr);
  return cudaGetLastError();
}

template <class T, int N, int CP = contract_ppt<T, N>(), int RB = 4>
cudaError_t staged_contract_n(const void* ch, int64_t K, int64_t mb, int R, const void* w,
                              int64_t ws, void* out, int64_t ntr, uint8_t* nf, cudaStream_t st) {
  const int64_t items = K * mb * mb;
  const size_t smem = (size_t)R * N * N * sizeof(T);
  auto kern = contract_dense_staged<T, N, CP, RB>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid((unsigned)((items + kThreads * CP - 1) / (kThreads * CP)),
            (unsigned)(ntr < 65535 ? ntr : 65535));
  kern<<<grid, kThreads, smem, st>>>((const T*)ch, (int)K, (int)mb, R, (const T*)w, ws, (T*)out, ntr, nf);
  return cudaGetLastError();
}

// Returns cudaErrorNotSupported when no staged instantiation applies.
template <class T>
cudaError_t staged_expand(int n, const void* x, int64_t xs, int64_t K, int64_t s, int R,
                          const void* c, int64_t cs, void* out, int64_t ntr, cudaStream_t st) {
  if ((size_t)R * n * n * sizeof(T) > 160 * 1024) return cudaErrorNotSupported;
  switch (n) {
    case 2: return staged_expand_n<T, 2>(x, xs, K, s, R, c, cs, out, ntr, st);
    case 3: return staged_expand_n<T, 3>(x, xs, K, s, R, c, cs, out, ntr, st);
    case 4: return staged_expand_n<T, 4>(x, xs, K, s, R, c, cs, out, ntr, st);
  }
  return cudaErrorNotSupported;
}

template <class T>
cudaError_t staged_contract(int n, const void* ch, int64_t K, int64_t mb, int R, const void* w,
                            int64_t ws, void* out, int64_t ntr, uint8_t* nf, cudaStream_t st) {
  if ((size_t)R * n * n * sizeof(T) > 160 * 1024) return cudaErrorNotSupported;
  // binary64 n = 3 (config 3's noisy Laderman): 2 positions per thread and
  // the children of 12 terms in flight (ms per launch: 4 terms 0.183, 8:
  // 0.175, 12: 0.164, 23: 0.201; 1 or 4 positions per thread no better)
  if (sizeof(T) == 8 && n == 3)
    return staged_contract_n<T, 3, 2, 12>(ch, K, mb, R, w, ws, out, ntr, nf, st);
  switch (n) {
    case 2: return staged_contract_n<T, 2>(ch, K, mb, R, w, ws, out, ntr, nf, st);
    case 3: return staged_contract_n<T, 3>(ch, K, mb, R, w, ws, out, ntr, nf, st);
  }
  return cudaErrorNotSupported;
}

inline dim3 grid_for(int64_t items, int64_t ntr) {
  const int64_t bx = (items + kThreads - 1) / kThreads;
  return dim3((unsigned)bx, (unsigned)(ntr < 65535 ? ntr : 65535), 1);
}

template <class T, int W>
cudaError_t expand_dense_w(const void* x, int64_t xs, int64_t K, int64_t s, int n, int R,
                           const void* c, int64_t cs, void* out, int64_t ntr, cudaStream_t st) {
  const int64_t mb = s / n;
  const dim3 grid = grid_for(K * (mb * mb / W), ntr);
  if (n <= 2)
    expand_dense_kernel<T, W, 2><<<grid, kThreads, 0, st>>>((const T*)x, xs, (int)K, (int)s, n, R,
                                                            (const T*)c, cs, (T*)out, ntr);
  else if (n <= 4)
    expand_dense_kernel<T, W, 4><<<grid, kThreads, 0, st>>>((const T*)x, xs, (int)K, (int)s, n, R,
                                                            (const T*)c, cs, (T*)out, ntr);
  else
    expand_dense_kernel<T, 1, kMaxDenseN><<<grid_for(K * mb * mb, ntr), kThreads, 0, st>>>(
        (const T*)x, xs, (int)K, (int)s, n, R, (const T*)c, cs, (T*)out, ntr);
  return cudaGetLastError();
}

template <class T>
cudaError_t expand_dense_t(int dtype, const void* x, int64_t xs, int64_t K, int64_t s, int n,
                           int R, const void* c, int64_t cs, void* out, int64_t ntr,
                           cudaStream_t st) {
  {
    cudaError_t e = staged_expand<T>(n, x, xs, K, s, R, c, cs, out, ntr, st);
    if (e != cudaErrorNotSupported) return e;
  }
  const int W = n > 4 ? 1 : pick_width(dtype, s / n, 8 / (int)sizeof(T));
  switch (W) {
    case 4: return expand_dense_w<T, (sizeof(T) == 2 ? 4 : 1)>(x, xs, K, s, n, R, c, cs, out, ntr, st);
    case 2: return expand_dense_w<T, (sizeof(T) <= 4 ? 2 : 1)>(x, xs, K, s, n, R, c, cs, out, ntr, st);
    default: return expand_dense_w<T, 1>(x, xs, K, s, n, R, c, cs, out, ntr, st);
  }
}

template <class T>
cudaError_t contract_dense_t(int dtype, const void* ch, int64_t K, int64_t mb, int n, int R,
                             const void* w, int64_t ws, void* out, int64_t ntr, uint8_t* nf,
                             cudaStream_t st) {
  {
    cudaError_t e = staged_contract<T>(n, ch, K, mb, R, w, ws, out, ntr, nf, st);
    if (e != cudaErrorNotSupported) return e;
  }
  const int W = pick_width(dtype, mb, 8 / (int)sizeof(T));
  if (W >= 2 && sizeof(T) <= 4) {
    constexpr int W2 = sizeof(T) <= 4 ? 2 : 1;
    contract_dense_kernel<T, W2><<<grid_for(K * (mb * mb / W2), ntr), kThreads, 0, st>>>(
        (const T*)ch, (int)K, (int)mb, n, R, (const T*)w, ws, (T*)out, ntr, nf);
  } else {
    contract_dense_kernel<T, 1><<<grid_for(K * mb * mb, ntr), kThreads, 0, st>>>(
        (const T*)ch, (int)K, (int)mb, n, R, (const T*)w, ws, (T*)out, ntr, nf);
  }
  return cudaGetLastError();
}

}  // namespace

int pick_width(int dtype, int64_t mb, int cap_elems) {
  (void)dtype;
  int W = 1;
  for (int c = 2; c <= cap_elems; c *= 2)
    if (mb % c == 0) W = c;
  return W;
}

cudaError_t launch_expand_dense(int dtype, const void* x, int64_t x_tstride, int64_t K, int64_t s,
                                int n, int R, const void* coeff, int64_t c_tstride, void* out,
                                int64_t ntr, cudaStream_t st) {
  if (n > kMaxDenseN) return cudaErrorInvalidValue;
  switch (dtype) {
    case kF64: return expand_dense_t<double>(dtype, x, x_tstride, K, s, n, R, coeff, c_tstride, out, ntr, st);
    case kF32: return expand_dense_t<float>(dtype, x, x_tstride, K, s, n, R, coeff, c_tstride, out, ntr, st);
    case kF16: return expand_dense_t<__half>(dtype, x, x_tstride, K, s, n, R, coeff, c_tstride, out, ntr, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_contract_dense(int dtype, const void* ch, int64_t K, int64_t mb, int n, int R,
                                  const void* w, int64_t w_tstride, void* out, int64_t ntr,
                                  uint8_t* nonfinite, cudaStream_t st) {
  if (n > kMaxDenseN) return cudaErrorInvalidValue;
  switch (dtype) {
    case kF64: return contract_dense_t<double>(dtype, ch, K, mb, n, R, w, w_tstride, out, ntr, nonfinite, st);
    case kF32: return contract_dense_t<float>(dtype, ch, K, mb, n, R, w, w_tstride, out, ntr, nonfinite, st);
    case kF16: return contract_dense_t<__half>(dtype, ch, K, mb, n, R, w, w_tstride, out, ntr, nonfinite, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace rbc
