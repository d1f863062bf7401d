// Microbenchmark of the exact-order multiply-add rate on the CUDA cores.
//
// The leaf products must round every multiply and every add separately
// (SURVEY §0.4), so their compute roofline is the FMUL+FADD (DMUL+DADD,
// HMUL2+HADD2) pair rate, not the FFMA rate.  Each thread runs 16
// independent chains a_i = mul(a_i, b); acc_i = add(acc_i, a_i): one
// separately rounded multiply and add per step, as in the leaf kernel.  flops = 2 per multiply-add (4 per half2 pair).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/fp_peak.cu -o tools/fp_peak
//   ./tools/fp_peak > profiles/fp_peaks.json
#include <cuda_fp16.h>
#include <cstdint>
#include <cstdio>

constexpr int kChains = 16;
constexpr int kIters = 8192;

template <class T> struct Ops;
template <> struct Ops<float> {
  static __device__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ float from(float x) { return x; }
  static constexpr double flops_per_op = 2.0;
};
template <> struct Ops<double> {
  static __device__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ double from(float x) { return x; }
  static constexpr double flops_per_op = 2.0;
};
template <> struct Ops<__half2> {
  // inline PTX so the chain is issued exactly as written (one HMUL2 and one
  // HADD2 per step)
  static __device__ __half2 mul(__half2 a, __half2 b) {
    uint32_t r, x = *reinterpret_cast<uint32_t*>(&a), y = *reinterpret_cast<uint32_t*>(&b);
    asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
    return *reinterpret_cast<__half2*>(&r);
  }
  static __device__ __half2 add(__half2 a, __half2 b) {
    uint32_t r, x = *reinterpret_cast<uint32_t*>(&a), y = *reinterpret_cast<uint32_t*>(&b);
    asm("add.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(y));
    return *reinterpret_cast<__half2*>(&r);
  }
  static __device__ __half2 from(float x) { return __float2half2_rn(x); }
  static constexpr double flops_per_op = 4.0;
};

template <class T>
__global__ void __launch_bounds__(256) mac_kernel(T* out, float seed) {
  using O = Ops<T>;
  T acc[kChains], a[kChains];
  const T b = O::from(1.0f - seed * 1e-6f);
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    acc[i] = O::from(0.0f);
    a[i] = O::from(1.0f + threadIdx.x * 1e-3f + i * 1e-4f);
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      a[i] = O::mul(a[i], b);
      acc[i] = O::add(acc[i], a[i]);
    }
  }
  T s = acc[0];
#pragma unroll
  for (int i = 1; i < kChains; ++i) s = O::add(s, acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) ffma_kernel(float* out, float seed) {
  float acc[kChains], a[kChains];
  const float b = seed * 1e-3f;
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    acc[i] = 0.f;
    a[i] = 1.0f + threadIdx.x * 1e-3f + i * 1e-4f;
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) acc[i] = __fmaf_rn(acc[i], b, a[i]);
  }
  float s = acc[0];
#pragma unroll
  for (int i = 1; i < kChains; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) dfma_kernel(double* out, float seed) {
  double acc[kChains], a[kChains];
  const double b = seed * 1e-3;
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    acc[i] = 0.0;
    a[i] = 1.0 + threadIdx.x * 1e-3 + i * 1e-4;
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) acc[i] = __fma_rn(acc[i], b, a[i]);
  }
  double s = acc[0];
#pragma unroll
  for (int i = 1; i < kChains; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Packed binary32 pairs (sm_100a FMUL2/FADD2 family).  ptxas contracts
// mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even with -fmad=false, so the
// multiply is issued as FFMA2 with an addend of (-0, -0) the compiler cannot
// see (a kernel argument): fl(a*b + -0) == fl(a*b) for every a, b (a +0
// product stays +0, a -0 product stays -0).  One FFMA2 + one FADD2 per two
// separately rounded multiply-adds.
typedef unsigned long long u64;
__device__ __forceinline__ u64 f2_mul(u64 a, u64 b, u64 negz) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(negz));
  return r;
}
__device__ __forceinline__ u64 f2_add(u64 a, u64 b) {
  u64 r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__global__ void __launch_bounds__(256) mac2_kernel(u64* out, float seed, u64 negz) {
  u64 acc[kChains], a[kChains];
  const float bf = 1.0f - seed * 1e-6f;
  const u64 b = ((u64)__float_as_uint(bf) << 32) | __float_as_uint(bf);
#pragma unroll
  for (int i = 0; i < kChains; ++i) {
    acc[i] = 0;
    float x = 1.0f + threadIdx.x * 1e-3f + i * 1e-4f;
    a[i] = ((u64)__float_as_uint(x) << 32) | __float_as_uint(x);
  }
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      a[i] = f2_mul(a[i], b, negz);
      acc[i] = f2_add(acc[i], a[i]);
    }
  }
  u64 s = acc[0];
#pragma unroll
  for (int i = 1; i < kChains; ++i) s = f2_add(s, acc[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <class K>
double time_kernel(K launch, int reps) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  const double ops = (double)blocks * threads * kIters * kChains;
  void* buf;
  cudaMalloc(&buf, (size_t)blocks * threads * 8);
  double f32 = time_kernel([&] { mac_kernel<float><<<blocks, threads>>>((float*)buf, 1.f); }, 5);
  double f64 = time_kernel([&] { mac_kernel<double><<<blocks, threads>>>((double*)buf, 1.f); }, 5);
  double f16 = time_kernel([&] { mac_kernel<__half2><<<blocks, threads>>>((__half2*)buf, 1.f); }, 5);
  double fma = time_kernel([&] { ffma_kernel<<<blocks, threads>>>((float*)buf, 1.f); }, 5);
  double dfma = time_kernel([&] { dfma_kernel<<<blocks, threads>>>((double*)buf, 1.f); }, 5);
  double f32x2 = time_kernel(
      [&] { mac2_kernel<<<blocks, threads>>>((u64*)buf, 1.f, 0x8000000080000000ull); }, 5);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e));
    return 1;
  }
  printf("{\"f32_tflops\": %.3f, \"f64_tflops\": %.3f, \"f16_tflops\": %.3f, "
         "\"ffma_f32_tflops\": %.3f, \"dfma_f64_tflops\": %.3f, \"f32x2_tflops\": %.3f, \"sms\": %d, "
         "\"how\": \"tools/fp_peak.cu: %d x 256 threads, 16 independent acc=add(acc,mul(a,b)) chains "
         "with separately rounded multiply and add (half2 counts 4 flops), best of 5, CUDA events\"}\n",
         ops * Ops<float>::flops_per_op / (f32 * 1e-3) / 1e12,
         ops * Ops<double>::flops_per_op / (f64 * 1e-3) / 1e12,
         ops * Ops<__half2>::flops_per_op / (f16 * 1e-3) / 1e12, ops * 2.0 / (fma * 1e-3) / 1e12,
         ops * 2.0 / (dfma * 1e-3) / 1e12, ops * 4.0 / (f32x2 * 1e-3) / 1e12, sms, blocks);
  return 0;
}
