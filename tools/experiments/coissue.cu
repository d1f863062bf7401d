// Do the FP64 pipe (DFMA: the binary64 truth) and the FMA pipe (packed
// FFMA2/FADD2: the exact-order binary32 leaf) run at their solo rates when
// warps of both kinds share an SM?  Warps with (warp % den) < num run the
// packed binary32 chains, the others the DFMA chains; each role's work is
// sized so both finish together if nothing is shared.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false tools/coissue.cu -o tools/coissue
#include <cstdint>
#include <cstdio>
typedef unsigned long long u64;
constexpr int kChains = 16;

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

__global__ void __launch_bounds__(256) mixed(u64* out, float seed, u64 negz, int num, int den,
                                             int it32, int it64) {
  const int warp = threadIdx.x >> 5;
  if ((warp % den) < num) {
    u64 acc[kChains], a[kChains];
    const float bf = 1.0f - seed * 1e-6f;
    const u64 b = ((u64)__float_as_uint(bf) << 32) | __float_as_uint(bf);
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      acc[i] = 0;
      float x = 1.0f + threadIdx.x * 1e-3f + i * 1e-4f;
      a[i] = ((u64)__float_as_uint(x) << 32) | __float_as_uint(x);
    }
    for (int it = 0; it < it32; ++it) {
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
  } else {
    double acc[kChains], a[kChains];
    const double b = seed * 1e-3;
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      acc[i] = 0.0;
      a[i] = 1.0 + threadIdx.x * 1e-3 + i * 1e-4;
    }
    for (int it = 0; it < it64; ++it) {
#pragma unroll
      for (int i = 0; i < kChains; ++i) acc[i] = __fma_rn(acc[i], b, a[i]);
    }
    double s = acc[0];
#pragma unroll
    for (int i = 1; i < kChains; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = __double_as_longlong(s);
  }
}

// same split, the non-DFMA warps run 32-bit integer multiply-add / xor chains
__global__ void __launch_bounds__(256) mixed_int(u64* out, unsigned seed, int num, int den, int iti,
                                                 int it64) {
  const int warp = threadIdx.x >> 5;
  if ((warp % den) < num) {
    unsigned a[kChains];
#pragma unroll
    for (int i = 0; i < kChains; ++i) a[i] = threadIdx.x * 2654435761u + i * 40503u + seed;
    for (int it = 0; it < iti; ++it) {
#pragma unroll
      for (int i = 0; i < kChains; ++i) {
        a[i] = a[i] * 1664525u + 1013904223u;  // IMAD
        a[i] ^= a[i] >> 7;                      // SHF + LOP3
      }
    }
    unsigned s = 0;
#pragma unroll
    for (int i = 0; i < kChains; ++i) s ^= a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    double acc[kChains], a[kChains];
    const double b = seed * 1e-3;
#pragma unroll
    for (int i = 0; i < kChains; ++i) {
      acc[i] = 0.0;
      a[i] = 1.0 + threadIdx.x * 1e-3 + i * 1e-4;
    }
    for (int it = 0; it < it64; ++it) {
#pragma unroll
      for (int i = 0; i < kChains; ++i) acc[i] = __fma_rn(acc[i], b, a[i]);
    }
    double s = acc[0];
#pragma unroll
    for (int i = 1; i < kChains; ++i) s += acc[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = __double_as_longlong(s);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 8, threads = 256;
  void* buf;
  cudaMalloc(&buf, (size_t)blocks * threads * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // rows: (num, den, it32, it64)
  const int cfg[][4] = {{1, 1, 8192, 0},    {0, 1, 0, 8192},    {1, 2, 8192, 8192},
                        {1, 2, 16384, 8192}, {1, 2, 8192, 4096}, {1, 2, 8192, 16384},
                        {1, 2, 8192, 0},    {1, 2, 0, 8192}};
  printf("[");
  for (int c = 0; c < 8; ++c) {
    const int num = cfg[c][0], den = cfg[c][1], it32 = cfg[c][2], it64 = cfg[c][3];
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      mixed<<<blocks, threads>>>((u64*)buf, 1.f, 0x8000000080000000ull, num, den, it32, it64);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    const double w32 = (double)blocks * threads * num / den, w64 = (double)blocks * threads * (den - num) / den;
    const double t32 = w32 * it32 * kChains * 4.0 / (best * 1e-3) / 1e12;
    const double t64 = w64 * it64 * kChains * 2.0 / (best * 1e-3) / 1e12;
    printf("%s{\"f32_warps\": \"%d/%d\", \"it32\": %d, \"it64\": %d, \"ms\": %.3f, \"f32x2_tflops\": %.2f, "
           "\"dfma_tflops\": %.2f}",
           c ? ",\n " : "", num, den, it32, it64, best, t32, t64);
  }
  printf("]\n");
  // DFMA beside integer chains: ms alone and mixed
  const int icfg[][4] = {{1, 2, 8192, 0}, {1, 2, 0, 8192}, {1, 2, 8192, 8192}, {1, 2, 16384, 8192},
                         {1, 2, 4096, 8192}};
  printf("[");
  for (int c = 0; c < 5; ++c) {
    const int num = icfg[c][0], den = icfg[c][1], iti = icfg[c][2], it64 = icfg[c][3];
    float best = 1e30f;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0);
      mixed_int<<<blocks, threads>>>((u64*)buf, 1u, num, den, iti, it64);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best) best = ms;
    }
    printf("%s{\"int_warps\": \"%d/%d\", \"it_int\": %d, \"it64\": %d, \"ms\": %.3f}", c ? ",\n " : "",
           num, den, iti, it64, best);
  }
  printf("]\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
