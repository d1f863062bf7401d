// DFMA throughput vs resident warps per SM and independent chains per thread
// (tuning aid for the binary64 truth kernel):  nvcc -arch=sm_100a -O3 dfma_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void dfma_chains(double* out, double b, int iters) {
  double acc[C];
#pragma unroll
  for (int i = 0; i < C; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i) acc[i] = __fma_rn(acc[i], b, 1.0 + i * 1e-7);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int C>
void run(double* buf, int sms, int warps) {
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_chains<C><<<sms, 32 * warps>>>(buf, 0.999, iters);
  cudaEventRecord(e0);
  dfma_chains<C><<<sms, 32 * warps>>>(buf, 0.999, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * C * iters * 32.0 * warps * sms;
  printf("chains %2d warps/SM %2d : %6.2f TFLOP/s\n", C, warps, flops / (ms * 1e-3) / 1e12);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* buf;
  cudaMalloc(&buf, sizeof(double) * sms * 1024);
  for (int w : {4, 8, 12, 16, 24, 32}) {
    run<8>(buf, sms, w);
    run<16>(buf, sms, w);
    run<32>(buf, sms, w);
  }
  return 0;
}
