// Experiment: 27x27 binary64 leaves (config 3), one warp per leaf, 9x3
// outputs per lane, leaves streamed through a CTA-wide ring of bulk-copy
// slots with full/empty mbarriers (no CTA barrier in the steady state).
//
//   nvcc -O3 -fmad=false -lineinfo -gencode arch=compute_100a,code=sm_100a \
//        -o tools/experiments/leaf27_warp tools/experiments/leaf27_warp.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../../paper_1905_07439_b200/csrc/bulk.cuh"

using namespace rbc;

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

constexpr int M = 27, E = M * M;
constexpr int SPAN = ((E * 8 + 16) + 15) / 16 * 16;  // 5856: enclosing 16-byte span

__global__ void ref_kernel(int64_t batch, const double* x, const double* y, double* out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= batch * E) return;
  const int64_t b = e / E;
  const int q = (int)(e - b * E), i = q / M, j = q % M;
  const double* X = x + b * E;
  const double* Y = y + b * E;
  double acc = __dmul_rn(X[i * M], Y[j]);
  for (int k = 1; k < M; ++k) acc = __dadd_rn(acc, __dmul_rn(X[i * M + k], Y[k * M + j]));
  out[e] = acc;
}

__global__ void cmp_kernel(int64_t n, const uint64_t* a, const uint64_t* b, unsigned long long* bad) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < n && a[e] != b[e]) {
    unsigned long long k = atomicAdd(bad, 1ull);
    if (k < 12) printf("  mismatch at leaf %lld row %d col %d\n", (long long)(e / E), (int)(e % E) / M, (int)(e % E) % M);
  }
}

// TM x TN outputs per lane; lanes (it, jt): rows TM*it .. TM*it+TM-1, columns
// jt + (M/TN)*j (strided, so a warp's stores of one register are contiguous
// runs).  TPL = (M/TM)*(M/TN) lanes per leaf must be <= 32.
template <int NW, int NSLOT, int TM, int TN, int UNR, int REL = 0>
__global__ void __launch_bounds__((NW + 1) * 32, 1)
    leaf27_warp_kernel(int64_t batch, const double* __restrict__ x, const double* __restrict__ y,
                       double* __restrict__ out) {
  constexpr int CJ = M / TN;  // column stride / lanes along N
  constexpr int TPL = (M / TM) * CJ;
  static_assert(TPL <= 32, "one warp per leaf");
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NSLOT * 2 * SPAN);
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
  const int64_t per = (batch + gridDim.x - 1) / gridDim.x;
  const int64_t lo = (int64_t)blockIdx.x * per;
  const int64_t hi = lo + per < batch ? lo + per : batch;
  const int n = hi > lo ? (int)(hi - lo) : 0;
  if (warp == NW) {
    if (lane == 0) {
      for (int i = 0; i < n; ++i) {
        const int s = i % NSLOT, r = i / NSLOT;
        if (r > 0) mbar_wait(&empty[s], (unsigned)((r - 1) & 1));
        const double* gx = x + (lo + i) * E;
        const double* gy = y + (lo + i) * E;
        const unsigned bx = span_bytes(gx, E * 8), by = span_bytes(gy, E * 8);
        mbar_expect_tx(&full[s], bx + by);
        unsigned char* slot = smem + (size_t)s * 2 * SPAN;
        bulk_g2s(slot, span_start(gx), bx, &full[s]);
        bulk_g2s(slot + SPAN, span_start(gy), by, &full[s]);
      }
    }
    return;
  }
  const int r = lane < TPL ? lane : 0;
  const int it = r / CJ, jt = r % CJ;
  for (int i = warp; i < n; i += NW) {
    const int s = i % NSLOT;
    mbar_wait(&full[s], (unsigned)((i / NSLOT) & 1));
    const double* gx = x + (lo + i) * E;
    const double* gy = y + (lo + i) * E;
    unsigned char* slot = smem + (size_t)s * 2 * SPAN;
    const double* Xr = reinterpret_cast<const double*>(slot + (reinterpret_cast<uintptr_t>(gx) & 15)) + TM * it * M;
    const double* Yc = reinterpret_cast<const double*>(slot + SPAN + (reinterpret_cast<uintptr_t>(gy) & 15)) + jt;
    double acc[TM][TN], a[2][TM], b[2][TN];
#pragma unroll
    for (int ii = 0; ii < TM; ++ii) a[0][ii] = Xr[ii * M];
#pragma unroll
    for (int j = 0; j < TN; ++j) b[0][j] = Yc[CJ * j];
#pragma unroll
    for (int ii = 0; ii < TM; ++ii) a[1][ii] = Xr[ii * M + 1];
#pragma unroll
    for (int j = 0; j < TN; ++j) b[1][j] = Yc[M + CJ * j];
#pragma unroll
    for (int ii = 0; ii < TM; ++ii)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[ii][j] = __dmul_rn(a[0][ii], b[0][j]);
    // steps 1 .. 26: operands of step k + 1 load while step k multiplies
#pragma unroll(UNR)
    for (int k = 1; k < M; k += 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kk = k + h;           // current step, operands in slot (kk & 1)
        const int c = (1 + h) & 1, nx = c ^ 1;
        if (kk + 1 < M) {
#pragma unroll
          for (int ii = 0; ii < TM; ++ii) a[nx][ii] = Xr[ii * M + kk + 1];
#pragma unroll
          for (int j = 0; j < TN; ++j) b[nx][j] = Yc[(kk + 1) * M + CJ * j];
        }
#pragma unroll
        for (int ii = 0; ii < TM; ++ii)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[ii][j] = __dadd_rn(acc[ii][j], __dmul_rn(a[c][ii], b[c][j]));
      }
    }
    // Release the slot before the stores, but not before every shared-memory
    // load of this leaf has returned: the arrive is predicated on a word
    // folded from all accumulators, so it cannot issue until they are
    // complete.  (Placed right after the last LDS issue, the refill overtook
    // loads still in flight: about one wrong row per 10^5 leaves.  Placed
    // after the stores, its release semantics wait for them: 3x slower.)
    if constexpr (REL == 0) {  // predicate folded from all accumulators
      unsigned dep = 0;
#pragma unroll
      for (int ii = 0; ii < TM; ++ii)
#pragma unroll
        for (int j = 0; j < TN; ++j) dep |= (unsigned)__double2hiint(acc[ii][j]);
      __syncwarp();
      if (lane == 0 && dep != 0x7ff00001u) mbar_arrive(&empty[s]);
    } else if constexpr (REL == 1) {  // cross-proxy fence, then arrive
      fence_proxy_async();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    } else if constexpr (REL == 2) {  // predicate folded from the last step's operands
      unsigned dep = 0;
#pragma unroll
      for (int ii = 0; ii < TM; ++ii) dep |= (unsigned)__double2hiint(a[0][ii]);
#pragma unroll
      for (int j = 0; j < TN; ++j) dep |= (unsigned)__double2hiint(b[0][j]);
      __syncwarp();
      if (lane == 0 && dep != 0x7ff00001u) mbar_arrive(&empty[s]);
    } else {  // the racy original
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (lane < TPL) {
      double* o = out + (lo + i) * E + TM * it * M + jt;
#pragma unroll
      for (int ii = 0; ii < TM; ++ii)
#pragma unroll
        for (int j = 0; j < TN; ++j) o[ii * M + CJ * j] = acc[ii][j];
    }
  }
}

template <int NW, int NSLOT, int TM, int TN, int UNR, int REL = 0>
float run(const char* name, int64_t batch, const double* x, const double* y, double* out,
          const double* ref, unsigned long long* bad) {
  auto kern = leaf27_warp_kernel<NW, NSLOT, TM, TN, UNR, REL>;
  const size_t smem = (size_t)NSLOT * 2 * SPAN + 2 * NSLOT * sizeof(uint64_t);
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  CK(cudaMemset(out, 0xff, batch * E * 8));
  kern<<<sms, (NW + 1) * 32, smem>>>(batch, x, y, out);
  CK(cudaDeviceSynchronize());
  CK(cudaMemset(bad, 0, 8));
  cmp_kernel<<<(unsigned)((batch * E + 255) / 256), 256>>>(batch * E, (const uint64_t*)out,
                                                          (const uint64_t*)ref, bad);
  unsigned long long hb = 0;
  CK(cudaMemcpy(&hb, bad, 8, cudaMemcpyDeviceToHost));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) kern<<<sms, (NW + 1) * 32, smem>>>(batch, x, y, out);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  printf("%-24s rel=%d NW=%2d NSLOT=%2d %dx%d unr=%2d  %8.3f ms  %6.2f TFLOP/s  %5.2f TB/s  mismatches=%llu\n",
         name, REL, NW, NSLOT, TM, TN, UNR, ms, 2.0 * batch * M * M * M / (ms * 1e-3) / 1e12,
         3.0 * batch * E * 8 / (ms * 1e-3) / 1e12, hb);
  fflush(stdout);
  return ms;
}

int main(int argc, char** argv) {
  const int64_t batch = argc > 1 ? atoll(argv[1]) : 12167LL * 16;
  double *x, *y, *out, *ref;
  unsigned long long* bad;
  const size_t bytes = (size_t)batch * E * 8;
  CK(cudaMalloc(&x, bytes + 16));
  CK(cudaMalloc(&y, bytes + 16));
  CK(cudaMalloc(&out, bytes));
  CK(cudaMalloc(&ref, bytes));
  CK(cudaMalloc(&bad, 8));
  double* h = (double*)malloc(bytes);
  uint64_t sd = 88172645463325252ull;
  for (int pass = 0; pass < 2; ++pass) {
    for (size_t i = 0; i < (size_t)batch * E; ++i) {
      sd ^= sd << 13; sd ^= sd >> 7; sd ^= sd << 17;
      h[i] = ((double)(sd >> 11) * (1.0 / 9007199254740992.0) - 0.5) * 4.0;
    }
    CK(cudaMemcpy(pass ? y : x, h, bytes, cudaMemcpyHostToDevice));
  }
  free(h);
  ref_kernel<<<(unsigned)((batch * E + 255) / 256), 256>>>(batch, x, y, ref);
  CK(cudaDeviceSynchronize());
  for (int rep = 0; rep < 4; ++rep) run<12, 16, 3, 9, 26, 3>("warp 3x9 racy", batch, x, y, out, ref, bad);
  for (int rep = 0; rep < 6; ++rep) run<12, 16, 3, 9, 26, 1>("warp 3x9 fence", batch, x, y, out, ref, bad);
  for (int rep = 0; rep < 6; ++rep) run<12, 16, 3, 9, 26, 2>("warp 3x9 opdep", batch, x, y, out, ref, bad);
  for (int rep = 0; rep < 3; ++rep) run<12, 16, 9, 3, 26, 0>("warp 9x3 accdep", batch, x, y, out, ref, bad);
  for (int rep = 0; rep < 3; ++rep) run<12, 16, 9, 3, 26, 1>("warp 9x3 fence", batch, x, y, out, ref, bad);
  for (int rep = 0; rep < 3; ++rep) run<12, 16, 9, 3, 26, 2>("warp 9x3 opdep", batch, x, y, out, ref, bad);
  run<10, 16, 9, 3, 26, 0>("warp 9x3 accdep", batch, x, y, out, ref, bad);
  run<14, 18, 9, 3, 26, 0>("warp 9x3 accdep", batch, x, y, out, ref, bad);
  return 0;
}
