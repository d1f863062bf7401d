// On-device seeded test matrices, bit-identical to the reference's host
// generators:
//
//   derive_rng(seed, *path) = Generator(Philox(SeedSequence(seed, spawn_key=path)))
//                                              (pkg/src/randbc/rng.py:20-23)
//   matgen.generate: A <- derive_rng(mseed, 0), B <- derive_rng(mseed, 1)
//                                              (pkg/src/randbc/matgen.py:55-97)
//
// The random streams are numpy's (pinned by numpy>=1.24, pkg/pyproject.toml:12;
// numpy 2.3 here).  The SeedSequence hashing runs on the host (numpy itself);
// the device reproduces, from the resulting 128-bit Philox key:
//
// * the raw stream: Philox4x64-10 (Salmon et al., SC'11), word i of the
//   stream = lane i % 4 of the block with counter (i / 4 + 1, 0, 0, 0) --
//   numpy advances the counter before its first block;
// * Generator.random(): (word >> 11) * 2^-53, one word per sample;
// * Generator.standard_normal(): the 256-strip Marsaglia-Tsang ziggurat in
//   numpy's formulation (random_standard_normal, 52-bit magnitude, sign bit
//   8, strip index in the low byte; wedge test against exp(-x^2/2); tail by
//   Marsaglia's exponential method) with numpy's own tables, read from the
//   installed numpy at build time (build.py: build/gen/ziggurat_tables.inc).
//
// A normal sample consumes a variable number of words (1 on the fast path,
// 2 per wedge attempt, 1 + 2m in the tail), so the stream is parsed in
// parallel: chunks of kChunk words are parsed from every possible entry
// offset (a map entry -> exit, count), the maps resolve each chunk's true
// entry (parses from different entries merge within a few words, so nearly
// every map is constant and a chunk's entry depends on its predecessor only),
// a scan of the counts gives output offsets, and the chunks are re-parsed
// writing their samples.  Tail samples (idx 0 past the base rectangle, about
// 2.5e-4 of the words) are evaluated on the host with the C library's log1p
// -- the very function numpy calls -- so their values and word counts are
// exact; the wedge test uses the device exp (< 1 ulp from glibc's; a
// decision could differ only if the uniform fell within that ulp, p < 1e-15
// per test).
//
// Memory shape of the parse (round 2: config 5's four 8192^2 matrices in 18.2
// instead of 59.7 ms).  One thread parses one chunk, so the raw
// words are stored chunk-interleaved: word p of chunk j lives at
// ((j / 32) * 64 + p) * 32 + j % 32, and the 32 lanes of a warp -- 32
// consecutive chunks, all near the same p -- read one 256-byte row per step
// instead of 32 separate lines.  The ziggurat tables sit in shared memory (a
// constant-memory lookup by a per-lane strip index serialises over the lanes),
// and the emitting kernel stages each CTA's samples in shared memory and
// writes its contiguous output range coalesced.
//
// Post-processing follows matgen.generate per family, in binary64, then one
// rounding into the mode (ScalarMode.array, precision.py:131-158): non-finite
// results set the matrix's flag (the host raises OverflowError).

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "kernels.h"
#include "ziggurat_tables.inc"

namespace rbc {

namespace {

__constant__ uint64_t c_ki[256] = RBC_ZIG_KI;
__constant__ double c_wi[256] = RBC_ZIG_WI;
__constant__ double c_fi[256] = RBC_ZIG_FI;

constexpr double kZigR = 3.6541528853610088;       // ziggurat_nor_r
constexpr double kZigInvR = 0.27366123732975828;   // ziggurat_nor_inv_r
constexpr uint64_t kMask52 = 0x000fffffffffffffull;
constexpr double kTwoM53 = 1.0 / 9007199254740992.0;
constexpr int kChunk = 64;     // words per parsed chunk
constexpr int kEntries = 8;    // entry offsets tabulated per chunk
constexpr int kTailWords = 64; // words fetched per tail candidate
constexpr int kScanThreads = 256;
constexpr int kGroup = 32;                       // chunks interleaved together (one warp)
constexpr int64_t kGroupWords = kGroup * kChunk;  // 2048: per-matrix word counts are multiples

// storage index of logical stream word i (chunk-interleaved, see above)
__device__ __forceinline__ int64_t wat(int64_t i) {
  const int64_t j = i >> 6;
  return ((j >> 5) << 11) | ((i & 63) << 5) | (j & 31);
}
// logical stream position of storage index q
__device__ __forceinline__ int64_t wlogical(int64_t q) {
  return ((((q >> 11) << 5) | (q & 31)) << 6) | ((q >> 5) & 63);
}

// ziggurat tables in shared memory (filled by zig_load at kernel start)
struct ZigTabs {
  const uint64_t* ki;
  const double* wi;
  const double* fi;
};
__device__ __forceinline__ ZigTabs zig_load(uint64_t* ski, double* swi, double* sfi) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    ski[i] = c_ki[i];
    swi[i] = c_wi[i];
    sfi[i] = c_fi[i];
  }
  __syncthreads();
  return ZigTabs{ski, swi, sfi};
}

__device__ __forceinline__ void philox4x64_10(uint64_t c[4], uint64_t k0, uint64_t k1) {
  constexpr uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  constexpr uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t lo0 = M0 * c[0], hi0 = __umul64hi(M0, c[0]);
    const uint64_t lo1 = M1 * c[2], hi1 = __umul64hi(M1, c[2]);
    const uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += W0;
    k1 += W1;
  }
}

__device__ __forceinline__ double unit_double(uint64_t w) {
  return __dmul_rn((double)(w >> 11), kTwoM53);
}

// ---- family post-processing (matgen.generate) + rounding into the mode ----
struct Post {
  int kind;   // MatgenKind
  int n;
  double tiny, huge, half;  // 1/(n*n), n*n, n/2
};

__device__ __forceinline__ double post_value(const Post& p, int which, int64_t e, double v) {
  const int row = (int)(e / p.n), col = (int)(e - (int64_t)row * p.n);
  const double i = row + 1.0, j = col + 1.0;  // 1-based index grids
  switch (p.kind) {
    case kMatUniformPm1:
      return __dsub_rn(__dmul_rn(2.0, v), 1.0);
    case kMatQuadrant100: {
      const int h = p.n / 2;
      const bool hit = which == 0 ? (row < h && col < h) : (row >= h && col >= h);
      return hit ? __dmul_rn(v, 100.0) : v;
    }
    case kMatAdv1: {
      const double s = which == 0 ? (j > p.half ? p.tiny : 1.0) : (i < p.half ? p.tiny : 1.0);
      return __dmul_rn(v, s);
    }
    case kMatAdv2: {
      const double s = which == 0 ? ((i < p.half && j > p.half) ? p.huge : 1.0)
                                  : (j < p.half ? p.tiny : 1.0);
      return __dmul_rn(v, s);
    }
    case kMatAdv3: {
      const bool band = (i < p.half && j > p.half) || (i >= p.half && j <= p.half);
      return __dmul_rn(v, band ? p.tiny : 1.0);
    }
    case kMatHilbert:
      return __ddiv_rn(1.0, __dsub_rn(__dadd_rn(i, j), 1.0));
    default:
      return v;
  }
}

template <class T>
__device__ __forceinline__ T round_into(double v);
template <> __device__ __forceinline__ double round_into<double>(double v) { return v; }
template <> __device__ __forceinline__ float round_into<float>(double v) { return __double2float_rn(v); }
template <> __device__ __forceinline__ __half round_into<__half>(double v) { return __double2half(v); }

template <class T>
__device__ __forceinline__ bool finite_of(T v) {
  return isfinite(static_cast<double>(v));
}
template <> __device__ __forceinline__ bool finite_of<__half>(__half v) {
  return isfinite(__half2float(v));
}

template <class T>
__device__ __forceinline__ void store_sample(T* out, uint8_t* flags, int m, int which,
                                             const Post& p, int64_t e, double v) {
  const T r = round_into<T>(post_value(p, which, e, v));
  out[e] = r;
  if (flags && !finite_of(r)) flags[m] = 1;
}

// ---- uniform families and Hilbert: one word per sample ---------------------
template <class T>
__global__ void __launch_bounds__(256) uniform_kernel(int64_t S, const uint64_t* __restrict__ keys,
                                                      const int* __restrict__ which, Post p,
                                                      T* __restrict__ out,
                                                      uint8_t* __restrict__ flags) {
  const int m = blockIdx.y;
  const uint64_t k0 = keys[2 * m], k1 = keys[2 * m + 1];
  T* o = out + (int64_t)m * S;
  const int w = which[m];
  for (int64_t blk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; blk * 4 < S;
       blk += (int64_t)gridDim.x * blockDim.x) {
    uint64_t c[4] = {(uint64_t)blk + 1, 0, 0, 0};
    if (p.kind != kMatHilbert) philox4x64_10(c, k0, k1);
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      const int64_t e = blk * 4 + l;
      if (e < S) store_sample<T>(o, flags, m, w, p, e, unit_double(c[l]));
    }
  }
}

// ---- standard normal ---------------------------------------------------------
__global__ void __launch_bounds__(256) fill_words_kernel(int64_t Wn, const uint64_t* __restrict__ keys,
                                                         uint64_t* __restrict__ W) {
  const int m = blockIdx.y;
  const uint64_t k0 = keys[2 * m], k1 = keys[2 * m + 1];
  uint64_t* o = W + (int64_t)m * Wn;
  // thread t -> (group g, block-in-chunk b4, lane l): Philox block (g*32+l)*16 + b4,
  // i.e. words 4*b4 .. 4*b4+3 of chunk g*32+l; a warp writes four 256-byte rows
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t * 4 < Wn;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = t >> 9;
    const int b4 = (int)((t >> 5) & 15), l = (int)(t & 31);
    const int64_t blk = ((g << 5) + l) * 16 + b4;
    uint64_t c[4] = {(uint64_t)blk + 1, 0, 0, 0};
    philox4x64_10(c, k0, k1);
    uint64_t* d = o + (g << 11) + ((int64_t)(4 * b4) << 5) + l;
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q << 5] = c[q];
  }
}

// positions of tail candidates (strip 0, outside the base rectangle); the
// words are scanned in storage order, the list holds logical positions
__global__ void __launch_bounds__(256) tail_candidates_kernel(int64_t Wn, int64_t Wparse,
                                                              const uint64_t* __restrict__ W,
                                                              int64_t* __restrict__ list,
                                                              unsigned long long* __restrict__ count,
                                                              int64_t cap) {
  const int m = blockIdx.y;
  const uint64_t* w = W + (int64_t)m * Wn;
  const uint64_t ki0 = c_ki[0];
  const int64_t Wscan = (Wparse + kGroupWords - 1) / kGroupWords * kGroupWords;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Wscan;
       q += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = w[q];
    if ((v & 0xff) == 0 && ((v >> 9) & kMask52) >= ki0) {
      const int64_t p = wlogical(q);
      if (p < Wparse) {
        const unsigned long long slot = atomicAdd(count, 1ull);
        if ((int64_t)slot < cap) list[slot] = (int64_t)m * Wn + p;
      }
    }
  }
}

// words p .. p+kTailWords-1 of every candidate: the r word (its bit 17 signs
// the tail sample) and the uniforms of the host tail loop
__global__ void __launch_bounds__(kTailWords) gather_tail_words_kernel(
    int64_t Wn, const uint64_t* __restrict__ W, const int64_t* __restrict__ list,
    uint64_t* __restrict__ words) {
  const int64_t c = blockIdx.x;
  const int64_t m = list[c] / Wn, p = list[c] - m * Wn;
  words[c * kTailWords + threadIdx.x] = W[m * Wn + wat(p + threadIdx.x)];
}

struct TailTab {
  const int64_t* pos;   // sorted global word positions m * Wn + p
  const int* used;      // words consumed by the sample starting there
  const double* value;  // its value
  int64_t count;
};

__device__ __forceinline__ int64_t tail_find(const TailTab& t, int64_t key) {
  int64_t lo = 0, hi = t.count - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (t.pos[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Parse one chunk's words [p, end) (p = the next r-read position, possibly
// past end).  Calls emit(k, x) for the k-th sample; returns the position of
// the next r-read (>= end).
template <class Emit>
__device__ __forceinline__ int64_t parse_words(const uint64_t* __restrict__ w, int64_t base,
                                               int64_t p, int64_t end, const TailTab& tt,
                                               const ZigTabs& z, int& cnt, Emit emit) {
  while (p < end) {
    const uint64_t r = w[wat(p)];
    const int idx = (int)(r & 0xff);
    const uint64_t rabs = (r >> 9) & kMask52;
    double x = __dmul_rn((double)rabs, z.wi[idx]);
    if ((r >> 8) & 1) x = -x;
    if (rabs < z.ki[idx]) {
      emit(cnt++, x);
      p += 1;
    } else if (idx == 0) {
      const int64_t t = tail_find(tt, base + p);
      emit(cnt++, tt.value[t]);
      p += tt.used[t];
    } else {
      const double u = unit_double(w[wat(p + 1)]);
      const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(z.fi[idx - 1], z.fi[idx]), u), z.fi[idx]);
      const double rhs = exp(__dmul_rn(__dmul_rn(-0.5, x), x));
      p += 2;
      if (lhs < rhs) emit(cnt++, x);
    }
  }
  return p;
}

struct NoEmit {
  __device__ void operator()(int, double) const {}
};

// per chunk: exit offset and sample count from each entry offset.  Entry 0
// is parsed in full, recording which chunk positions it reads an r word at
// (rmask) and which of those emitted a sample (emask); a parse from entry e
// stops as soon as it reads an r word at one of those positions -- from there
// on it is entry 0's parse -- so nearly every extra entry costs a step or two.
static_assert(kChunk == 64, "position masks are 64-bit");
__global__ void __launch_bounds__(256) chunk_maps_kernel(int64_t Wn, int64_t J,
                                                         const uint64_t* __restrict__ W, TailTab tt,
                                                         int* __restrict__ exits,
                                                         int* __restrict__ cnts) {
  __shared__ uint64_t ski[256];
  __shared__ double swi[256], sfi[256];
  const ZigTabs z = zig_load(ski, swi, sfi);
  const int m = blockIdx.y;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  const uint64_t* w = W + (int64_t)m * Wn;
  const int64_t base = (int64_t)m * Wn;
  const int64_t c0 = j * kChunk, end = c0 + kChunk;
  const int64_t o = ((int64_t)m * J + j) * kEntries;
  uint64_t rmask = 0, emask = 0;
  int cnt0 = 0;
  int64_t p = c0;
  // entry 0, recording its r-read positions
  while (p < end) {
    const int at = (int)(p - c0);
    rmask |= 1ull << at;
    int one = 0;
    const int64_t q = parse_words(w, base, p, p + 1, tt, z, one, NoEmit{});
    if (one) emask |= 1ull << at;
    cnt0 += one;
    p = q;
  }
  const int exit0 = (int)(p - end);
  exits[o] = exit0;
  cnts[o] = cnt0;
  for (int e = 1; e < kEntries; ++e) {
    int cnt = 0;
    int64_t q = c0 + e;
    bool merged = false;
    while (q < end) {
      const int at = (int)(q - c0);
      if ((rmask >> at) & 1) {
        cnt += __popcll(emask >> at);
        merged = true;
        break;
      }
      q = parse_words(w, base, q, q + 1, tt, z, cnt, NoEmit{});
    }
    exits[o + e] = merged ? exit0 : (int)(q - end);
    cnts[o + e] = cnt;
  }
}

__device__ __forceinline__ bool map_constant(const int* ex) {
#pragma unroll
  for (int e = 1; e < kEntries; ++e)
    if (ex[e] != ex[0]) return false;
  return true;
}

// Entry of chunk j: walk back to the nearest chunk with a constant map (its
// exit does not depend on its entry), then forward through the maps.
// Entries >= kEntries (a long tail spilling over) are parsed directly.
__device__ int chunk_entry(const uint64_t* __restrict__ w, int64_t base, int64_t j,
                           const int* __restrict__ exits, const TailTab& tt, const ZigTabs& z) {
  int64_t i = j - 1;
  while (i >= 0 && !map_constant(exits + i * kEntries)) --i;
  int entry = i >= 0 ? exits[i * kEntries] : 0;
  for (int64_t k = i + 1; k < j; ++k) {
    if (entry < kEntries) {
      entry = exits[k * kEntries + entry];
    } else {
      int cnt = 0;
      const int64_t end = (k + 1) * kChunk;
      entry = (int)(parse_words(w, base, k * kChunk + entry, end, tt, z, cnt, NoEmit{}) - end);
    }
  }
  return entry;
}

// per chunk: resolved entry and count; per block of kScanThreads chunks: sum
__global__ void __launch_bounds__(kScanThreads) chunk_entries_kernel(
    int64_t Wn, int64_t J, const uint64_t* __restrict__ W, TailTab tt,
    const int* __restrict__ exits, const int* __restrict__ cnts, int* __restrict__ entry_out,
    int* __restrict__ cnt_out, long long* __restrict__ bsum) {
  __shared__ uint64_t ski[256];
  __shared__ double swi[256], sfi[256];
  const ZigTabs z = zig_load(ski, swi, sfi);
  const int m = blockIdx.y;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t* w = W + (int64_t)m * Wn;
  const int* ex = exits + (int64_t)m * J * kEntries;
  const int* ct = cnts + (int64_t)m * J * kEntries;
  int cnt = 0;
  if (j < J) {
    const int entry = chunk_entry(w, (int64_t)m * Wn, j, ex, tt, z);
    if (entry < kEntries) {
      cnt = ct[j * kEntries + entry];
    } else {
      parse_words(w, (int64_t)m * Wn, j * kChunk + entry, (j + 1) * kChunk, tt, z, cnt, NoEmit{});
    }
    entry_out[(int64_t)m * J + j] = entry;
    cnt_out[(int64_t)m * J + j] = cnt;
  }
  __shared__ long long red[kScanThreads];
  red[threadIdx.x] = cnt;
  __syncthreads();
  for (int s = kScanThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) bsum[(int64_t)m * gridDim.x + blockIdx.x] = red[0];
}

// exclusive scan of the block sums of one matrix (one CTA per matrix);
// total[m] = samples available
__global__ void __launch_bounds__(1024) scan_bsum_kernel(int nblk, long long* __restrict__ bsum,
                                                         long long* __restrict__ total) {
  const int m = blockIdx.x;
  long long* b = bsum + (int64_t)m * nblk;
  const int per = (nblk + blockDim.x - 1) / blockDim.x;
  const int lo = threadIdx.x * per, hi = min(nblk, lo + per);
  long long s = 0;
  for (int i = lo; i < hi; ++i) s += b[i];
  __shared__ long long part[1024];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const long long v = part[t];
      part[t] = run;
      run += v;
    }
    total[m] = run;
  }
  __syncthreads();
  long long run = part[threadIdx.x];
  for (int i = lo; i < hi; ++i) {
    const long long v = b[i];
    b[i] = run;
    run += v;
  }
}

// Emits the samples of emit_threads<T>() consecutive chunks.  Their outputs form
// one contiguous range of the matrix (the scan gives its start), so each
// thread stages its samples -- post-processed and rounded into the mode -- in
// shared memory at their offset inside the range, and the CTA then writes the
// range with coalesced stores.
template <class T>
constexpr int emit_threads() { return sizeof(T) == 8 ? 64 : 128; }  // 32 KB of staged samples
template <class T>
__global__ void __launch_bounds__(emit_threads<T>()) emit_normals_kernel(
    int64_t Wn, int64_t J, int64_t S, const uint64_t* __restrict__ W, TailTab tt,
    const int* __restrict__ entries, const int* __restrict__ cnts,
    const long long* __restrict__ bsum, const int* __restrict__ which, Post p, T* __restrict__ out,
    uint8_t* __restrict__ flags) {
  constexpr int kEmitThreads = emit_threads<T>();
  static_assert(kScanThreads % kEmitThreads == 0, "emit CTAs subdivide the scan blocks");
  constexpr int kSub = kScanThreads / kEmitThreads;
  __shared__ uint64_t ski[256];
  __shared__ double swi[256], sfi[256];
  __shared__ int sc[kEmitThreads];
  __shared__ long long sbase;
  __shared__ T stage[kEmitThreads * kChunk];
  const ZigTabs z = zig_load(ski, swi, sfi);
  const int m = blockIdx.y;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int cnt = j < J ? cnts[(int64_t)m * J + j] : 0;
  // block-exclusive scan of the chunk counts
  sc[threadIdx.x] = cnt;
  __syncthreads();
  for (int s = 1; s < kEmitThreads; s <<= 1) {
    const int v = threadIdx.x >= s ? sc[threadIdx.x - s] : 0;
    __syncthreads();
    sc[threadIdx.x] += v;
    __syncthreads();
  }
  // start of this CTA's range: the scan block's offset plus the counts of the
  // emit CTAs before this one inside the scan block
  if (threadIdx.x == 0)
    sbase = bsum[(int64_t)m * ((gridDim.x + kSub - 1) / kSub) + blockIdx.x / kSub];
  __syncthreads();
  {
    const int64_t j0 = (int64_t)(blockIdx.x / kSub) * kScanThreads;
    int pre = 0;
    for (int64_t k = j0 + threadIdx.x; k < (int64_t)blockIdx.x * kEmitThreads && k < J;
         k += kEmitThreads)
      pre += cnts[(int64_t)m * J + k];
    if (pre) atomicAdd(reinterpret_cast<unsigned long long*>(&sbase), (unsigned long long)pre);
  }
  __syncthreads();
  const long long base = sbase;
  const int total = sc[kEmitThreads - 1];
  const int loc = sc[threadIdx.x] - cnt;
  if (base >= S || total == 0) return;  // CTA-uniform
  const uint64_t* w = W + (int64_t)m * Wn;
  const int wh = which[m];
  if (j < J && cnt > 0) {
    int k = 0;
    parse_words(w, (int64_t)m * Wn, j * kChunk + entries[(int64_t)m * J + j], (j + 1) * kChunk, tt, z,
                k, [&](int q, double x) {
                  const int64_t e = base + loc + q;
                  if (e < S) {
                    const T r = round_into<T>(post_value(p, wh, e, x));
                    stage[loc + q] = r;
                    if (flags && !finite_of(r)) flags[m] = 1;
                  }
                });
  }
  __syncthreads();
  T* o = out + (int64_t)m * S + base;
  const int lim = (int)(S - base < total ? S - base : total);
  for (int t = threadIdx.x; t < lim; t += kEmitThreads) o[t] = stage[t];
}

// Host half of the tail: numpy's loop
//   xx = -inv_r * log1p(-U); yy = -log1p(-U); until yy + yy > xx * xx
// with the C library's log1p, over the words after the candidate r = win[0].
bool host_tail(const uint64_t* win, int* used, double* value) {
  const uint64_t rabs = (win[0] >> 9) & kMask52;
  for (int it = 0; 2 * it + 2 < kTailWords; ++it) {
    const double u1 = (double)(win[1 + 2 * it] >> 11) * kTwoM53;
    const double u2 = (double)(win[2 + 2 * it] >> 11) * kTwoM53;
    const double xx = -kZigInvR * std::log1p(-u1);
    const double yy = -std::log1p(-u2);
    if (yy + yy > xx * xx) {
      *used = 1 + 2 * (it + 1);
      *value = ((rabs >> 8) & 0x1) ? -(kZigR + xx) : kZigR + xx;
      return true;
    }
  }
  return false;
}

template <class T>
int run_normals(int64_t count, int64_t n, const uint64_t* dkeys, const int* dwhich, const Post& post,
                void* out, uint8_t* flags, cudaStream_t st) {
  const int64_t S = n * n;
  // expected consumption is ~1.0125 words per sample; 1/32 + 4096 spare
  int64_t Wparse = ((S + S / 32 + 4096) + kChunk - 1) / kChunk * kChunk;
  for (int attempt = 0; attempt < 4; ++attempt, Wparse *= 2) {
    // readable past the last chunk; whole interleave groups per matrix
    const int64_t Wn = (Wparse + 2 * kTailWords + 64 + kGroupWords - 1) / kGroupWords * kGroupWords;
    const int64_t J = Wparse / kChunk;
    const int nblk = (int)((J + kScanThreads - 1) / kScanThreads);
    const int64_t cap = std::max<int64_t>(4096, count * Wparse / 512);
    // scratch: W | exits | cnts | entries | counts | bsum | total | list | ctr | tail words
    size_t off = 0;
    auto take = [&](size_t bytes) {
      const size_t o = off;
      off += (bytes + 255) / 256 * 256;
      return o;
    };
    const size_t oW = take(sizeof(uint64_t) * count * Wn);
    const size_t oEx = take(sizeof(int) * count * J * kEntries);
    const size_t oCt = take(sizeof(int) * count * J * kEntries);
    const size_t oEn = take(sizeof(int) * count * J);
    const size_t oCn = take(sizeof(int) * count * J);
    const size_t oBs = take(sizeof(long long) * count * nblk);
    const size_t oTo = take(sizeof(long long) * count);
    const size_t oLi = take(sizeof(int64_t) * cap);
    const size_t oCr = take(sizeof(unsigned long long));
    char* scratch = nullptr;
    {
      int dev = 0;
      CUDA_TRY(cudaGetDevice(&dev));
      CUDA_TRY(keep_pool(dev));  // repeated draws reuse the scratch
    }
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&scratch), off, st));
    auto at = [&](size_t o) { return scratch + o; };
    uint64_t* W = reinterpret_cast<uint64_t*>(at(oW));
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(at(oCr));
    int64_t* list = reinterpret_cast<int64_t*>(at(oLi));
    const unsigned gx = (unsigned)std::min<int64_t>((Wn / 4 + 255) / 256, 148 * 8);
    fill_words_kernel<<<dim3(gx, (unsigned)count), 256, 0, st>>>(Wn, dkeys, W);
    CUDA_TRY(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long), st));
    const unsigned gc = (unsigned)std::min<int64_t>((Wparse + 255) / 256, 148 * 8);
    tail_candidates_kernel<<<dim3(gc, (unsigned)count), 256, 0, st>>>(Wn, Wparse, W, list, ctr, cap);
    unsigned long long ncand = 0;
    CUDA_TRY(cudaMemcpyAsync(&ncand, ctr, sizeof(ncand), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if ((int64_t)ncand > cap) {  // far beyond expectation: not a ziggurat stream
      cudaFreeAsync(scratch, st);
      return fail_cuda(cudaErrorUnknown, "tail candidate overflow", __FILE__, __LINE__);
    }
    // host tail loop over the sorted candidates
    const size_t nc = std::max<size_t>(1, ncand);
    std::vector<int64_t> pos(ncand);
    std::vector<uint64_t> words(ncand * kTailWords);
    std::vector<int> used(ncand);
    std::vector<double> val(ncand);
    int64_t* tpos = nullptr;
    int* tused = nullptr;
    double* tval = nullptr;
    uint64_t* twords = nullptr;
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&twords), sizeof(uint64_t) * nc * kTailWords, st));
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tpos), sizeof(int64_t) * nc, st));
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tused), sizeof(int) * nc, st));
    CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tval), sizeof(double) * nc, st));
    if (ncand > 0) {
      CUDA_TRY(cudaMemcpyAsync(pos.data(), list, sizeof(int64_t) * ncand, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      std::sort(pos.begin(), pos.end());
      CUDA_TRY(cudaMemcpyAsync(tpos, pos.data(), sizeof(int64_t) * ncand, cudaMemcpyHostToDevice, st));
      gather_tail_words_kernel<<<(unsigned)ncand, kTailWords, 0, st>>>(Wn, W, tpos, twords);
      CUDA_TRY(cudaMemcpyAsync(words.data(), twords, sizeof(uint64_t) * ncand * kTailWords,
                               cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      for (size_t c = 0; c < ncand; ++c) {
        if (!host_tail(&words[c * kTailWords], &used[c], &val[c])) {
          cudaFreeAsync(scratch, st);
          return fail_cuda(cudaErrorUnknown, "ziggurat tail did not accept", __FILE__, __LINE__);
        }
      }
      CUDA_TRY(cudaMemcpyAsync(tused, used.data(), sizeof(int) * ncand, cudaMemcpyHostToDevice, st));
      CUDA_TRY(cudaMemcpyAsync(tval, val.data(), sizeof(double) * ncand, cudaMemcpyHostToDevice, st));
    }
    const TailTab tt{tpos, tused, tval, (int64_t)ncand};
    int* exits = reinterpret_cast<int*>(at(oEx));
    int* cnts = reinterpret_cast<int*>(at(oCt));
    int* ent = reinterpret_cast<int*>(at(oEn));
    int* cn = reinterpret_cast<int*>(at(oCn));
    long long* bsum = reinterpret_cast<long long*>(at(oBs));
    long long* total = reinterpret_cast<long long*>(at(oTo));
    const dim3 gj((unsigned)nblk, (unsigned)count);
    chunk_maps_kernel<<<gj, kScanThreads, 0, st>>>(Wn, J, W, tt, exits, cnts);
    chunk_entries_kernel<<<gj, kScanThreads, 0, st>>>(Wn, J, W, tt, exits, cnts, ent, cn, bsum);
    scan_bsum_kernel<<<(unsigned)count, 1024, 0, st>>>(nblk, bsum, total);
    std::vector<long long> tot(count);
    CUDA_TRY(cudaMemcpyAsync(tot.data(), total, sizeof(long long) * count, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const bool enough = std::all_of(tot.begin(), tot.end(), [&](long long t) { return t >= S; });
    if (enough) {
      constexpr int kEmitThreads = emit_threads<T>();
      const dim3 ge((unsigned)((J + kEmitThreads - 1) / kEmitThreads), (unsigned)count);
      emit_normals_kernel<T><<<ge, kEmitThreads, 0, st>>>(Wn, J, S, W, tt, ent, cn, bsum, dwhich,
                                                          post, static_cast<T*>(out), flags);
    }
    const cudaError_t e = cudaGetLastError();
    cudaFreeAsync(twords, st);
    cudaFreeAsync(tpos, st);
    cudaFreeAsync(tused, st);
    cudaFreeAsync(tval, st);
    cudaFreeAsync(scratch, st);
    if (e != cudaSuccess) return fail_cuda(e, "matgen normals", __FILE__, __LINE__);
    if (enough) return RBC_OK;
  }
  return fail_cuda(cudaErrorUnknown, "normal stream shorter than needed", __FILE__, __LINE__);
}

template <class T>
int matgen_typed(int kind, int64_t count, int64_t n, const uint64_t* dkeys, const int* dwhich,
                 void* out, uint8_t* flags, cudaStream_t st) {
  Post p;
  p.kind = kind;
  p.n = (int)n;
  p.tiny = 1.0 / (double)(n * n);
  p.huge = (double)(n * n);
  p.half = (double)n / 2.0;
  const int64_t S = n * n;
  if (kind == kMatGaussian || kind == kMatQuadrant100)
    return run_normals<T>(count, n, dkeys, dwhich, p, out, flags, st);
  const unsigned gx = (unsigned)std::min<int64_t>((S / 4 + 256) / 256, 148 * 8);
  uniform_kernel<T><<<dim3(gx, (unsigned)count), 256, 0, st>>>(S, dkeys, dwhich, p,
                                                               static_cast<T*>(out), flags);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RBC_OK : fail_cuda(e, "matgen uniform", __FILE__, __LINE__);
}

}  // namespace

int matgen(int kind, int dtype, int64_t count, int64_t n, const uint64_t* keys, const int* which,
           void* out, uint8_t* flags, cudaStream_t st) {
  // keys / which: host arrays (count x 2, count), uploaded here
  uint64_t* dk = nullptr;
  int* dw = nullptr;
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dk), sizeof(uint64_t) * 2 * count, st));
  CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&dw), sizeof(int) * count, st));
  CUDA_TRY(cudaMemcpyAsync(dk, keys, sizeof(uint64_t) * 2 * count, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(dw, which, sizeof(int) * count, cudaMemcpyHostToDevice, st));
  int rc;
  if (dtype == kF64) rc = matgen_typed<double>(kind, count, n, dk, dw, out, flags, st);
  else if (dtype == kF32) rc = matgen_typed<float>(kind, count, n, dk, dw, out, flags, st);
  else rc = matgen_typed<__half>(kind, count, n, dk, dw, out, flags, st);
  cudaFreeAsync(dk, st);
  cudaFreeAsync(dw, st);
  // the host copies of keys/which must outlive the uploads
  const cudaError_t e = cudaStreamSynchronize(st);
  if (rc == RBC_OK && e != cudaSuccess) return fail_cuda(e, "matgen", __FILE__, __LINE__);
  return rc;
}

}  // namespace rbc
