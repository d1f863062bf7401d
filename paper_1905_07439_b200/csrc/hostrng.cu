// Host-side seed derivation and plan draws of the reference's RNG layout, in
// C++ ("port numpy's SeedSequence pool hashing
// to vectorised C, so generating a pair's keys costs microseconds").
//
// The reference keys every stream as
//   derive_rng(seed, *path) = Generator(Philox(SeedSequence(seed, spawn_key=path)))
//   derive_seed(seed, *path) = SeedSequence(seed, spawn_key=path).generate_state(1, u64)[0]
// (pkg/src/randbc/rng.py:20-29), and draws a randomization plan as
//   signs = 1 - 2 * gen.integers(0, 2, (3, n)); perms = 3 x gen.permutation(n)
// (randomize.py:118-127).  Python's SeedSequence construction costs ~15 us
// per stream, which made host key derivation the bound on fresh inputs
// (1000 pairs of configuration 2: ~30 ms).  This file restates the published
// numpy algorithms (numpy >= 1.17, pinned numpy>=1.24 by the reference's
// pyproject.toml:12; bit-for-bit checked against numpy by
// tests/test_hostrng.py):
//   * SeedSequence: 32-bit entropy words (an integer splits into little-endian
//     32-bit words, 0 -> [0]); with a spawn key the run entropy is zero-padded
//     to the 4-word pool; pool mixing with the hashmix / mix functions
//     (INIT_A, MULT_A, MIX_MULT_L, MIX_MULT_R, XSHIFT 16); generate_state
//     cycles the pool through the INIT_B / MULT_B hash, u64 = two
//     little-endian u32 words;
//   * Philox4x64-10 (Salmon et al., SC'11), counter starting at 0 and
//     incremented before each 4-word block;
//   * next_uint32 = low half of a 64-bit word, then its high half;
//   * integers(0, 2): Lemire's bounded 32-bit method (range 1: the top bit
//     of one 32-bit draw);
//   * permutation(n): Fisher-Yates from the end, j = random_interval(i)
//     (smallest all-ones mask >= i, redraw 32-bit words until <= i).

#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "../../include/rbc.h"

namespace {

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;
constexpr int kXShift = 16, kPool = 4;

inline uint32_t hashmix(uint32_t v, uint32_t& h) {
  v ^= h;
  h *= kMultA;
  v *= h;
  v ^= v >> kXShift;
  return v;
}
inline uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> kXShift;
  return r;
}

inline void push_int(std::vector<uint32_t>& w, uint64_t x) {
  if (x == 0) {
    w.push_back(0);
    return;
  }
  while (x) {
    w.push_back((uint32_t)x);
    x >>= 32;
  }
}

// SeedSequence(seed, spawn_key=path).generate_state(nwords, u32)
void seed_state(uint64_t seed, int depth, const uint64_t* path, int nwords, uint32_t* out) {
  std::vector<uint32_t> ent;
  ent.reserve(kPool + 2 * depth);
  push_int(ent, seed);
  if (depth > 0)
    while ((int)ent.size() < kPool) ent.push_back(0);
  for (int i = 0; i < depth; ++i) push_int(ent, path[i]);
  uint32_t pool[kPool];
  uint32_t h = kInitA;
  for (int i = 0; i < kPool; ++i) pool[i] = hashmix(i < (int)ent.size() ? ent[i] : 0u, h);
  for (int s = 0; s < kPool; ++s)
    for (int d = 0; d < kPool; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], h));
  for (size_t s = kPool; s < ent.size(); ++s)
    for (int d = 0; d < kPool; ++d) pool[d] = mix(pool[d], hashmix(ent[s], h));
  uint32_t hb = kInitB;
  for (int i = 0; i < nwords; ++i) {
    uint32_t v = pool[i % kPool];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> kXShift;
    out[i] = v;
  }
}

struct Philox {
  uint64_t ctr[4] = {0, 0, 0, 0};
  uint64_t key[2];
  uint64_t buf[4];
  int pos = 4;
  bool has32 = false;
  uint32_t half = 0;

  void block() {
    if (++ctr[0] == 0)
      if (++ctr[1] == 0)
        if (++ctr[2] == 0) ++ctr[3];
    uint64_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint64_t k0 = key[0], k1 = key[1];
    const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
    for (int r = 0; r < 10; ++r) {
      const unsigned __int128 p0 = (unsigned __int128)M0 * c[0];
      const unsigned __int128 p1 = (unsigned __int128)M1 * c[2];
      const uint64_t n0 = (uint64_t)(p1 >> 64) ^ c[1] ^ k0;
      const uint64_t n2 = (uint64_t)(p0 >> 64) ^ c[3] ^ k1;
      c[0] = n0;
      c[1] = (uint64_t)p1;
      c[2] = n2;
      c[3] = (uint64_t)p0;
      k0 += W0;
      k1 += W1;
    }
    memcpy(buf, c, sizeof c);
    pos = 0;
  }
  uint64_t next64() {
    if (pos >= 4) block();
    return buf[pos++];
  }
  uint32_t next32() {
    if (has32) {
      has32 = false;
      return half;
    }
    const uint64_t w = next64();
    has32 = true;
    half = (uint32_t)(w >> 32);
    return (uint32_t)w;
  }
  // Lemire's bounded draw on [0, rng] (rng < 2^32 - 1)
  uint32_t bounded(uint32_t rng) {
    const uint32_t excl = rng + 1;
    uint64_t m = (uint64_t)next32() * excl;
    uint32_t left = (uint32_t)m;
    if (left < excl) {
      const uint32_t thr = (UINT32_MAX - rng) % excl;
      while (left < thr) {
        m = (uint64_t)next32() * excl;
        left = (uint32_t)m;
      }
    }
    return (uint32_t)(m >> 32);
  }
  // random_interval(max): masked rejection on 32-bit draws (max < 2^32)
  uint64_t interval(uint64_t mx) {
    if (mx == 0) return 0;
    uint64_t mask = mx;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    mask |= mask >> 32;
    uint64_t v;
    while ((v = (next32() & mask)) > mx) {
    }
    return v;
  }
};

void philox_key(uint64_t seed, int depth, const uint64_t* path, uint64_t key[2]) {
  uint32_t w[4];
  seed_state(seed, depth, path, 4, w);
  key[0] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  key[1] = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
}

template <class F>
void parallel_for(int64_t count, F fn) {
  const int64_t per = 2048;
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  const int64_t chunks = (count + per - 1) / per;
  if (chunks <= 1 || nt == 1) {
    for (int64_t i = 0; i < count; ++i) fn(i);
    return;
  }
  const unsigned use = (unsigned)std::min<int64_t>(chunks, nt > 16 ? 16 : nt);
  std::vector<std::thread> th;
  for (unsigned t = 0; t < use; ++t)
    th.emplace_back([&, t] {
      for (int64_t c = t; c < chunks; c += use)
        for (int64_t i = c * per; i < std::min(count, (c + 1) * per); ++i) fn(i);
    });
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

int rbc_derive_seeds(const uint64_t* seeds, int64_t seed_stride, int depth,
                     const uint64_t* paths, int64_t count, uint64_t* out) {
  if (depth < 0 || count < 0 || seed_stride < 0) return RBC_EVALUE;
  parallel_for(count, [&](int64_t i) {
    uint32_t w[2];
    seed_state(seeds[i * seed_stride], depth, paths + i * depth, 2, w);
    out[i] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  });
  return RBC_OK;
}

int rbc_philox_keys(const uint64_t* seeds, int64_t seed_stride, int depth, const uint64_t* paths,
                    int64_t count, uint64_t* keys) {
  if (depth < 0 || count < 0 || seed_stride < 0) return RBC_EVALUE;
  parallel_for(count, [&](int64_t i) {
    philox_key(seeds[i * seed_stride], depth, paths + i * depth, keys + 2 * i);
  });
  return RBC_OK;
}

int rbc_draw_plans(int n, const uint64_t* seeds, int64_t seed_stride, int depth,
                   const uint64_t* paths, int64_t count, int64_t* perms, double* signs) {
  if (n < 1 || n > 64 || depth < 0 || count < 0 || seed_stride < 0) return RBC_EVALUE;
  parallel_for(count, [&](int64_t i) {
    Philox g;
    philox_key(seeds[i * seed_stride], depth, paths + i * depth, g.key);
    double* s = signs + i * 3 * n;
    int64_t* p = perms + i * 3 * n;
    for (int k = 0; k < 3 * n; ++k) s[k] = 1.0 - 2.0 * (double)g.bounded(1);
    for (int r = 0; r < 3; ++r) {
      int64_t* row = p + r * n;
      for (int k = 0; k < n; ++k) row[k] = k;
      for (int k = n - 1; k >= 1; --k) {
        const int64_t j = (int64_t)g.interval((uint64_t)k);
        const int64_t t = row[j];
        row[j] = row[k];
        row[k] = t;
      }
    }
  });
  return RBC_OK;
}

}  // extern "C"
