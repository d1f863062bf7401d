// Common device helpers for the B200 BC-multiply engine.
//
// Every arithmetic operation on the data path goes through the Arith<T>
// traits below, which use the explicitly rounded intrinsics (__fmul_rn,
// __fadd_rn, __dmul_rn, __dadd_rn, __hmul_rn, __hadd_rn, and the half2
// forms).  These are never contracted into FMA, so each multiply and each
// add rounds once (IEEE RNE), which is the per-element rounding sequence of
// the reference engine (pkg/src/randbc/_engine.py:3-18).  The library is
// also compiled with -fmad=false as a second line of defence.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace rbc {

// ---------------------------------------------------------------- arith ----
template <class T> struct Arith;

template <> struct Arith<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float neg(float a) { return -a; }
  static __device__ __forceinline__ bool finite(float a) { return isfinite(a); }
  static __device__ __forceinline__ double widen(float a) { return (double)a; }
};

template <> struct Arith<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double neg(double a) { return -a; }
  static __device__ __forceinline__ bool finite(double a) { return isfinite(a); }
  static __device__ __forceinline__ double widen(double a) { return a; }
};

template <> struct Arith<__half> {
  static __device__ __forceinline__ __half mul(__half a, __half b) { return __hmul_rn(a, b); }
  static __device__ __forceinline__ __half add(__half a, __half b) { return __hadd_rn(a, b); }
  static __device__ __forceinline__ __half sub(__half a, __half b) { return __hsub_rn(a, b); }
  static __device__ __forceinline__ __half neg(__half a) { return __hneg(a); }
  static __device__ __forceinline__ bool finite(__half a) { return !(__hisinf(a) || __hisnan(a)); }
  static __device__ __forceinline__ double widen(__half a) { return (double)__half2float(a); }
};

template <> struct Arith<__half2> {
  static __device__ __forceinline__ __half2 mul(__half2 a, __half2 b) { return __hmul2_rn(a, b); }
  static __device__ __forceinline__ __half2 add(__half2 a, __half2 b) { return __hadd2_rn(a, b); }
  static __device__ __forceinline__ __half2 sub(__half2 a, __half2 b) { return __hsub2_rn(a, b); }
  static __device__ __forceinline__ __half2 neg(__half2 a) { return __hneg2(a); }
};

// ------------------------------------------------ packed binary32 pairs ----
// sm_100a issues two binary32 lanes per instruction (FFMA2 / FADD2 on
// 64-bit register pairs).  The FMA pipe takes them at half the scalar
// instruction rate, so the element rate is unchanged (tools/fp_peak.cu:
// 37.1 vs 35.1 TFLOP/s exact-order), but every packed instruction frees an
// issue slot -- the limit of the exact-order leaf, which needs a separate
// FMUL and FADD per multiply-add.
//
// ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under
// -fmad=false (and folds an fma with a literal -0 addend the same way), so
// the rounded multiply is issued as fma.rn.f32x2(a, b, z) with z = (-0, -0)
// passed in at run time, which the compiler cannot see through:
// fl(a*b + -0) == fl(a*b) for every a, b (a +0 product stays +0, -0 stays
// -0; no flush to zero).  Pass kF2NegZero as a kernel argument.
constexpr uint64_t kF2NegZero = 0x8000000080000000ull;

__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float f2_lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2_hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
// (a, a) * (b.lo, b.hi), each product rounded once; ptxas encodes the
// broadcast as a scalar .F32 operand (no MOV)
__device__ __forceinline__ uint64_t f2_mul_bcast(float a, uint64_t b, uint64_t negz) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(f2_pack(a, a)), "l"(b), "l"(negz));
  return r;
}
__device__ __forceinline__ uint64_t f2_add(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

// Bit-exact sign flip (used for the signed permutations of a plan).
__device__ __forceinline__ float flip_sign(float x, uint32_t m) {
  return __uint_as_float(__float_as_uint(x) ^ m);
}
__device__ __forceinline__ double flip_sign(double x, uint32_t m) {
  return __longlong_as_double(__double_as_longlong(x) ^ ((unsigned long long)m << 32));
}
__device__ __forceinline__ __half flip_sign(__half x, uint32_t m) {
  return __ushort_as_half((unsigned short)(__half_as_ushort(x) ^ (m >> 16)));
}
// mask for a sign: 0 (positive) or the sign bit of a 32-bit word
__device__ __forceinline__ uint32_t sign_mask(int negative) { return negative ? 0x80000000u : 0u; }

// ----------------------------------------------------------------- pack ----
// W consecutive elements handled by one thread; loaded and stored with one
// vector access when the address is sizeof(Pack)-aligned (power-of-two W;
// other widths are register-only packs).
template <class T, int W>
struct alignas((W & (W - 1)) == 0 ? sizeof(T) * W : sizeof(T)) Pack {
  T v[W];
};

template <class T, int W>
__device__ __forceinline__ Pack<T, W> pload(const T* p) {
  return *reinterpret_cast<const Pack<T, W>*>(p);
}
template <class T, int W>
__device__ __forceinline__ void pstore(T* p, const Pack<T, W>& x) {
  *reinterpret_cast<Pack<T, W>*>(p) = x;
}

// Elementwise ops on packs.  Half packs with an even width use half2 SIMD
// (HADD2/HMUL2), which rounds each lane exactly like the scalar forms.
template <class T, int W> struct PackOps {
  using P = Pack<T, W>;
  static __device__ __forceinline__ P add(const P& a, const P& b) {
    P r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = Arith<T>::add(a.v[i], b.v[i]);
    return r;
  }
  static __device__ __forceinline__ P sub(const P& a, const P& b) {
    P r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = Arith<T>::sub(a.v[i], b.v[i]);
    return r;
  }
  static __device__ __forceinline__ P neg(const P& a) {
    P r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = Arith<T>::neg(a.v[i]);
    return r;
  }
  static __device__ __forceinline__ P mul_scalar(T c, const P& a) {
    P r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = Arith<T>::mul(c, a.v[i]);
    return r;
  }
  static __device__ __forceinline__ P flip(const P& a, uint32_t m) {
    P r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = flip_sign(a.v[i], m);
    return r;
  }
  static __device__ __forceinline__ P select(bool c, const P& a, const P& b) {
    P r;
#pragma unroll
    for (int i = 0; i < W; ++i) r.v[i] = c ? a.v[i] : b.v[i];
    return r;
  }
  static __device__ __forceinline__ bool all_finite(const P& a) {
    bool ok = true;
#pragma unroll
    for (int i = 0; i < W; ++i) ok = ok && Arith<T>::finite(a.v[i]);
    return ok;
  }
};

// binary32 packs of three (the 3 x 3 leaf rows of the fused subtree): elements
// 0 and 1 travel as one f32x2 pair, element 2 as a scalar, so an add or a
// subtract of a pack is two instructions instead of three.  Each packed lane
// rounds exactly like the scalar instruction.  Negation of the pair is
// fma(a, (-1, -1), (-0, -0)): exact, signed zeros included; the two constants
// sit in constant memory so that ptxas sees run-time values (it would fold a
// literal -0 addend and contract a packed multiply into the next add).
__device__ __constant__ uint64_t kcF2NegZero = 0x8000000080000000ull;
__device__ __constant__ uint64_t kcF2MinusOne = 0xbf800000bf800000ull;

__device__ __forceinline__ uint64_t f2_sub(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t f2_fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

#ifndef RBC_NO_F32X2_PACK3
template <> struct PackOps<float, 3> {
  using P = Pack<float, 3>;
  static __device__ __forceinline__ uint64_t pr(const P& a) { return f2_pack(a.v[0], a.v[1]); }
  static __device__ __forceinline__ P un(uint64_t p01, float c) {
    P r;
    r.v[0] = f2_lo(p01);
    r.v[1] = f2_hi(p01);
    r.v[2] = c;
    return r;
  }
  static __device__ __forceinline__ P add(const P& a, const P& b) {
    return un(f2_add(pr(a), pr(b)), __fadd_rn(a.v[2], b.v[2]));
  }
  static __device__ __forceinline__ P sub(const P& a, const P& b) {
    return un(f2_sub(pr(a), pr(b)), __fsub_rn(a.v[2], b.v[2]));
  }
  static __device__ __forceinline__ P neg(const P& a) {
    return un(f2_fma(pr(a), kcF2MinusOne, kcF2NegZero), -a.v[2]);
  }
  static __device__ __forceinline__ P mul_scalar(float c, const P& a) {
    return un(f2_mul_bcast(c, pr(a), kcF2NegZero), __fmul_rn(c, a.v[2]));
  }
  static __device__ __forceinline__ P flip(const P& a, uint32_t m) {
    P r;
#pragma unroll
    for (int i = 0; i < 3; ++i) r.v[i] = flip_sign(a.v[i], m);
    return r;
  }
  static __device__ __forceinline__ P select(bool c, const P& a, const P& b) {
    P r;
#pragma unroll
    for (int i = 0; i < 3; ++i) r.v[i] = c ? a.v[i] : b.v[i];
    return r;
  }
  static __device__ __forceinline__ bool all_finite(const P& a) {
    return isfinite(a.v[0]) && isfinite(a.v[1]) && isfinite(a.v[2]);
  }
};
#endif

#define RBC_HALF2_PACK(W)                                                              \
  template <> struct PackOps<__half, W> {                                              \
    using P = Pack<__half, W>;                                                         \
    static __device__ __forceinline__ const __half2* h2(const P& a) {                  \
      return reinterpret_cast<const __half2*>(a.v);                                    \
    }                                                                                  \
    static __device__ __forceinline__ __half2* h2(P& a) {                              \
      return reinterpret_cast<__half2*>(a.v);                                          \
    }                                                                                  \
    static __device__ __forceinline__ P add(const P& a, const P& b) {                  \
      P r;                                                                             \
      _Pragma("unroll") for (int i = 0; i < W / 2; ++i) h2(r)[i] = __hadd2_rn(h2(a)[i], h2(b)[i]); \
      return r;                                                                        \
    }                                                                                  \
    static __device__ __forceinline__ P sub(const P& a, const P& b) {                  \
      P r;                                                                             \
      _Pragma("unroll") for (int i = 0; i < W / 2; ++i) h2(r)[i] = __hsub2_rn(h2(a)[i], h2(b)[i]); \
      return r;                                                                        \
    }                                                                                  \
    static __device__ __forceinline__ P neg(const P& a) {                              \
      P r;                                                                             \
      _Pragma("unroll") for (int i = 0; i < W / 2; ++i) h2(r)[i] = __hneg2(h2(a)[i]);  \
      return r;                                                                        \
    }                                                                                  \
    static __device__ __forceinline__ P mul_scalar(__half c, const P& a) {             \
      P r;                                                                             \
      __half2 cc = __half2half2(c);                                                    \
      _Pragma("unroll") for (int i = 0; i < W / 2; ++i) h2(r)[i] = __hmul2_rn(cc, h2(a)[i]); \
      return r;                                                                        \
    }                                                                                  \
    static __device__ __forceinline__ P flip(const P& a, uint32_t m) {                 \
      P r;                                                                             \
      const uint32_t* s = reinterpret_cast<const uint32_t*>(a.v);                      \
      uint32_t* d = reinterpret_cast<uint32_t*>(r.v);                                  \
      uint32_t mm = m ? 0x80008000u : 0u;                                              \
      _Pragma("unroll") for (int i = 0; i < W / 2; ++i) d[i] = s[i] ^ mm;              \
      return r;                                                                        \
    }                                                                                  \
    static __device__ __forceinline__ P select(bool c, const P& a, const P& b) {       \
      P r;                                                                             \
      const uint32_t* x = reinterpret_cast<const uint32_t*>(a.v);                      \
      const uint32_t* y = reinterpret_cast<const uint32_t*>(b.v);                      \
      uint32_t* d = reinterpret_cast<uint32_t*>(r.v);                                  \
      _Pragma("unroll") for (int i = 0; i < W / 2; ++i) d[i] = c ? x[i] : y[i];        \
      return r;                                                                        \
    }                                                                                  \
    static __device__ __forceinline__ bool all_finite(const P& a) {                    \
      bool ok = true;                                                                  \
      _Pragma("unroll") for (int i = 0; i < W; ++i) ok = ok && Arith<__half>::finite(a.v[i]); \
      return ok;                                                                       \
    }                                                                                  \
  };
RBC_HALF2_PACK(2)
RBC_HALF2_PACK(4)
RBC_HALF2_PACK(8)
#undef RBC_HALF2_PACK

// Three-term left fold whose order is a runtime choice: the two elements
// that come first are added first (addition commutes, so their order does
// not matter) and the element named by `last` (0, 1 or 2) is added last.
template <class T, int W>
__device__ __forceinline__ Pack<T, W> fold3(const Pack<T, W>& a, const Pack<T, W>& b,
                                            const Pack<T, W>& c, int last) {
  using O = PackOps<T, W>;
  Pack<T, W> p = O::select(last == 0, b, a);
  Pack<T, W> q = O::select(last == 2, b, c);
  Pack<T, W> r = O::select(last == 0, a, O::select(last == 1, b, c));
  return O::add(O::add(p, q), r);
}

// -------------------------------------------------------------- plans ----
// Per (trial, level) randomization plan, packed for the device
// (reference RandomizationPlan, randomize.py:58-85).  perm[i][hat] is the
// base block index that hatted block index `hat` reads (perms[i][j] in the
// reference); inv[i][base] is its inverse; neg[i][hat] is 1 where
// signs[i][hat] == -1.
constexpr int kMaxPlanN = 4;
struct PlanLevel {
  int8_t perm[3][kMaxPlanN];
  int8_t inv[3][kMaxPlanN];
  int8_t neg[3][kMaxPlanN];
  int8_t pad[4];
};
static_assert(sizeof(PlanLevel) == 40, "PlanLevel layout");

}  // namespace rbc
