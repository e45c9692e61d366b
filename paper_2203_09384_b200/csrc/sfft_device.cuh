// Device primitives for the batched C2C FFT: complex arithmetic, compile-time
// twiddles and fully unrolled in-register DFTs.
//
// Replaces the per-stage numpy arithmetic of the reference butterfly engine:
//   kernels.py:98-104  (_dft4: radix-4 DFT with rot = -i)
//   kernels.py:126-151 (radix8_stage: two DFT-4s + eighth-root constants)
// Here a radix-r DFT (r <= 64) is a radix-2 decision-in-frequency network over
// r registers; every twiddle inside it is a compile-time constant, and the
// +-1, +-i and (+-1 +- i)/sqrt(2) factors are strength-reduced exactly like the
// reference's radix-8 constants (kernels.py:136-141).  Only forward kernels
// exist; the inverse uses IDFT(x) = swap(DFT(swap(x))) with swap(a+bi) = b+ai,
// which is exact, so "conjugate twiddles" (kernels.py:70-71) costs nothing.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>
#include <utility>

namespace sfft {

template <typename T> struct CxOf;
template <> struct CxOf<float> { using type = float2; };
template <> struct CxOf<double> { using type = double2; };
template <typename T> using cx_t = typename CxOf<T>::type;

// ---------------------------------------------------------------- static_for
template <int I, int END, typename F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < END) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, END>(f);
  }
}

__host__ __device__ constexpr int ilog2(int n) { return n <= 1 ? 0 : 1 + ilog2(n >> 1); }

__host__ __device__ constexpr int bitrev(int k, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((k >> b) & 1) << (bits - 1 - b);
  return r;
}

// cos(2*pi*j/64), j in [0, 64), correctly rounded doubles (50-digit mpmath
// reference, rounded once).  Radix-r DFTs use the r-th roots, r <= 64.
__host__ __device__ constexpr double cos64(int j) {
  j &= 63;
  if (j > 32) j = 64 - j;  // cos is even
  bool neg = false;
  if (j > 16) { j = 32 - j; neg = true; }  // cos(pi - x) = -cos(x)
  double c = 0.0;
  switch (j) {
    case 0: c = 1.0; break;
    case 1: c = 0.9951847266721969; break;
    case 2: c = 0.9807852804032304; break;
    case 3: c = 0.9569403357322088; break;
    case 4: c = 0.9238795325112867; break;
    case 5: c = 0.881921264348355; break;
    case 6: c = 0.8314696123025452; break;
    case 7: c = 0.773010453362737; break;
    case 8: c = 0.7071067811865476; break;
    case 9: c = 0.6343932841636455; break;
    case 10: c = 0.5555702330196022; break;
    case 11: c = 0.47139673682599764; break;
    case 12: c = 0.3826834323650898; break;
    case 13: c = 0.2902846772544624; break;
    case 14: c = 0.19509032201612828; break;
    case 15: c = 0.0980171403295606; break;
    default: c = 0.0; break;
  }
  return neg ? -c : c;
}
__host__ __device__ constexpr double sin64(int j) { return cos64(16 - j + 64); }

// ------------------------------------------------------------ complex helpers
// fp64: scalar DADD/DFMA.  fp32: Blackwell's packed FP32x2 pipe (FADD2 /
// FMUL2 / FFMA2): one instruction updates re and im together.  Swaps and
// single-lane negations written as make_float2(-b.y, b.x) cost nothing --
// ptxas folds them into the .F32x2.LO_HI / .NP operand modifiers, and
// make_float2(c, c) becomes a scalar-broadcast operand (.F32, immediate or
// register) -- so +-i rotations stay free and a complex multiply is 2
// instructions.
template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return C{a.x + b.x, a.y + b.y}; }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { return C{a.x - b.x, a.y - b.y}; }
template <typename C> __device__ __forceinline__ C cmul(C a, C w) {
  return C{a.x * w.x - a.y * w.y, a.x * w.y + a.y * w.x};
}
// fp64: the FMA structure is spelled out (__fma_rn / __dmul_rn) instead of
// left to contraction, so every kernel instantiation rounds identically --
// e.g. the real-input loader (imaginary parts known zero in pass 0) stays
// bit-identical to widening the input to complex first.
template <> __device__ __forceinline__ double2 cmul<double2>(double2 a, double2 w) {
  return double2{__fma_rn(a.x, w.x, -__dmul_rn(a.y, w.y)), __fma_rn(a.x, w.y, __dmul_rn(a.y, w.x))};
}

// CUDA's sm_100 float2 intrinsics (crt/sm_100_rt.h) keep (re, im) in one
// register pair; hand-packing through a u64 (shift/or) instead costs a MOV /
// LOP3 / zeroing per operand (1440 -> 856 SASS instructions per thread for
// the fp32 N=1024 kernel).
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
template <> __device__ __forceinline__ float2 cadd<float2>(float2 a, float2 b) { return add2(a, b); }
template <> __device__ __forceinline__ float2 csub<float2>(float2 a, float2 b) { return sub2(a, b); }
// a*w = (a.x, a.y)*w.x + (-a.y, a.x)*w.y: w.x / w.y are scalar-broadcast
// operands and i*a is an operand modifier (.LO_HI.NP), so 2 instructions and
// no register shuffles.
template <> __device__ __forceinline__ float2 cmul<float2>(float2 a, float2 w) {
  return fma2(make_float2(-a.y, a.x), make_float2(w.y, w.y), mul2(a, make_float2(w.x, w.x)));
}

template <typename C> __device__ __forceinline__ C cswap(C a) { return C{a.y, a.x}; }
template <typename C> __device__ __forceinline__ C mul_minus_i(C a) { return C{a.y, -a.x}; }
template <typename C> __device__ __forceinline__ C mul_plus_i(C a) { return C{-a.y, a.x}; }

// a * exp(-2*pi*i*J/L) with J, L compile-time, L a power of two <= 64.
template <int J, int L, typename C>
__device__ __forceinline__ C twiddle_const(C a) {
  using T = decltype(a.x);
  constexpr int j = ((J % L) + L) % L;
  constexpr T h = T(0.7071067811865476);
  if constexpr (j == 0) {
    return a;
  } else if constexpr (2 * j == L) {
    return C{-a.x, -a.y};
  } else if constexpr (4 * j == L) {
    return mul_minus_i(a);
  } else if constexpr (4 * j == 3 * L) {
    return mul_plus_i(a);
  } else if constexpr (std::is_same_v<C, float2>) {
    // eighth roots: h*(a + rot*a) with rot in {-i, +i}; others: 2-op cmul
    if constexpr (8 * j == L) {  // (1 - i)/sqrt2
      return mul2(add2(a, mul_minus_i(a)), make_float2(h, h));
    } else if constexpr (8 * j == 3 * L) {  // (-1 - i)/sqrt2 = -i * (1 - i)/sqrt2 ... = h*(-a - i a)
      return mul2(add2(mul_minus_i(a), C{-a.x, -a.y}), make_float2(h, h));
    } else if constexpr (8 * j == 5 * L) {  // (-1 + i)/sqrt2
      return mul2(add2(mul_plus_i(a), C{-a.x, -a.y}), make_float2(h, h));
    } else if constexpr (8 * j == 7 * L) {  // (1 + i)/sqrt2
      return mul2(add2(a, mul_plus_i(a)), make_float2(h, h));
    } else {
      constexpr int j64 = j * (64 / L);
      constexpr T c = T(cos64(j64));
      constexpr T s = T(-sin64(j64));
      return fma2(make_float2(-a.y, a.x), make_float2(s, s), mul2(a, make_float2(c, c)));  // immediates
    }
  } else {
    // __dmul_rn: the products must not be contracted into the butterfly
    // adds that consume them (see cmul<double2>)
    if constexpr (8 * j == L) {  // (1 - i)/sqrt2
      return C{__dmul_rn(a.x + a.y, h), __dmul_rn(a.y - a.x, h)};
    } else if constexpr (8 * j == 3 * L) {  // (-1 - i)/sqrt2
      return C{__dmul_rn(a.y - a.x, h), -__dmul_rn(a.x + a.y, h)};
    } else if constexpr (8 * j == 5 * L) {  // (-1 + i)/sqrt2
      return C{-__dmul_rn(a.x + a.y, h), __dmul_rn(a.x - a.y, h)};
    } else if constexpr (8 * j == 7 * L) {  // (1 + i)/sqrt2
      return C{__dmul_rn(a.x - a.y, h), __dmul_rn(a.x + a.y, h)};
    } else {
      constexpr int j64 = j * (64 / L);
      constexpr T c = T(cos64(j64));
      constexpr T s = T(-sin64(j64));
      return cmul(a, C{c, s});
    }
  }
}

// In-place forward DFT of R registers, natural order in and out.
template <int R, typename C>
__device__ __forceinline__ void dft_regs(C (&v)[R]) {
  static_assert((R & (R - 1)) == 0 && R >= 1 && R <= 64, "radix");
  if constexpr (R == 1) {
    return;
  } else {
    constexpr int LOG = ilog2(R);
    static_for<0, LOG>([&](auto S) {
      constexpr int len = R >> decltype(S)::value;
      constexpr int half = len / 2;
      static_for<0, R / len>([&](auto B) {
        static_for<0, half>([&](auto J) {
          constexpr int ia = decltype(B)::value * len + decltype(J)::value;
          constexpr int ib = ia + half;
          const C a = v[ia];
          const C b = v[ib];
          v[ia] = cadd(a, b);
          v[ib] = twiddle_const<decltype(J)::value, len>(csub(a, b));
        });
      });
    });
    C t[R];
    static_for<0, R>([&](auto K) { t[decltype(K)::value] = v[bitrev(decltype(K)::value, LOG)]; });
    static_for<0, R>([&](auto K) { v[decltype(K)::value] = t[decltype(K)::value]; });
  }
}

// ----------------------------------------------------- global memory streams
// Streaming (evict-first) accesses: every element is read once and written once.
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }
__device__ __forceinline__ double ld_stream(const double* p) { return __ldcs(p); }
__device__ __forceinline__ float2 ld_stream(const float2* p) { return __ldcs(p); }
__device__ __forceinline__ double2 ld_stream(const double2* p) { return __ldcs(p); }
__device__ __forceinline__ float4 ld_stream(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_stream(float2* p, float2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(double2* p, double2 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float4* p, float4 v) { __stcs(p, v); }

// Non-finite detection (executor.py:72-73 raises DomainError on NaN/Inf
// input).  The kernels OR a sticky bit per thread and publish it once.
__device__ __forceinline__ uint32_t nonfinite_bits(float2 v) {
  const uint32_t a = __float_as_uint(v.x) & 0x7f800000u;
  const uint32_t b = __float_as_uint(v.y) & 0x7f800000u;
  return (a == 0x7f800000u) | (b == 0x7f800000u);
}
__device__ __forceinline__ uint32_t nonfinite_bits(double2 v) {
  const uint32_t a = uint32_t(__double2hiint(v.x)) & 0x7ff00000u;
  const uint32_t b = uint32_t(__double2hiint(v.y)) & 0x7ff00000u;
  return (a == 0x7ff00000u) | (b == 0x7ff00000u);
}

template <typename C, typename T>
__device__ __forceinline__ C cscale(C a, T s) { return C{a.x * s, a.y * s}; }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return mul2(a, make_float2(s, s)); }

}  // namespace sfft
