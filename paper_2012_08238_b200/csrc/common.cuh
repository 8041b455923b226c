// Shared device/host helpers for the sm_100a sparse-FFT hot path.
//
// Complex values are double2 (re, im).  Every decision-relevant quantity is
// fp64, in both the complex64 (input rounded to float2, fp64 accumulation) and
// the complex128 mode (SURVEY.md §7 hard part 1).
#pragma once

#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <string>

#ifndef SFFT_HD
#define SFFT_HD __host__ __device__ __forceinline__

// Checked build (-DSFFT_CHECKED, libsfft_b200_checked.so): device-side bounds
// asserts on the indices of the hot kernels -- the stand-in for
// compute-sanitizer memcheck where the tool is unavailable.  A failed check
// prints its location and traps (the launch then fails loudly).
#ifdef SFFT_CHECKED
#define SFFT_DASSERT(c)                                                          \
  do {                                                                           \
    if (!(c)) {                                                                  \
      printf("SFFT_DASSERT %s:%d: %s\n", __FILE__, __LINE__, #c);                \
      __trap();                                                                  \
    }                                                                            \
  } while (0)
#else
#define SFFT_DASSERT(c) \
  do {                  \
  } while (0)
#endif
#endif

namespace sfft {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);
const char* last_error();
void count_launch();   // running total of this library's kernel launches

#define SFFT_CHECK_LAUNCH(what)                                                  \
  do {                                                                           \
    ::sfft::count_launch();                                                      \
    cudaError_t _e = cudaGetLastError();                                         \
    if (_e != cudaSuccess) {                                                     \
      ::sfft::set_error(std::string(what) + ": " + cudaGetErrorString(_e));     \
      return -3;                                                                 \
    }                                                                            \
  } while (0)

#define SFFT_CUDA(call)                                                          \
  do {                                                                           \
    cudaError_t _e = (call);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::sfft::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));    \
      return -3;                                                                 \
    }                                                                            \
  } while (0)

#define SFFT_REQUIRE(cond, msg)                                                  \
  do {                                                                           \
    if (!(cond)) {                                                               \
      ::sfft::set_error(msg);                                                    \
      return -2;                                                                 \
    }                                                                            \
  } while (0)

// ----------------------------------------------------------------- complex
SFFT_HD double2 cmk(double r, double i) { return make_double2(r, i); }
SFFT_HD double2 cadd(double2 a, double2 b) { return cmk(a.x + b.x, a.y + b.y); }
SFFT_HD double2 csub(double2 a, double2 b) { return cmk(a.x - b.x, a.y - b.y); }
SFFT_HD double2 cmul(double2 a, double2 b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
SFFT_HD double2 cconj(double2 a) { return cmk(a.x, -a.y); }
SFFT_HD double2 cscale(double2 a, double s) { return cmk(a.x * s, a.y * s); }
SFFT_HD double2 cdivr(double2 a, double s) { return cmk(a.x / s, a.y / s); }

#ifdef __CUDACC__
// Products/sums without FMA contraction, where the reference's rounding
// sequence is cheap to reproduce exactly (elementwise numpy products).
__device__ __forceinline__ double2 cmul_rn(double2 a, double2 b) {
  return cmk(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
             __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 csub_rn(double2 a, double2 b) {
  return cmk(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 cadd_rn(double2 a, double2 b) {
  return cmk(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
#endif

// |z| as numpy's vectorised np.abs(complex128 array): larger*sqrt(fma(r,r,1)),
// r = smaller/larger (numpy universal-intrinsics loop; bit-exact with it).
// Used wherever the reference takes np.abs of an array.
#ifdef __CUDA_ARCH__
__device__ __forceinline__ double cabs_(double2 a) {
  double re = fabs(a.x), im = fabs(a.y);
  if (isinf(re) || isinf(im)) return CUDART_INF;
  if (isnan(re) || isnan(im)) return CUDART_NAN;
  const double lg = fmax(re, im), sm = fmin(re, im);
  if (lg == 0.0) return 0.0;
  const double r = __ddiv_rn(sm, lg);
  return __dmul_rn(__dsqrt_rn(__fma_rn(r, r, 1.0)), lg);
}
// glibc 2.35+ hypot (dbl-64 e_hypot.c, non-FMA kernel): what abs() of a
// numpy complex128 scalar and of a Python complex return.
__device__ __forceinline__ double hypot_glibc_kernel(double ax, double ay) {
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    const double d = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, d), ax));
    t2 = __dmul_rn(__dsub_rn(d, __dmul_rn(2.0, __dsub_rn(ax, ay))), d);
  } else {
    const double d = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, d), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, d), ay), ay), __dmul_rn(d, d));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}
__device__ __forceinline__ double cabs_scalar(double2 a) {
  double x = fabs(a.x), y = fabs(a.y);
  if (isinf(x) || isinf(y)) return CUDART_INF;
  if (isnan(x) || isnan(y)) return CUDART_NAN;
  const double ax = x < y ? y : x, ay = x < y ? x : y;
  const double SCALE = 0x1p-600, LARGE = 0x1p+511, TINY = 0x1p-511, EPS = 0x1p-54;
  if (ax > LARGE) {
    if (ay <= __dmul_rn(ax, EPS)) return __dadd_rn(ax, ay);
    return __ddiv_rn(hypot_glibc_kernel(__dmul_rn(ax, SCALE), __dmul_rn(ay, SCALE)), SCALE);
  }
  if (ay < TINY) {
    if (ax >= __ddiv_rn(ay, EPS)) return __dadd_rn(ax, ay);
    return __dmul_rn(hypot_glibc_kernel(__ddiv_rn(ax, SCALE), __ddiv_rn(ay, SCALE)), SCALE);
  }
  if (ay <= __dmul_rn(ax, EPS)) return __dadd_rn(ax, ay);
  return hypot_glibc_kernel(ax, ay);
}
#else
inline double cabs_(double2 a) { return std::hypot(a.x, a.y); }
inline double cabs_scalar(double2 a) { return std::hypot(a.x, a.y); }
#endif

// Complex division with Smith's scaling (numpy's complex128 divide).
SFFT_HD double2 cdiv(double2 a, double2 b) {
  const double br = b.x, bi = b.y;
  const double abs_br = fabs(br), abs_bi = fabs(bi);
  if (abs_br >= abs_bi) {
    if (abs_br == 0.0 && abs_bi == 0.0) {
      return cmk(a.x / abs_br, a.y / abs_br);
    }
    const double rat = bi / br;
    const double scl = 1.0 / (br + bi * rat);
    return cmk((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
  }
  const double rat = br / bi;
  const double scl = 1.0 / (bi + br * rat);
  return cmk((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}

// ----------------------------------------------------------------- modular
SFFT_HD int64_t pmod(int64_t a, int64_t n) {
  // power-of-two n (every flat-window config): a mask, also for negative a
  // (two's complement); 64-bit division costs ~50 instructions on the GPU
  if ((n & (n - 1)) == 0) return a & (n - 1);
  int64_t r = a % n;
  return r < 0 ? r + n : r;
}
// (a*b) mod n for 0 <= a,b < n < 2^31 (products stay below 2^62).
SFFT_HD int64_t mulmod(int64_t a, int64_t b, int64_t n) { return pmod(a * b, n); }

// w_n^e = exp(-2*pi*i*(e mod n)/n), with the angle formed as the reference
// forms it ((-2*pi*e)/n, sfft/signal.py:50-57).
SFFT_HD double2 unit_root(int64_t n, int64_t e) {
  const double th = (-6.283185307179586 * (double)pmod(e, n)) / (double)n;
  double s, c;
  sincos(th, &s, &c);
  return cmk(c, s);
}

// ----------------------------------------------------------------- loads
// Permuted signal gathers: ld.global.cg (cache at L2, bypass L1).  The
// read-only texture path (ld.global.nc) fills L1 at 128-byte granularity,
// which for a random 8-byte gather quadruples the L2->SM and DRAM sector
// traffic (measured with ncu: lts sectors 4.3x l1tex sectors); .cg requests
// single 32-byte sectors.
//
// L2 eviction policy: the flat response table is read with evict_last (every
// subtraction re-reads it) so the streaming gathers do not push it out of L2.
// (evict_first on the gathers was measured slower: it cuts the L2 reuse
// between the concurrently running shifted measurements.)
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ unsigned long long policy_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// response-table read (read-only path, evict_last)
__device__ __forceinline__ double2 ld_table(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(policy_evict_last()));
  return v;
}

template <typename T>
struct Sample;
template <>
struct Sample<float2> {
  static __device__ __forceinline__ double2 load(const float2* p, int64_t i) {
    const float2 v = __ldcg(p + i);
    return cmk((double)v.x, (double)v.y);
  }
};
template <>
struct Sample<double2> {
  static __device__ __forceinline__ double2 load(const double2* p, int64_t i) {
    return __ldcg(p + i);
  }
};

__device__ __forceinline__ double2 to_d2_(float2 v) { return cmk((double)v.x, (double)v.y); }
__device__ __forceinline__ double2 to_d2_(double2 v) { return v; }

// ----------------------------------------------------------------- misc
SFFT_HD int64_t cdiv_up(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Non-negative doubles order like their bit patterns.
SFFT_HD unsigned long long dbits(double v) {
#ifdef __CUDA_ARCH__
  return (unsigned long long)__double_as_longlong(v);
#else
  unsigned long long u;
  memcpy(&u, &v, 8);
  return u;
#endif
}

}  // namespace sfft
