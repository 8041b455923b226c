// Shared-memory mixed-radix FFT for one CTA (forward, w = exp(-2*pi*i/M)).
//
// In-place decimation-in-frequency over G independent segments of length M,
// radices 2/3/4/5/7/11/13 (B = 2^8..2^17 for the flat
// configs, 3^5*5^3 / 2^7*3^5 / 2^7*5^3 for the FFAST stages).  Output k of a
// segment lands at smem position fft_pos(k) (mixed-radix digit reversal); the
// caller gathers it back to natural order while writing to HBM, so no second
// buffer is needed and B = 8192 complex128 fits in 128 KB of shared memory.
//
// Twiddles come from one table W[e] = w_Wn^e (complex128, L1/L2 resident);
// a transform of length M | Wn reads W[e * (Wn / M)].
#pragma once

#include "common.cuh"

namespace sfft {

constexpr int kMaxStages = 28;
constexpr int kFusedMaxB = 8192;   // one-CTA fold+FFT up to this many buckets

struct FftPlan {
  int n;
  int nst;
  int rad[kMaxStages];
};

// Host: factor n into supported radices (4s first).  false if a prime factor
// above 13 remains (the caller then uses the direct-DFT path).
inline bool make_plan(int64_t n, FftPlan* p) {
  p->n = (int)n;
  p->nst = 0;
  int64_t m = n;
  auto push = [&](int r) { p->rad[p->nst++] = r; m /= r; };
  while (m % 4 == 0 && p->nst < kMaxStages) push(4);
  while (m % 2 == 0 && p->nst < kMaxStages) push(2);
  const int primes[] = {3, 5, 7, 11, 13};
  for (int r : primes)
    while (m % r == 0 && p->nst < kMaxStages) push(r);
  return m == 1;
}

__device__ __forceinline__ int fft_pos(int k, const FftPlan& P) {
  int pos = 0, span = P.n;
#pragma unroll 1
  for (int st = 0; st < P.nst; ++st) {
    const int r = P.rad[st];
    span /= r;
    pos += (k % r) * span;
    k /= r;
  }
  return pos;
}

template <int R>
__device__ __forceinline__ void bfly(double2* __restrict__ s, int base, int Mp, int j,
                                     const double2* __restrict__ W, int ws, int wsr) {
  double2 a[R];
#pragma unroll
  for (int p = 0; p < R; ++p) a[p] = s[base + p * Mp];
  if constexpr (R == 2) {
    s[base] = cadd(a[0], a[1]);
    const double2 d = csub(a[0], a[1]);
    s[base + Mp] = j ? cmul(d, __ldg(W + j * ws)) : d;
  } else if constexpr (R == 4) {
    const double2 t0 = cadd(a[0], a[2]), t1 = csub(a[0], a[2]);
    const double2 t2 = cadd(a[1], a[3]), t3 = csub(a[1], a[3]);
    s[base] = cadd(t0, t2);
    const double2 b1 = cmk(t1.x + t3.y, t1.y - t3.x);
    const double2 b2 = csub(t0, t2);
    const double2 b3 = cmk(t1.x - t3.y, t1.y + t3.x);
    if (j) {
      s[base + Mp] = cmul(b1, __ldg(W + j * ws));
      s[base + 2 * Mp] = cmul(b2, __ldg(W + 2 * j * ws));
      s[base + 3 * Mp] = cmul(b3, __ldg(W + 3 * j * ws));
    } else {
      s[base + Mp] = b1;
      s[base + 2 * Mp] = b2;
      s[base + 3 * Mp] = b3;
    }
  } else if constexpr (R == 3) {
    // X0 = a0 + t, X1/X2 = (a0 - t/2) -/+ i sin(2 pi/3) (a1 - a2), t = a1 + a2
    constexpr double s3 = 0.86602540378443864676;
    const double2 t = cadd(a[1], a[2]), d = csub(a[1], a[2]);
    const double2 m = cmk(a[0].x - 0.5 * t.x, a[0].y - 0.5 * t.y);
    const double2 x1 = cmk(m.x + s3 * d.y, m.y - s3 * d.x);
    const double2 x2 = cmk(m.x - s3 * d.y, m.y + s3 * d.x);
    s[base] = cadd(a[0], t);
    if (j) {
      s[base + Mp] = cmul(x1, __ldg(W + j * ws));
      s[base + 2 * Mp] = cmul(x2, __ldg(W + 2 * j * ws));
    } else {
      s[base + Mp] = x1;
      s[base + 2 * Mp] = x2;
    }
  } else if constexpr (R == 5) {
    // t1 = a1 + a4, t2 = a2 + a3, d1 = a1 - a4, d2 = a2 - a3;
    // X1/X4 = (a0 + c1 t1 + c2 t2) -/+ i (s1 d1 + s2 d2),
    // X2/X3 = (a0 + c2 t1 + c1 t2) -/+ i (s2 d1 - s1 d2)
    constexpr double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
    constexpr double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;
    const double2 t1 = cadd(a[1], a[4]), t2 = cadd(a[2], a[3]);
    const double2 d1 = csub(a[1], a[4]), d2 = csub(a[2], a[3]);
    const double2 m1 = cmk(a[0].x + c1 * t1.x + c2 * t2.x, a[0].y + c1 * t1.y + c2 * t2.y);
    const double2 m2 = cmk(a[0].x + c2 * t1.x + c1 * t2.x, a[0].y + c2 * t1.y + c1 * t2.y);
    const double2 n1 = cmk(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y);
    const double2 n2 = cmk(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y);
    const double2 x1 = cmk(m1.x + n1.y, m1.y - n1.x), x4 = cmk(m1.x - n1.y, m1.y + n1.x);
    const double2 x2 = cmk(m2.x + n2.y, m2.y - n2.x), x3 = cmk(m2.x - n2.y, m2.y + n2.x);
    s[base] = cadd(a[0], cadd(t1, t2));
    if (j) {
      s[base + Mp] = cmul(x1, __ldg(W + j * ws));
      s[base + 2 * Mp] = cmul(x2, __ldg(W + 2 * j * ws));
      s[base + 3 * Mp] = cmul(x3, __ldg(W + 3 * j * ws));
      s[base + 4 * Mp] = cmul(x4, __ldg(W + 4 * j * ws));
    } else {
      s[base + Mp] = x1;
      s[base + 2 * Mp] = x2;
      s[base + 3 * Mp] = x3;
      s[base + 4 * Mp] = x4;
    }
  } else {
    // generic odd radix: all inputs are in registers, so each output can be
    // formed and stored in turn (no second register array)
#pragma unroll 1
    for (int q = 0; q < R; ++q) {
      double2 acc = a[0];
#pragma unroll
      for (int p = 1; p < R; ++p) {
        const double2 w = __ldg(W + ((p * q) % R) * wsr);
        acc.x = fma(a[p].x, w.x, fma(-a[p].y, w.y, acc.x));
        acc.y = fma(a[p].x, w.y, fma(a[p].y, w.x, acc.y));
      }
      s[base + q * Mp] = (j && q) ? cmul(acc, __ldg(W + j * q * ws)) : acc;
    }
  }
}

// G segments of length P.n at s + g*seg.  Block-wide; ends with __syncthreads.
__device__ __forceinline__ void fft_dif(double2* s, int G, int seg, const FftPlan& P,
                                        const double2* __restrict__ W, int Wn, int tid,
                                        int nt) {
  const int M = P.n;
  int Mb = M;
#pragma unroll 1
  for (int st = 0; st < P.nst; ++st) {
    const int r = P.rad[st];
    const int Mp = Mb / r;
    const int nb = M / r;
    const int ws = Wn / Mb;
    const int wsr = Wn / r;
#pragma unroll 1
    for (int t = tid; t < G * nb; t += nt) {
      const int g = t / nb;
      const int tt = t - g * nb;
      const int blk = tt / Mp;
      const int j = tt - blk * Mp;
      const int base = g * seg + blk * Mb + j;
      switch (r) {
        case 4: bfly<4>(s, base, Mp, j, W, ws, wsr); break;
        case 2: bfly<2>(s, base, Mp, j, W, ws, wsr); break;
        case 3: bfly<3>(s, base, Mp, j, W, ws, wsr); break;
        case 5: bfly<5>(s, base, Mp, j, W, ws, wsr); break;
        case 7: bfly<7>(s, base, Mp, j, W, ws, wsr); break;
        case 11: bfly<11>(s, base, Mp, j, W, ws, wsr); break;
        default: bfly<13>(s, base, Mp, j, W, ws, wsr); break;
      }
    }
    __syncthreads();
    Mb = Mp;
  }
}

// ---------------------------------------------------------------- pow2 FFT
// Radix-8 register butterflies for power-of-two lengths M = 2^LG (then one
// radix-2/4 stage when LG % 3 != 0), NI segments of length M at s + i*M,
// every butterfly of a stage on its own thread.  Output k of a segment lands
// at pow2_pos<M>(k).
__device__ __forceinline__ void dft4_(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 t0 = cadd(x0, x2), t1 = csub(x0, x2);
  const double2 t2 = cadd(x1, x3), d = csub(x1, x3);
  const double2 t3 = cmk(d.y, -d.x);  // (x1 - x3) * (-i)
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

// X_m = sum_p a_p w8^{pm}, natural order
__device__ __forceinline__ void dft8_(double2* a) {
  constexpr double r = 0.70710678118654752440;
  double2 b[4], c[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    b[k] = cadd(a[k], a[k + 4]);
    c[k] = csub(a[k], a[k + 4]);
  }
  c[1] = cmk(r * (c[1].x + c[1].y), r * (c[1].y - c[1].x));   // * w8
  c[2] = cmk(c[2].y, -c[2].x);                                // * w8^2 = -i
  c[3] = cmk(r * (c[3].y - c[3].x), -r * (c[3].x + c[3].y));  // * w8^3
  dft4_(b[0], b[1], b[2], b[3]);
  dft4_(c[0], c[1], c[2], c[3]);
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    a[2 * m] = b[m];
    a[2 * m + 1] = c[m];
  }
}

template <int M>
struct Pow2 {
  static constexpr int LG = (M >= 2) ? 1 + Pow2<M / 2>::LG : 0;
  static constexpr int N8 = LG / 3;
  static constexpr int RL = 1 << (LG - 3 * N8);  // last radix 1, 2 or 4
};
template <>
struct Pow2<1> {
  static constexpr int LG = 0, N8 = 0, RL = 1;
};

template <int M>
__device__ __forceinline__ int pow2_pos(int k) {
  // digit reversal of the DIF stages (8, ..., 8, RL)
  int pos = 0, span = M;
#pragma unroll
  for (int st = 0; st < Pow2<M>::N8; ++st) {
    span >>= 3;
    pos += (k & 7) * span;
    k >>= 3;
  }
  if (Pow2<M>::RL > 1) pos += k;  // span == RL, digit k < RL, weight 1
  return pos;
}

// tw: the stage twiddles laid out [stage][q][j], tw[off_st + (q - 1) Mp + j] =
// w_M^{j q (M / Mb)} with Mb = M / 8^st, Mp = Mb / 8 (fewer than M entries in
// all): the threads of a warp read consecutive j for every q, where a flat
// table w_M^e made the few j of a late stage collide on one bank group.
template <int M, int NI, int NT>
__device__ __forceinline__ void fft_pow2(double2* __restrict__ s, const double2* __restrict__ tw) {
  int Mb = M;
#pragma unroll 1
  for (int st = 0; st < Pow2<M>::N8; ++st) {
    const int Mp = Mb >> 3;
#pragma unroll 1
    for (int t = threadIdx.x; t < NI * (M / 8); t += NT) {
      const int seg = t / (M / 8), tt = t - seg * (M / 8);
      const int blk = tt / Mp, j = tt - blk * Mp;
      double2* x = s + seg * M + blk * Mb + j;
      double2 a[8];
#pragma unroll
      for (int p = 0; p < 8; ++p) a[p] = x[p * Mp];
      dft8_(a);
      x[0] = a[0];
#pragma unroll
      for (int q = 1; q < 8; ++q) x[q * Mp] = j ? cmul(a[q], tw[(q - 1) * Mp + j]) : a[q];
    }
    __syncthreads();
    tw += 7 * Mp;
    Mb = Mp;
  }
  if (Pow2<M>::RL == 4) {
    for (int t = threadIdx.x; t < NI * (M / 4); t += NT) {
      double2* x = s + 4 * t;
      dft4_(x[0], x[1], x[2], x[3]);
    }
    __syncthreads();
  } else if (Pow2<M>::RL == 2) {
    for (int t = threadIdx.x; t < NI * (M / 2); t += NT) {
      double2* x = s + 2 * t;
      const double2 u = x[0], v = x[1];
      x[0] = cadd(u, v);
      x[1] = csub(u, v);
    }
    __syncthreads();
  }
}

}  // namespace sfft
