// Block-level building blocks shared by the decode and runner kernels:
// reductions, scans, MSB-first radix select on 64-bit keys, the exact numpy
// median of |v|, and a shared-memory bitonic sort on (key, tiebreak) pairs.
#pragma once

#include "common.cuh"

namespace sfft {

// ================================================================ block utils

template <int NT>
__device__ __forceinline__ double block_max(double v, double* red) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < NT / 32) ? red[l] : 0.0;
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  const double r = red[0];
  __syncthreads();
  return r;
}

template <int NT>
__device__ __forceinline__ unsigned long long block_min_u64(unsigned long long v,
                                                            unsigned long long* red) {
  for (int o = 16; o; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t < v ? t : v;
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < NT / 32) ? red[l] : ~0ull;
    for (int o = 16; o; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, v, o);
      v = t < v ? t : v;
    }
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  const unsigned long long r = red[0];
  __syncthreads();
  return r;
}

template <int NT>
__device__ __forceinline__ int block_sum_int(int v, int* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = (l < NT / 32) ? red[l] : 0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  const int r = red[0];
  __syncthreads();
  return r;
}

// Exclusive block scan of one int per thread; returns the total in *total.
template <int NT>
__device__ __forceinline__ int block_exscan(int v, int* red, int* total) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  int x = v;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, x, o);
    if (l >= o) x += t;
  }
  __syncthreads();
  if (l == 31) red[w] = x;
  __syncthreads();
  if (w == 0) {
    int y = (l < NT / 32) ? red[l] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, y, o);
      if (l >= o) y += t;
    }
    if (l < NT / 32) red[l] = y;
  }
  __syncthreads();
  const int base = w ? red[w - 1] : 0;
  const int tot = red[NT / 32 - 1];
  __syncthreads();
  *total = tot;
  return base + x - v;
}

// k-th smallest (0-indexed) of the keys key(i), i < cnt, restricted to keys
// >= lo; MSB-first 8-bit radix select.  Returns the key bits; *below = number
// of included keys strictly smaller, *equal = number equal.
template <int NT, typename KeyF>
__device__ unsigned long long block_radix_select(KeyF key, int64_t cnt, unsigned long long lo,
                                                 int64_t k, unsigned* hist, long long* sh,
                                                 long long* below, long long* equal) {
  unsigned long long prefix = 0;
  long long kk = k;
  long long nbelow = 0;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < cnt; i += NT) {
      const unsigned long long u = key(i);
      if (u < lo) continue;
      if (pass == 0 || (u >> (shift + 8)) == (prefix >> (shift + 8)))
        atomicAdd(&hist[(u >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x < 32) {
      const int l = threadIdx.x;
      long long loc = 0;
      for (int j = 0; j < 8; ++j) loc += hist[l * 8 + j];
      long long inc = loc;
      for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, inc, o);
        if (l >= o) inc += t;
      }
      const long long exc = inc - loc;
      const unsigned ballot = __ballot_sync(0xffffffffu, inc > kk);
      const int owner = __ffs(ballot) - 1;
      if (l == owner) {
        long long c = exc;
        int d = l * 8;
        for (int j = 0; j < 8; ++j) {
          const long long h = hist[l * 8 + j];
          if (c + h > kk) { d = l * 8 + j; break; }
          c += h;
        }
        sh[0] = d;
        sh[1] = kk - c;
        sh[2] = c;
        sh[3] = hist[d];
      }
    }
    __syncthreads();
    prefix |= (unsigned long long)sh[0] << shift;
    kk = sh[1];
    nbelow += sh[2];
    const long long eq = sh[3];
    __syncthreads();
    if (pass == 7) {
      *below = nbelow;
      *equal = eq;
    }
  }
  return prefix;
}

// ================================================================ floor (A8)

struct MagKey {
  const double2* v;
  __device__ __forceinline__ unsigned long long operator()(int64_t i) const {
    return dbits(cabs_(v[i]));
  }
};

template <int NT, typename KeyF>
__device__ void median_and_peak_k(KeyF key, int64_t B, double* med, double* peak, unsigned* hist,
                                  long long* sh, double* redd, unsigned long long* redu);

struct SmemKey {
  const unsigned long long* k;
  __device__ __forceinline__ unsigned long long operator()(int64_t i) const { return k[i]; }
};

// median of |v| (numpy: mean of the two middle values for even counts) and max.
template <int NT>
__device__ void median_and_peak(const double2* v, int64_t B, double* med, double* peak,
                                unsigned* hist, long long* sh, double* redd,
                                unsigned long long* redu) {
  MagKey key{v};
  median_and_peak_k<NT>(key, B, med, peak, hist, sh, redd, redu);
}

template <int NT, typename KeyF>
__device__ void median_and_peak_k(KeyF key, int64_t B, double* med, double* peak, unsigned* hist,
                                  long long* sh, double* redd, unsigned long long* redu) {
  unsigned long long mx = 0;
  for (int64_t i = threadIdx.x; i < B; i += NT) {
    const unsigned long long u = key(i);
    mx = u > mx ? u : mx;
  }
  *peak = __longlong_as_double((long long)(~block_min_u64<NT>(~mx, redu)));
  const int64_t k1 = (B - 1) / 2;
  long long below, equal;
  const unsigned long long u1 = block_radix_select<NT>(key, B, 0ull, k1, hist, sh, &below, &equal);
  const double v1 = __longlong_as_double((long long)u1);
  if (B % 2) {
    *med = v1;
    return;
  }
  double v2;
  if (below + equal >= k1 + 2) {
    v2 = v1;
  } else {
    unsigned long long mn = ~0ull;
    for (int64_t i = threadIdx.x; i < B; i += NT) {
      const unsigned long long u = key(i);
      if (u > u1 && u < mn) mn = u;
    }
    v2 = __longlong_as_double((long long)block_min_u64<NT>(mn, redu));
  }
  *med = (v1 + v2) / 2.0;
}


// Bitonic sort of cnt <= cap (power of two) entries in shared memory,
// ascending by (k1, k2); padding entries get k1 = ~0.  payload follows.
template <int NT>
__device__ void block_bitonic(unsigned long long* k1, long long* k2, int* pay, int cnt,
                              int cap) {
  for (int i = cnt + threadIdx.x; i < cap; i += NT) {
    k1[i] = ~0ull;
    k2[i] = 0x7fffffffffffffffll;
    pay[i] = -1;
  }
  __syncthreads();
  for (int size = 2; size <= cap; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < cap / 2; t += NT) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const bool gt = (k1[lo] > k1[hi]) || (k1[lo] == k1[hi] && k2[lo] > k2[hi]);
        if (gt == up) {
          const unsigned long long a = k1[lo]; k1[lo] = k1[hi]; k1[hi] = a;
          const long long b = k2[lo]; k2[lo] = k2[hi]; k2[hi] = b;
          const int c = pay[lo]; pay[lo] = pay[hi]; pay[hi] = c;
        }
      }
      __syncthreads();
    }
  }
}

}  // namespace sfft
