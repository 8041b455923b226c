// Result truncation shared by the runners: drop exact zeros, keep the k
// largest |c| with ties to the smaller position (sfft/frameworks.py:151-155,
// sfft/signal.py:142-145; |c| is Python's complex abs = glibc hypot).
#pragma once

#include "block.cuh"

namespace sfft {

constexpr int kFinNT = 512;

struct FinMagKey {
  const double2* rc;
  __device__ __forceinline__ unsigned long long operator()(int64_t i) const {
    return dbits(cabs_scalar(rc[i]));
  }
};

struct FinPosKey {  // f+1 of the entries whose |c| bits equal u; else 0
  const double2* rc;
  const int64_t* rp;
  unsigned long long u;
  __device__ __forceinline__ unsigned long long operator()(int64_t i) const {
    return dbits(cabs_scalar(rc[i])) == u ? (unsigned long long)(rp[i] + 1) : 0ull;
  }
};

// One CTA per signal; dynamic smem kFusedMaxB * 20 bytes; k <= kFusedMaxB.
// gate (optional): only slots with gate[s] != 0; rows (optional): output row
// of slot s (default s).
static __global__ void __launch_bounds__(kFinNT) k_finalize(const int64_t* rec_pos,
                                                            const double2* rec_coef,
                                                            const int32_t* rec_count, int cap,
                                                            int64_t k, int64_t* out_pos,
                                                            double2* out_coef, int32_t* out_n,
                                                            const int32_t* gate = nullptr,
                                                            const int32_t* rows = nullptr) {
  extern __shared__ unsigned char fsm[];
  __shared__ int redi[32];
  __shared__ unsigned hist[256];
  __shared__ long long sh[4];
  const int s = blockIdx.x;
  if (gate && !gate[s]) return;
  const int64_t row = rows ? rows[s] : s;
  const int T = rec_count[s];
  const int64_t* rp = rec_pos + (int64_t)s * cap;
  const double2* rc = rec_coef + (int64_t)s * cap;
  unsigned long long* k1 = (unsigned long long*)fsm;
  long long* k2 = (long long*)(k1 + kFusedMaxB);
  int* pay = (int*)(k2 + kFusedMaxB);
  FinMagKey mag{rc};
  // nonzero entries (c != 0  <=>  |c| > 0  <=>  bits >= 1)
  int nz = 0;
  for (int t = threadIdx.x; t < T; t += kFinNT) nz += mag(t) >= 1ull;
  const int tot = block_sum_int<kFinNT>(nz, redi);
  const int kk = (int)(k < (int64_t)tot ? k : (int64_t)tot);
  // selection predicate: all nonzero when they fit, else the top kk
  unsigned long long thr = 1ull, fthr = ~0ull;
  bool all = tot <= kFusedMaxB;
  if (!all) {
    long long below, equal;
    thr = block_radix_select<kFinNT>(mag, T, 1ull, (int64_t)tot - kk, hist, sh, &below, &equal);
    const long long above = (long long)tot - below - equal;
    const long long need_eq = kk - above;
    FinPosKey pk{rc, rp, thr};
    long long b2, e2;
    fthr = need_eq > 0 ? block_radix_select<kFinNT>(pk, T, 1ull, need_eq - 1, hist, sh, &b2, &e2)
                       : 0ull;
  }
  const int per = (T + kFinNT - 1) / kFinNT;
  const int t0 = threadIdx.x * per, t1 = min(T, t0 + per);
  int mine = 0;
  for (int t = t0; t < t1; ++t) {
    const unsigned long long u = mag(t);
    mine += all ? (u >= 1ull) : (u > thr || (u == thr && (unsigned long long)(rp[t] + 1) <= fthr));
  }
  int cnt;
  int off = block_exscan<kFinNT>(mine, redi, &cnt);
  for (int t = t0; t < t1; ++t) {
    const unsigned long long u = mag(t);
    const bool sel = all ? (u >= 1ull)
                         : (u > thr || (u == thr && (unsigned long long)(rp[t] + 1) <= fthr));
    if (sel) {
      k1[off] = ~u;
      k2[off] = rp[t];
      pay[off] = t;
      ++off;
    }
  }
  __syncthreads();
  int capp = 1;
  while (capp < cnt) capp <<= 1;
  block_bitonic<kFinNT>(k1, k2, pay, cnt, capp);
  for (int i = threadIdx.x; i < kk; i += kFinNT) {
    out_pos[row * k + i] = rp[pay[i]];
    out_coef[row * k + i] = rc[pay[i]];
  }
  if (threadIdx.x == 0) out_n[row] = kk;
}

}  // namespace sfft
