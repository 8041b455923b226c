// Decode-stage kernels (sm_100a): robust noise floor, heavy-bucket selection,
// hash-inverse voting + vote selection, bucket-energy estimates, the trimmed
// mean over rounds and the bucket-domain forward-model subtraction.
//
// All arithmetic that feeds a discrete decision is fp64 and follows the
// reference's formulas and tie rules:
//   floor      max(min(3*median|v|, peak/4), 1e-9*peak, 1e-300)   sfft/reconstruct.py:119-133
//   heavy      |v| >= max(thr,0), order (-|v|, idx), first h       sfft/reconstruct.py:171-177
//   votes      +1 per round whose heavy set holds f's flat bucket  sfft/reconstruct.py:158-179
//   select     count >= max(frac*R, 1e-12), order (-count, pos)    sfft/reconstruct.py:182-194
//   estimates  y[b] / (G[bL-m] * w^{tau m}), NaN under 0.05*max|G| sfft/frameworks.py:321-332
//   trimmed    median / lower-quartile / keep / nanmean            sfft/frameworks.py:335-351
//   subtract   y[b] - sum_f c_f G[(bL - sigma f)] w^{tau_tot sigma f} sfft/frameworks.py:423-436
#include "kernels.cuh"
#include "block.cuh"
#include "robust.cuh"

namespace sfft {

constexpr int kFloorNT = 256;

// One CTA per bucket set: floor[i] and peak[i] of values[i][0..B).
constexpr int kFloorBigNT = 1024;
constexpr int64_t kFloorCache = 24576;  // |v| bits cached in shared memory up to this B

template <int NT>
__global__ void __launch_bounds__(NT) k_floor(const double2* __restrict__ values, int64_t B,
                                              double mult, const int32_t* item_sig,
                                              const int32_t* active, double* floor_out,
                                              double* peak_out) {
  extern __shared__ unsigned long long fcache[];
  __shared__ unsigned hist[256];
  __shared__ long long sh[4];
  __shared__ double redd[32];
  __shared__ unsigned long long redu[32];
  const int item = blockIdx.x;
  if (active) {
    const int sig = item_sig ? item_sig[item] : item;
    if (!active[sig]) return;
  }
  double med, peak;
  const double2* v = values + (int64_t)item * B;
  if (B <= kFloorCache) {
    for (int64_t i = threadIdx.x; i < B; i += NT) fcache[i] = dbits(cabs_(v[i]));
    __syncthreads();
    median_and_peak_k<NT>(SmemKey{fcache}, B, &med, &peak, hist, sh, redd, redu);
  } else {
    median_and_peak<NT>(v, B, &med, &peak, hist, sh, redd, redu);
  }
  if (threadIdx.x == 0) {
    const double fl = fmax(fmax(fmin(mult * med, 0.25 * peak), 1e-9 * peak), 1e-300);
    floor_out[item] = fl;
    if (peak_out) peak_out[item] = peak;
  }
}

int run_floor(const double2* values, int64_t nsets, int64_t B, double mult,
              const int32_t* item_sig, const int32_t* active, double* floor_out, double* peak_out,
              cudaStream_t st) {
  if (nsets <= 0) return 0;
  const size_t sm = B <= kFloorCache ? (size_t)B * 8 : 0;
  if (B > 2048) {
    SFFT_CUDA(cudaFuncSetAttribute(k_floor<kFloorBigNT>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sm ? sm : 1)));
    k_floor<kFloorBigNT><<<(unsigned)nsets, kFloorBigNT, sm, st>>>(values, B, mult, item_sig,
                                                                   active, floor_out, peak_out);
  } else {
    k_floor<kFloorNT><<<(unsigned)nsets, kFloorNT, sm, st>>>(values, B, mult, item_sig, active,
                                                             floor_out, peak_out);
  }
  SFFT_CHECK_LAUNCH("k_floor");
  return 0;
}

// ================================================================ heavy set (A9)

// Heavy bitmap of one round: the first `hc` eligible buckets in (-|v|, idx)
// order.  bits[B/32 words].  One CTA per item.
// Heavy bitmap of one set from its keys (|v| bits): the first hc eligible
// buckets (|v| >= thr) in (-|v|, idx) order; *nheavy_out = their count.
template <int NT, typename KeyF>
__device__ void heavy_bits_k(KeyF key, int64_t B, double thr, int64_t hc, uint32_t* bw,
                             int32_t* nheavy_out, unsigned* hist, long long* sh, int* redi) {
  const int64_t words = (B + 31) / 32;
  const double t = fmax(thr, 0.0);
  const unsigned long long lo = dbits(t);
  // eligible count
  int e = 0;
  for (int64_t i = threadIdx.x; i < B; i += NT) e += key(i) >= lo;
  const int E = block_sum_int<NT>(e, redi);
  for (int64_t w = threadIdx.x; w < words; w += NT) bw[w] = 0u;
  __syncthreads();
  if (E <= hc) {
    for (int64_t i = threadIdx.x; i < B; i += NT)
      if (key(i) >= lo) atomicOr(&bw[i >> 5], 1u << (i & 31));
    if (threadIdx.x == 0 && nheavy_out) *nheavy_out = E;
    return;
  }
  // threshold: the (E-hc)-th smallest eligible key; above it all heavy, at it
  // the smallest indices first.
  long long below, equal;
  const unsigned long long ut =
      block_radix_select<NT>(key, B, lo, E - hc, hist, sh, &below, &equal);
  const long long above = (long long)E - below - equal;
  const long long need_eq = hc - above;
  // ties in index order: each thread scans a contiguous index range
  const int64_t per = (B + NT - 1) / NT;
  const int64_t i0 = threadIdx.x * per, i1 = min(B, i0 + per);
  int my_eq = 0;
  for (int64_t i = i0; i < i1; ++i) my_eq += key(i) == ut;
  int tot;
  int rank = block_exscan<NT>(my_eq, redi, &tot);
  for (int64_t i = i0; i < i1; ++i) {
    const unsigned long long u = key(i);
    bool h = u > ut;
    if (u == ut) {
      h = rank < need_eq;
      ++rank;
    }
    if (h) atomicOr(&bw[i >> 5], 1u << (i & 31));
  }
  if (threadIdx.x == 0 && nheavy_out) *nheavy_out = (int)hc;
}

__global__ void __launch_bounds__(kFloorNT) k_heavy_bitmap(const double2* __restrict__ values,
                                                           int64_t B, const double* thr,
                                                           int64_t hc, const int32_t* item_sig,
                                                           const int32_t* active,
                                                           uint32_t* __restrict__ bits,
                                                           int32_t* nheavy) {
  constexpr int NT = kFloorNT;
  __shared__ unsigned hist[256];
  __shared__ long long sh[4];
  __shared__ int redi[32];
  const int item = blockIdx.x;
  if (active) {
    const int sig = item_sig ? item_sig[item] : item;
    if (!active[sig]) return;
  }
  const int64_t words = (B + 31) / 32;
  heavy_bits_k<NT>(MagKey{values + (int64_t)item * B}, B, thr[item], hc,
                   bits + (int64_t)item * words, nheavy ? nheavy + item : nullptr, hist, sh, redi);
}

// Floor (A8) and heavy bitmap (A9) of one set in one CTA from |v| bits cached
// in shared memory (each |v| computed once instead of once per radix pass).
__global__ void __launch_bounds__(kFloorBigNT) k_floor_heavy(const double2* __restrict__ values,
                                                             int64_t B, double mult, int64_t hc,
                                                             double* floor_out,
                                                             uint32_t* __restrict__ bits,
                                                             int32_t* nheavy) {
  constexpr int NT = kFloorBigNT;
  extern __shared__ unsigned long long fcache[];
  __shared__ unsigned hist[256];
  __shared__ long long sh[4];
  __shared__ double redd[32];
  __shared__ unsigned long long redu[32];
  __shared__ int redi[32];
  const int item = blockIdx.x;
  const double2* v = values + (int64_t)item * B;
  for (int64_t i = threadIdx.x; i < B; i += NT) fcache[i] = dbits(cabs_(v[i]));
  __syncthreads();
  double med, peak;
  median_and_peak_k<NT>(SmemKey{fcache}, B, &med, &peak, hist, sh, redd, redu);
  const double fl = fmax(fmax(fmin(mult * med, 0.25 * peak), 1e-9 * peak), 1e-300);
  if (threadIdx.x == 0) floor_out[item] = fl;
  const int64_t words = (B + 31) / 32;
  heavy_bits_k<NT>(SmemKey{fcache}, B, fl, hc, bits + (int64_t)item * words,
                   nheavy ? nheavy + item : nullptr, hist, sh, redi);
}

int run_floor_heavy(const double2* values, int64_t nsets, int64_t B, double mult, int64_t hc,
                    double* floor_out, uint32_t* bits, int32_t* nheavy, cudaStream_t st) {
  if (nsets <= 0) return 0;
  // small sets: the two 256-thread kernels are faster than one 1024-thread CTA
  if (B > kFloorCache || B < 4096) {
    int rc = run_floor(values, nsets, B, mult, nullptr, nullptr, floor_out, nullptr, st);
    return rc ? rc : run_heavy_bitmap(values, nsets, B, floor_out, hc, nullptr, nullptr, bits,
                                      nheavy, st);
  }
  const size_t sm = (size_t)B * 8;
  SFFT_CUDA(cudaFuncSetAttribute(k_floor_heavy, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sm ? sm : 1)));
  k_floor_heavy<<<(unsigned)nsets, kFloorBigNT, sm, st>>>(values, B, mult, hc, floor_out, bits,
                                                         nheavy);
  SFFT_CHECK_LAUNCH("k_floor_heavy");
  return 0;
}

int run_heavy_bitmap(const double2* values, int64_t nsets, int64_t B, const double* thr,
                     int64_t hc, const int32_t* item_sig, const int32_t* active, uint32_t* bits,
                     int32_t* nheavy, cudaStream_t st) {
  if (nsets <= 0) return 0;
  k_heavy_bitmap<<<(unsigned)nsets, kFloorNT, 0, st>>>(values, B, thr, hc, item_sig, active,
                                                       bits, nheavy);
  SFFT_CHECK_LAUNCH("k_heavy_bitmap");
  return 0;
}

// ================================================================ votes (A10, A11)

__device__ __forceinline__ int vote_count(const VoteRounds& vr, const uint32_t* bits_s,
                                          const int64_t* sig_s, const int64_t* bp_s, int64_t f) {
  int cnt = 0;
  const int64_t n = vr.n;
  for (int r = 0; r < vr.R; ++r) {
    const int64_t bp = bp_s ? bp_s[r] : 0;
    const int64_t m = mulmod(sig_s[r], pmod(f - bp, n), n);
    int64_t b = pmod(m - vr.cs + vr.L / 2, n) / vr.L;
    if (b >= vr.B) b -= vr.B;
    cnt += (bits_s[(int64_t)r * vr.words + (b >> 5)] >> (b & 31)) & 1u;
  }
  return cnt;
}

constexpr int kVoteNT = 512;
constexpr int kVoteChunk = 4096;  // positions per CTA

// Pass 1: counts (optionally stored) and, per chunk, a histogram of counts.
__global__ void __launch_bounds__(kVoteNT) k_votes_hist(VoteRounds vr, const int64_t* counts_in,
                                                        int64_t* counts_out, int nchunks,
                                                        int* chist /*[S][nchunks][R+1]*/) {
  extern __shared__ uint32_t sbits[];
  __shared__ int h[kMaxVoteRounds + 1];
  const int s = blockIdx.y;
  const int chunk = blockIdx.x;
  const int R = vr.R;
  const int64_t* sig_s = vr.sigma ? vr.sigma + (int64_t)s * R : nullptr;
  const int64_t* bp_s = vr.bprime ? vr.bprime + (int64_t)s * R : nullptr;
  const uint32_t* bits_s = vr.bits_global ? vr.bits + (int64_t)s * R * vr.words : sbits;
  if (!counts_in && !vr.bits_global) {
    const uint32_t* g = vr.bits + (int64_t)s * R * vr.words;
    for (int64_t i = threadIdx.x; i < (int64_t)R * vr.words; i += kVoteNT) sbits[i] = g[i];
  }
  for (int i = threadIdx.x; i <= R; i += kVoteNT) h[i] = 0;
  __syncthreads();
  const int64_t p0 = (int64_t)chunk * kVoteChunk;
  for (int64_t p = p0 + threadIdx.x; p < min(vr.n, p0 + kVoteChunk); p += kVoteNT) {
    int c;
    if (counts_in) c = (int)counts_in[(int64_t)s * vr.n + p];
    else c = vote_count(vr, bits_s, sig_s, bp_s, p);
    if (counts_out) counts_out[(int64_t)s * vr.n + p] = c;
    if (c > 0) atomicAdd(&h[c], 1);
  }
  __syncthreads();
  int* o = chist + ((int64_t)s * nchunks + chunk) * (R + 1);
  for (int i = threadIdx.x; i <= R; i += kVoteNT) o[i] = h[i];
}

// Pass 2: base[s][chunk][c] = (#positions with count > c) + (#count==c in
// earlier chunks); ntot[s] = #positions with count >= need (capped at keep).
__global__ void k_votes_scan(int nchunks, int R, int need, int keep, int* chist,
                             int32_t* ncand) {
  const int s = blockIdx.x;
  int* hs = chist + (int64_t)s * nchunks * (R + 1);
  __shared__ long long tot[kMaxVoteRounds + 1];
  for (int c = threadIdx.x; c <= R; c += blockDim.x) {
    long long run = 0;
    for (int k = 0; k < nchunks; ++k) {
      const int v = hs[(int64_t)k * (R + 1) + c];
      hs[(int64_t)k * (R + 1) + c] = (int)run;
      run += v;
    }
    tot[c] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long above = 0, sel = 0;
    for (int c = R; c >= 0; --c) {
      const long long t = tot[c];
      tot[c] = above;
      if (c >= need && c > 0) sel += t;
      above += t;
    }
    ncand[s] = (int)(sel < keep ? sel : keep);
  }
  __syncthreads();
  for (int c = threadIdx.x; c <= R; c += blockDim.x) {
    const long long a = tot[c];
    for (int k = 0; k < nchunks; ++k) hs[(int64_t)k * (R + 1) + c] += (int)a;
  }
}

// Pass 3: each chunk ranks its candidates (count >= need) in position order
// within their count class and writes those with rank < keep.
__global__ void __launch_bounds__(kVoteNT) k_votes_emit(VoteRounds vr, const int64_t* counts_in,
                                                        int nchunks, const int* chist, int need,
                                                        int keep, int64_t* cand,
                                                        int32_t* cand_count) {
  extern __shared__ uint32_t sbits[];
  __shared__ int red[32];
  __shared__ int64_t lpos[kVoteChunk];
  __shared__ uint8_t lcnt[kVoteChunk];
  __shared__ int run[kMaxVoteRounds + 1];
  const int s = blockIdx.y;
  const int chunk = blockIdx.x;
  const int R = vr.R;
  const int64_t* sig_s = vr.sigma ? vr.sigma + (int64_t)s * R : nullptr;
  const int64_t* bp_s = vr.bprime ? vr.bprime + (int64_t)s * R : nullptr;
  const uint32_t* bits_s = vr.bits_global ? vr.bits + (int64_t)s * R * vr.words : sbits;
  if (!counts_in && !vr.bits_global) {
    const uint32_t* g = vr.bits + (int64_t)s * R * vr.words;
    for (int64_t i = threadIdx.x; i < (int64_t)R * vr.words; i += kVoteNT) sbits[i] = g[i];
  }
  const int* base = chist + ((int64_t)s * nchunks + chunk) * (R + 1);
  for (int i = threadIdx.x; i <= R; i += kVoteNT) run[i] = base[i];
  __syncthreads();
  // each thread owns 8 consecutive positions (kVoteChunk = 8 * kVoteNT)
  const int64_t p0 = (int64_t)chunk * kVoteChunk + threadIdx.x * 8;
  int cnts[8];
  int mine = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int64_t p = p0 + j;
    int c = 0;
    if (p < vr.n) {
      if (counts_in) c = (int)counts_in[(int64_t)s * vr.n + p];
      else c = vote_count(vr, bits_s, sig_s, bp_s, p);
    }
    cnts[j] = c;
    mine += (c >= need && c > 0);
  }
  int total;
  int off = block_exscan<kVoteNT>(mine, red, &total);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (cnts[j] >= need && cnts[j] > 0) {
      lpos[off] = p0 + j;
      lcnt[off] = (uint8_t)cnts[j];
      ++off;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t* cs = cand + (int64_t)s * keep;
    for (int i = 0; i < total; ++i) {
      const int c = lcnt[i];
      const int rk = run[c]++;
      if (rk < keep) cs[rk] = lpos[i];
    }
  }
  (void)cand_count;
}

// ---------------------------------------------------------------- general tally

// vote_tally over any bucket sets (sfft/reconstruct.py:158-179): position f
// scores one in round r iff its bucket under round r's hash view
// (sfft/bucketize.py:81-90) is heavy.  m = sigma_r (f - b'_r) mod n, L_r = n/B_r:
//   kind 0 (flat, or Dirichlet with half offset): ((m - cs_r + L_r/2) mod n) / L_r mod B_r
//   kind 1 (spike):                                m mod B_r
//   kind 2 (Dirichlet, no half offset):           ((m - cs_r) mod n) / L_r mod B_r
// This is the reference's preimage scatter evaluated per position (no atomics).
__global__ void k_vote_tally(int64_t n, int R, const int64_t* __restrict__ Bs,
                             const int64_t* __restrict__ boff, const uint32_t* __restrict__ bits,
                             const int64_t* __restrict__ sigma, const int64_t* __restrict__ bprime,
                             const int32_t* __restrict__ kind, const int64_t* __restrict__ cs,
                             int64_t* __restrict__ counts) {
  const int64_t f = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= n) return;
  int64_t c = 0;
  for (int r = 0; r < R; ++r) {
    const int64_t B = Bs[r], L = n / B;
    const int64_t m = mulmod(pmod(sigma[r], n), pmod(f - (bprime ? bprime[r] : 0), n), n);
    const int kd = kind ? kind[r] : 0;
    const int64_t sh = cs ? cs[r] : 0;
    int64_t b;
    if (kd == 1) b = m % B;
    else if (kd == 2) b = (pmod(m - sh, n) / L) % B;
    else b = (pmod(m - sh + L / 2, n) / L) % B;
    c += (__ldg(bits + boff[r] + (b >> 5)) >> (b & 31)) & 1u;
  }
  counts[f] = c;
}

int run_vote_tally(int64_t n, int R, const int64_t* Bs, const int64_t* boff, const uint32_t* bits,
                   const int64_t* sigma, const int64_t* bprime, const int32_t* kind,
                   const int64_t* cs, int64_t* counts, cudaStream_t st) {
  if (n <= 0) return 0;
  k_vote_tally<<<(unsigned)cdiv_up(n, 256), 256, 0, st>>>(n, R, Bs, boff, bits, sigma, bprime,
                                                            kind, cs, counts);
  SFFT_CHECK_LAUNCH("k_vote_tally");
  return 0;
}

// ---------------------------------------------------------------- fast path

__device__ __forceinline__ int64_t modinv_dev(int64_t a, int64_t n) {
  int64_t t = 0, nt = 1, r = n, nr = pmod(a, n);
  while (nr) {
    const int64_t q = r / nr;
    int64_t tmp = t - q * nt; t = nt; nt = tmp;
    tmp = r - q * nr; r = nr; nr = tmp;
  }
  return t < 0 ? t + n : t;
}

constexpr int kVoteCap = 8192;  // candidates sorted in shared memory per signal

struct FastVote {
  int64_t nmask;  // n - 1 when n is a power of two, else -1
  int logL;       // log2 L when L is a power of two, else -1
};

__device__ __forceinline__ int64_t vbucket(const VoteRounds& vr, const FastVote& fv,
                                           int64_t sg, int64_t bp, int64_t f) {
  if (fv.nmask >= 0 && fv.logL >= 0 && bp == 0 && vr.cs == 0) {
    const int64_t m = (sg * f) & fv.nmask;
    return ((m + (vr.L >> 1)) & fv.nmask) >> fv.logL;
  }
  const int64_t m = mulmod(sg, pmod(f - bp, vr.n), vr.n);
  int64_t b = pmod(m - vr.cs + vr.L / 2, vr.n) / vr.L;
  return b >= vr.B ? b - vr.B : b;
}

__device__ __forceinline__ bool vheavy(const uint32_t* bits_r, int64_t b) {
  return (bits_r[b >> 5] >> (b & 31)) & 1u;
}

// Per (signal, round): heavy bucket list from the bitmap, and sigma^-1.
__global__ void k_vote_lists(VoteRounds vr, int64_t hc, int32_t* hl, int32_t* nh,
                             int64_t* sinv) {
  __shared__ int cnt;
  const int s = blockIdx.y, r = blockIdx.x;
  const int64_t sr = (int64_t)s * vr.R + r;
  const uint32_t* bw = vr.bits + sr * vr.words;
  if (threadIdx.x == 0) {
    cnt = 0;
    sinv[sr] = modinv_dev(vr.sigma[sr], vr.n);
  }
  __syncthreads();
  for (int64_t w = threadIdx.x; w < vr.words; w += blockDim.x) {
    uint32_t v = bw[w];
    while (v) {
      const int bit = __ffs(v) - 1;
      v &= v - 1;
      const int idx = atomicAdd(&cnt, 1);
      if (idx < hc) hl[sr * hc + idx] = (int32_t)(w * 32 + bit);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) nh[sr] = cnt < hc ? cnt : (int)hc;
}

// Warp-aggregated append of (R - score, f) keys.
__device__ __forceinline__ void vappend(bool take, unsigned long long key, int s,
                                        int32_t* cnt, unsigned long long* buf) {
  const unsigned mask = __ballot_sync(0xffffffffu, take);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(mask) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(cnt + s, __popc(mask));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (take) {
    const int idx = base + __popc(mask & ((1u << lane) - 1));
    if (idx < kVoteCap) buf[(int64_t)s * kVoteCap + idx] = key;
  }
}

// Bit-sliced vote scan (power-of-two N and B, no b' and no centre shift: the
// runners' case).  sigma (f0 + j L) = sigma f0 + (sigma j mod B) L, so the
// bucket of position f0 + j L in round r is (b_r(f0) + sigma_r j) mod B: with
// the round's heavy bitmap permuted once, P_r[i] = heavy_r[(sigma_r i) mod B],
// the B positions {f0 + j L} hit exactly the bits of P_r rotated by
// c_r = sigma_r^-1 b_r(f0) mod B.  A warp takes 1024 of them at a time (one
// 32-bit word per lane), rotates each round's vector out of shared memory
// (two conflict-free loads and a funnel shift) and adds it into bit-sliced
// counters (two logic ops per slice): ~25 instructions per round for 1024
// positions instead of a multiply, a shuffle and a test per position and
// round.  Positions whose counter reaches `need` (a sliced comparison) are
// appended with their exact count, as the scan does.
template <int NS>
__global__ void __launch_bounds__(256) k_vote_sliced(VoteRounds vr, FastVote fv, int need,
                                                     int32_t* cnt, unsigned long long* buf) {
  extern __shared__ uint32_t vsp[];  // [R][W] permuted bitmaps
  __shared__ uint32_t vsig[kMaxVoteRounds], vinv[kMaxVoteRounds];
  const int s = blockIdx.y;
  const int R = vr.R;
  const int W = (int)vr.words;
  const uint32_t Bm = (uint32_t)vr.B - 1u;
  const uint32_t* gb = vr.bits + (int64_t)s * R * W;
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const uint32_t sg = (uint32_t)vr.sigma[(int64_t)s * R + r];
    uint32_t x = sg;  // Newton: inverse of an odd number mod 2^32
    for (int it = 0; it < 5; ++it) x *= 2u - sg * x;
    vsig[r] = sg;
    vinv[r] = x;
  }
  __syncthreads();
  for (int wi = threadIdx.x; wi < R * W; wi += blockDim.x) {
    const int r = wi / W, k = wi - r * W;
    const uint32_t sg = vsig[r];
    const uint32_t* bw = gb + (int64_t)r * W;
    uint32_t word = 0;
    for (int t = 0; t < 32; ++t) {
      const uint32_t src = (sg * (uint32_t)(32 * k + t)) & Bm;
      word |= ((__ldg(bw + (src >> 5)) >> (src & 31)) & 1u) << t;
    }
    vsp[wi] = word;
  }
  __syncthreads();
  const uint32_t nmask = (uint32_t)fv.nmask, half = (uint32_t)(vr.L >> 1);
  const int lg = fv.logL;
  const int lane = threadIdx.x & 31;
  const int nchunk = W >= 32 ? W / 32 : 1;
  const int64_t items = vr.L * nchunk;
  const int wpb = blockDim.x >> 5;
  for (int64_t item = (int64_t)blockIdx.x * wpb + (threadIdx.x >> 5); item < items;
       item += (int64_t)gridDim.x * wpb) {
    const uint32_t f0 = (uint32_t)(item / nchunk);
    const int k = (int)(item % nchunk) * 32 + lane;  // this lane's word of the vector
    uint32_t sl[NS];
#pragma unroll
    for (int i = 0; i < NS; ++i) sl[i] = 0u;
    for (int r = 0; r < R; ++r) {
      const uint32_t b0 = ((((vsig[r] * f0) & nmask) + half) & nmask) >> lg;
      const uint32_t c = (vinv[r] * b0) & Bm;
      const int cw = (int)(c >> 5);
      const uint32_t* pr = vsp + r * W;
      const uint32_t lo = pr[(k + cw) & (W - 1)], hi = pr[(k + cw + 1) & (W - 1)];
      uint32_t carry = lane < W ? __funnelshift_r(lo, hi, c & 31u) : 0u;
#pragma unroll
      for (int i = 0; i < NS; ++i) {
        const uint32_t t = sl[i] & carry;
        sl[i] ^= carry;
        carry = t;
      }
    }
    uint32_t gt = 0u, eq = ~0u;
#pragma unroll
    for (int i = NS - 1; i >= 0; --i) {
      const uint32_t nb = ((need >> i) & 1) ? ~0u : 0u;
      gt |= eq & sl[i] & ~nb;
      eq &= ~(sl[i] ^ nb);
    }
    uint32_t ge = gt | eq;
    while (__any_sync(0xffffffffu, ge != 0u)) {
      const bool take = ge != 0u;
      unsigned long long key = 0ull;
      if (take) {
        const int t = __ffs(ge) - 1;
        ge &= ge - 1u;
        int c = 0;
#pragma unroll
        for (int i = 0; i < NS; ++i) c |= (int)((sl[i] >> t) & 1u) << i;
        const int64_t f = (int64_t)f0 + (int64_t)(32 * k + t) * vr.L;
        key = ((unsigned long long)(R - c) << 40) | (unsigned long long)f;
      }
      vappend(take, key, s, cnt, buf);
    }
  }
}

// mode 0: every position; mode 1: preimages of the heavy buckets of rounds
// 0..R-need (every position with >= need votes is heavy in one of them),
// each position counted from its first heavy round only.
template <int MODE>
__global__ void __launch_bounds__(256) k_vote_collect(VoteRounds vr, FastVote fv, int need,
                                                      int64_t hc, const int32_t* hl,
                                                      const int32_t* nh, const int64_t* sinv,
                                                      int32_t* cnt, unsigned long long* buf) {
  extern __shared__ uint32_t sbm[];
  __shared__ int64_t ssig[kMaxVoteRounds];
  const int s = blockIdx.y;
  const int R = vr.R;
  const uint32_t* gb = vr.bits + (int64_t)s * R * vr.words;
  const uint32_t* sb = vr.bits_global ? gb : sbm;
  if (!vr.bits_global)
    for (int64_t i = threadIdx.x; i < (int64_t)R * vr.words; i += blockDim.x) sbm[i] = gb[i];
  for (int r = threadIdx.x; r < R; r += blockDim.x) ssig[r] = vr.sigma[(int64_t)s * R + r];
  __syncthreads();
  const int64_t* bps = vr.bprime ? vr.bprime + (int64_t)s * R : nullptr;
  const bool fast32 = MODE == 0 && fv.nmask >= 0 && fv.logL >= 0 && !bps && vr.cs == 0 &&
                      vr.n <= (int64_t(1) << 32) && vr.words <= 64 * 1024;
  if (fast32 && vr.words <= 32 && R <= 32) {
    // B <= 1024: lane w keeps word w of every round's heavy bitmap in a
    // register and a look-up is one shuffle — no shared-memory bank conflicts
    // (32 random words over 32 banks serialise ~3.5x).  Two positions per
    // thread; the warp leaves the round loop once none of its 64 positions can
    // still reach `need` (a candidate keeps its warp in the loop to the last
    // round, so its count is complete).
    const uint32_t mask = (uint32_t)fv.nmask, half = (uint32_t)(vr.L >> 1);
    const int lg = fv.logL;
    const int words = (int)vr.words;
    const int lane = threadIdx.x & 31;
    uint32_t w[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) w[r] = (r < R && lane < words) ? sb[r * words + lane] : 0u;
    // t = (sigma f + L/2) mod N: word = t >> (lg + 5), bit = (t >> lg) & 31
    // (the funnel shift takes its count mod 32)
    constexpr int P = 4;  // positions per thread
    const int64_t step = (int64_t)gridDim.x * blockDim.x * P;
    for (int64_t f0 = (int64_t)blockIdx.x * blockDim.x * P; f0 < vr.n; f0 += step) {
      uint32_t u[P];
      int c[P];
#pragma unroll
      for (int q = 0; q < P; ++q) {
        u[q] = (uint32_t)(f0 + threadIdx.x + (int64_t)q * blockDim.x);
        c[q] = 0;
      }
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        if (r >= R) break;
        const uint32_t sg = (uint32_t)ssig[r];
#pragma unroll
        for (int q = 0; q < P; ++q) {
          const uint32_t t = (sg * u[q] + half) & mask;
          const uint32_t wv = __shfl_sync(0xffffffffu, w[r], t >> (lg + 5));
          c[q] += __funnelshift_r(wv, 0u, t >> lg) & 1u;
        }
        if (r & 1) {  // every second round is often enough
          const int left = R - 1 - r;
          int best = c[0];
#pragma unroll
          for (int q = 1; q < P; ++q) best = max(best, c[q]);
          if (!__any_sync(0xffffffffu, best + left >= need)) break;
        }
      }
#pragma unroll
      for (int q = 0; q < P; ++q) {
        const int64_t f = f0 + threadIdx.x + (int64_t)q * blockDim.x;
        vappend(f < vr.n && c[q] >= need,
                ((unsigned long long)(R - c[q]) << 40) | (unsigned long long)f, s, cnt, buf);
      }
    }
  } else if (fast32) {
    // power-of-two N: bucket of f in round r is ((sigma_r f mod 2^32 & (N-1)) + L/2 & (N-1)) >> log2 L
    const uint32_t mask = (uint32_t)fv.nmask, half = (uint32_t)(vr.L >> 1);
    const int lg = fv.logL;
    const int words = (int)vr.words;
    for (int64_t f0 = (int64_t)blockIdx.x * blockDim.x; f0 < vr.n;
         f0 += (int64_t)gridDim.x * blockDim.x) {
      const int64_t f = f0 + threadIdx.x;
      const uint32_t fu = (uint32_t)f;
      int c = 0;
      if (f < vr.n) {
        // stop once the remaining rounds cannot lift the count to `need`
        // (the count itself only matters for candidates)
        for (int r = 0; r < R; ++r) {
          const uint32_t m = ((uint32_t)ssig[r] * fu) & mask;
          const uint32_t b = ((m + half) & mask) >> lg;
          c += (sb[r * words + (b >> 5)] >> (b & 31)) & 1u;
          if (c + (R - 1 - r) < need) break;
        }
      }
      vappend(f < vr.n && c >= need, ((unsigned long long)(R - c) << 40) | (unsigned long long)f,
              s, cnt, buf);
    }
  } else if (MODE == 0) {
    for (int64_t f0 = (int64_t)blockIdx.x * blockDim.x; f0 < vr.n;
         f0 += (int64_t)gridDim.x * blockDim.x) {
      const int64_t f = f0 + threadIdx.x;
      int c = 0;
      if (f < vr.n)
        for (int r = 0; r < R; ++r)
          c += vheavy(sb + (int64_t)r * vr.words, vbucket(vr, fv, ssig[r], bps ? bps[r] : 0, f));
      vappend(f < vr.n && c >= need, ((unsigned long long)(R - c) << 40) | (unsigned long long)f,
              s, cnt, buf);
    }
  } else {
    const int R0 = R - need + 1;
    const int64_t per_round = hc * vr.L;
    const int64_t total = (int64_t)R0 * per_round;
    for (int64_t e0 = (int64_t)blockIdx.x * blockDim.x; e0 < total;
         e0 += (int64_t)gridDim.x * blockDim.x) {
      const int64_t e = e0 + threadIdx.x;
      bool take = false;
      unsigned long long key = 0;
      if (e < total) {
        const int r0 = (int)(e / per_round);
        const int64_t rem = e - (int64_t)r0 * per_round;
        const int64_t hi = rem / vr.L, j = rem - hi * vr.L;
        const int64_t sr = (int64_t)s * R + r0;
        if (hi < nh[sr]) {
          const int64_t b = hl[sr * hc + hi];
          const int64_t m = pmod(b * vr.L + vr.cs - vr.L / 2 + j, vr.n);
          const int64_t f = pmod(mulmod(sinv[sr], m, vr.n) + (bps ? bps[r0] : 0), vr.n);
          bool first = true;
          for (int r = 0; r < r0 && first; ++r)
            first = !vheavy(sb + (int64_t)r * vr.words, vbucket(vr, fv, ssig[r], bps ? bps[r] : 0, f));
          if (first) {
            int c = 1;
            for (int r = r0 + 1; r < R; ++r)
              c += vheavy(sb + (int64_t)r * vr.words, vbucket(vr, fv, ssig[r], bps ? bps[r] : 0, f));
            take = c >= need;
            key = ((unsigned long long)(R - c) << 40) | (unsigned long long)f;
          }
        }
      }
      vappend(take, key, s, cnt, buf);
    }
  }
}

// Per signal: sort the (R - score, f) keys, keep the first `keep`.
__global__ void __launch_bounds__(1024) k_vote_sort(const int32_t* cnt,
                                                    const unsigned long long* buf, int keep,
                                                    int64_t* cand, int32_t* ncand,
                                                    int32_t* overflow) {
  extern __shared__ unsigned long long ks[];
  const int s = blockIdx.x;
  const int c = cnt[s];
  if (c > kVoteCap) {
    if (threadIdx.x == 0) {
      *overflow = 1;
      ncand[s] = 0;
    }
    return;
  }
  int capp = 1;
  while (capp < c) capp <<= 1;
  for (int i = threadIdx.x; i < capp; i += blockDim.x)
    ks[i] = i < c ? buf[(int64_t)s * kVoteCap + i] : ~0ull;
  __syncthreads();
  for (int size = 2; size <= capp; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < capp / 2; t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        if ((ks[lo] > ks[hi]) == up) {
          const unsigned long long x = ks[lo];
          ks[lo] = ks[hi];
          ks[hi] = x;
        }
      }
      __syncthreads();
    }
  const int kk = c < keep ? c : keep;
  for (int i = threadIdx.x; i < kk; i += blockDim.x)
    cand[(int64_t)s * keep + i] = (int64_t)(ks[i] & ((1ull << 40) - 1));
  if (threadIdx.x == 0) ncand[s] = kk;
}

size_t votes_fast_ws_bytes(int S, int R, int64_t hc) {
  return (size_t)S * kVoteCap * 8 + (size_t)S * 4 + 256 + (size_t)S * R * hc * 4 +
         (size_t)S * R * 4 + (size_t)S * R * 8 + 1024;
}

int run_votes_fast(const VoteRounds& vr, int S, int need, int keep, int64_t hc, int64_t* cand,
                   int32_t* ncand, void* ws, size_t ws_bytes, int* overflow_host,
                   cudaStream_t st) {
  SFFT_REQUIRE(vr.R >= 1 && vr.R <= kMaxVoteRounds && need >= 1, "votes_fast: bad rounds");
  SFFT_REQUIRE(ws_bytes >= votes_fast_ws_bytes(S, vr.R, hc), "votes_fast: workspace too small");
  char* w = (char*)ws;
  unsigned long long* buf = (unsigned long long*)w;
  w += (size_t)S * kVoteCap * 8;
  int32_t* cnt = (int32_t*)w;
  w += (size_t)S * 4;
  int32_t* ovf = (int32_t*)w;
  w += 256;
  int32_t* hl = (int32_t*)w;
  w += (size_t)S * vr.R * hc * 4;
  int32_t* nh = (int32_t*)w;
  w += (size_t)S * vr.R * 4;
  w = (char*)(((uintptr_t)w + 7) & ~(uintptr_t)7);
  int64_t* sinv = (int64_t*)w;
  SFFT_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * S, st));
  SFFT_CUDA(cudaMemsetAsync(ovf, 0, sizeof(int32_t), st));
  FastVote fv;
  fv.nmask = (vr.n & (vr.n - 1)) == 0 ? vr.n - 1 : -1;
  fv.logL = (vr.L & (vr.L - 1)) == 0 ? __builtin_ctzll((unsigned long long)vr.L) : -1;
  // heavy bitmaps in shared memory when they fit, else read from global memory
  VoteRounds vg = vr;
  vg.bits_global = (size_t)vr.R * vr.words * sizeof(uint32_t) > 200 * 1024;
  const size_t sm = vg.bits_global ? 0 : (size_t)vr.R * vr.words * sizeof(uint32_t);
  const int R0 = vr.R - need + 1;
  const bool pre = R0 >= 1 && (double)R0 * hc * vr.L < 0.5 * (double)vr.n;
  // SFFT_NO_VOTE_SLICED=1 keeps the per-position scans (A/B and the parity test)
  const bool sliced = !getenv("SFFT_NO_VOTE_SLICED") && fv.nmask >= 0 && fv.logL >= 0 &&
                      !vr.bprime && vr.cs == 0 && vr.n <= (int64_t(1) << 32) && vr.B >= 32 &&
                      (vr.B & (vr.B - 1)) == 0 && vr.words * 32 == vr.B && sm > 0 && need >= 1 &&
                      need <= vr.R;
  if (sliced) {
    const int64_t items = vr.L * std::max<int64_t>(1, vr.words / 32);
    // a CTA permutes the R bitmaps once (~0.04 R B instructions per thread): give
    // each warp enough 1024-position items (>= B/128) to amortise that
    const int64_t per_warp = std::max<int64_t>(16, vr.B / 128);
    const unsigned gx =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(items / (8 * per_warp), 64));
    if (vr.R <= 31) {
      SFFT_CUDA(cudaFuncSetAttribute(k_vote_sliced<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sm));
      k_vote_sliced<5><<<dim3(gx, S), 256, sm, st>>>(vg, fv, need, cnt, buf);
    } else {
      SFFT_CUDA(cudaFuncSetAttribute(k_vote_sliced<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sm));
      k_vote_sliced<8><<<dim3(gx, S), 256, sm, st>>>(vg, fv, need, cnt, buf);
    }
    SFFT_CHECK_LAUNCH("k_vote_sliced");
  } else if (pre) {
    k_vote_lists<<<dim3(vr.R, S), 256, 0, st>>>(vr, hc, hl, nh, sinv);
    SFFT_CHECK_LAUNCH("k_vote_lists");
    SFFT_CUDA(cudaFuncSetAttribute(k_vote_collect<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sm ? sm : 1)));
    const int64_t total = (int64_t)R0 * hc * vr.L;
    const unsigned gx = (unsigned)std::min<int64_t>(cdiv_up(total, 256), 512);
    k_vote_collect<1><<<dim3(gx, S), 256, sm, st>>>(vg, fv, need, hc, hl, nh, sinv, cnt, buf);
    SFFT_CHECK_LAUNCH("k_vote_collect<pre>");
  } else {
    SFFT_CUDA(cudaFuncSetAttribute(k_vote_collect<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sm ? sm : 1)));
    // >= 16 positions per thread: the per-block bitmap copy is amortised
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv_up(vr.n, 256 * 16), 1024));
    k_vote_collect<0><<<dim3(gx, S), 256, sm, st>>>(vg, fv, need, hc, hl, nh, sinv, cnt, buf);
    SFFT_CHECK_LAUNCH("k_vote_collect<scan>");
  }
  SFFT_CUDA(cudaFuncSetAttribute(k_vote_sort, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kVoteCap * 8));
  k_vote_sort<<<S, 1024, kVoteCap * 8, st>>>(cnt, buf, keep, cand, ncand, ovf);
  SFFT_CHECK_LAUNCH("k_vote_sort");
  SFFT_CUDA(cudaMemcpyAsync(overflow_host, ovf, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SFFT_CUDA(cudaStreamSynchronize(st));
  return 0;
}

int run_votes(const VoteRounds& vr, int S, const int64_t* counts_in, int64_t* counts_out,
              int need, int keep, int64_t* cand, int32_t* ncand, int* chist, bool emit,
              cudaStream_t st) {
  SFFT_REQUIRE(vr.R >= 0 && vr.R <= kMaxVoteRounds, "votes: rounds must be <= 255");
  const int nchunks = (int)cdiv_up(vr.n, kVoteChunk);
  const size_t static3 = kVoteChunk * (8 + 1) + (kMaxVoteRounds + 1) * 4 + 32 * 4;
  VoteRounds vg = vr;
  vg.bits_global = !counts_in && (size_t)vr.R * vr.words * sizeof(uint32_t) + static3 > 220 * 1024;
  const size_t sm = (counts_in || vg.bits_global) ? 0 : (size_t)vr.R * vr.words * sizeof(uint32_t);
  SFFT_CUDA(cudaFuncSetAttribute(k_votes_hist, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sm ? sm : 1)));
  dim3 g(nchunks, S);
  k_votes_hist<<<g, kVoteNT, sm, st>>>(vg, counts_in, counts_out, nchunks, chist);
  SFFT_CHECK_LAUNCH("k_votes_hist");
  if (!emit) return 0;
  k_votes_scan<<<S, 64, 0, st>>>(nchunks, vr.R, need, keep, chist, ncand);
  SFFT_CHECK_LAUNCH("k_votes_scan");
  const size_t sm3 = sm;
  SFFT_CUDA(cudaFuncSetAttribute(k_votes_emit, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)(sm3 ? sm3 : 1)));
  k_votes_emit<<<g, kVoteNT, sm3, st>>>(vg, counts_in, nchunks, chist, need, keep, cand, ncand);
  SFFT_CHECK_LAUNCH("k_votes_emit");
  return 0;
}

size_t votes_ws_bytes(int64_t n, int S, int R) {
  return (size_t)cdiv_up(n, kVoteChunk) * S * (R + 1) * sizeof(int);
}

// ================================================================ estimates (A12, A13)

// est[item][c] for item = (s, r): y[b]/(G[bL-m] * w^{tau m}); (NaN, 0) when
// |G| < 0.05 * gmax (numpy assigns a real NaN into the complex array).
__device__ __forceinline__ double2 energy_est_one(const double2* y, const double2* gt,
                                                  double gfloor, int64_t n, int64_t B,
                                                  int64_t L, int64_t sigma, int64_t tau,
                                                  int64_t f) {
  const int64_t m = mulmod(sigma, pmod(f, n), n);
  const int64_t b = pmod(m + L / 2, n) / L;
  const int64_t e = pmod(b * L - m, n);
  const double2 w = gt[(e % L) * B + e / L];
  if (cabs_(w) < gfloor) return cmk(CUDART_NAN, 0.0);
  const double2 ph = unit_root(n, mulmod(tau % n, m, n));
  return cdiv(y[b], cmul(w, ph));
}

__global__ void k_trimmed_mean(const double2* __restrict__ est, int R, int64_t C,
                               double2* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  out[c] = trimmed_mean_col(est + c, C, R);
}

int run_trimmed_mean(const double2* est, int R, int64_t C, double2* out, cudaStream_t st) {
  SFFT_REQUIRE(R >= 1 && R <= kMaxRounds, "trimmed_mean: 1 <= rounds <= 255");
  if (C <= 0) return 0;
  k_trimmed_mean<<<(unsigned)cdiv_up(C, 128), 128, 0, st>>>(est, R, C, out);
  SFFT_CHECK_LAUNCH("k_trimmed_mean");
  return 0;
}

__global__ void k_energy_est(const double2* __restrict__ y, int64_t B, const double2* gt,
                             const double* gmax, int64_t n, int R, const int64_t* sigma,
                             const int64_t* tau, const int64_t* cand, int64_t C,
                             double2* __restrict__ est) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y;
  if (c >= C) return;
  const int64_t L = n / B;
  est[(int64_t)r * C + c] = energy_est_one(y + (int64_t)r * B, gt, 0.05 * gmax[0], n, B, L,
                                           sigma[r], tau[r], cand[c]);
}

int run_energy_est(const double2* y, int64_t B, const double2* gt, const double* gmax, int64_t n,
                   int R, const int64_t* sigma, const int64_t* tau, const int64_t* cand,
                   int64_t C, double2* est, cudaStream_t st) {
  if (C <= 0 || R <= 0) return 0;
  dim3 g((unsigned)cdiv_up(C, 128), R);
  k_energy_est<<<g, 128, 0, st>>>(y, B, gt, gmax, n, R, sigma, tau, cand, C, est);
  SFFT_CHECK_LAUNCH("k_energy_est");
  return 0;
}

// ================================================================ subtraction (A14)

// out[item][i] = y[item][bk] - sum_t c_t * G[(bk*L - m_t) mod n] * w^{(tau_tot m_t) mod n},
// bk = i (full) or blist[item*nb + i]; tones of signal item_sig[item] in order.
constexpr int kSubNT = 256;
constexpr int kSubChunk = 256;

// Two buckets per thread, kSubNT apart (each warp load instruction reads 32
// consecutive table entries: measured 16 -> 8 L1 sectors per request); a_t = c_t * w^{tau m_t} is formed once
// per tone in shared memory (the reference forms (c*w)*phase: same value up
// to rounding).
constexpr int kSubBPT = 2;
constexpr int kSubPerSplit = 128;  // tones per split

__device__ __forceinline__ int sub_splits(int64_t T, int maxTS) {
  const int64_t z = (T + kSubPerSplit - 1) / kSubPerSplit;
  return (int)(z < 1 ? 1 : (z > maxTS ? maxTS : z));
}

#ifndef SFFT_SUB_MINB
#define SFFT_SUB_MINB 4
#endif
#ifndef SFFT_SUB_BATCH
#define SFFT_SUB_BATCH 8   // tones whose table reads are in flight together (real form)
#endif
template <bool REAL>
__global__ void __launch_bounds__(kSubNT, SFFT_SUB_MINB) k_subtract(
    const double2* __restrict__ y, double2* __restrict__ out, int64_t B, int64_t nb,
    const int32_t* blist, const double2* __restrict__ gt, int64_t n, const int32_t* item_sig,
    const int64_t* sigma, const int64_t* tau_tot, const int64_t* tpos, const double2* tcoef,
    const int32_t* tcount, int64_t tstride, const int32_t* gate, double2* __restrict__ part,
    RealTab rt, const int32_t* __restrict__ list) {
  __shared__ int32_t s_row[kSubChunk];
  __shared__ int32_t s_q[kSubChunk];
  __shared__ double2 s_a[kSubChunk];     // complex: c w^{tau m}; real: beta = c w^{tau m} w^{-m h} / B
  __shared__ double2 s_al[kSubChunk];    // real: alpha = c w^{tau m} t0 / B
  __shared__ double2 s_alsum;
  const int item = list ? list[blockIdx.y] : blockIdx.y;
  const int sig = item_sig ? item_sig[item] : item;
  if (gate && !gate[sig]) return;
  const int64_t L = n / B;
  const int64_t sg = sigma[item];
  const int64_t tt = tau_tot[item];
  const int64_t Tall = tcount[sig];
  // tone split z < TS of this item's own tone count (gridDim.z = the largest
  // split count); with one split the running value starts at y and the tones
  // are subtracted in order (reference order)
  const int TS = sub_splits(Tall, gridDim.z);
  if ((int)blockIdx.z >= TS) return;
  const int64_t per = (Tall + TS - 1) / TS;
  const int64_t tb = (int64_t)blockIdx.z * per;
  const int64_t te = (tb + per < Tall) ? tb + per : Tall;
  const int64_t T = te > tb ? te - tb : 0;
  const int64_t* tp = tpos + (int64_t)sig * tstride + tb;
  const double2* tc = tcoef + (int64_t)sig * tstride + tb;
  // bucket u of this thread: i0 + u * kSubNT, so every load instruction of a
  // warp reads 32 consecutive table entries (full 32-byte sectors)
  const int64_t i0 = (int64_t)blockIdx.x * kSubNT * kSubBPT + threadIdx.x;
  int bk[kSubBPT];
  bool live[kSubBPT];
  double2 acc[kSubBPT];
#pragma unroll
  for (int u = 0; u < kSubBPT; ++u) {
    const int64_t i = i0 + u * kSubNT;
    live[u] = i < nb;
    bk[u] = live[u] ? (int)(blist ? blist[(int64_t)item * nb + i] : i) : 0;
    acc[u] = (live[u] && TS == 1 && !REAL) ? y[(int64_t)item * B + bk[u]] : cmk(0.0, 0.0);
  }
  const int Bi = (int)B;
  const double t0v = REAL ? rt.taps[0] : 0.0;
  const double invB = 1.0 / (double)B;
  if (REAL && threadIdx.x == 0) s_alsum = cmk(0.0, 0.0);
  for (int64_t t0 = 0; t0 < T; t0 += kSubChunk) {
    __syncthreads();
    for (int j = threadIdx.x; j < kSubChunk && t0 + j < T; j += kSubNT) {
      const int64_t m = mulmod(sg, pmod(tp[t0 + j], n), n);
      s_row[j] = (int)((L - m % L) % L);
      s_q[j] = (int)((m + L - 1) / L);
      const double2 cp = cmul(tc[t0 + j], unit_root(n, mulmod(tt, m, n)));
      if (REAL) {
        s_a[j] = cscale(cmul(cp, unit_root(n, pmod(-mulmod(m, rt.h % n, n), n))), invB);
        s_al[j] = cscale(cp, t0v * invB);
      } else {
        s_a[j] = cp;
      }
    }
    __syncthreads();
    if (REAL && threadIdx.x < 32) {
      // alpha is bucket-independent: one warp sums the chunk
      const int tn = (int)((T - t0 < kSubChunk) ? (T - t0) : kSubChunk);
      double2 z = cmk(0.0, 0.0);
      for (int j = threadIdx.x; j < tn; j += 32) z = cadd(z, s_al[j]);
      for (int o = 16; o; o >>= 1) {
        z.x += __shfl_xor_sync(0xffffffffu, z.x, o);
        z.y += __shfl_xor_sync(0xffffffffu, z.y, o);
      }
      if (threadIdx.x == 0) s_alsum = cadd(s_alsum, z);
    }
    if (REAL) {
      if (live[0]) {
        const int tn = (int)((T - t0 < kSubChunk) ? (T - t0) : kSubChunk);
        int j = 0;
        for (; j + SFFT_SUB_BATCH <= tn; j += SFFT_SUB_BATCH) {
          double w[SFFT_SUB_BATCH][kSubBPT];
#pragma unroll
          for (int v = 0; v < SFFT_SUB_BATCH; ++v) {
            const double* row = rt.at + (int64_t)s_row[j + v] * B;
#pragma unroll
            for (int u = 0; u < kSubBPT; ++u) {
              int col = bk[u] - s_q[j + v];
              col += (col < 0) ? Bi : 0;
              SFFT_DASSERT(col >= 0 && col < Bi && s_row[j + v] >= 0 && s_row[j + v] < n / B);
              w[v][u] = __ldg(row + col);
            }
          }
#pragma unroll
          for (int v = 0; v < SFFT_SUB_BATCH; ++v)
#pragma unroll
            for (int u = 0; u < kSubBPT; ++u) {
              acc[u].x = fma(s_a[j + v].x, w[v][u], acc[u].x);
              acc[u].y = fma(s_a[j + v].y, w[v][u], acc[u].y);
            }
        }
        for (; j < tn; ++j) {
          const double* row = rt.at + (int64_t)s_row[j] * B;
#pragma unroll
          for (int u = 0; u < kSubBPT; ++u) {
            int col = bk[u] - s_q[j];
            col += (col < 0) ? Bi : 0;
            const double w = __ldg(row + col);
            acc[u].x = fma(s_a[j].x, w, acc[u].x);
            acc[u].y = fma(s_a[j].y, w, acc[u].y);
          }
        }
      }
      continue;
    }
    if (live[0]) {
      const int tn = (int)((T - t0 < kSubChunk) ? (T - t0) : kSubChunk);
      // 4 tones x 2 buckets of table reads in flight, then the ordered updates
      int j = 0;
      for (; j + 4 <= tn; j += 4) {
        double2 w[4][kSubBPT];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const double2* row = gt + (int64_t)s_row[j + v] * B;
#pragma unroll
          for (int u = 0; u < kSubBPT; ++u) {
            int col = bk[u] - s_q[j + v];
            col += (col < 0) ? Bi : 0;
            w[v][u] = ld_table(row + col);
          }
        }
#pragma unroll
        for (int v = 0; v < 4; ++v)
#pragma unroll
          for (int u = 0; u < kSubBPT; ++u) acc[u] = csub(acc[u], cmul(s_a[j + v], w[v][u]));
      }
      for (; j < tn; ++j) {
        const double2* row = gt + (int64_t)s_row[j] * B;
#pragma unroll
        for (int u = 0; u < kSubBPT; ++u) {
          int col = bk[u] - s_q[j];
          col += (col < 0) ? Bi : 0;
          acc[u] = csub(acc[u], cmul(s_a[j], ld_table(row + col)));
        }
      }
    }
  }
  if (REAL) {
    // model = alpha_total + w^{b L h} S_b; running value y - model
    __syncthreads();
    const double2 al = s_alsum;
#pragma unroll
    for (int u = 0; u < kSubBPT; ++u) {
      if (!live[u]) continue;
      const double2 pb = unit_root(n, mulmod(mulmod(bk[u], L, n), rt.h % n, n));
      const double2 model = cadd(al, cmul(pb, acc[u]));
      acc[u] = TS == 1 ? csub(y[(int64_t)item * B + bk[u]], model) : cmk(-model.x, -model.y);
    }
  }
#pragma unroll
  for (int u = 0; u < kSubBPT; ++u) {
    if (!live[u]) continue;
    const int64_t i = i0 + u * kSubNT;
    if (TS == 1) out[(int64_t)item * nb + i] = acc[u];
    else part[((int64_t)item * gridDim.z + blockIdx.z) * nb + i] = acc[u];
  }
}

// out = y + sum of the (negated) split partial sums, in split order.
__global__ void k_sub_reduce(const double2* __restrict__ y, double2* __restrict__ out, int64_t B,
                             int64_t nb, const int32_t* blist, const int32_t* item_sig,
                             const int32_t* gate, const double2* __restrict__ part, int maxTS,
                             const int32_t* tcount, const int32_t* __restrict__ list) {
  const int item = list ? list[blockIdx.y] : blockIdx.y;
  const int sig = item_sig ? item_sig[item] : item;
  if (gate && !gate[sig]) return;
  const int TS = sub_splits(tcount[sig], maxTS);
  if (TS == 1) return;  // written in place by k_subtract
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const int64_t bk = blist ? blist[(int64_t)item * nb + i] : i;
  double2 acc = cmk(0.0, 0.0);
  for (int t = 0; t < TS; ++t) acc = cadd(acc, part[((int64_t)item * maxTS + t) * nb + i]);
  out[(int64_t)item * nb + i] = cadd(y[(int64_t)item * B + bk], acc);
}

// A_f = Re((B G_f - t0) w^{-f h}) in the transposed layout (f = rho + j L at
// rho * B + j); the imaginary part is rounding noise for a symmetric window.
__global__ void k_real_table(const double2* __restrict__ gt, const double* __restrict__ taps,
                             int64_t n, int64_t B, int64_t h, double* __restrict__ at) {
  const int64_t L = n / B;
  const double t0 = taps[0];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rho = e / B, j = e - rho * B;
    const int64_t f = rho + j * L;
    const double2 g = gt[e];
    const double2 w = unit_root(n, pmod(-mulmod(f, h % n, n), n));
    at[e] = (g.x * (double)B - t0) * w.x - (g.y * (double)B) * w.y;
  }
}

bool real_table_ok(int64_t omega) { return omega >= 2 && omega % 2 == 0 && !getenv("SFFT_NO_REAL_TABLE"); }

int build_real_table(const double2* gt, const double* taps, int64_t n, int64_t B, int64_t omega,
                     double* at, cudaStream_t st) {
  k_real_table<<<(unsigned)std::min<int64_t>(4096, cdiv_up(n, 256)), 256, 0, st>>>(gt, taps, n, B,
                                                                                 omega / 2, at);
  SFFT_CHECK_LAUNCH("k_real_table");
  return 0;
}

int run_subtract_gated(const double2* y, double2* out, int64_t B, int64_t nb,
                       const int32_t* blist, int64_t nitems, const double2* gt, int64_t n,
                       const int32_t* item_sig, const int64_t* sigma, const int64_t* tau_tot,
                       const int64_t* tpos, const double2* tcoef, const int32_t* tcount,
                       int64_t tstride, const int32_t* gate, cudaStream_t st, int TS,
                       double2* part, const RealTab* rt, const int32_t* list, int64_t nlist) {
  // list: the items to process (grid over the list instead of every item)
  if (list) nitems = nlist;
  if (nitems <= 0 || nb <= 0) return 0;
  if (TS < 1 || !part) TS = 1;
  dim3 g((unsigned)cdiv_up(nb, (int64_t)kSubNT * kSubBPT), (unsigned)nitems, (unsigned)TS);
  if (rt && rt->at) {
    k_subtract<true><<<g, kSubNT, 0, st>>>(y, out, B, nb, blist, gt, n, item_sig, sigma,
                                           tau_tot, tpos, tcoef, tcount, tstride, gate, part,
                                           *rt, list);
  } else {
    k_subtract<false><<<g, kSubNT, 0, st>>>(y, out, B, nb, blist, gt, n, item_sig, sigma,
                                            tau_tot, tpos, tcoef, tcount, tstride, gate, part,
                                            RealTab{}, list);
  }
  SFFT_CHECK_LAUNCH("k_subtract");
  if (TS > 1) {
    dim3 g2((unsigned)cdiv_up(nb, 256), (unsigned)nitems);
    k_sub_reduce<<<g2, 256, 0, st>>>(y, out, B, nb, blist, item_sig, gate, part, TS, tcount, list);
    SFFT_CHECK_LAUNCH("k_sub_reduce");
  }
  return 0;
}

int run_subtract(const double2* y, double2* out, int64_t B, int64_t nb, const int32_t* blist,
                 int64_t nitems, const double2* gt, int64_t n, const int32_t* item_sig,
                 const int64_t* sigma, const int64_t* tau_tot, const int64_t* tpos,
                 const double2* tcoef, const int32_t* tcount, int64_t tstride, cudaStream_t st) {
  return run_subtract_gated(y, out, B, nb, blist, nitems, gt, n, item_sig, sigma, tau_tot, tpos,
                            tcoef, tcount, tstride, nullptr, st);
}

}  // namespace sfft
