// Read schedules of the runners and the samples_read count.
//
// The reference marks a bool map per gathered index (sfft/signal.py:82-86)
// and counts it at the end (RecoveryResult.samples_read, sfft/frameworks.py:
// 151-155).  Here each signal logs its measurement groups instead — a flat
// group is one permutation sigma with a handful of extra shifts (the phase
// ladder, or the polish shifts 0/1/2; kind 2: an arithmetic shift set), a
// spike group one (stride, tau):
//   flat group g reads {sigma_g * t : t in U_g},  U_g = union_d [-tau-d, Omega-tau-d) mod n
// and k_mark_count_smem counts |union of read indices| exactly from bitmaps
// in shared memory.  No bookkeeping store touches HBM during the gathers.
#pragma once

#include "block.cuh"

namespace sfft {

constexpr int kMaxShifts = 16;
constexpr int kMaxGroups = 64;
constexpr int kMaxPieces = 2 * kMaxShifts;

// kind 2 (flat, arithmetic shifts): the split-location measurements of one
// loop iteration, shifts k*sh[0] for k < nsh (sfft/frameworks.py:524-529:
// d*(n/step) for d < step); nsh may exceed kMaxShifts.
struct Group {
  int64_t a;     // flat: sigma | spike: stride L
  int64_t tau;   // base shift
  int64_t cnt;   // flat: Omega | spike: number of samples
  int32_t kind;  // 0 flat, 1 spike, 2 flat with shifts k*sh[0], k < nsh
  int32_t nsh;   // extra shifts (flat) | shift count (kind 2)
  int64_t sh[kMaxShifts];
};

SFFT_HD int64_t modinv(int64_t a, int64_t n) {
  int64_t t = 0, nt = 1, r = n, nr = pmod(a, n);
  while (nr) {
    const int64_t q = r / nr;
    int64_t tmp = t - q * nt; t = nt; nt = tmp;
    tmp = r - q * nr; r = nr; nr = tmp;
  }
  return t < 0 ? t + n : t;
}

struct GroupSh {
  int64_t lo[kMaxPieces];
  int64_t hi[kMaxPieces];
  int np;
  int64_t total;
  int64_t ainv;
};

// Merge the circular intervals [s_d, s_d + omega) (mod n) into disjoint
// linear pieces of [0, n).  Single thread.
__device__ inline void merge_pieces(const Group& g, int64_t n, GroupSh* out) {
  int64_t lo[kMaxPieces], hi[kMaxPieces];
  int m = 0;
  if (g.kind == 1) {
    out->np = 0;
    out->total = g.cnt;
    out->ainv = 0;
    return;
  }
  const int64_t w = g.cnt >= n ? n : g.cnt;
  if (g.kind == 2) {  // arcs [-tau - k*step, +w): disjoint when step >= w, else one run
    const int64_t step = g.sh[0], c = g.nsh;
    out->np = 0;
    out->total = step >= w ? min(n, c * w) : min(n, (c - 1) * step + w);
    out->ainv = modinv(g.a, n);
    return;
  }
  for (int d = 0; d < g.nsh; ++d) {
    const int64_t s = pmod(-g.tau - g.sh[d], n);
    if (w >= n) { lo[m] = 0; hi[m] = n; ++m; continue; }
    if (s + w <= n) { lo[m] = s; hi[m] = s + w; ++m; }
    else { lo[m] = s; hi[m] = n; ++m; lo[m] = 0; hi[m] = s + w - n; ++m; }
  }
  // insertion sort by lo
  for (int i = 1; i < m; ++i) {
    const int64_t a = lo[i], b = hi[i];
    int j = i - 1;
    while (j >= 0 && lo[j] > a) { lo[j + 1] = lo[j]; hi[j + 1] = hi[j]; --j; }
    lo[j + 1] = a; hi[j + 1] = b;
  }
  int k = 0;
  int64_t tot = 0;
  for (int i = 0; i < m; ++i) {
    if (k > 0 && lo[i] <= out->hi[k - 1]) {
      if (hi[i] > out->hi[k - 1]) out->hi[k - 1] = hi[i];
    } else {
      out->lo[k] = lo[i];
      out->hi[k] = hi[i];
      ++k;
    }
  }
  for (int i = 0; i < k; ++i) tot += out->hi[i] - out->lo[i];
  out->np = k;
  out->total = tot;
  out->ainv = modinv(g.a, n);
}

// (a * b) mod n with a, b < n < 2^31; a mask when n is a power of two.
__device__ __forceinline__ int64_t mulmod_n(int64_t a, int64_t b, int64_t n, int64_t mask) {
  return mask >= 0 ? ((a * b) & mask) : (a * b) % n;
}

// e of element j of group g (j < gs.total)
__device__ __forceinline__ int64_t group_elem(const Group& g, const GroupSh& gs, int64_t n,
                                              int64_t j, int64_t mask) {
  if (g.kind == 1) return pmod(g.a * j - g.tau, n);
  if (g.kind == 2) {
    const int64_t w = g.cnt >= n ? n : g.cnt;
    const int64_t step = g.sh[0], c = g.nsh;
    int64_t u;
    if (w >= n) u = j;
    else if (step >= w) u = -g.tau - (j / w) * step + (j % w);
    else u = -g.tau - (c - 1) * step + j;
    return mulmod_n(g.a, pmod(u, n), n, mask);
  }
  for (int i = 0; i < gs.np; ++i) {
    const int64_t len = gs.hi[i] - gs.lo[i];
    if (j < len) return mulmod_n(g.a, gs.lo[i] + j, n, mask);
    j -= len;
  }
  return 0;
}

constexpr int kSchedWords = 5 + kMaxShifts;  // kind, a, tau, cnt, nsh, sh[]

// Export the groups as int64 records [S][kMaxGroups][kSchedWords].
static __global__ void k_export_groups(const Group* __restrict__ groups, const int32_t* ngroups,
                                       int S, int64_t* out, const int32_t* gate = nullptr,
                                       const int32_t* rows = nullptr) {
  const int s = blockIdx.x;
  if (gate && !gate[s]) return;
  const int64_t row = rows ? rows[s] : s;
  const int G = min(ngroups[s], kMaxGroups);
  for (int g = threadIdx.x; g < kMaxGroups; g += blockDim.x) {
    int64_t* o = out + (row * kMaxGroups + g) * kSchedWords;
    if (g >= G) {
      o[0] = -1;
      continue;
    }
    const Group& q = groups[(int64_t)s * kMaxGroups + g];
    o[0] = q.kind;
    o[1] = q.a;
    o[2] = q.tau;
    o[3] = q.cnt;
    o[4] = q.nsh;
    const int ns = q.kind == 2 ? 1 : q.nsh;
    for (int i = 0; i < kMaxShifts; ++i) o[5 + i] = i < ns ? q.sh[i] : 0;
  }
}

// samples[row of s] = 0 for the gated signals (before the count accumulates).
static __global__ void k_zero_rows(int64_t* v, int S, const int32_t* gate, const int32_t* rows) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S || (gate && !gate[s])) return;
  v[rows ? rows[s] : s] = 0;
}

// samples_read: CTA r of a finishing slot owns the index range
// [r R, (r+1) R) as an R-bit map in shared memory, walks every read of the
// slot's groups, sets the bits that fall in its range (shared atomics) and
// popcounts its map; samples[row] accumulates the CTAs' counts.  No global
// bitmap, no global atomics per read.
constexpr int kMarkNT = 1024;
constexpr int64_t kMarkBits = 176 * 1024 * 8;  // 176 KB of shared memory per CTA (N = 2^22: 3 CTAs)

static __global__ void __launch_bounds__(kMarkNT) k_mark_count_smem(
    const Group* __restrict__ groups, const int32_t* ngroups, int gstride, int64_t n,
    const int32_t* gate, const int32_t* rows, unsigned long long* samples) {
  extern __shared__ uint32_t mbits[];
  __shared__ Group sg[kMaxGroups];
  __shared__ GroupSh sp[kMaxGroups];
  __shared__ unsigned long long red[32];
  const int s = blockIdx.y;
  if (gate && !gate[s]) return;
  const int64_t r0 = (int64_t)blockIdx.x * kMarkBits;
  if (r0 >= n) return;
  const int64_t r1 = min(n, r0 + kMarkBits);
  const int64_t words = (r1 - r0 + 31) / 32;
  const int G = min(ngroups[s], kMaxGroups);
  const Group* gs = groups + (int64_t)s * gstride;
  const int64_t mask = (n & (n - 1)) == 0 ? n - 1 : -1;
  for (int i = threadIdx.x; i < G; i += kMarkNT) sg[i] = gs[i];
  for (int64_t w = threadIdx.x; w < words; w += kMarkNT) mbits[w] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < G; i += kMarkNT) merge_pieces(sg[i], n, &sp[i]);
  __syncthreads();
  for (int g = 0; g < G; ++g) {
    if (sg[g].kind == 0) {
      // flat pieces [lo, hi) of u: e = sigma u mod n, advanced incrementally
      const int64_t sig = sg[g].a;
      const int64_t step = mulmod(sig, kMarkNT % n, n);
      for (int i = 0; i < sp[g].np; ++i) {
        const int64_t lo = sp[g].lo[i], hi = sp[g].hi[i];
        int64_t u = lo + threadIdx.x;
        if (u >= hi) continue;
        int64_t e = mulmod(sig, u, n);
        for (; u < hi; u += kMarkNT) {
          if (e >= r0 && e < r1) {
            const int64_t o = e - r0;
            atomicOr(&mbits[o >> 5], 1u << (o & 31));
          }
          e += step;
          e -= (e >= n) ? n : 0;
        }
      }
      continue;
    }
    const int64_t tot = sp[g].total;
    for (int64_t j = threadIdx.x; j < tot; j += kMarkNT) {
      const int64_t e = group_elem(sg[g], sp[g], n, j, mask);
      if (e >= r0 && e < r1) {
        const int64_t o = e - r0;
        atomicOr(&mbits[o >> 5], 1u << (o & 31));
      }
    }
  }
  __syncthreads();
  unsigned long long c = 0;
  for (int64_t w = threadIdx.x; w < words; w += kMarkNT) c += __popc(mbits[w]);
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < kMarkNT / 32; ++i) t += red[i];
    if (t) atomicAdd(samples + (rows ? rows[s] : s), t);
  }
}

inline int run_union_smem(const Group* groups, const int32_t* ngroups, int S, int64_t n,
                          int64_t* samples, const int32_t* gate, const int32_t* rows,
                          cudaStream_t st) {
  k_zero_rows<<<(unsigned)((S + 127) / 128), 128, 0, st>>>(samples, S, gate, rows);
  SFFT_CHECK_LAUNCH("k_zero_rows");
  const size_t sm = (size_t)(std::min<int64_t>(n, kMarkBits) + 31) / 32 * sizeof(uint32_t);
  SFFT_CUDA(cudaFuncSetAttribute(k_mark_count_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
  dim3 g((unsigned)((n + kMarkBits - 1) / kMarkBits), S);
  k_mark_count_smem<<<g, kMarkNT, sm, st>>>(groups, ngroups, kMaxGroups, n, gate, rows,
                                            (unsigned long long*)samples);
  SFFT_CHECK_LAUNCH("k_mark_count_smem");
  return 0;
}

}  // namespace sfft
