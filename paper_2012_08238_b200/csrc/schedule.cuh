// Read schedules of the runners and the samples_read count.
//
// The reference marks a bool map per gathered index (sfft/signal.py:82-86)
// and counts it at the end (RecoveryResult.samples_read, sfft/frameworks.py:
// 151-155).  Here each signal logs its measurement groups instead — a flat
// group is one permutation sigma with a handful of extra shifts (the phase
// ladder, or the polish shifts 0/1/2; kind 2: an arithmetic shift set), a
// spike group one (stride, tau):
//   flat group g reads {sigma_g * t : t in U_g},  U_g = union_d [-tau-d, Omega-tau-d) mod n
// and k_union_excl(_p2) counts |union of read indices| exactly by exclusion
// (no bitmap).  No bookkeeping store touches HBM during the gathers.
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

// Is index e read by group g?  (The inverse of group_elem.)
__device__ __forceinline__ bool group_has(const Group& g, const GroupSh& gs, int64_t n, int64_t e,
                                          int64_t mask) {
  if (g.kind == 1) {  // e = a j - tau, j < cnt (a cnt <= n)
    const int64_t v = pmod(e + g.tau, n);
    return v % g.a == 0 && v / g.a < g.cnt;
  }
  const int64_t u = mulmod_n(gs.ainv, e, n, mask);
  if (g.kind == 2) {
    const int64_t w = g.cnt >= n ? n : g.cnt;
    if (w >= n) return true;
    const int64_t step = g.sh[0], c = g.nsh;
    if (step < w) return pmod(u + g.tau + (c - 1) * step, n) < (c - 1) * step + w;
    // arcs [-tau - k step, +w), k < c, c step <= n: v = u + tau, v + k step in [0, w) mod n
    const int64_t v = pmod(u + g.tau, n);
    if (v < w) return true;
    const int64_t k = (n - v + step - 1) / step;
    return k < c && k * step < n - v + w;
  }
  for (int i = 0; i < gs.np; ++i)
    if (u >= gs.lo[i] && u < gs.hi[i]) return true;
  return false;
}

// samples_read without a bitmap: |U_g P_g| = sum_g |P_g \ U_{h<g} P_h|.  Each
// element of group g (its reads are distinct) is tested against the groups
// before it with the inverse map (one modular multiply and a few interval
// compares per test); no shared-memory atomics, no bitmap.  The CTAs of a
// slot split its elements; samples[row] accumulates their counts.
constexpr int kUxNT = 256;

static __global__ void __launch_bounds__(kUxNT) k_union_excl(
    const Group* __restrict__ groups, const int32_t* ngroups, int gstride, int64_t n,
    const int32_t* gate, const int32_t* rows, unsigned long long* samples) {
  __shared__ Group sg[kMaxGroups];
  __shared__ GroupSh sp[kMaxGroups];
  __shared__ unsigned long long red[kUxNT / 32];
  const int s = blockIdx.y;
  if (gate && !gate[s]) return;
  const int G = min(ngroups[s], kMaxGroups);
  const Group* gs = groups + (int64_t)s * gstride;
  const int64_t mask = (n & (n - 1)) == 0 ? n - 1 : -1;
  for (int i = threadIdx.x; i < G; i += kUxNT) sg[i] = gs[i];
  __syncthreads();
  for (int i = threadIdx.x; i < G; i += kUxNT) merge_pieces(sg[i], n, &sp[i]);
  __syncthreads();
  unsigned long long c = 0;
  const int64_t stride = (int64_t)gridDim.x * kUxNT;
  const int64_t t0 = (int64_t)blockIdx.x * kUxNT + threadIdx.x;
  bool full = false;
  for (int g = 0; g < G; ++g) full |= sp[g].total >= n;
  if (full) {
    if (t0 == 0) c = n;
  } else {
    if (t0 == 0 && G > 0) c = sp[0].total;
    for (int g = 1; g < G; ++g) {
      const int64_t tot = sp[g].total;
      for (int64_t j = t0; j < tot; j += stride) {
        const int64_t e = group_elem(sg[g], sp[g], n, j, mask);
        bool seen = false;
        for (int h = 0; h < g && !seen; ++h) seen = group_has(sg[h], sp[h], n, e, mask);
        c += !seen;
      }
    }
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < kUxNT / 32; ++i) t += red[i];
    if (t) atomicAdd(samples + (rows ? rows[s] : s), t);
  }
}

// Power-of-two n with flat groups only (the phase-location runners): the same
// exclusion count in 32-bit arithmetic, since (a b) mod 2^m is the low m bits
// of the wrapping 32-bit product.  Per test: one multiply, one mask and an
// unsigned compare per merged piece.  A slot with another group kind sets
// *fallback and is left to k_union_excl.
constexpr int kUxPieces = 8;

static __global__ void __launch_bounds__(kUxNT) k_union_excl_p2(
    const Group* __restrict__ groups, const int32_t* ngroups, int gstride, int64_t n,
    const int32_t* gate, const int32_t* rows, unsigned long long* samples, int32_t* fallback) {
  __shared__ uint32_t f_sig[kMaxGroups], f_inv[kMaxGroups];
  __shared__ int32_t f_np[kMaxGroups];
  __shared__ uint32_t f_lo[kMaxGroups][kUxPieces], f_len[kMaxGroups][kUxPieces];
  __shared__ int s_bad;
  __shared__ unsigned long long red[kUxNT / 32];
  const int s = blockIdx.y;
  if (gate && !gate[s]) return;
  const int G = min(ngroups[s], kMaxGroups);
  const Group* gs = groups + (int64_t)s * gstride;
  const uint32_t mask = (uint32_t)(n - 1);
  if (threadIdx.x == 0) s_bad = 0;
  __syncthreads();
  for (int g = threadIdx.x; g < G; g += kUxNT) {
    const Group q = gs[g];
    GroupSh p;
    if (q.kind != 0) {
      s_bad = 1;
      continue;
    }
    merge_pieces(q, n, &p);
    if (p.np > kUxPieces || p.total >= n) {
      s_bad = 1;
      continue;
    }
    f_sig[g] = (uint32_t)q.a;
    f_inv[g] = (uint32_t)p.ainv;
    f_np[g] = p.np;
    for (int i = 0; i < p.np; ++i) {
      f_lo[g][i] = (uint32_t)p.lo[i];
      f_len[g][i] = (uint32_t)(p.hi[i] - p.lo[i]);
    }
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0 && blockIdx.x == 0) fallback[s] = 1;
    return;
  }
  const uint32_t stride = gridDim.x * kUxNT;
  const uint32_t t0 = blockIdx.x * kUxNT + threadIdx.x;
  unsigned long long c = 0;
  if (t0 == 0 && G > 0)
    for (int i = 0; i < f_np[0]; ++i) c += f_len[0][i];
  // kUxE elements per thread in registers; each earlier group's parameters are
  // read from shared memory once per batch (not once per test)
  constexpr int kUxE = 16;
  for (int g = 1; g < G; ++g) {
    const uint32_t sg = f_sig[g];
    for (int i = 0; i < f_np[g]; ++i) {
      const uint32_t lo = f_lo[g][i], len = f_len[g][i];
      for (uint32_t o0 = t0; o0 < len; o0 += kUxE * stride) {
        uint32_t e[kUxE];
        uint32_t live = 0;
#pragma unroll
        for (int k = 0; k < kUxE; ++k) {
          const uint32_t o = o0 + k * stride;
          e[k] = (sg * (lo + o)) & mask;
          live |= (o < len ? 1u : 0u) << k;
        }
        uint32_t seen = 0;
        for (int h = 0; h < g; ++h) {
          const uint32_t inv = f_inv[h];
          const int np = f_np[h];
          const uint32_t l0 = f_lo[h][0], n0 = f_len[h][0];
          const uint32_t l1 = np > 1 ? f_lo[h][1] : 0u, n1 = np > 1 ? f_len[h][1] : 0u;
#pragma unroll
          for (int k = 0; k < kUxE; ++k) {
            const uint32_t u = (inv * e[k]) & mask;
            const bool in = (((u - l0) & mask) < n0) | (((u - l1) & mask) < n1);
            seen |= (in ? 1u : 0u) << k;
          }
          for (int p = 2; p < np; ++p) {
            const uint32_t lp = f_lo[h][p], npl = f_len[h][p];
#pragma unroll
            for (int k = 0; k < kUxE; ++k) {
              const uint32_t u = (inv * e[k]) & mask;
              seen |= ((((u - lp) & mask) < npl) ? 1u : 0u) << k;
            }
          }
        }
        c += __popc(live & ~seen);
      }
    }
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int i = 0; i < kUxNT / 32; ++i) t += red[i];
    if (t) atomicAdd(samples + (rows ? rows[s] : s), t);
  }
}

// fallback[s] set by k_union_excl_p2: this slot takes the general kernel.
static __global__ void k_union_gate(int S, const int32_t* gate, const int32_t* fallback,
                                    int32_t* out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < S) out[s] = (!gate || gate[s]) && fallback[s];
}

// Scratch for run_union_count's fallback gate: 2 ints per slot.
// (a third int per slot is the caller's: the voting runner keeps its
// shared-schedule gate there)
inline size_t union_scratch_bytes(int S) { return sizeof(int32_t) * 3 * (size_t)S; }

inline int run_union_count(const Group* groups, const int32_t* ngroups, int S, int64_t n,
                          int64_t* samples, const int32_t* gate, const int32_t* rows,
                          cudaStream_t st, int32_t* scratch = nullptr, int ctas_min = 1) {
  k_zero_rows<<<(unsigned)((S + 127) / 128), 128, 0, st>>>(samples, S, gate, rows);
  SFFT_CHECK_LAUNCH("k_zero_rows");
  const unsigned ctas = (unsigned)std::max<int64_t>(
      ctas_min, std::min<int64_t>(8, std::max<int64_t>(1, n >> 20)));
  const bool p2 = (n & (n - 1)) == 0 && n <= (int64_t(1) << 31) && scratch;
  const int32_t* g2 = gate;
  if (p2) {
    SFFT_CUDA(cudaMemsetAsync(scratch, 0, sizeof(int32_t) * S, st));
    k_union_excl_p2<<<dim3(ctas, S), kUxNT, 0, st>>>(groups, ngroups, kMaxGroups, n, gate, rows,
                                                     (unsigned long long*)samples, scratch);
    SFFT_CHECK_LAUNCH("k_union_excl_p2");
    k_union_gate<<<(unsigned)((S + 127) / 128), 128, 0, st>>>(S, gate, scratch, scratch + S);
    SFFT_CHECK_LAUNCH("k_union_gate");
    g2 = scratch + S;
  }
  k_union_excl<<<dim3(ctas, S), kUxNT, 0, st>>>(groups, ngroups, kMaxGroups, n, g2, rows,
                                                (unsigned long long*)samples);
  SFFT_CHECK_LAUNCH("k_union_excl");
  return 0;
}

}  // namespace sfft
