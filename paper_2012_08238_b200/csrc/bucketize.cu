// Bucketization (the encode stage), sm_100a.
//
// Flat window (sfft/bucketize.py:142-161):
//   y[j] = FFT_B( fold_B( g[i] * x[sigma*(i - tau_tot) mod N] * w_N^{b'sigma*i} ) )[j] / B
// Spike train (sfft/bucketize.py:164-178):
//   y[j] = FFT_B( x[(N/B)*i - tau mod N] )[j] / B
// Response table (sfft/filters.py:146-149, transposed to [L][B]):
//   T[rho][j] = G[rho + j*L] = FFT_B( fold_B( g[i] * w_N^{rho*i} ) )[j] / B
//
// One CTA owns one bucketization (item) when B <= kFusedMaxB: every thread
// owns whole slots s and sums the ceil(Omega/B) rows of its slot in row
// order (the reference's fold order, no atomics), the slots land in shared
// memory, and the CTA runs the B-point FFT in place.  Larger B (config 5,
// FFAST stages) use a four-step split B = B1*B2 whose column pass produces
// the slots directly (no z round trip) and whose row pass writes y.
#include <cooperative_groups.h>

#include <mutex>

#include "kernels.cuh"

namespace sfft {

struct ItemCtx {
  const void* xs;
  int64_t a, b, c;
  int64_t step;    // flat: sigma*B mod n
  int64_t estep;   // flat: bsig*B mod n
  bool skip;
};

template <int MODE>
__device__ __forceinline__ ItemCtx item_ctx(const Prod& p, int item, int elem_bytes) {
  ItemCtx c;
  const int sig = p.item_sig ? p.item_sig[item] : item;
  c.skip = (p.active && !p.active[sig]) || (p.item_active && !p.item_active[item]);
  c.xs = p.x ? (const char*)p.x + (int64_t)sig * p.xstride * elem_bytes : nullptr;
  c.a = p.item_a ? p.item_a[item] : 0;
  c.b = p.item_b ? p.item_b[item] : 0;
  c.c = p.item_c ? p.item_c[item] : 0;
  c.step = 0;
  c.estep = 0;
  if (MODE == PROD_FLAT) {
    c.step = mulmod(c.a, p.B % p.n, p.n);
    c.estep = mulmod(c.c, p.B % p.n, p.n);
  }
  return c;
}

template <typename Tin, int MODE>
__device__ __forceinline__ double2 produce(const Prod& p, const ItemCtx& c, int item,
                                           int64_t s) {
  const int64_t n = p.n;
  if (MODE == PROD_FLAT) {
    const Tin* xs = (const Tin*)c.xs;
    int64_t idx = mulmod(c.a, pmod(s - c.b, n), n);
    double2 acc = cmk(0.0, 0.0);
    if (c.c == 0) {
      // rows in order, 4 gathers in flight per step
      int64_t i = s;
      for (; i + 3 * p.B < p.omega; i += 4 * p.B) {
        int64_t i1 = idx + c.step; i1 -= (i1 >= n) ? n : 0;
        int64_t i2 = i1 + c.step;  i2 -= (i2 >= n) ? n : 0;
        int64_t i3 = i2 + c.step;  i3 -= (i3 >= n) ? n : 0;
        const double2 v0 = Sample<Tin>::load(xs, idx);
        const double2 v1 = Sample<Tin>::load(xs, i1);
        const double2 v2 = Sample<Tin>::load(xs, i2);
        const double2 v3 = Sample<Tin>::load(xs, i3);
        const double g0 = __ldg(p.taps + i), g1 = __ldg(p.taps + i + p.B);
        const double g2 = __ldg(p.taps + i + 2 * p.B), g3 = __ldg(p.taps + i + 3 * p.B);
        acc = cadd_rn(acc, cmk(__dmul_rn(g0, v0.x), __dmul_rn(g0, v0.y)));
        acc = cadd_rn(acc, cmk(__dmul_rn(g1, v1.x), __dmul_rn(g1, v1.y)));
        acc = cadd_rn(acc, cmk(__dmul_rn(g2, v2.x), __dmul_rn(g2, v2.y)));
        acc = cadd_rn(acc, cmk(__dmul_rn(g3, v3.x), __dmul_rn(g3, v3.y)));
        idx = i3 + c.step;
        idx -= (idx >= n) ? n : 0;
      }
      for (; i < p.omega; i += p.B) {
        const double2 v = Sample<Tin>::load(xs, idx);
        const double g = __ldg(p.taps + i);
        acc = cadd_rn(acc, cmk(__dmul_rn(g, v.x), __dmul_rn(g, v.y)));
        idx += c.step;
        idx -= (idx >= n) ? n : 0;
      }
    } else {
      int64_t e = mulmod(c.c, s % n, n);
      for (int64_t i = s; i < p.omega; i += p.B) {
        const double2 v = Sample<Tin>::load(xs, idx);
        const double g = __ldg(p.taps + i);
        const double2 z = cmk(__dmul_rn(g, v.x), __dmul_rn(g, v.y));
        acc = cadd_rn(acc, cmul_rn(z, unit_root(n, e)));
        idx += c.step;
        idx -= (idx >= n) ? n : 0;
        e += c.estep;
        e -= (e >= n) ? n : 0;
      }
    }
    return acc;
  } else if (MODE == PROD_SPIKE) {
    const Tin* xs = (const Tin*)c.xs;
    const int64_t L = n / p.B;
    return Sample<Tin>::load(xs, pmod(L * s - c.a, n));
  } else if (MODE == PROD_DIRICHLET) {
    // conj of the folded box window: sum over rows r of
    // (taps[i] * x[(t - i) mod n]) * hm_i, i = s + r B < L, hm_i = w^{-(L/2) i}
    // unless half_offset (the forward FFT of the conjugate is the inverse one)
    const Tin* xs = (const Tin*)c.xs;
    const int64_t L = p.omega, t = pmod(c.a, n);
    double2 acc = cmk(0.0, 0.0);
    for (int64_t i = s; i < L; i += p.B) {
      double2 w = cmul_rn(p.ctaps[i], Sample<Tin>::load(xs, pmod(t - i, n)));
      if (!p.half_offset) w = cmul_rn(w, unit_root(n, pmod(-mulmod((L / 2) % n, i % n, n), n)));
      acc = cadd_rn(acc, w);
    }
    return cmk(acc.x, -acc.y);
  } else if (MODE == PROD_GTAB) {
    double2 acc = cmk(0.0, 0.0);
    int64_t e = mulmod(c.a, s % n, n);
    const int64_t estep = mulmod(c.a, p.B % n, n);
    for (int64_t i = s; i < p.omega; i += p.B) {
      const double g = __ldg(p.taps + i);
      const double2 w = unit_root(n, e);
      acc.x += g * w.x;
      acc.y += g * w.y;
      e += estep;
      e -= (e >= n) ? n : 0;
    }
    return acc;
  } else {
    return p.z[out_row(p, item) * p.B + s];
  }
}

// Two flat slots at once (8 gathers in flight per thread): slot s0 of item
// ca and slot s1 >= s0 of item cb (the same or another item).  Each slot's
// rows are still summed in row order without FMA contraction.
template <typename Tin>
__device__ __forceinline__ void produce_flat2(const Prod& p, const ItemCtx& ca, int64_t s0,
                                              const ItemCtx& cb, int64_t s1, double2* o0,
                                              double2* o1) {
  const int64_t n = p.n;
  const Tin* xa = (const Tin*)ca.xs;
  const Tin* xb = (const Tin*)cb.xs;
  int64_t ia = mulmod(ca.a, pmod(s0 - ca.b, n), n);
  int64_t ib = mulmod(cb.a, pmod(s1 - cb.b, n), n);
  double2 aa = cmk(0.0, 0.0), ab = cmk(0.0, 0.0);
  int64_t i = s0, k = s1;
  const int64_t B = p.B;
  // s1 > s0, so slot s1 runs out of rows first or at the same time
  for (; k + 3 * B < p.omega; i += 4 * B, k += 4 * B) {
    int64_t ia1 = ia + ca.step; ia1 -= (ia1 >= n) ? n : 0;
    int64_t ia2 = ia1 + ca.step; ia2 -= (ia2 >= n) ? n : 0;
    int64_t ia3 = ia2 + ca.step; ia3 -= (ia3 >= n) ? n : 0;
    int64_t ib1 = ib + cb.step; ib1 -= (ib1 >= n) ? n : 0;
    int64_t ib2 = ib1 + cb.step; ib2 -= (ib2 >= n) ? n : 0;
    int64_t ib3 = ib2 + cb.step; ib3 -= (ib3 >= n) ? n : 0;
    const double2 va0 = Sample<Tin>::load(xa, ia), va1 = Sample<Tin>::load(xa, ia1);
    const double2 va2 = Sample<Tin>::load(xa, ia2), va3 = Sample<Tin>::load(xa, ia3);
    const double2 vb0 = Sample<Tin>::load(xb, ib), vb1 = Sample<Tin>::load(xb, ib1);
    const double2 vb2 = Sample<Tin>::load(xb, ib2), vb3 = Sample<Tin>::load(xb, ib3);
    const double ga0 = __ldg(p.taps + i), ga1 = __ldg(p.taps + i + B);
    const double ga2 = __ldg(p.taps + i + 2 * B), ga3 = __ldg(p.taps + i + 3 * B);
    const double gb0 = __ldg(p.taps + k), gb1 = __ldg(p.taps + k + B);
    const double gb2 = __ldg(p.taps + k + 2 * B), gb3 = __ldg(p.taps + k + 3 * B);
    aa = cadd_rn(aa, cmk(__dmul_rn(ga0, va0.x), __dmul_rn(ga0, va0.y)));
    aa = cadd_rn(aa, cmk(__dmul_rn(ga1, va1.x), __dmul_rn(ga1, va1.y)));
    aa = cadd_rn(aa, cmk(__dmul_rn(ga2, va2.x), __dmul_rn(ga2, va2.y)));
    aa = cadd_rn(aa, cmk(__dmul_rn(ga3, va3.x), __dmul_rn(ga3, va3.y)));
    ab = cadd_rn(ab, cmk(__dmul_rn(gb0, vb0.x), __dmul_rn(gb0, vb0.y)));
    ab = cadd_rn(ab, cmk(__dmul_rn(gb1, vb1.x), __dmul_rn(gb1, vb1.y)));
    ab = cadd_rn(ab, cmk(__dmul_rn(gb2, vb2.x), __dmul_rn(gb2, vb2.y)));
    ab = cadd_rn(ab, cmk(__dmul_rn(gb3, vb3.x), __dmul_rn(gb3, vb3.y)));
    ia = ia3 + ca.step; ia -= (ia >= n) ? n : 0;
    ib = ib3 + cb.step; ib -= (ib >= n) ? n : 0;
  }
  // tails (slot a: at most 4 rows left, slot b: at most 3): every load in
  // flight at once, then the adds in row order
  Tin ta[4], tb[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (i + u * B < p.omega) ta[u] = __ldcg(xa + ia);
    if (k + u * B < p.omega) tb[u] = __ldcg(xb + ib);
    ia += ca.step;
    ia -= (ia >= n) ? n : 0;
    ib += cb.step;
    ib -= (ib >= n) ? n : 0;
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (i + u * B < p.omega) {
      const double2 v = to_d2_(ta[u]);
      const double g = __ldg(p.taps + i + u * B);
      aa = cadd_rn(aa, cmk(__dmul_rn(g, v.x), __dmul_rn(g, v.y)));
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (k + u * B < p.omega) {
      const double2 v = to_d2_(tb[u]);
      const double g = __ldg(p.taps + k + u * B);
      ab = cadd_rn(ab, cmk(__dmul_rn(g, v.x), __dmul_rn(g, v.y)));
    }
  }
  // rows beyond those (only when s1 - s0 >= B; no caller does that)
  for (i += 4 * B; i < p.omega; i += B) {
    const double2 v = Sample<Tin>::load(xa, ia);
    const double g = __ldg(p.taps + i);
    aa = cadd_rn(aa, cmk(__dmul_rn(g, v.x), __dmul_rn(g, v.y)));
    ia += ca.step;
    ia -= (ia >= n) ? n : 0;
  }
  for (k += 4 * B; k < p.omega; k += B) {
    const double2 v = Sample<Tin>::load(xb, ib);
    const double g = __ldg(p.taps + k);
    ab = cadd_rn(ab, cmk(__dmul_rn(g, v.x), __dmul_rn(g, v.y)));
    ib += cb.step;
    ib -= (ib >= n) ? n : 0;
  }
  *o0 = aa;
  *o1 = ab;
}

constexpr int kNT = 512;

template <typename Tin, int MODE>
__global__ void __launch_bounds__(kNT) k_fused(Prod p, FftPlan P, const double2* __restrict__ W,
                                               double2* __restrict__ out) {
  extern __shared__ double2 sm[];
  const int item = blockIdx.x;
  const ItemCtx c = item_ctx<MODE>(p, item, sizeof(Tin));
  if (c.skip) return;
  if (p.prof_items && threadIdx.x == 0) atomicAdd(p.prof_items, 1ull);
  const int B = (int)p.B;
  for (int s = threadIdx.x; s < B; s += kNT) sm[s] = produce<Tin, MODE>(p, c, item, s);
  __syncthreads();
  fft_dif(sm, 1, B, P, W, B, threadIdx.x, kNT);
  double2* o = out + out_row(p, item) * B;
  const double bd = (double)B;
  for (int k = threadIdx.x; k < B; k += kNT) o[k] = cdivr(sm[fft_pos(k, P)], bd);
}

// Cluster path (B = CL * M, power of two, CL in {2,4,8}, M in {256, 512,
// 1024}): the CL CTAs of a thread-block cluster own NI consecutive items (see
// cluster_items).  CTA q folds slots
// [qM, qM + M) of every item into shared memory (rows in reference order,
// fp64, no atomics); the radix-CL first DIF stage reads the CL slot slices
// over DSMEM (b_q[j] = w_B^{jq} sum_p a_p[j] w_CL^{pq}, q = cluster rank);
// each CTA then runs the NI length-M sub-transforms with radix-8 register
// butterflies (twiddles in shared memory, digit reversal by shifts):
// y[q + CL k] = FFT_M(b_q)[k] / B.  A 77k-sample gather is spread over CL SMs.
constexpr int kClNT = 256;

// the complex64 flat gather is latency bound: cap registers at 64 so that 4
// CTAs (1024 threads) share an SM; other instantiations keep their registers
template <typename Tin, int MODE>
constexpr int cluster_min_blocks() {
  return (MODE == PROD_FLAT && sizeof(Tin) == 8) ? 4 : 1;
}

// items per cluster: one for the gathering producers (the 8 measurements of a
// slot then run in 8 clusters side by side and share their L2 lines), 2048/M
// (one butterfly per thread and FFT stage) for the gather-free ones
template <int MODE, int M>
constexpr int cluster_items() {
  return (MODE == PROD_FLAT || MODE == PROD_SPIKE) ? 1 : 2048 / M;
}

template <typename Tin, int MODE, int CL, int M>
__global__ void __launch_bounds__(kClNT, cluster_min_blocks<Tin, MODE>())
    k_cluster(Prod p, int64_t nitems, const double2* __restrict__ W, double2* __restrict__ out,
              int strided_off) {
  constexpr int NI = cluster_items<MODE, M>();
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  extern __shared__ double2 sm[];
  __shared__ int s_live[NI];
  __shared__ ItemCtx s_ctx[NI];
  const int q = (int)cl.block_rank();
  const int64_t item0 = (int64_t)(blockIdx.x / CL) * NI;
  const int B = CL * M;
  double2* a = sm;               // [NI][M] folded slots of this CTA
  double2* bq = sm + NI * M;     // [NI][M] sub-transform inputs
  double2* tw = bq + NI * M;     // [M] w_M^e
  if (threadIdx.x < NI) {
    const int64_t it = item0 + threadIdx.x;
    const bool in = it < nitems;
    const ItemCtx c = item_ctx<MODE>(p, in ? (int)it : 0, sizeof(Tin));
    s_ctx[threadIdx.x] = c;
    s_live[threadIdx.x] = in && !c.skip;
  }
  for (int e = threadIdx.x; e < M; e += kClNT) tw[e] = __ldg(W + (int64_t)e * CL);
  __syncthreads();
  int nl = 0;
#pragma unroll
  for (int i = 0; i < NI; ++i) nl += s_live[i];
  if (nl == 0) return;  // uniform over the cluster (same items)
  if (p.prof_items && threadIdx.x == 0 && q == 0) atomicAdd(p.prof_items, (unsigned long long)nl);
  constexpr int NJ = M / CL;
  // ---- strided-ownership fold (flat gathers, one item): CTA q folds the
  // slots n1 M + n2 for every n1 < CL and its own n2 slice [q NJ, (q+1) NJ),
  // so the radix-CL stage over n1 is local; its CL outputs (times w_B^{n2 k1})
  // go straight to CTA k1.  One cluster barrier instead of two, and every
  // folded value crosses the cluster once.  Bit-identical to the pull form.
  if (NI == 1 && MODE == PROD_FLAT && s_ctx[0].c == 0 && (M / 2) % kClNT == 0 &&
      !strided_off) {
    const ItemCtx c = s_ctx[0];
    // every CTA of the cluster must have started before any DSMEM access: a
    // relaxed arrive now, its wait after the fold (overlapped with the gathers)
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    // local index j = n1 NJ + jj  ->  slot n1 M + q NJ + jj; pairs (j, j + M/2)
    for (int j = threadIdx.x; j < M / 2; j += kClNT) {
      const int j2 = j + M / 2;
      const int64_t s0 = (int64_t)(j / NJ) * M + q * NJ + (j % NJ);
      const int64_t s1 = (int64_t)(j2 / NJ) * M + q * NJ + (j2 % NJ);
      produce_flat2<Tin>(p, c, s0, c, s1, &a[j], &a[j2]);
    }
    __syncthreads();
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    for (int jj = threadIdx.x; jj < NJ; jj += kClNT) {
      const int n2 = q * NJ + jj;
      double2 v[8];
#pragma unroll
      for (int r = 0; r < CL; ++r) v[r] = a[r * NJ + jj];
      if (CL == 8) {
        dft8_(v);
      } else if (CL == 4) {
        dft4_(v[0], v[1], v[2], v[3]);
      } else {
        const double2 u = v[0];
        v[0] = cadd(u, v[1]);
        v[1] = csub(u, v[1]);
      }
#pragma unroll
      for (int r = 0; r < CL; ++r)
        cl.map_shared_rank(bq, r)[n2] = (n2 * r) ? cmul(v[r], __ldg(W + n2 * r)) : v[r];
    }
  } else {
    // ---- fold: every slot of the NI items in turn, item pairs side by side, so
    // the shifted measurements of one signal re-read their samples from L2
    if (NI == 1 && MODE == PROD_FLAT && M % (2 * kClNT) == 0 && s_ctx[0].c == 0) {
      // two slots per call, 8 gathers in flight
      const ItemCtx c = s_ctx[0];
      for (int j = threadIdx.x; j < M; j += 2 * kClNT)
        produce_flat2<Tin>(p, c, (int64_t)q * M + j, c, (int64_t)q * M + j + kClNT, &a[j],
                           &a[j + kClNT]);
    } else {
      for (int j = threadIdx.x; j < M; j += kClNT) {
        const int64_t sl = (int64_t)q * M + j;
#pragma unroll
        for (int i = 0; i < NI; ++i)
          if (s_live[i]) a[i * M + j] = produce<Tin, MODE>(p, s_ctx[i], (int)(item0 + i), sl);
      }
    }
    cl.sync();
    // ---- radix-CL stage over DSMEM: CTA q takes slots j in [q M/CL, (q+1) M/CL)
    // of every CTA, forms the CL-point DFT over the CTAs and scatters output
    // q' (times w_B^{j q'}) to CTA q' -- every folded value crosses the cluster
    // once
    for (int t = threadIdx.x; t < NI * NJ; t += kClNT) {
      const int i = t / NJ;
      const int j = q * NJ + (t - i * NJ);
      double2 v[8];
#pragma unroll
      for (int r = 0; r < CL; ++r) v[r] = cl.map_shared_rank(a, r)[i * M + j];
      if (CL == 8) {
        dft8_(v);
      } else if (CL == 4) {
        dft4_(v[0], v[1], v[2], v[3]);
      } else {
        const double2 u = v[0];
        v[0] = cadd(u, v[1]);
        v[1] = csub(u, v[1]);
      }
#pragma unroll
      for (int r = 0; r < CL; ++r)
        cl.map_shared_rank(bq, r)[i * M + j] = (j * r) ? cmul(v[r], __ldg(W + j * r)) : v[r];
    }
  }
  cl.sync();  // all slices scattered (and all remote reads of a done)
  // ---- NI sub-transforms of length M
  fft_pow2<M, NI, kClNT>(bq, tw);
  const double bd = (double)B;
  for (int t = threadIdx.x; t < NI * M; t += kClNT) {
    const int i = t / M, k = t - i * M;
    if (!s_live[i]) continue;
    out[out_row(p, item0 + i) * B + q + (int64_t)CL * k] = cdivr(bq[i * M + pow2_pos<M>(k)], bd);
  }
}

template <typename Tin, int MODE, int CL, int M>
static int launch_cluster_m(const Prod& p, int64_t nitems, const double2* W, double2* out,
                            cudaStream_t st) {
  constexpr int NI = cluster_items<MODE, M>();
  const size_t sm = (size_t)(2 * NI * M + M) * sizeof(double2);
  auto kern = k_cluster<Tin, MODE, CL, M>;
  SFFT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(cdiv_up(nitems, NI) * CL));
  cfg.blockDim = dim3(kClNT);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const int strided_off = getenv("SFFT_NO_STRIDED_FOLD") ? 1 : 0;
  SFFT_CUDA(cudaLaunchKernelEx(&cfg, kern, p, nitems, W, out, strided_off));
  SFFT_CHECK_LAUNCH("k_cluster");
  return 0;
}

template <typename Tin, int MODE, int CL>
static int launch_cluster(const Prod& p, int64_t nitems, const double2* W, double2* out,
                          cudaStream_t st) {
  const int64_t M = p.B / CL;
  if (M == 256) return launch_cluster_m<Tin, MODE, CL, 256>(p, nitems, W, out, st);
  if (M == 512) return launch_cluster_m<Tin, MODE, CL, 512>(p, nitems, W, out, st);
  if (M == 1024) return launch_cluster_m<Tin, MODE, CL, 1024>(p, nitems, W, out, st);
  set_error("bucketize: cluster slice must be 256, 512 or 1024 slots");
  return -2;
}

// cluster size for B (0: use the one-CTA path)
static int cluster_size(int64_t B) {
  if (B < 1024 || B > kFusedMaxB || (B & (B - 1))) return 0;
  const int64_t M = std::max<int64_t>(256, B / 8);
  return (int)(B / M);
}

// Four-step column pass: DFT_B1 over n1 of z[n1*B2 + n2] for CG columns, times
// w_B^{n2*k1}, stored at ws[k1*B2 + n2].
template <typename Tin, int MODE>
__global__ void __launch_bounds__(kNT) k_cols(Prod p, FftPlan P1, int B1, int B2, int CG,
                                              const double2* __restrict__ W,
                                              double2* __restrict__ ws) {
  extern __shared__ double2 sm[];
  const int item = blockIdx.y;
  const ItemCtx c = item_ctx<MODE>(p, item, sizeof(Tin));
  if (c.skip) return;
  if (p.prof_items && threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p.prof_items, 1ull);
  const int c0 = blockIdx.x * CG;
  const int seg = B1 + 1;
  const int B = (int)p.B;
  for (int t = threadIdx.x; t < CG * B1; t += kNT) {
    const int g = t % CG, n1 = t / CG;
    const int n2 = c0 + g;
    sm[g * seg + n1] = (n2 < B2) ? produce<Tin, MODE>(p, c, item, (int64_t)n1 * B2 + n2)
                                 : cmk(0.0, 0.0);
  }
  __syncthreads();
  fft_dif(sm, CG, seg, P1, W, B, threadIdx.x, kNT);
  double2* o = ws + (int64_t)item * B;
  for (int t = threadIdx.x; t < CG * B1; t += kNT) {
    const int g = t % CG, k1 = t / CG;
    const int n2 = c0 + g;
    if (n2 >= B2) continue;
    const double2 v = sm[g * seg + fft_pos(k1, P1)];
    const int64_t e = ((int64_t)n2 * k1) % B;
    o[(int64_t)k1 * B2 + n2] = e ? cmul(v, __ldg(W + e)) : v;
  }
}

// Four-step row pass: DFT_B2 over n2 of ws[k1*B2 + n2]; y[k1 + B1*k2] = . / B.
__global__ void __launch_bounds__(kNT) k_rows(const double2* __restrict__ ws, FftPlan P2, int B1,
                                              int B2, int RG, const double2* __restrict__ W,
                                              const int32_t* item_sig, const int32_t* active,
                                              double2* __restrict__ out, int out_M,
                                              int64_t out_S, const int32_t* item_active,
                                              const int32_t* item_row) {
  extern __shared__ double2 sm[];
  const int item = blockIdx.y;
  if (item_active && !item_active[item]) return;
  if (active) {
    const int sig = item_sig ? item_sig[item] : item;
    if (!active[sig]) return;
  }
  const int r0 = blockIdx.x * RG;
  const int seg = B2 + 1;
  const int B = B1 * B2;
  const double2* in = ws + (int64_t)item * B;
  for (int t = threadIdx.x; t < RG * B2; t += kNT) {
    const int g = t / B2, n2 = t - g * B2;
    const int k1 = r0 + g;
    sm[g * seg + n2] = (k1 < B1) ? in[(int64_t)k1 * B2 + n2] : cmk(0.0, 0.0);
  }
  __syncthreads();
  fft_dif(sm, RG, seg, P2, W, B, threadIdx.x, kNT);
  const int64_t row = item_row ? item_row[item]
                                 : (out_M > 0 ? (item % out_M) * out_S + item / out_M : item);
  double2* o = out + row * B;
  const double bd = (double)B;
  for (int t = threadIdx.x; t < RG * B2; t += kNT) {
    const int g = t % RG, k2 = t / RG;
    const int k1 = r0 + g;
    if (k1 >= B1) continue;
    o[k1 + (int64_t)B1 * k2] = cdivr(sm[g * seg + fft_pos(k2, P2)], bd);
  }
}

// Four-step flat path, fold pass: the folded slots of every item, two per
// thread (8 gathers in flight, rows in reference order), written to the item's
// output row, which the column pass then reads coalesced (PROD_LOAD) before the
// row pass overwrites it.  Small blocks and few registers keep many gathers in
// flight per SM, which the column pass (86 registers, one block per SM) cannot.
constexpr int kFrNT = 256;
template <typename Tin>
__global__ void __launch_bounds__(kFrNT) k_fold_rows(Prod p, double2* __restrict__ out) {
  const int item = blockIdx.y;
  const ItemCtx c = item_ctx<PROD_FLAT>(p, item, sizeof(Tin));
  if (c.skip) return;
  if (p.prof_items && threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(p.prof_items, 1ull);
  const int64_t s0 = (int64_t)blockIdx.x * 2 * kFrNT + threadIdx.x;
  const int64_t s1 = s0 + kFrNT;
  double2* o = out + out_row(p, item) * p.B;
  if (s1 < p.B && c.c == 0) {
    double2 a0, a1;
    produce_flat2<Tin>(p, c, s0, c, s1, &a0, &a1);
    o[s0] = a0;
    o[s1] = a1;
  } else {
    if (s0 < p.B) o[s0] = produce<Tin, PROD_FLAT>(p, c, item, s0);
    if (s1 < p.B) o[s1] = produce<Tin, PROD_FLAT>(p, c, item, s1);
  }
}

// ---- permutation runs: the shifted measurements of one (signal, sigma) share
// their samples.  Item j of a run reads x[sigma (s + rB - tau_j)] for slot s,
// row r; with tau_j = tau_0 + a_j B + c_j (0 <= c_j < B) and column
// col = (s - c_j) mod B that is U[col + (r - o_j) B], U[u] = x[sigma (u - tau_0)],
// o_j = a_j + (col + c_j >= B).  So one thread owns one column: it gathers the
// column's rows v in [-max o_j, R) ONCE into its private shared-memory column
// and folds every item of the run from there (virtual slot s_j = col + c_j
// mod B, taps g[s_j + rB], rows in reference order, no FMA contraction, so
// bit-identical to the per-item fold).  Items too far back for the window
// (o_j > wrows - R) are folded by the per-item path, slot = col.  The ladder
// of a C3 loop iteration (shifts 0,1,8,64,512,4096,32768) gathers 27 rows per
// column instead of 7 x 19, the polish shifts (0,1,2) 20 instead of 57.
// Folded slots go to each item's output row; the in-place FFT pass follows.
constexpr int kRfNT = 256;
constexpr int kRfMaxBack = 8;  // window reaches at most this many rows back
constexpr int kRfT = 22;       // tap registers: items of up to kRfT - 1 rows share them

template <typename Tin>
__global__ void __launch_bounds__(kRfNT, 3)
    k_run_fold(Prod p, const int32_t* __restrict__ run_first, const int32_t* __restrict__ run_cnt,
               int wrows, double2* __restrict__ out, int async, int prefetch) {
  extern __shared__ __align__(16) unsigned char rf_smem[];
  Tin* V = reinterpret_cast<Tin*>(rf_smem);  // [wrows][kRfNT], column = thread
  const int run = blockIdx.y;
  const int rfirst = run_first[run], rcnt = run_cnt[run];
  if (p.prof_items && threadIdx.x == 0 && blockIdx.x == 0)
    atomicAdd(p.prof_items, (unsigned long long)rcnt);
  // B, Omega < 2^31 (launcher); index arithmetic mod n stays 64-bit
  const int B = (int)p.B, omega = (int)p.omega;
  const int64_t n = p.n;
  const int col = blockIdx.x * kRfNT + threadIdx.x;
  if (col >= B) return;
  const int R = (omega + B - 1) / B;  // < kRfT (launcher)
  const int A = wrows - R;            // largest o_j a window item may have
  if (prefetch) {
    // the lead run of a signal (its first in the list; runs are slot-major)
    // asks L2 for the whole signal in bulk, at streaming efficiency, so the
    // gathers of all its runs find their lines there
    const int pr = run + prefetch - 1;
    if (pr < gridDim.y) {
      const int f0 = run_first[pr];
      const int sg0 = p.item_sig ? p.item_sig[f0] : f0;
      const int sgp = pr == 0 ? -1 : (p.item_sig ? p.item_sig[run_first[pr - 1]] : run_first[pr - 1]);
      if (sg0 != sgp) {
        const size_t bytes = (size_t)n * sizeof(Tin);
        const size_t per = (bytes / (gridDim.x * kRfNT)) & ~(size_t)15;
        const char* base = (const char*)p.x + (size_t)sg0 * p.xstride * sizeof(Tin) +
                           (size_t)(blockIdx.x * kRfNT + threadIdx.x) * per;
        if (per)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(base), "r"((uint32_t)per)
                       : "memory");
      }
    }
  }
  for (int first = rfirst; first < rfirst + rcnt; first += 32) {
    const int cnt = min(32, rfirst + rcnt - first);
    uint32_t left = cnt == 32 ? 0xffffffffu : ((1u << cnt) - 1u);
    // windows: the first item left is the base (its signal, sigma, tau_h);
    // every item of the same signal and sigma within A rows behind it joins;
    // the rest (the ladder's N/16 shift) forms the next window
    while (left) {
      const int h = first + __ffs(left) - 1;
      const int sigh = p.item_sig ? p.item_sig[h] : h;
      const int64_t sgm = p.item_a[h], tau_h = p.item_b[h];
      uint32_t win = 0;
      int maxo = -1, vhi = 0;
      for (uint32_t m = left; m; m &= m - 1) {
        const int j = __ffs(m) - 1;
        const int it = first + j;
        if ((p.item_sig ? p.item_sig[it] : it) != sigh || p.item_a[it] != sgm) continue;
        const int64_t d = pmod(p.item_b[it] - tau_h, n);
        const int cj = (int)(d % B);
        const int64_t o = d / B + (col + cj >= B);
        if (o > A) continue;
        const int s = col + cj - ((col + cj >= B) ? B : 0);
        const int nr = s < omega ? (omega - s + B - 1) / B : 0;
        win |= 1u << j;
        maxo = max(maxo, (int)o);
        vhi = max(vhi, nr - (int)o);
      }
      left &= ~win;
      // gather the column's window rows once, a chunk of loads in flight, raw
      // samples to shared memory (the column is this thread's own: no barrier)
      {
        constexpr int CH = sizeof(Tin) == 8 ? 8 : 4;
        const Tin* xs = (const Tin*)p.x + (int64_t)sigh * p.xstride;
        const int64_t step = mulmod(sgm, (int64_t)B % n, n);
        int64_t idx = mulmod(sgm, pmod((int64_t)col - (int64_t)maxo * B - tau_h, n), n);
        Tin* vc = V + threadIdx.x;
        const int nv = vhi + maxo;
        if (async) {
          // every row of the window in flight at once, no registers held:
          // asynchronous copies straight into the thread's column
          uint32_t sa = (uint32_t)__cvta_generic_to_shared(vc);
          for (int v = 0; v < nv; ++v) {
            if (sizeof(Tin) == 8)
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(xs + idx)
                           : "memory");
            else
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(xs + idx)
                           : "memory");
            sa += kRfNT * (uint32_t)sizeof(Tin);
            idx += step;
            idx -= (idx >= n) ? n : 0;
          }
          asm volatile("cp.async.commit_group;\n" ::: "memory");
          asm volatile("cp.async.wait_all;\n" ::: "memory");
        }
        for (int v = 0; v < (async ? 0 : nv); v += CH) {
          Tin t[CH];
#pragma unroll
          for (int u = 0; u < CH; ++u) {
            if (v + u < nv) t[u] = __ldcg(xs + idx);
            idx += step;
            idx -= (idx >= n) ? n : 0;
          }
#pragma unroll
          for (int u = 0; u < CH; ++u)
            if (v + u < nv) vc[(v + u) * kRfNT] = t[u];
        }
      }
      // the window's items, grouped by c = shift mod B: the items of one c
      // read the same taps g[col + c + tB] (t = r - wrap), held in registers
      uint32_t todo = win;
      while (todo) {
        const int c = (int)(pmod(p.item_b[first + __ffs(todo) - 1] - tau_h, n) % B);
        const int w = (col + c >= B);
        const int s = col + c - (w ? B : 0);
        const int nr = s < omega ? (omega - s + B - 1) / B : 0;
        double T[kRfT];  // T[t + 1] = g[col + c + tB], t = -1 .. kRfT - 2
        {
          const double* tp = p.taps + (col + c - B);
          const int tcnt = (omega - (col + c) + 2 * B - 1) / B;  // valid: t < tcnt
#pragma unroll
          for (int t = 0; t < kRfT; ++t)
            T[t] = (t >= 1 - w && t < tcnt) ? __ldg(tp + t * B) : 0.0;
        }
        for (uint32_t m = todo; m; m &= m - 1) {
          const int j = __ffs(m) - 1;
          const int it = first + j;
          const int64_t d = pmod(p.item_b[it] - tau_h, n);
          if ((int)(d % B) != c) continue;
          todo &= ~(1u << j);
          const int o = (int)(d / B) + w;
          const Tin* vc = V + (maxo - o) * kRfNT + threadIdx.x;  // row r at vc[r NT]
          double2 acc = cmk(0.0, 0.0);
          if (w) {
#pragma unroll
            for (int r = 0; r < kRfT; ++r)
              if (r < nr) {
                const double2 v = to_d2_(vc[r * kRfNT]);
                acc = cadd_rn(acc, cmk(__dmul_rn(T[r], v.x), __dmul_rn(T[r], v.y)));
              }
          } else {
#pragma unroll
            for (int r = 0; r + 1 < kRfT; ++r)
              if (r < nr) {
                const double2 v = to_d2_(vc[r * kRfNT]);
                acc = cadd_rn(acc, cmk(__dmul_rn(T[r + 1], v.x), __dmul_rn(T[r + 1], v.y)));
              }
          }
          out[out_row(p, it) * p.B + s] = acc;
        }
      }
    }
  }
}

// Fallback for B with a prime factor above 13: slots to HBM, O(B^2) DFT.
template <typename Tin, int MODE>
__global__ void __launch_bounds__(256) k_slots(Prod p, double2* __restrict__ z) {
  const int item = blockIdx.y;
  const ItemCtx c = item_ctx<MODE>(p, item, sizeof(Tin));
  if (c.skip) return;
  const int64_t s = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (s < p.B) z[(int64_t)item * p.B + s] = produce<Tin, MODE>(p, c, item, s);
}

__global__ void __launch_bounds__(256) k_dft_direct(const double2* __restrict__ z, int64_t B,
                                                    const double2* __restrict__ W,
                                                    const int32_t* item_sig,
                                                    const int32_t* active,
                                                    double2* __restrict__ out, int out_M,
                                                    int64_t out_S, const int32_t* item_active,
                                                    const int32_t* item_row) {
  const int item = blockIdx.y;
  if (item_active && !item_active[item]) return;
  if (active) {
    const int sig = item_sig ? item_sig[item] : item;
    if (!active[sig]) return;
  }
  const int64_t k = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (k >= B) return;
  const double2* zi = z + (int64_t)item * B;
  double2 acc = cmk(0.0, 0.0);
  int64_t e = 0;
  for (int64_t s = 0; s < B; ++s) {
    const double2 w = __ldg(W + e);
    const double2 v = zi[s];
    acc.x += v.x * w.x - v.y * w.y;
    acc.y += v.x * w.y + v.y * w.x;
    e += k;
    if (e >= B) e -= B;
  }
  const int64_t row = item_row ? item_row[item]
                                 : (out_M > 0 ? (item % out_M) * out_S + item / out_M : item);
  out[row * B + k] = cdivr(acc, (double)B);
}

__global__ void k_twiddle(double2* W, int64_t B) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B) return;
  double s, c;
  sincospi(-2.0 * (double)e / (double)B, &s, &c);
  W[e] = cmk(c, s);
}

// Flat-window taps (sfft/filters.py:125-151): sinc(u/B)/B-normalised times a
// Gaussian, u = i - Omega/2, centre tap 1/B.
__global__ void k_flat_taps(double* taps, int64_t omega, int64_t B, double gsig) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= omega) return;
  const double u = (double)i - (double)omega / 2.0;
  const double core = (u == 0.0) ? 1.0 / (double)B
                                 : sin(3.141592653589793 * u / (double)B) /
                                       (3.141592653589793 * u);
  const double r = u / gsig;
  taps[i] = core * exp(-0.5 * (r * r));
}

// max |T| over the response table (sfft/frameworks.py:331, :463).
__global__ void k_absmax(const double2* __restrict__ v, int64_t count,
                         unsigned long long* out_bits) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, cabs_(v[i]));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out_bits, dbits(m));
}

// ----------------------------------------------------------------- host side

template <typename K>
static int ensure_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) {
    SFFT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)bytes));
  }
  return 0;
}

// Choose B = B1*B2 for the four-step path: both plan-able and <= kFusedMaxB,
// B2 the smallest such divisor >= sqrt(B).
static bool split_plan(int64_t B, int64_t* B1, int64_t* B2) {
  int64_t best = 0;
  for (int64_t d = 1; d * d <= B; ++d) {
    if (B % d) continue;
    const int64_t a = d, b = B / d;
    FftPlan pa, pb;
    if (a <= kFusedMaxB && b <= kFusedMaxB && make_plan(a, &pa) && make_plan(b, &pb)) best = a;
  }
  if (!best) return false;
  *B1 = best;
  *B2 = B / best;
  return true;
}

// SFFT_NO_CLUSTER=1 forces the one-CTA path (A/B measurements).
static bool cluster_disabled() {
  static const bool off = [] {
    const char* e = getenv("SFFT_NO_CLUSTER");
    return e && e[0] == '1';
  }();
  return off;
}

size_t bucketize_ws_bytes(int64_t B, int64_t nitems) {
  FftPlan P;
  if (B <= 4096 && make_plan(B, &P)) return 0;  // flat B > 4096 takes the four-step path
  return (size_t)nitems * (size_t)B * sizeof(double2);
}

template <typename Tin, int MODE>
static int run_bucketize_t(const Prod& p, int64_t nitems, const double2* W, double2* out,
                           void* ws, size_t ws_bytes, cudaStream_t st) {
  if (nitems <= 0) return 0;
  const int64_t B = p.B;
  FftPlan P;
  // flat windows with B > 4096: the fold pass + four-step FFT beats the
  // 1024-slot cluster slices (env SFFT_FLAT_FOURSTEP_MIN overrides the bound)
  static const int64_t fs_min =
      getenv("SFFT_FLAT_FOURSTEP_MIN") ? atoll(getenv("SFFT_FLAT_FOURSTEP_MIN")) : 4097;
  const bool four = MODE == PROD_FLAT && B >= fs_min;
  const int CL = four ? 0 : cluster_size(B);
  if (CL > 1 && !cluster_disabled()) {
    if (CL == 8) return launch_cluster<Tin, MODE, 8>(p, nitems, W, out, st);
    if (CL == 4) return launch_cluster<Tin, MODE, 4>(p, nitems, W, out, st);
    return launch_cluster<Tin, MODE, 2>(p, nitems, W, out, st);
  }
  if (!four && B <= kFusedMaxB && make_plan(B, &P)) {
    const size_t sm = (size_t)B * sizeof(double2);
    if (ensure_smem(k_fused<Tin, MODE>, sm)) return -3;
    SFFT_CUDA(cudaFuncSetAttribute(k_fused<Tin, MODE>,
                                   cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    k_fused<Tin, MODE><<<(unsigned)nitems, kNT, sm, st>>>(p, P, W, out);
    SFFT_CHECK_LAUNCH("k_fused");
    return 0;
  }
  SFFT_REQUIRE(ws && ws_bytes >= bucketize_ws_bytes(B, nitems),
               "bucketize: workspace too small for the four-step path");
  double2* z = (double2*)ws;
  int64_t B1, B2;
  if (split_plan(B, &B1, &B2)) {
    FftPlan P1, P2;
    make_plan(B1, &P1);
    make_plan(B2, &P2);
    const int CG = (int)std::max<int64_t>(1, std::min<int64_t>(B2, kFusedMaxB / (B1 + 1)));
    const int RG = (int)std::max<int64_t>(1, std::min<int64_t>(B1, kFusedMaxB / (B2 + 1)));
    const size_t smc = (size_t)CG * (B1 + 1) * sizeof(double2);
    const size_t smr = (size_t)RG * (B2 + 1) * sizeof(double2);
    if (ensure_smem(k_cols<Tin, MODE>, smc)) return -3;
    if (ensure_smem(k_rows, smr)) return -3;
    dim3 gc((unsigned)cdiv_up(B2, CG), (unsigned)nitems);
    if (MODE == PROD_FLAT) {
      // fold into the output rows, then the column pass from there
      dim3 gf((unsigned)cdiv_up(B, 2 * kFrNT), (unsigned)nitems);
      k_fold_rows<Tin><<<gf, kFrNT, 0, st>>>(p, out);
      SFFT_CHECK_LAUNCH("k_fold_rows");
      Prod pz = p;
      pz.z = out;
      pz.prof_items = nullptr;
      if (ensure_smem(k_cols<Tin, PROD_LOAD>, smc)) return -3;
      k_cols<Tin, PROD_LOAD><<<gc, kNT, smc, st>>>(pz, P1, (int)B1, (int)B2, CG, W, z);
    } else {
      k_cols<Tin, MODE><<<gc, kNT, smc, st>>>(p, P1, (int)B1, (int)B2, CG, W, z);
    }
    SFFT_CHECK_LAUNCH("k_cols");
    dim3 gr((unsigned)cdiv_up(B1, RG), (unsigned)nitems);
    k_rows<<<gr, kNT, smr, st>>>(z, P2, (int)B1, (int)B2, RG, W, p.item_sig, p.active, out,
                                 p.out_M, p.out_S, p.item_active, p.item_row);
    SFFT_CHECK_LAUNCH("k_rows");
    return 0;
  }
  dim3 g((unsigned)cdiv_up(B, 256), (unsigned)nitems);
  k_slots<Tin, MODE><<<g, 256, 0, st>>>(p, z);
  SFFT_CHECK_LAUNCH("k_slots");
  k_dft_direct<<<g, 256, 0, st>>>(z, B, W, p.item_sig, p.active, out, p.out_M, p.out_S,
                                  p.item_active, p.item_row);
  SFFT_CHECK_LAUNCH("k_dft_direct");
  return 0;
}

static int run_bucketize_inner(int dtype, int mode, const Prod& p, int64_t nitems,
                               const double2* W, double2* out, void* ws, size_t ws_bytes,
                               cudaStream_t st) {
  if (mode == PROD_FLAT)
    return dtype == 0 ? run_bucketize_t<float2, PROD_FLAT>(p, nitems, W, out, ws, ws_bytes, st)
                      : run_bucketize_t<double2, PROD_FLAT>(p, nitems, W, out, ws, ws_bytes, st);
  if (mode == PROD_SPIKE)
    return dtype == 0 ? run_bucketize_t<float2, PROD_SPIKE>(p, nitems, W, out, ws, ws_bytes, st)
                      : run_bucketize_t<double2, PROD_SPIKE>(p, nitems, W, out, ws, ws_bytes, st);
  if (mode == PROD_GTAB)
    return run_bucketize_t<double2, PROD_GTAB>(p, nitems, W, out, ws, ws_bytes, st);
  if (mode == PROD_DIRICHLET)
    return dtype == 0
               ? run_bucketize_t<float2, PROD_DIRICHLET>(p, nitems, W, out, ws, ws_bytes, st)
               : run_bucketize_t<double2, PROD_DIRICHLET>(p, nitems, W, out, ws, ws_bytes, st);
  return run_bucketize_t<double2, PROD_LOAD>(p, nitems, W, out, ws, ws_bytes, st);
}

// out[k] = (sum_t B conj(y_t[k]) w^{c_k t}) / T over the offsets in order,
// c_k = (k L + base + center) mod n (bucket_centers, sfft/filters.py:92-100)
__global__ void k_dirichlet_combine(const double2* __restrict__ y, int64_t noff,
                                    const int64_t* __restrict__ offsets, int64_t n, int64_t L,
                                    int64_t B, int half, int64_t center, double2* out) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= B) return;
  const int64_t c = pmod(k * L + (half ? 0 : L / 2) + center, n);
  const double bd = (double)B;
  double2 tot = cmk(0.0, 0.0);
  for (int64_t t = 0; t < noff; ++t) {
    const double2 v = y[t * B + k];                           // FFT(conj z)[k] / B
    const double2 vb = cmul(cmk(bd, 0.0), cmk(v.x, -v.y));   // b * ifft(z)[k]
    tot = cadd(tot, cmul(vb, unit_root(n, mulmod(c, pmod(offsets[t], n), n))));
  }
  out[k] = cdiv(tot, cmk((double)noff, 0.0));
}

int run_dirichlet_combine(const double2* y, int64_t noff, const int64_t* offsets, int64_t n,
                          int64_t L, int64_t B, int half_offset, int64_t center_offset,
                          double2* out, cudaStream_t st) {
  k_dirichlet_combine<<<(unsigned)cdiv_up(B, 256), 256, 0, st>>>(y, noff, offsets, n, L, B,
                                                                  half_offset,
                                                                  pmod(center_offset, n), out);
  SFFT_CHECK_LAUNCH("k_dirichlet_combine");
  return 0;
}

// mean_i x[idx_i] w^{f idx_i} (sfft/reconstruct.py:356-371): block partial
// sums over contiguous index ranges, then an ordered sum of the partials
constexpr int kFsBlocks = 256, kFsNT = 256;

template <typename Tin>
__global__ void __launch_bounds__(kFsNT) k_freqshift_part(const Tin* __restrict__ x, int64_t n,
                                                          const int64_t* __restrict__ idx,
                                                          int64_t count, int64_t f,
                                                          double2* partial) {
  __shared__ double2 red[kFsNT / 32];
  const int64_t per = (count + gridDim.x - 1) / gridDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(count, i0 + per);
  double2 acc = cmk(0.0, 0.0);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += kFsNT) {
    const int64_t e = pmod(idx[i], n);
    acc = cadd(acc, cmul(Sample<Tin>::load(x, e), unit_root(n, mulmod(pmod(f, n), e, n))));
  }
  for (int o = 16; o; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double2 t = red[0];
    for (int w = 1; w < kFsNT / 32; ++w) t = cadd(t, red[w]);
    partial[blockIdx.x] = t;
  }
}

__global__ void k_freqshift_final(const double2* partial, int nb, int64_t count, double2* out) {
  double2 t = cmk(0.0, 0.0);
  for (int b = 0; b < nb; ++b) t = cadd(t, partial[b]);
  out[0] = cdiv(t, cmk((double)count, 0.0));
}

int run_freqshift(int dtype, const void* x, int64_t n, const int64_t* idx, int64_t count,
                  int64_t f, double2* partial, double2* out, cudaStream_t st) {
  const int nb = (int)std::min<int64_t>(kFsBlocks, cdiv_up(count, kFsNT));
  if (dtype == 0)
    k_freqshift_part<float2><<<nb, kFsNT, 0, st>>>((const float2*)x, n, idx, count, f, partial);
  else
    k_freqshift_part<double2><<<nb, kFsNT, 0, st>>>((const double2*)x, n, idx, count, f, partial);
  SFFT_CHECK_LAUNCH("k_freqshift_part");
  k_freqshift_final<<<1, 1, 0, st>>>(partial, nb, count, out);
  SFFT_CHECK_LAUNCH("k_freqshift_final");
  return 0;
}

BucketProf& bucket_prof() {
  static BucketProf p;
  return p;
}

int prof_begin(cudaStream_t st, cudaEvent_t* ev0) {
  SFFT_CUDA(cudaEventCreate(ev0));
  SFFT_CUDA(cudaEventRecord(*ev0, st));
  return 0;
}

int prof_end(cudaStream_t st, cudaEvent_t ev0) {
  cudaEvent_t ev1;
  SFFT_CUDA(cudaEventCreate(&ev1));
  SFFT_CUDA(cudaEventRecord(ev1, st));
  std::lock_guard<std::mutex> lk(bucket_prof().mu);
  bucket_prof().pending.push_back({ev0, ev1});
  bucket_prof().launches += 1;
  return 0;
}

int prof_collect() {
  BucketProf& p = bucket_prof();
  std::lock_guard<std::mutex> lk(p.mu);
  for (auto& e : p.pending) {
    SFFT_CUDA(cudaEventSynchronize(e.second));
    float ms = 0.f;
    SFFT_CUDA(cudaEventElapsedTime(&ms, e.first, e.second));
    p.ms += ms;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  p.pending.clear();
  return 0;
}

// Flat and spike bucketizations of the runners and the C ABI go through here;
// with profiling on, each launch is bracketed by CUDA events on its stream.
// Random 8-byte gathers: ask L2 to fetch single 32-byte sectors from HBM
// instead of the default 64/128-byte promotion (measured: 4 DRAM sectors per
// gathered sample without this).  Once per device; SFFT_L2_FETCH overrides.
static void gather_fetch_granularity() {
  static std::mutex mu;
  static bool done[64] = {false};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return;
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return;
  const char* e = getenv("SFFT_L2_FETCH");
  const size_t g = e ? (size_t)atoi(e) : 32;
  if (g > 0) cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
  cudaGetLastError();
  done[dev] = true;
}

int run_bucketize(int dtype, int mode, const Prod& p0, int64_t nitems, const double2* W,
                  double2* out, void* ws, size_t ws_bytes, cudaStream_t st) {
  gather_fetch_granularity();
  BucketProf& bp = bucket_prof();
  if (!bp.on || (mode != PROD_FLAT && mode != PROD_SPIKE))
    return run_bucketize_inner(dtype, mode, p0, nitems, W, out, ws, ws_bytes, st);
  Prod p = p0;
  p.prof_items = bp.d_items;
  cudaEvent_t ev0;
  int rc = prof_begin(st, &ev0);
  if (rc) return rc;
  rc = run_bucketize_inner(dtype, mode, p, nitems, W, out, ws, ws_bytes, st);
  if (rc) return rc;
  return prof_end(st, ev0);
}

// Flat bucketizations grouped in permutation runs (items [run_first[r],
// run_first[r] + run_cnt[r]) share signal and sigma; b' = 0, no gates): the
// run fold into each item's output row, then the FFT of every row in place.
// Profiled (when on) as one bucketization launch of nitems items.
int run_flat_runs(int dtype, const Prod& p0, const int32_t* run_first, const int32_t* run_cnt,
                  int64_t nruns, int64_t nitems, const double2* W, double2* out, void* ws,
                  size_t ws_bytes, cudaStream_t st) {
  if (nruns <= 0 || nitems <= 0) return 0;
  SFFT_REQUIRE(!p0.item_c && !p0.active && !p0.item_active && p0.item_row,
               "run fold: needs an ungated item list with output rows and b' = 0");
  gather_fetch_granularity();
  BucketProf& bp = bucket_prof();
  Prod p = p0;
  p.prof_items = bp.on ? bp.d_items : nullptr;
  cudaEvent_t ev0{};
  if (bp.on) {
    int rc = prof_begin(st, &ev0);
    if (rc) return rc;
  }
  const int R = (int)cdiv_up(p.omega, p.B);
  if (R >= kRfT || p.B >= (1 << 30) || p.omega >= (1 << 30))  // per-item kernels
    return run_bucketize(dtype, PROD_FLAT, p0, nitems, W, out, ws, ws_bytes, st);
  const int wrows = R + (int)std::min<int64_t>(kRfMaxBack, std::max(R - 1, 0));
  const dim3 g((unsigned)cdiv_up(p.B, kRfNT), (unsigned)nruns);
  // SFFT_RF_SMEM=<bytes>: pad the dynamic shared memory (occupancy experiments)
  const size_t pad = getenv("SFFT_RF_SMEM") ? (size_t)atoll(getenv("SFFT_RF_SMEM")) : 0;
  const int async = getenv("SFFT_RF_ASYNC") ? atoi(getenv("SFFT_RF_ASYNC")) : 0;
  const int prefetch = getenv("SFFT_RF_PREFETCH") ? atoi(getenv("SFFT_RF_PREFETCH")) : 0;
  if (dtype == 0) {
    const size_t sm = std::max(pad, (size_t)wrows * kRfNT * sizeof(float2));
    if (ensure_smem(k_run_fold<float2>, sm)) return -3;
    k_run_fold<float2><<<g, kRfNT, sm, st>>>(p, run_first, run_cnt, wrows, out, async, prefetch);
  } else {
    const size_t sm = std::max(pad, (size_t)wrows * kRfNT * sizeof(double2));
    if (ensure_smem(k_run_fold<double2>, sm)) return -3;
    k_run_fold<double2><<<g, kRfNT, sm, st>>>(p, run_first, run_cnt, wrows, out, async, prefetch);
  }
  SFFT_CHECK_LAUNCH("k_run_fold");
  Prod pl = p;
  pl.z = out;
  pl.prof_items = nullptr;
  int rc = run_bucketize_inner(dtype, PROD_LOAD, pl, nitems, W, out, ws, ws_bytes, st);
  if (rc) return rc;
  return bp.on ? prof_end(st, ev0) : 0;
}

int run_twiddle(double2* W, int64_t B, cudaStream_t st) {
  k_twiddle<<<(unsigned)cdiv_up(B, 256), 256, 0, st>>>(W, B);
  SFFT_CHECK_LAUNCH("k_twiddle");
  return 0;
}

int run_flat_taps(double* taps, int64_t omega, int64_t B, double gsig, cudaStream_t st) {
  k_flat_taps<<<(unsigned)cdiv_up(omega, 256), 256, 0, st>>>(taps, omega, B, gsig);
  SFFT_CHECK_LAUNCH("k_flat_taps");
  return 0;
}

int run_absmax(const double2* v, int64_t count, double* out, cudaStream_t st) {
  SFFT_CUDA(cudaMemsetAsync(out, 0, sizeof(double), st));
  const int blocks = (int)std::min<int64_t>(1184, cdiv_up(count, 256));
  k_absmax<<<blocks, 256, 0, st>>>(v, count, (unsigned long long*)out);
  SFFT_CHECK_LAUNCH("k_absmax");
  return 0;
}

}  // namespace sfft
