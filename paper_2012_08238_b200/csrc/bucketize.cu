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
#include <cuda.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "kernels.cuh"

namespace sfft {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*TensorMapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                      const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static TensorMapEncodeFn tensor_map_encoder() {
  static TensorMapEncodeFn fn = []() -> TensorMapEncodeFn {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return (TensorMapEncodeFn)f;
  }();
  return fn;
}

// The signals as a 3-D tensor of 8-byte words: [signal][row j < L][B eb / 8],
// boxes of one 128-byte line x up to 256 rows.
static int stream_tensor_map(const void* x, int64_t xstride, int64_t n, int64_t B, int64_t eb,
                             CUtensorMap* tm) {
  TensorMapEncodeFn enc = tensor_map_encoder();
  SFFT_REQUIRE(enc, "stream fold: cuTensorMapEncodeTiled not available");
  const int64_t L = n / B;
  const cuuint64_t dims[3] = {(cuuint64_t)(B * eb / 8), (cuuint64_t)L, (cuuint64_t)1 << 20};
  const cuuint64_t strides[2] = {(cuuint64_t)(B * eb), (cuuint64_t)(xstride * eb)};
  const cuuint32_t box[3] = {16, (cuuint32_t)std::min<int64_t>(L, 256), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const char* pe = getenv("SFFT_SF_PROMO");
  const int promo = pe ? atoi(pe) : 0;
  const CUtensorMapL2promotion l2 = promo == 64    ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : promo == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                    : promo == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                   : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  const CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void*>(x), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, l2, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("stream fold: cuTensorMapEncodeTiled failed");
    return -3;
  }
  return 0;
}

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
    SFFT_DASSERT(idx >= 0 && idx < n && s >= 0 && s < p.B);
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
  double2* tw = bq + NI * M;     // [< M] stage twiddles of fft_pow2
  if (threadIdx.x < NI) {
    const int64_t it = item0 + threadIdx.x;
    const bool in = it < nitems;
    const ItemCtx c = item_ctx<MODE>(p, in ? (int)it : 0, sizeof(Tin));
    s_ctx[threadIdx.x] = c;
    s_live[threadIdx.x] = in && !c.skip;
  }
  // stage twiddles of fft_pow2 laid out [stage][q][j] (see fft.cuh): w_M^e = W[e CL]
  {
    int off = 0, Mbs = M;
    for (int st = 0; st < Pow2<M>::N8; ++st) {
      const int Mps = Mbs >> 3;
      for (int e = threadIdx.x; e < 7 * Mps; e += kClNT) {
        const int q = e / Mps + 1, j = e - (q - 1) * Mps;
        tw[off + e] = __ldg(W + (int64_t)j * q * (M / Mbs) * CL);
      }
      off += 7 * Mps;
      Mbs = Mps;
    }
  }
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
      SFFT_DASSERT(n2 < M);
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
__global__ void __launch_bounds__(kNT, 2) k_cols(Prod p, FftPlan P1, int B1, int B2, int CG,
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
  if (MODE == PROD_SPIKE) {
    // strided samples x[(L s - a) mod n], s = n1 B2 + n2 < B so L s < n: the
    // index needs one conditional add, not a 64-bit modulo per sample, and
    // (g, n1) advance incrementally; four gathers are in flight per thread
    // before the first is stored (the kernel is bound by their latency)
    const Tin* xs = (const Tin*)c.xs;
    const int64_t n = p.n, Ls = n / p.B, am = pmod(c.a, n);
    const int dg = kNT % CG, dn = kNT / CG;
    int g = threadIdx.x % CG, n1 = threadIdx.x / CG;
    for (int t = threadIdx.x; t < CG * B1; t += 4 * kNT) {
      double2 v[4];
      int at[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        at[u] = -1;
        v[u] = cmk(0.0, 0.0);
        if (t + u * kNT < CG * B1) {
          at[u] = g * seg + n1;
          const int n2 = c0 + g;
          if (n2 < B2) {
            int64_t idx = Ls * ((int64_t)n1 * B2 + n2) - am;
            idx += (idx < 0) ? n : 0;
            v[u] = Sample<Tin>::load(xs, idx);
          }
        }
        g += dg;
        n1 += dn;
        if (g >= CG) {
          g -= CG;
          ++n1;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (at[u] >= 0) sm[at[u]] = v[u];
    }
  } else {
    for (int t = threadIdx.x; t < CG * B1; t += kNT) {
      const int g = t % CG, n1 = t / CG;
      const int n2 = c0 + g;
      sm[g * seg + n1] = (n2 < B2) ? produce<Tin, MODE>(p, c, item, (int64_t)n1 * B2 + n2)
                                   : cmk(0.0, 0.0);
    }
  }
  // digit-reversed positions once per CTA (behind the CG segments)
  int* pos = (int*)(sm + CG * seg);
  for (int k = threadIdx.x; k < B1; k += kNT) pos[k] = fft_pos(k, P1);
  __syncthreads();
  fft_dif(sm, CG, seg, P1, W, B, threadIdx.x, kNT);
  double2* o = ws + (int64_t)item * B;
  {
    const int dg = kNT % CG, dk = kNT / CG;  // (g, k1) of t = k1 CG + g, advanced by kNT
    int g = threadIdx.x % CG, k1 = threadIdx.x / CG;
    for (int t = threadIdx.x; t < CG * B1; t += kNT) {
      const int n2 = c0 + g;
      if (n2 < B2) {
        const double2 v = sm[g * seg + pos[k1]];
        const int e = n2 * k1;  // n2 < B2, k1 < B1: below B, no reduction needed
        o[(int64_t)k1 * B2 + n2] = e ? cmul(v, __ldg(W + e)) : v;
      }
      g += dg;
      k1 += dk;
      if (g >= CG) {
        g -= CG;
        ++k1;
      }
    }
  }
}

// Four-step row pass: DFT_B2 over n2 of ws[k1*B2 + n2]; y[k1 + B1*k2] = . / B.
__global__ void __launch_bounds__(kNT, 2) k_rows(const double2* __restrict__ ws, FftPlan P2, int B1,
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
  {
    const int dn = kNT % B2, dg = kNT / B2;  // (g, n2) of t = g B2 + n2, advanced by kNT
    int g = threadIdx.x / B2, n2 = threadIdx.x % B2;
    for (int t = threadIdx.x; t < RG * B2; t += kNT) {
      const int k1 = r0 + g;
      sm[g * seg + n2] = (k1 < B1) ? in[(int64_t)k1 * B2 + n2] : cmk(0.0, 0.0);
      n2 += dn;
      g += dg;
      if (n2 >= B2) {
        n2 -= B2;
        ++g;
      }
    }
  }
  int* pos = (int*)(sm + RG * seg);
  for (int k = threadIdx.x; k < B2; k += kNT) pos[k] = fft_pos(k, P2);
  __syncthreads();
  fft_dif(sm, RG, seg, P2, W, B, threadIdx.x, kNT);
  const int64_t row = item_row ? item_row[item]
                                 : (out_M > 0 ? (item % out_M) * out_S + item / out_M : item);
  double2* o = out + row * B;
  const double bd = (double)B;
  {
    const int dg = kNT % RG, dk = kNT / RG;  // (g, k2) of t = k2 RG + g, advanced by kNT
    int g = threadIdx.x % RG, k2 = threadIdx.x / RG;
    for (int t = threadIdx.x; t < RG * B2; t += kNT) {
      const int k1 = r0 + g;
      if (k1 < B1) o[k1 + (int64_t)B1 * k2] = cdivr(sm[g * seg + pos[k2]], bd);
      g += dg;
      k2 += dk;
      if (g >= RG) {
        g -= RG;
        ++k2;
      }
    }
  }
}

// ---- power-of-two four-step passes (flat B = 2^13 .. 2^18: the config-5 grid)
// Both passes transform G lines of length M (64..512) per CTA in shared
// memory, line g at s + g*(M+1): thread t works on line t % G, so the eight
// threads of a 16-byte shared-memory phase always sit on eight different lines
// (odd line pitch: no bank conflicts at any butterfly stride) while global
// loads and stores run along the contiguous axis (G x 16 bytes or a whole
// line).  Radix-8 register butterflies (dft8_, then one radix-4/2 stage),
// stage twiddles w_M^e in shared memory, digit reversal by pow2_pos.
//   pass 1 (columns): DFT_B1 over n1 of z[n1 B2 + n2], times w_B^{n2 k1},
//                     stored at ws[k1 B2 + n2]
//   pass 2 (rows):    DFT_B2 over n2 of ws[k1 B2 + n2]; y[k1 + B1 k2] = ./B
constexpr int kF4NT = 512;
constexpr int fs_lines(int M) { return M <= 128 ? 32 : (M == 256 ? 16 : 8); }

template <int M, int G>
__device__ __forceinline__ void fs_lines_fft(double2* __restrict__ s,
                                             const double2* __restrict__ tw) {
  constexpr int NB = kF4NT / G;  // butterflies of a line side by side
  const int g = threadIdx.x % G, bi = threadIdx.x / G;
  double2* line = s + g * (M + 1);
  int Mb = M;
#pragma unroll
  for (int st = 0; st < Pow2<M>::N8; ++st) {
    const int Mp = Mb >> 3;
    const int tstr = M / Mb;
    for (int tt = bi; tt < M / 8; tt += NB) {
      const int blk = tt / Mp, j = tt - blk * Mp;
      double2* x = line + blk * Mb + j;
      double2 a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = x[q * Mp];
      dft8_(a);
      x[0] = a[0];
#pragma unroll
      for (int q = 1; q < 8; ++q) x[q * Mp] = j ? cmul(a[q], tw[j * q * tstr]) : a[q];
    }
    __syncthreads();
    Mb = Mp;
  }
  if (Pow2<M>::RL == 4) {
    for (int tt = bi; tt < M / 4; tt += NB) {
      double2* x = line + 4 * tt;
      dft4_(x[0], x[1], x[2], x[3]);
    }
    __syncthreads();
  } else if (Pow2<M>::RL == 2) {
    for (int tt = bi; tt < M / 2; tt += NB) {
      double2* x = line + 2 * tt;
      const double2 u = x[0], v = x[1];
      x[0] = cadd(u, v);
      x[1] = csub(u, v);
    }
    __syncthreads();
  }
}

template <int M>
__global__ void __launch_bounds__(kF4NT) k_fs_cols(Prod p, int B2, const double2* __restrict__ W,
                                                   double2* __restrict__ ws) {
  constexpr int G = fs_lines(M);
  extern __shared__ double2 fs_s[];
  double2* tw = fs_s + G * (M + 1);
  const int item = blockIdx.y;
  const int sig = p.item_sig ? p.item_sig[item] : item;
  if ((p.active && !p.active[sig]) || (p.item_active && !p.item_active[item])) return;
  const int B = M * B2;
  const int c0 = blockIdx.x * G;
  const double2* in = p.z + out_row(p, item) * (int64_t)B;
  for (int e = threadIdx.x; e < M; e += kF4NT) tw[e] = __ldg(W + (int64_t)e * B2);
  for (int t = threadIdx.x; t < G * M; t += kF4NT) {
    const int g = t % G, n1 = t / G;
    fs_s[g * (M + 1) + n1] = in[(int64_t)n1 * B2 + c0 + g];
  }
  __syncthreads();
  fs_lines_fft<M, G>(fs_s, tw);
  double2* o = ws + (int64_t)item * B;
  for (int t = threadIdx.x; t < G * M; t += kF4NT) {
    const int g = t % G, k1 = t / G;
    const int n2 = c0 + g;
    const double2 v = fs_s[g * (M + 1) + pow2_pos<M>(k1)];
    const int e = n2 * k1;  // < B
    o[(int64_t)k1 * B2 + n2] = e ? cmul(v, __ldg(W + e)) : v;
  }
}

template <int M>
__global__ void __launch_bounds__(kF4NT) k_fs_rows(Prod p, int B1, const double2* __restrict__ W,
                                                   const double2* __restrict__ ws,
                                                   double2* __restrict__ out) {
  constexpr int G = fs_lines(M);
  extern __shared__ double2 fs_s[];
  double2* tw = fs_s + G * (M + 1);
  const int item = blockIdx.y;
  const int sig = p.item_sig ? p.item_sig[item] : item;
  if ((p.active && !p.active[sig]) || (p.item_active && !p.item_active[item])) return;
  const int B = M * B1;
  const int r0 = blockIdx.x * G;
  const double2* in = ws + (int64_t)item * B + (int64_t)r0 * M;
  for (int e = threadIdx.x; e < M; e += kF4NT) tw[e] = __ldg(W + (int64_t)e * B1);
  for (int t = threadIdx.x; t < G * M; t += kF4NT) {
    const int g = t / M, n2 = t - g * M;
    fs_s[g * (M + 1) + n2] = in[t];
  }
  __syncthreads();
  fs_lines_fft<M, G>(fs_s, tw);
  double2* o = out + out_row(p, item) * (int64_t)B;
  const double bd = (double)B;
  for (int t = threadIdx.x; t < G * M; t += kF4NT) {
    const int g = t % G, k2 = t / G;
    o[r0 + g + (int64_t)B1 * k2] = cdivr(fs_s[g * (M + 1) + pow2_pos<M>(k2)], bd);
  }
}

template <int M>
static int launch_fs_cols(const Prod& p, int64_t nitems, int64_t B2, const double2* W, double2* ws,
                          cudaStream_t st) {
  constexpr int G = fs_lines(M);
  const size_t sm = (size_t)(G * (M + 1) + M) * sizeof(double2);
  SFFT_CUDA(cudaFuncSetAttribute(k_fs_cols<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
  k_fs_cols<M><<<dim3((unsigned)(B2 / G), (unsigned)nitems), kF4NT, sm, st>>>(p, (int)B2, W, ws);
  SFFT_CHECK_LAUNCH("k_fs_cols");
  return 0;
}

template <int M>
static int launch_fs_rows(const Prod& p, int64_t nitems, int64_t B1, const double2* W,
                          const double2* ws, double2* out, cudaStream_t st) {
  constexpr int G = fs_lines(M);
  const size_t sm = (size_t)(G * (M + 1) + M) * sizeof(double2);
  SFFT_CUDA(cudaFuncSetAttribute(k_fs_rows<M>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sm));
  k_fs_rows<M><<<dim3((unsigned)(B1 / G), (unsigned)nitems), kF4NT, sm, st>>>(p, (int)B1, W, ws,
                                                                             out);
  SFFT_CHECK_LAUNCH("k_fs_rows");
  return 0;
}

// B = B1*B2 with B1 = 2^floor(lg/2); both in 64..512 for B = 2^12 .. 2^18.
static bool fs_pow2_split(int64_t B, int64_t* B1, int64_t* B2) {
  if (B < 4096 || B > (1 << 18) || (B & (B - 1))) return false;
  int lg = 0;
  while (((int64_t)1 << lg) < B) ++lg;
  *B1 = (int64_t)1 << (lg / 2);
  *B2 = B / *B1;
  return true;
}

// The two passes over rows already in natural order at p.z (row of item i =
// out_row(p, i)); ws holds the intermediate, results land in out's rows.
static int run_fs_pow2(const Prod& p, int64_t nitems, int64_t B1, int64_t B2, const double2* W,
                       double2* ws, double2* out, cudaStream_t st) {
  int rc;
  switch (B1) {
    case 64: rc = launch_fs_cols<64>(p, nitems, B2, W, ws, st); break;
    case 128: rc = launch_fs_cols<128>(p, nitems, B2, W, ws, st); break;
    case 256: rc = launch_fs_cols<256>(p, nitems, B2, W, ws, st); break;
    default: rc = launch_fs_cols<512>(p, nitems, B2, W, ws, st); break;
  }
  if (rc) return rc;
  switch (B2) {
    case 64: return launch_fs_rows<64>(p, nitems, B1, W, ws, out, st);
    case 128: return launch_fs_rows<128>(p, nitems, B1, W, ws, out, st);
    case 256: return launch_fs_rows<256>(p, nitems, B1, W, ws, out, st);
    default: return launch_fs_rows<512>(p, nitems, B1, W, ws, out, st);
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

// ---- item groups: the shifted measurements of one (signal, sigma) share
// their samples.  Item j reads x[sigma (s + rB - tau_j)] for slot s, row r;
// with tau_j = tau_h + a_j B + c_j (0 <= c_j < B, tau_h the window head's) and
// column col = (s - c_j) mod B that is U[col + (r - o_j) B], U[u] =
// x[sigma (u - tau_h)], o_j = a_j + (col + c_j >= B).  A CTA owns kGfCols
// columns of a group of up to kGfItems items (whole permutation runs of one
// slot, packed by the planner): every sample of a window (head + the items
// within kGfBack rows behind it) is gathered ONCE into shared memory, then
// warp j folds item j for 32 of the columns from there (virtual slot s_j =
// col + c_j mod B, taps g[s_j + rB], rows in reference order, no FMA
// contraction: bit-identical to the per-item fold).  The C3 loop ladder
// (shifts 0,1,8,...,32768 in one window, N/16 in a second) gathers 27 + 19
// rows per column instead of 8 x 19; two polish permutations (0,1,2 each)
// 2 x 20 instead of 6 x 19.  About one slot's groups are in flight at a time,
// so the granules a slot touches stay in L2 across its windows.  Folded slots
// go to each item's output row; the in-place FFT pass follows.
constexpr int kGfCols = 32;    // columns per CTA (one per lane)
constexpr int kGfNT = 256;     // 8 warps: warp j folds item j
constexpr int kGfRows = 48;    // window rows held in shared memory at once
constexpr int kGfBack = 8;     // a window reaches at most this many rows back
constexpr int kGfTapRegs = 20; // most rows per slot (taps of a slot)
#ifndef SFFT_GF_HALF
#define SFFT_GF_HALF 10
#endif
constexpr int kGfTapHalf = SFFT_GF_HALF; // taps in registers at once
#ifndef SFFT_GF_MINB
#define SFFT_GF_MINB 5         // CTAs per SM the register budget is set for (4: 64 regs, no spills; 5 measured 7 % faster)
#endif

// Per group: its windows (head item, rows gathered before row 0, the batch
// and first shared-memory row they occupy) and per item the window, rows back
// a_j and column shift c_j -- formed once per group by k_gf_prep (the 64 CTAs
// of a group then load it in one round trip).
struct GfDesc {
  int32_t nwin, nbatch;
  int32_t win[kGfItems], a[kGfItems], c[kGfItems];
  int32_t head[kGfItems], back[kGfItems], row0[kGfItems], batch[kGfItems];
};
constexpr int kGfDescWords = (int)(sizeof(GfDesc) / sizeof(int32_t));

__global__ void k_gf_prep(Prod p, const int32_t* __restrict__ gfirst,
                          const int32_t* __restrict__ gcnt, int64_t ngroups, GfDesc* desc) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  const int first = gfirst[g];
  const int cnt = min(gcnt[g], kGfItems);
  const int64_t n = p.n, B = p.B;
  const int R = (int)((p.omega + B - 1) / B);
  const int A = min(kGfBack, R - 1);
  GfDesc d{};
  int nw = 0;
  for (int j = 0; j < cnt; ++j) {
    const int it = first + j;
    const int sg = p.item_sig ? p.item_sig[it] : it;
    const int64_t sm = p.item_a[it], tau = p.item_b[it];
    int w = -1;
    for (int q = 0; q < nw && w < 0; ++q) {
      const int h = first + d.head[q];
      if ((p.item_sig ? p.item_sig[h] : h) != sg || p.item_a[h] != sm) continue;
      const int64_t dd = pmod(tau - p.item_b[h], n);
      if (dd / B <= A) {
        w = q;
        d.a[j] = (int)(dd / B);
        d.c[j] = (int)(dd % B);
      }
    }
    if (w < 0) {
      w = nw++;
      d.head[w] = j;
      d.back[w] = 0;
      d.a[j] = 0;
      d.c[j] = 0;
    }
    d.win[j] = w;
    d.back[w] = max(d.back[w], d.a[j] + (d.c[j] > 0));
  }
  int nb = 0, used = kGfRows + 1;
  for (int w = 0; w < nw; ++w) {
    const int rows = R + d.back[w];
    if (used + rows > kGfRows) {
      ++nb;
      used = 0;
    }
    d.batch[w] = nb - 1;
    d.row0[w] = used;
    used += rows;
  }
  d.nwin = nw;
  d.nbatch = nb;
  desc[g] = d;
}

template <typename Tin>
__global__ void __launch_bounds__(kGfNT, SFFT_GF_MINB)
    k_group_fold(Prod p, const int32_t* __restrict__ gfirst, const int32_t* __restrict__ gcnt,
                 const GfDesc* __restrict__ desc, double2* __restrict__ out, int g0) {
  extern __shared__ __align__(16) unsigned char gf_smem[];
  Tin* V = reinterpret_cast<Tin*>(gf_smem);  // [kGfRows][kGfCols]
  __shared__ GfDesc sd;
  __shared__ int s_isig[kGfItems];
  __shared__ int64_t s_isgm[kGfItems], s_itau[kGfItems];
  const int g = g0 + blockIdx.y;
  const int first = gfirst[g];
  const int cnt = min(gcnt[g], kGfItems);
  const int B = (int)p.B, omega = (int)p.omega;
  const int64_t n = p.n;
  const int R = (omega + B - 1) / B;
  const int tail = omega - (R - 1) * B;  // slots s < tail have R rows, the rest R - 1
  const int col0 = blockIdx.x * kGfCols;
  if (p.prof_items && threadIdx.x == 0 && blockIdx.x == 0)
    atomicAdd(p.prof_items, (unsigned long long)cnt);
  // ---- the group's descriptor and items (one load each, in parallel)
  if (threadIdx.x < kGfDescWords)
    reinterpret_cast<int32_t*>(&sd)[threadIdx.x] =
        reinterpret_cast<const int32_t*>(desc + g)[threadIdx.x];
  if (threadIdx.x >= 128 && threadIdx.x < 128 + cnt) {
    const int j = threadIdx.x - 128, it = first + j;
    s_isig[j] = p.item_sig ? p.item_sig[it] : it;
    s_isgm[j] = p.item_a[it];
    s_itau[j] = p.item_b[it];
  }
  __syncthreads();
  const int nw = sd.nwin;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int bt = 0; bt < sd.nbatch; ++bt) {
    // ---- gather every needed sample of the batch's windows: asynchronous
    // 8/16-byte copies straight into shared memory, all in flight at once;
    // thread = (column lane, row phase)
    for (int w = 0; w < nw; ++w) {
      if (sd.batch[w] != bt) continue;
      const int h = sd.head[w];
      const Tin* xs = (const Tin*)p.x + (int64_t)s_isig[h] * p.xstride;
      const int64_t sm = s_isgm[h], tau = s_itau[h];
      const int back = sd.back[w], rows = R + back;
      // rows [-lo, hi) any item of the window needs in this lane's column
      int lo = 0, hi = 0;
      {
        const int gc = col0 + lane;
        if (gc < B)
          for (int j = 0; j < cnt; ++j) {
            if (sd.win[j] != w) continue;
            const int wrap = gc + sd.c[j] >= B;
            const int o = sd.a[j] + wrap;
            const int s = gc + sd.c[j] - (wrap ? B : 0);
            const int nr = R - (s >= tail);  // rows with s + rB < Omega (s < B)
            if (nr > 0) {
              lo = max(lo, o);
              hi = max(hi, nr - o);
            }
          }
      }
      Tin* vw = V + (int64_t)sd.row0[w] * kGfCols + lane;
      const int64_t base = (int64_t)(col0 + lane) - tau;
      for (int vr = warp; vr < rows; vr += kGfNT / 32) {
        const int v = vr - back;
        if (v < -lo || v >= hi) continue;
        const int64_t idx = mulmod(sm, pmod(base + (int64_t)v * B, n), n);
        SFFT_DASSERT(idx >= 0 && idx < n && sd.row0[w] + vr < kGfRows);
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(vw + vr * kGfCols);
        if (sizeof(Tin) == 8)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(xs + idx)
                       : "memory");
        else
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(xs + idx)
                       : "memory");
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    // ---- warp j folds item j (of this batch) for its 32 columns; its taps
    // are requested before the wait, so their L2 round trip overlaps the
    // gathers' DRAM one
    const int j = warp;
    const bool act = j < cnt && sd.batch[sd.win[j]] == bt && col0 + lane < B;
    int s = 0, nr = 0;
    const Tin* vc = V;
    // the first kGfTapHalf taps of the slot are requested before the wait, the
    // rest after the first half is folded: 20 doubles at once do not fit the
    // 48 registers of 5 CTAs per SM (80 bytes of spills per thread were 6.7 GB
    // of local-memory traffic per 512-slot launch, 6x the folded-slot stores)
    double t[kGfTapHalf];
    const double* tg = p.taps;
    if (act) {
      const int w = sd.win[j];
      const int gc = col0 + lane;
      const int cj = sd.c[j];
      const int wrap = gc + cj >= B;
      const int o = sd.a[j] + wrap;
      s = gc + cj - (wrap ? B : 0);
      nr = R - (s >= tail);
      vc = V + (int64_t)(sd.row0[w] + sd.back[w] - o) * kGfCols + lane;  // row r at vc[r C]
      SFFT_DASSERT(sd.row0[w] + sd.back[w] - o >= 0 && sd.row0[w] + sd.back[w] - o + nr <= kGfRows);
      SFFT_DASSERT(s >= 0 && s < B && nr <= kGfTapRegs);
      tg = p.taps + s;
#pragma unroll
      for (int r = 0; r < kGfTapHalf; ++r) t[r] = r < nr ? __ldg(tg + r * B) : 0.0;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    if (act) {
      double2 acc = cmk(0.0, 0.0);
#pragma unroll
      for (int h = 0; h < kGfTapRegs; h += kGfTapHalf) {
        if (h > 0) {
#pragma unroll
          for (int r = 0; r < kGfTapHalf; ++r) t[r] = h + r < nr ? __ldg(tg + (h + r) * B) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < kGfTapHalf; ++r)
          if (h + r < nr) {
            const double2 v = to_d2_(vc[(h + r) * kGfCols]);
            acc = cadd_rn(acc, cmk(__dmul_rn(t[r], v.x), __dmul_rn(t[r], v.y)));
          }
      }
      out[out_row(p, first + j) * p.B + s] = acc;
    }
    if (bt + 1 < sd.nbatch) __syncthreads();  // the next batch reuses the shared memory
  }
}

// ---- stream fold (opt-in, SFFT_STREAM_FOLD=1): a slot whose round reads a
// large part of its signal (the first loop round of the iterative engine with
// its speculative rows: 31 bucketizations over 7 permutations touch 18 % of
// the samples and 80 % of the 64-byte granules of a C3 signal) reads the
// signal ONCE, sequentially, instead of gathering.  With B | n the sample
// x[sigma (s + rB - tau)] of folded slot s lives in address column
// c = sigma (s - tau) mod B whatever the row r (sigma B = (sigma mod L) B mod
// n, L = n/B), and s <-> c is a bijection per item: the signal seen as X[j][c]
// (j < L rows of B samples), a CTA that holds address columns [c0, c0 + CW)
// for every j can form, for EVERY item of the slot, the complete folded slot
// of each of its columns -- rows in reference order from j0 + r (sigma mod L)
// mod L, taps g[s + rB], no FMA contraction, so bit-identical to the per-item
// fold.
//
// Persistent CTAs (one per SM) walk the (slot, column block) units; a unit is
// the 128-byte line [c0, c0 + CW) of every signal row.  One producer thread
// moves it with TMA tile loads (128 B x 256 rows per box) through a 7-box
// shared-memory ring (full/empty mbarriers; a unit of L = 1024 rows holds 4
// boxes, 3 more are in flight); the 512 consumer threads are the unit's
// (item, column) pairs: each reads its taps from the round's permuted tap
// table (k_sf_taps: T[item][r][c] = g[s_item(c) + rB], so a unit's taps are
// contiguous instead of one sector per tap; every first-round slot runs the
// same items, the permutation stream being shared), waits for the unit's
// boxes, folds from shared memory and writes its slot.
//
// Measured (profiles/r2_stream_fold_experiments.md): correct and
// bit-identical, but not faster than the group fold on this part -- both end
// at ~4.4 TB/s of mixed DRAM traffic (the scattered 16-byte folded-slot
// stores cost read-modify-write sectors, the tap table competes with the
// streamed signal for L2), 9.6 vs 8.6 us per slot -- so the group fold stays
// the default.
constexpr int kSfStages = 7;                       // ring of TMA boxes
constexpr int kSfCons = 512;                       // consumer threads
constexpr int kSfNT = kSfCons + 32;                // + the producer warp
constexpr int kSfGranule = 128;                    // bytes per signal row and unit: one line
constexpr int kSfMaxL = 1024;                      // rows
constexpr int kSfBoxRows = 256;                    // rows per TMA box (32 KB per stage)

bool stream_fold_ok(int dtype, const void* x, int64_t xstride, int64_t n, int64_t B,
                    int64_t omega) {
  const int64_t eb = dtype == 0 ? 8 : 16;
  if (n <= 0 || B <= 0 || (n & (n - 1)) || (B & (B - 1)) || B > n) return false;
  const int64_t L = n / B;
  if (L > kSfMaxL || L < 4 || B * eb < kSfGranule) return false;
  if (cdiv_up(omega, B) > kGfTapRegs || omega < B) return false;
  if (((uintptr_t)x % 128) || ((xstride * eb) % 128)) return false;
  return B < (1 << 30) && omega < (1 << 30) && tensor_map_encoder() != nullptr;
}

size_t stream_fold_taps_bytes(int64_t B, int64_t nitems) {
  return sizeof(double) * (size_t)kGfTapRegs * (size_t)B * (size_t)nitems;
}

// T[i][r][c] = g[s_i(c) + rB] (0 past Omega) for the lead slot's items i
__global__ void k_sf_taps(Prod p, const int4* __restrict__ dense, int R, double* __restrict__ T) {
  const int4 dd = __ldg(dense);
  const int i = blockIdx.y / R, r = blockIdx.y % R;
  if (i >= dd.z) return;
  const unsigned B = (unsigned)p.B;
  const uint64_t sg = (uint64_t)p.item_a[dd.y + i], tau = (uint64_t)p.item_b[dd.y + i];
  uint64_t inv = sg;
#pragma unroll
  for (int q = 0; q < 5; ++q) inv *= 2 - sg * inv;
  for (unsigned c = blockIdx.x * blockDim.x + threadIdx.x; c < B; c += gridDim.x * blockDim.x) {
    const unsigned s = (unsigned)((tau + inv * (uint64_t)c) & (B - 1));
    const int64_t idx = (int64_t)s + (int64_t)r * B;
    T[((size_t)i * R + r) * B + c] = idx < p.omega ? __ldg(p.taps + idx) : 0.0;
  }
}

__device__ __forceinline__ void sf_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(bar), "r"(parity)
      : "memory");
}

template <typename Tin>
__global__ void __launch_bounds__(kSfNT, 1)
    k_stream_fold(const __grid_constant__ CUtensorMap tmap, Prod p, const int4* __restrict__ dense,
                  int64_t nunits, const double* __restrict__ tperm, double2* __restrict__ out,
                  int lgB, int mode) {
  constexpr int CW = kSfGranule / (int)sizeof(Tin);
  extern __shared__ __align__(128) unsigned char sf_smem[];
  __shared__ __align__(8) uint64_t sf_full[kSfStages], sf_empty[kSfStages];
  const unsigned B = (unsigned)p.B, omega = (unsigned)p.omega;
  const unsigned L = (unsigned)(p.n >> lgB);
  const int R = (int)((omega + B - 1) / B);
  const unsigned tail = omega - (unsigned)(R - 1) * B;  // slots s < tail have R rows
  const unsigned nblk = B / CW;                         // units per slot
  const unsigned RB = L < (unsigned)kSfBoxRows ? L : (unsigned)kSfBoxRows;  // rows per box
  const unsigned NB = L / RB;                                               // boxes per unit
  const unsigned lgRB = 31 - __clz(RB);
  const unsigned stage_bytes = RB * kSfGranule;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(sf_smem);
  const uint32_t fb = (uint32_t)__cvta_generic_to_shared(sf_full);
  const uint32_t eb = (uint32_t)__cvta_generic_to_shared(sf_empty);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSfStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(fb + 8 * i));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(eb + 8 * i), "r"(kSfCons));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= kSfCons) {
    // ---- producer: box q of the CTA's k-th unit goes to ring position k NB + q
    if (threadIdx.x == kSfCons) {
      uint64_t pol;
      if (mode & 1)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
      else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(pol));
      unsigned pos = 0;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int4 dd = __ldg(dense + u / nblk);
        const int cx = (int)((u % nblk) * (kSfGranule / 8));  // in 8-byte words
        for (unsigned q = 0; q < NB; ++q, ++pos) {
          const unsigned st = pos % kSfStages;
          sf_mbar_wait(eb + 8 * st, ((pos / kSfStages) & 1) ^ 1);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(
                           fb + 8 * st),
                       "r"(stage_bytes)
                       : "memory");
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(
                  sbase + st * stage_bytes),
              "l"(&tmap), "r"(cx), "r"((int)(q * RB)), "r"(dd.w), "r"(fb + 8 * st), "l"(pol)
              : "memory");
        }
      }
    }
    return;
  }
  // ---- consumers: thread (item, column) of every unit
  const int t = threadIdx.x;
  unsigned pos0 = 0;  // ring position of the unit's first box
  for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x, pos0 += NB) {
    const int4 dd = __ldg(dense + u / nblk);  // slot, first item, items, signal
    const int first = dd.y, cnt = dd.z;
    const unsigned c0 = (unsigned)(u % nblk) * CW;
    if (p.prof_items && t == 0 && c0 == 0) atomicAdd(p.prof_items, (unsigned long long)cnt);
    const unsigned st0 = pos0 % kSfStages;
    const int total = cnt * CW;
    const int npass = (total + kSfCons - 1) / kSfCons;
    for (int pass = 0; pass < npass; ++pass) {
      const int w = pass * kSfCons + t;
      const bool act = w < total;
      unsigned s = 0, j = 0, jstep = 0, cc = 0;
      int nr = 0, item = first;
      double tp[kGfTapRegs];
      if (act) {
        const int i = w / CW;
        item = first + i;
        cc = (unsigned)(w % CW);
        const uint64_t sg = (uint64_t)p.item_a[item], tau = (uint64_t)p.item_b[item];
        uint64_t inv = sg;  // sigma^-1 mod 2^64 (sigma odd): Newton, 3 -> 96 bits
#pragma unroll
        for (int q = 0; q < 5; ++q) inv *= 2 - sg * inv;
        s = (unsigned)((tau + inv * (uint64_t)(c0 + cc)) & (B - 1));
        const uint64_t idx0 = (sg * ((uint64_t)s - tau)) & (uint64_t)(p.n - 1);
        SFFT_DASSERT((unsigned)(idx0 & (B - 1)) == c0 + cc);
        j = (unsigned)(idx0 >> lgB);
        jstep = (unsigned)(sg & (L - 1));
        nr = R - (s >= tail);
        const double* tg = tperm + (size_t)i * R * B + c0 + cc;
#pragma unroll
        for (int r = 0; r < kGfTapRegs; ++r) tp[r] = r < nr ? __ldg(tg + (size_t)r * B) : 0.0;
      }
      if (pass == 0)
        for (unsigned q = 0; q < NB; ++q)
          sf_mbar_wait(fb + 8 * ((pos0 + q) % kSfStages), ((pos0 + q) / kSfStages) & 1);
      double2 acc = cmk(0.0, 0.0);
      if (act) {
        const unsigned char* vc = sf_smem + cc * sizeof(Tin);
#pragma unroll
        for (int r = 0; r < kGfTapRegs; ++r)
          if (r < nr) {
            SFFT_DASSERT(j < L);
            unsigned st = st0 + (j >> lgRB);
            st -= st >= (unsigned)kSfStages ? (unsigned)kSfStages : 0u;
            const double2 v = to_d2_(*reinterpret_cast<const Tin*>(
                vc + st * stage_bytes + (j & (RB - 1)) * kSfGranule));
            acc = cadd_rn(acc, cmk(__dmul_rn(tp[r], v.x), __dmul_rn(tp[r], v.y)));
            j = (j + jstep) & (L - 1);
          }
      }
      if (pass == npass - 1)  // done with the unit's boxes: the producer may refill them
        for (unsigned q = 0; q < NB; ++q)
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(
                           eb + 8 * ((pos0 + q) % kSfStages))
                       : "memory");
      if (act) out[out_row(p, item) * p.B + s] = acc;
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
  // power-of-two B >= 8192 (flat fold pass or rows already folded): the
  // line-per-thread radix-8 passes; SFFT_NO_FS_POW2=1 keeps the generic ones
  static const bool fs_pow2_on = !getenv("SFFT_NO_FS_POW2");
  if (fs_pow2_on && (MODE == PROD_FLAT || MODE == PROD_LOAD) && B >= 8192 &&
      fs_pow2_split(B, &B1, &B2)) {
    Prod pz = p;
    if (MODE == PROD_FLAT) {
      dim3 gf((unsigned)cdiv_up(B, 2 * kFrNT), (unsigned)nitems);
      k_fold_rows<Tin><<<gf, kFrNT, 0, st>>>(p, out);
      SFFT_CHECK_LAUNCH("k_fold_rows");
      pz.z = out;
      pz.prof_items = nullptr;
    }
    return run_fs_pow2(pz, nitems, B1, B2, W, z, out, st);
  }
  if (split_plan(B, &B1, &B2)) {
    FftPlan P1, P2;
    make_plan(B1, &P1);
    make_plan(B2, &P2);
    // columns / rows per CTA: SFFT_FS_CAP shared-memory entries per CTA.  4096
    // (64 KB) with the passes capped at 64 registers puts two CTAs on an SM: the
    // passes are latency-bound (strided spike gathers, one barrier per stage),
    // measured 34.1k -> 38.2k C4 transforms/s against 8192 / one CTA
    static const int64_t fs_cap =
        getenv("SFFT_FS_CAP") ? std::max<int64_t>(256, atoll(getenv("SFFT_FS_CAP"))) : 4096;
    const int CG = (int)std::max<int64_t>(1, std::min<int64_t>(B2, fs_cap / (B1 + 1)));
    const int RG = (int)std::max<int64_t>(1, std::min<int64_t>(B1, fs_cap / (B2 + 1)));
    const size_t smc = (size_t)CG * (B1 + 1) * sizeof(double2) + (size_t)B1 * sizeof(int);
    const size_t smr = (size_t)RG * (B2 + 1) * sizeof(double2) + (size_t)B2 * sizeof(int);
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

// In-place FFT of folded rows (the group fold's second pass), power-of-two
// B <= 4096: one CTA per row, the row in shared memory (coalesced in and
// out), radix-8 DIF stages (the same butterflies and twiddles as fft_pow2, so
// the values are bit-identical to the cluster path), twiddles read through
// L1.  Shared-memory index i lives at i + i/8 + i/512: conflict-free for the
// unit-stride stage loads, the stride-8 last stage and the stride-512
// digit-reversed read-out.
constexpr int kFrowNT = 512;
__device__ __forceinline__ int frow_pad(int i) { return i + (i >> 3) + (i >> 9); }

template <int M>
__global__ void __launch_bounds__(kFrowNT) k_fft_rows(const int32_t* __restrict__ item_row,
                                                     const double2* __restrict__ W,
                                                     double2* __restrict__ y,
                                                     const int32_t* __restrict__ gfirst, int g_lo,
                                                     int g_hi, int nitems) {
  extern __shared__ double2 fr_s[];
  double2* tw8 = fr_s + frow_pad(M - 1) + 1;  // tw8[e] = W[8 e], e < M/8 (stages >= 2)
  // items [gfirst[g_lo], gfirst[g_hi]) (or all when gfirst is null)
  int item = blockIdx.x;
  if (gfirst) {
    item += gfirst[g_lo];
    if (item >= (g_hi >= 0 ? gfirst[g_hi] : nitems)) return;
  }
  SFFT_DASSERT(item >= 0 && (gfirst || item < (int)gridDim.x));
  double2* row = y + (int64_t)item_row[item] * M;
  // stage twiddles laid out [stage][q][j] (j contiguous): thread j of a warp
  // reads consecutive entries for every q.  The flat table tw8[j q 8^(st-1)]
  // made the eight j of the Mp = 8 stage hit one bank group for every q (8-way
  // conflicts on 7 loads per butterfly; ncu: L1/TEX 91 % busy, DRAM 38 %).
  // Same table values, so the results are unchanged bit for bit.
  {
    int off = 0, Mbs = M / 8;
    for (int st = 1; st < Pow2<M>::N8; ++st) {
      const int Mps = Mbs >> 3;
      for (int e = threadIdx.x; e < 7 * Mps; e += kFrowNT) {
        const int q = e / Mps + 1, j = e - (q - 1) * Mps;
        tw8[off + e] = __ldg(W + (int64_t)j * q * (M / Mbs));
      }
      off += 7 * Mps;
      Mbs = Mps;
    }
  }
  // stage 1 straight from global memory: the 8 inputs of a butterfly and its
  // twiddles are all requested at once (one round trip), then written to
  // shared memory already transformed
  constexpr int Mp1 = M / 8;
  for (int j = threadIdx.x; j < Mp1; j += kFrowNT) {
    double2 a[8], w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = row[j + q * Mp1];
#pragma unroll
    for (int q = 1; q < 8; ++q) w[q] = __ldg(W + j * q);
    dft8_(a);
    fr_s[frow_pad(j)] = a[0];
#pragma unroll
    for (int q = 1; q < 8; ++q) fr_s[frow_pad(j + q * Mp1)] = j ? cmul(a[q], w[q]) : a[q];
  }
  __syncthreads();
  int Mb = Mp1;
  int toff = 0;
#pragma unroll 1
  for (int st = 1; st < Pow2<M>::N8; ++st) {
    const int Mp = Mb >> 3;
    const double2* tws = tw8 + toff;  // tws[(q - 1) Mp + j] = w_M^{j q (M / Mb)}
    for (int t = threadIdx.x; t < M / 8; t += kFrowNT) {
      const int blk = t / Mp, j = t - blk * Mp;
      const int base = blk * Mb + j;
      double2 a[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) a[q] = fr_s[frow_pad(base + q * Mp)];
      dft8_(a);
      fr_s[frow_pad(base)] = a[0];
#pragma unroll
      for (int q = 1; q < 8; ++q)
        fr_s[frow_pad(base + q * Mp)] = j ? cmul(a[q], tws[(q - 1) * Mp + j]) : a[q];
    }
    __syncthreads();
    toff += 7 * Mp;
    Mb = Mp;
  }
  if (Pow2<M>::RL == 4) {
    for (int t = threadIdx.x; t < M / 4; t += kFrowNT) {
      double2 x0 = fr_s[frow_pad(4 * t)], x1 = fr_s[frow_pad(4 * t + 1)];
      double2 x2 = fr_s[frow_pad(4 * t + 2)], x3 = fr_s[frow_pad(4 * t + 3)];
      dft4_(x0, x1, x2, x3);
      fr_s[frow_pad(4 * t)] = x0;
      fr_s[frow_pad(4 * t + 1)] = x1;
      fr_s[frow_pad(4 * t + 2)] = x2;
      fr_s[frow_pad(4 * t + 3)] = x3;
    }
    __syncthreads();
  } else if (Pow2<M>::RL == 2) {
    for (int t = threadIdx.x; t < M / 2; t += kFrowNT) {
      const double2 u = fr_s[frow_pad(2 * t)], v = fr_s[frow_pad(2 * t + 1)];
      fr_s[frow_pad(2 * t)] = cadd(u, v);
      fr_s[frow_pad(2 * t + 1)] = csub(u, v);
    }
    __syncthreads();
  }
  const double bd = (double)M;
  for (int k = threadIdx.x; k < M; k += kFrowNT)
    row[k] = cdivr(fr_s[frow_pad(pow2_pos<M>(k))], bd);
}

static int launch_fft_rows(const int32_t* item_row, int64_t nitems, int64_t B, const double2* W,
                           double2* y, cudaStream_t st, const int32_t* gfirst = nullptr,
                           int g_lo = 0, int g_hi = -1, int64_t ntot = 0) {
  const size_t sm = (size_t)(B + B / 8 + B / 512 + 1 + B / 8) * sizeof(double2);
  switch (B) {
    case 4096:
      SFFT_CUDA(cudaFuncSetAttribute(k_fft_rows<4096>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      k_fft_rows<4096><<<(unsigned)nitems, kFrowNT, sm, st>>>(item_row, W, y, gfirst, g_lo, g_hi, (int)ntot);
      break;
    case 2048:
      if (ensure_smem(k_fft_rows<2048>, sm)) return -3;
      k_fft_rows<2048><<<(unsigned)nitems, kFrowNT, sm, st>>>(item_row, W, y, gfirst, g_lo, g_hi, (int)ntot);
      break;
    case 1024:
      if (ensure_smem(k_fft_rows<1024>, sm)) return -3;
      k_fft_rows<1024><<<(unsigned)nitems, kFrowNT, sm, st>>>(item_row, W, y, gfirst, g_lo, g_hi, (int)ntot);
      break;
    default:
      return 1;  // not handled here
  }
  SFFT_CHECK_LAUNCH("k_fft_rows");
  return 0;
}

// Flat bucketizations in item groups (items [gfirst[g], gfirst[g] + gcnt[g]),
// at most kGfItems, whole permutation runs of one slot; b' = 0, no gates):
// the group fold into each item's output row, then the FFT of every row in
// place.  Profiled (when on) as one bucketization launch of nitems items.
size_t flat_groups_desc_bytes(int64_t ngroups) { return (size_t)ngroups * sizeof(GfDesc); }

int run_flat_groups(int dtype, const Prod& p0, const int32_t* gfirst, const int32_t* gcnt,
                    int64_t ngroups, int64_t nitems, const double2* W, double2* out, void* ws,
                    size_t ws_bytes, void* desc_ws, cudaStream_t st, const int32_t* dense,
                    int64_t ndense, void* taps_ws, int max_items) {
  if ((ngroups <= 0 && ndense <= 0) || nitems <= 0) return 0;
  SFFT_REQUIRE(ndense <= 0 || (dense &&
                               stream_fold_ok(dtype, p0.x, p0.xstride, p0.n, p0.B, p0.omega)),
               "stream fold: streamed slots on a problem it cannot take");
  SFFT_REQUIRE(!p0.item_c && !p0.active && !p0.item_active && p0.item_row,
               "group fold: needs an ungated item list with output rows and b' = 0");
  const int R = (int)cdiv_up(p0.omega, p0.B);
  if (R + std::min(kGfBack, R - 1) + 1 > kGfRows || R > kGfTapRegs || p0.B >= (1 << 30) ||
      p0.omega >= (1 << 30))
    return run_bucketize(dtype, PROD_FLAT, p0, nitems, W, out, ws, ws_bytes, st);
  gather_fetch_granularity();
  BucketProf& bp = bucket_prof();
  Prod p = p0;
  p.prof_items = bp.on ? bp.d_items : nullptr;
  cudaEvent_t ev0{};
  if (bp.on) {
    int rc = prof_begin(st, &ev0);
    if (rc) return rc;
  }
  GfDesc* desc = (GfDesc*)desc_ws;
  if (ngroups > 0) {
    k_gf_prep<<<(unsigned)cdiv_up(ngroups, 128), 128, 0, st>>>(p, gfirst, gcnt, ngroups, desc);
    SFFT_CHECK_LAUNCH("k_gf_prep");
  }
  if (ndense > 0) {
    // streamed slots first: their FFT rows are the bulk of the row pass
    SFFT_REQUIRE(taps_ws, "stream fold: no tap table scratch");
    const int64_t L = p.n / p.B;
    const size_t ssm = (size_t)kSfStages * std::min<int64_t>(L, kSfBoxRows) * kSfGranule;
    int lgB = 0;
    while (((int64_t)1 << lgB) < p.B) ++lgB;
    const int64_t eb = dtype == 0 ? 8 : 16;
    const int64_t nunits = ndense * (p.B * eb / kSfGranule);
    CUtensorMap tmap;
    if (stream_tensor_map(p.x, p.xstride, p.n, p.B, eb, &tmap)) return -3;
    const int4* dp = reinterpret_cast<const int4*>(dense);
    double* tperm = (double*)taps_ws;
    k_sf_taps<<<dim3((unsigned)cdiv_up(p.B, 256), (unsigned)(max_items * R)), 256, 0, st>>>(
        p, dp, R, tperm);
    SFFT_CHECK_LAUNCH("k_sf_taps");
    int dev = 0, sms = 0, per = 0;
    SFFT_CUDA(cudaGetDevice(&dev));
    SFFT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (dtype == 0) {
      SFFT_CUDA(cudaFuncSetAttribute(k_stream_fold<float2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
      SFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stream_fold<float2>, kSfNT,
                                                              ssm));
    } else {
      SFFT_CUDA(cudaFuncSetAttribute(k_stream_fold<double2>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
      SFFT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_stream_fold<double2>, kSfNT,
                                                              ssm));
    }
    const unsigned grid = (unsigned)std::min<int64_t>(nunits, (int64_t)sms * std::max(per, 1));
    const char* me = getenv("SFFT_SF_MODE");
    const int mode = me ? atoi(me) : 1;  // bit 0: evict_first on the streamed lines
    if (dtype == 0)
      k_stream_fold<float2><<<grid, kSfNT, ssm, st>>>(tmap, p, dp, nunits, tperm, out, lgB, mode);
    else
      k_stream_fold<double2><<<grid, kSfNT, ssm, st>>>(tmap, p, dp, nunits, tperm, out, lgB, mode);
    SFFT_CHECK_LAUNCH("k_stream_fold");
  }
  const size_t sm = (size_t)kGfRows * kGfCols * (dtype == 0 ? sizeof(float2) : sizeof(double2));
  if (dtype == 0)
    SFFT_CUDA(cudaFuncSetAttribute(k_group_fold<float2>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  else
    SFFT_CUDA(cudaFuncSetAttribute(k_group_fold<double2>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  auto fold = [&](int64_t g0, int64_t ng, cudaStream_t s2) -> int {
    const dim3 g((unsigned)cdiv_up(p.B, kGfCols), (unsigned)ng);
    if (dtype == 0)
      k_group_fold<float2><<<g, kGfNT, sm, s2>>>(p, gfirst, gcnt, desc, out, (int)g0);
    else
      k_group_fold<double2><<<g, kGfNT, sm, s2>>>(p, gfirst, gcnt, desc, out, (int)g0);
    SFFT_CHECK_LAUNCH("k_group_fold");
    return 0;
  };
  // SFFT_GF_FFT=cluster keeps the cluster FFT pass (A/B measurements)
  const char* fe = getenv("SFFT_GF_FFT");
  const bool rows = !(fe && !strcmp(fe, "cluster")) && (p.B == 4096 || p.B == 2048 || p.B == 1024);
  int rc = 0;
  {
    if (ngroups > 0 && (rc = fold(0, ngroups, st))) return rc;
    rc = rows ? launch_fft_rows(p.item_row, nitems, p.B, W, out, st) : 1;
    if (rc > 0) {
      Prod pl = p;
      pl.z = out;
      pl.prof_items = nullptr;
      rc = run_bucketize_inner(dtype, PROD_LOAD, pl, nitems, W, out, ws, ws_bytes, st);
    }
  }
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
