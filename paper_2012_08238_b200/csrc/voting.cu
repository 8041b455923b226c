// Batched voting framework (sfft/frameworks.py:354-417), device-resident.
//
// S signals x R rounds in one pass of launches, no host synchronisation:
//   y[s][r]    = bucketize(x_s, sigma_r, tau_r)                     (A5)
//   thr[s][r]  = robust_noise_floor(y[s][r])                         (A8)
//   heavy bits = first 2K eligible buckets in (-|y|, b) order         (A9)
//   cand[s]    = positions with >= R/2 votes, (-votes, pos), first 2K (A10, A11)
//   [optional spike pre-stage: keep candidates whose f mod B_pre bucket is heavy]
//   est        = y[b]/(G w^{tau m}), NaN under 0.05 max|G|          (A12)
//   coef       = trimmed mean over rounds                            (A13)
//   2 x: safe = finite(coef) ? coef : 0; est of y - model(safe) at the
//        candidate buckets (A14 restricted); coef = safe + trimmed mean
//   entries    = finite coefficients, top K by (-|c|, f)
#include "kernels.cuh"
#include "schedule.cuh"
#include "finalize.cuh"
#include "robust.cuh"

namespace sfft {

struct VoteArgs {
  int64_t n, B, L, omega, k;
  int S, R, C;                   // C = 2k candidate capacity
  const int64_t* psig;           // [S][R]
  const int64_t* ptau;           // [S][R]
  const double2* gt;
  const double* gmax;
  double2* y;                    // [S*R][B]
  int64_t* cand;                 // [S][C]
  int32_t* ncand;                // [S]
  int64_t* m;                    // [S][R][C]  sigma_r * f mod n
  int32_t* bk;                   // [S][R][C]  candidate bucket
  double2* w;                    // [S][R][C]  own weight G[bL - m]
  double2* ph;                   // [S][R][C]  w^{tau_r m}
  double2* est;                  // [S][R][C]
  double2* coef;                 // [S][C]
  double2* safe;                 // [S][C]
};

__global__ void k_vo_prep(VoteArgs a) {
  const int s = blockIdx.z, r = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.ncand[s]) return;
  const int64_t n = a.n, L = a.L, B = a.B;
  const int64_t i = ((int64_t)s * a.R + r) * a.C + c;
  const int64_t sg = a.psig[(int64_t)s * a.R + r];
  const int64_t tau = a.ptau[(int64_t)s * a.R + r];
  const int64_t m = mulmod(sg, pmod(a.cand[(int64_t)s * a.C + c], n), n);
  const int64_t b = pmod(m + L / 2, n) / L;
  const int64_t e = pmod(b * L - m, n);
  a.m[i] = m;
  a.bk[i] = (int32_t)b;
  a.w[i] = a.gt[(e % L) * B + e / L];
  a.ph[i] = unit_root(n, mulmod(tau, m, n));
}

// est[s][r][c] of y (pass 0) or of y - model(safe) (refinement passes).
constexpr int kVoNT = 128;
constexpr int kVoChunk = 128;

__global__ void __launch_bounds__(kVoNT) k_vo_est(VoteArgs a, int refine) {
  __shared__ int64_t u_row[kVoChunk], u_q[kVoChunk];
  __shared__ double2 u_cp[kVoChunk];
  const int s = blockIdx.z, r = blockIdx.y;
  const int C = a.ncand[s];
  const int c0 = blockIdx.x * kVoNT;
  if (c0 >= C) return;
  const int c = c0 + threadIdx.x;
  const bool live = c < C;
  const int64_t n = a.n, L = a.L, B = a.B;
  const int64_t base = ((int64_t)s * a.R + r) * a.C;
  int64_t b = 0;
  double2 v = cmk(0.0, 0.0);
  if (live) {
    b = a.bk[base + c];
    v = a.y[((int64_t)s * a.R + r) * B + b];
  }
  if (refine) {
    const double2* sf = a.safe + (int64_t)s * a.C;
    for (int u0 = 0; u0 < C; u0 += kVoChunk) {
      __syncthreads();
      for (int q = threadIdx.x; q < kVoChunk && u0 + q < C; q += kVoNT) {
        const int64_t mu = a.m[base + u0 + q];
        u_row[q] = (L - mu % L) % L;
        u_q[q] = (mu + L - 1) / L;
        u_cp[q] = sf[u0 + q];
      }
      __syncthreads();
      if (live) {
        const int un = min(kVoChunk, C - u0);
        // (c * w) * phase, subtracted in model order (frameworks.py:432-435);
        // 8 table reads in flight
        int q = 0;
        for (; q + 8 <= un; q += 8) {
          double2 wq[8], pq[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            int64_t col = b - u_q[q + u];
            col += (col < 0) ? B : 0;
            wq[u] = ld_table(a.gt + u_row[q + u] * B + col);
            pq[u] = a.ph[base + u0 + q + u];
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) v = csub(v, cmul(cmul(u_cp[q + u], wq[u]), pq[u]));
        }
        for (; q < un; ++q) {
          int64_t col = b - u_q[q];
          col += (col < 0) ? B : 0;
          const double2 wq = ld_table(a.gt + u_row[q] * B + col);
          v = csub(v, cmul(cmul(u_cp[q], wq), a.ph[base + u0 + q]));
        }
      }
    }
  }
  if (!live) return;
  const double2 w = a.w[base + c];
  a.est[base + c] = (cabs_(w) < 0.05 * a.gmax[0]) ? cmk(CUDART_NAN, 0.0)
                                                  : cdiv(v, cmul(w, a.ph[base + c]));
}


// coef = [safe +] trimmed mean over rounds; next safe = finite ? coef : 0.
__global__ void k_vo_tmean(VoteArgs a, int refine, int last) {
  const int s = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= a.ncand[s]) return;
  const int64_t i = (int64_t)s * a.C + c;
  const double2 tm = trimmed_mean_col(a.est + (int64_t)s * a.R * a.C + c, a.C, a.R);
  const double2 cf = refine ? cadd(a.safe[i], tm) : tm;
  const bool fin = isfinite(cf.x) && isfinite(cf.y);
  a.coef[i] = (last && !fin) ? cmk(0.0, 0.0) : cf;  // non-finite entries are dropped
  a.safe[i] = fin ? cf : cmk(0.0, 0.0);
}

// Spike pre-stage filter (frameworks.py:373-382, :396-397): stable compaction
// of the candidates whose bucket f mod B_pre is among the pre-stage's heavy.
__global__ void k_vo_prefilter(VoteArgs a, const uint32_t* pbits, int64_t Bpre) {
  __shared__ int red[32];
  const int s = blockIdx.x;
  const int C = a.ncand[s];
  int64_t* cs = a.cand + (int64_t)s * a.C;
  const int64_t words = (Bpre + 31) / 32;
  const uint32_t* bw = pbits + (int64_t)s * words;
  const int per = (C + blockDim.x - 1) / blockDim.x;
  const int i0 = threadIdx.x * per, i1 = min(C, i0 + per);
  int64_t keep[32];
  int nk = 0;
  for (int i = i0; i < i1; ++i) {
    const int64_t f = cs[i];
    const int64_t bb = f % Bpre;
    if ((bw[bb >> 5] >> (bb & 31)) & 1u) keep[nk++] = f;
  }
  int tot;
  int off = block_exscan<256>(nk, red, &tot);
  __syncthreads();
  for (int j = 0; j < nk; ++j) cs[off + j] = keep[j];
  if (threadIdx.x == 0) a.ncand[s] = tot;
}

// gate[s] = 1 for signal 0 and for every signal whose (sigma, tau) rows differ
// from signal 0's; the others take signal 0's samples_read.
__global__ void k_vo_same(const int64_t* __restrict__ psig, const int64_t* __restrict__ ptau,
                          int S, int R, int32_t* gate) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  bool diff = false;
  for (int r = 0; r < R; ++r)
    diff |= psig[(int64_t)s * R + r] != psig[r] || ptau[(int64_t)s * R + r] != ptau[r];
  gate[s] = (s == 0 || diff) ? 1 : 0;
}

__global__ void k_vo_samples(int64_t* samples, const int32_t* gate, int S) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < S && !gate[s]) samples[s] = samples[0];
}

__global__ void k_vo_groups(Group* groups, int32_t* ngroups, const int64_t* psig,
                            const int64_t* ptau, int S, int R, int64_t omega, int64_t pre_L,
                            int64_t pre_B) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  Group* g = groups + (int64_t)s * kMaxGroups;
  int ng = 0;
  if (pre_B > 0) {
    g[ng].kind = 1;
    g[ng].a = pre_L;
    g[ng].tau = 0;
    g[ng].cnt = pre_B;
    g[ng].nsh = 1;
    g[ng].sh[0] = 0;
    ++ng;
  }
  for (int r = 0; r < R && ng < kMaxGroups; ++r, ++ng) {
    g[ng].kind = 0;
    g[ng].a = psig[(int64_t)s * R + r];
    g[ng].tau = ptau[(int64_t)s * R + r];
    g[ng].cnt = omega;
    g[ng].nsh = 1;
    g[ng].sh[0] = 0;
  }
  ngroups[s] = ng;
}

__global__ void k_vo_items(int S, int R, int32_t* item_sig) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < S * R) item_sig[i] = i / R;
}

struct VoteLayout {
  size_t off[24];
  size_t total;
};

static size_t alv(size_t x) { return (x + 255) & ~size_t(255); }

static VoteLayout vote_layout(int64_t n, int64_t B, int S, int R, int C, int64_t Bpre) {
  VoteLayout L{};
  const size_t SRC = (size_t)S * R * C;
  const int64_t words = (B + 31) / 32;
  size_t sizes[] = {
      sizeof(double2) * (size_t)S * R * B,        // 0 y
      sizeof(double) * (size_t)S * R,             // 1 thr
      sizeof(uint32_t) * (size_t)S * R * words,   // 2 heavy bits
      sizeof(int64_t) * (size_t)S * C,            // 3 cand
      sizeof(int32_t) * (size_t)S,                // 4 ncand
      sizeof(int64_t) * SRC,                      // 5 m
      sizeof(int32_t) * SRC,                      // 6 bk
      sizeof(double2) * SRC,                      // 7 w
      sizeof(double2) * SRC,                      // 8 ph
      sizeof(double2) * SRC,                      // 9 est
      sizeof(double2) * (size_t)S * C,            // 10 coef
      sizeof(double2) * (size_t)S * C,            // 11 safe
      votes_ws_bytes(n, S, R),                    // 12 chist
      sizeof(Group) * (size_t)S * kMaxGroups,     // 13 groups
      sizeof(int32_t) * (size_t)S,                // 14 ngroups
      sizeof(int32_t) * (size_t)S * R,            // 15 item_sig
      sizeof(double2) * (size_t)S * (Bpre > 0 ? Bpre : 1),            // 16 pre y
      sizeof(uint32_t) * (size_t)S * ((Bpre > 0 ? Bpre : 1) + 31) / 32 + 64,  // 17 pre bits
      sizeof(double) * (size_t)S,                 // 18 pre thr
      sizeof(int64_t) * (size_t)S,                // 19 pre tau (zeros)
      votes_fast_ws_bytes(S, R, 2 * (int64_t)(C / 2)),  // 20 fast vote workspace
      union_scratch_bytes(S),                     // 21 union-count fallback gate
  };
  size_t o = 0;
  const int cnt = sizeof(sizes) / sizeof(sizes[0]);
  for (int i = 0; i < cnt; ++i) {
    L.off[i] = o;
    o += alv(sizes[i]);
  }
  L.total = o;
  return L;
}

size_t voting_ws_bytes(int64_t n, int64_t B, int S, int R, int C, int64_t Bpre) {
  return vote_layout(n, B, S, R, C, Bpre).total +
         std::max(bucketize_ws_bytes(B, (int64_t)S * R),
                  Bpre > 0 ? bucketize_ws_bytes(Bpre, S) : (size_t)0);
}

int run_voting(int dtype, const void* x, int64_t n, int64_t xstride, int S, const double* taps,
               int64_t omega, int64_t B, const double2* gt, const double* gmax, const double2* W,
               const int64_t* psig, const int64_t* ptau, int R, int64_t k, int need,
               int64_t Bpre, const double2* Wpre, int64_t* out_pos, double2* out_coef,
               int32_t* out_n, int64_t* out_samples, int64_t* out_sched, void* ws,
               size_t ws_bytes, cudaStream_t st) {
  SFFT_REQUIRE(R >= 1 && R <= kMaxVoteRounds, "voting: 1 <= rounds <= 255");
  const int C = (int)(2 * k);
  SFFT_REQUIRE(C >= 1 && C <= kFusedMaxB, "voting: 2k must be <= 8192");
  SFFT_REQUIRE(ws_bytes >= voting_ws_bytes(n, B, S, R, C, Bpre), "voting: workspace too small");
  const VoteLayout Lo = vote_layout(n, B, S, R, C, Bpre);
  char* w = (char*)ws;
  VoteArgs a{};
  a.n = n;
  a.B = B;
  a.L = n / B;
  a.omega = omega;
  a.k = k;
  a.S = S;
  a.R = R;
  a.C = C;
  a.psig = psig;
  a.ptau = ptau;
  a.gt = gt;
  a.gmax = gmax;
  a.y = (double2*)(w + Lo.off[0]);
  double* thr = (double*)(w + Lo.off[1]);
  uint32_t* bits = (uint32_t*)(w + Lo.off[2]);
  a.cand = (int64_t*)(w + Lo.off[3]);
  a.ncand = (int32_t*)(w + Lo.off[4]);
  a.m = (int64_t*)(w + Lo.off[5]);
  a.bk = (int32_t*)(w + Lo.off[6]);
  a.w = (double2*)(w + Lo.off[7]);
  a.ph = (double2*)(w + Lo.off[8]);
  a.est = (double2*)(w + Lo.off[9]);
  a.coef = (double2*)(w + Lo.off[10]);
  a.safe = (double2*)(w + Lo.off[11]);
  int* chist = (int*)(w + Lo.off[12]);
  Group* groups = (Group*)(w + Lo.off[13]);
  int32_t* ngroups = (int32_t*)(w + Lo.off[14]);
  int32_t* item_sig = (int32_t*)(w + Lo.off[15]);
  void* fastws = w + Lo.off[20];
  void* bws = w + Lo.total;
  const size_t bws_bytes = ws_bytes - Lo.total;

  k_vo_items<<<(unsigned)cdiv_up((int64_t)S * R, 256), 256, 0, st>>>(S, R, item_sig);
  SFFT_CHECK_LAUNCH("k_vo_items");
  Prod p{};
  p.x = x;
  p.xstride = xstride;
  p.n = n;
  p.taps = taps;
  p.omega = omega;
  p.B = B;
  p.item_sig = item_sig;
  p.item_a = psig;
  p.item_b = ptau;
  int rc = run_bucketize(dtype, PROD_FLAT, p, (int64_t)S * R, W, a.y, bws, bws_bytes, st);
  if (rc) return rc;
  rc = run_floor_heavy(a.y, (int64_t)S * R, B, 3.0, 2 * k, thr, bits, nullptr, st);
  if (rc) return rc;
  VoteRounds vr{};
  vr.bits = bits;
  vr.sigma = psig;
  vr.bprime = nullptr;
  vr.n = n;
  vr.B = B;
  vr.L = n / B;
  vr.words = (B + 31) / 32;
  vr.cs = 0;
  vr.R = R;
  {
    int overflow = 0;
    rc = run_votes_fast(vr, S, need, C, 2 * k, a.cand, a.ncand, fastws, votes_fast_ws_bytes(S, R, 2 * k),
                        &overflow, st);
    if (rc) return rc;
    if (overflow) {  // some signal has > 8192 candidates: exact chunked ranking
      rc = run_votes(vr, S, nullptr, nullptr, need, C, a.cand, a.ncand, chist, true, st);
      if (rc) return rc;
    }
  }

  int64_t pre_L = 0;
  if (Bpre > 0) {
    double2* py = (double2*)(w + Lo.off[16]);
    uint32_t* pbits = (uint32_t*)(w + Lo.off[17]);
    double* pthr = (double*)(w + Lo.off[18]);
    int64_t* ptz = (int64_t*)(w + Lo.off[19]);
    SFFT_CUDA(cudaMemsetAsync(ptz, 0, sizeof(int64_t) * S, st));
    Prod q{};
    q.x = x;
    q.xstride = xstride;
    q.n = n;
    q.B = Bpre;
    q.item_a = ptz;
    rc = run_bucketize(dtype, PROD_SPIKE, q, S, Wpre, py, bws, bws_bytes, st);
    if (rc) return rc;
    rc = run_floor_heavy(py, S, Bpre, 3.0, 2 * k, pthr, pbits, nullptr, st);
    if (rc) return rc;
    k_vo_prefilter<<<S, 256, 0, st>>>(a, pbits, Bpre);
    SFFT_CHECK_LAUNCH("k_vo_prefilter");
    pre_L = n / Bpre;
  }

  const dim3 gp((unsigned)cdiv_up(C, 128), R, S);
  k_vo_prep<<<gp, 128, 0, st>>>(a);
  SFFT_CHECK_LAUNCH("k_vo_prep");
  const dim3 ge((unsigned)cdiv_up(C, kVoNT), R, S);
  const dim3 gt2((unsigned)cdiv_up(C, 128), S);
  for (int pass = 0; pass < 3; ++pass) {
    k_vo_est<<<ge, kVoNT, 0, st>>>(a, pass > 0);
    SFFT_CHECK_LAUNCH("k_vo_est");
    k_vo_tmean<<<gt2, 128, 0, st>>>(a, pass > 0, pass == 2);
    SFFT_CHECK_LAUNCH("k_vo_tmean");
  }
  const size_t dsm = (size_t)kFusedMaxB * (8 + 8 + 4);
  SFFT_CUDA(cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  k_finalize<<<S, kFinNT, dsm, st>>>(a.cand, a.coef, a.ncand, C, k, out_pos, out_coef, out_n);
  SFFT_CHECK_LAUNCH("k_finalize");
  k_vo_groups<<<(unsigned)cdiv_up(S, 128), 128, 0, st>>>(groups, ngroups, psig, ptau, S, R, omega,
                                                         pre_L, Bpre);
  SFFT_CHECK_LAUNCH("k_vo_groups");
  // signals that share signal 0's permutations read the same samples (the
  // batched runner draws one seeded stream for the whole batch): those are
  // counted once, by more CTAs, and copied
  int32_t* same_gate = (int32_t*)(w + Lo.off[21]) + 2 * (size_t)S;
  k_vo_same<<<(unsigned)cdiv_up(S, 128), 128, 0, st>>>(psig, ptau, S, R, same_gate);
  SFFT_CHECK_LAUNCH("k_vo_same");
  rc = run_union_count(groups, ngroups, S, n, out_samples, same_gate, nullptr, st,
                      (int32_t*)(w + Lo.off[21]), 32);
  if (rc) return rc;
  k_vo_samples<<<(unsigned)cdiv_up(S, 128), 128, 0, st>>>(out_samples, same_gate, S);
  SFFT_CHECK_LAUNCH("k_vo_samples");
  if (out_sched) {
    k_export_groups<<<S, 64, 0, st>>>(groups, ngroups, S, out_sched);
    SFFT_CHECK_LAUNCH("k_export_groups");
  }
  return 0;
}

}  // namespace sfft
