// Batched one-shot framework (sfft/frameworks.py:216-311), device-resident.
//
//   meas[t]  = bucketize_spike(x, B, shift_t) for the shifts
//              0..2a_max-1, the phase-ladder rungs not among them, and the
//              seeded pursuit shifts                                    (A7)
//   floor    = robust_noise_floor(|meas[0]|)                            (A8)
//   counts   = count_collisions: singular values of every bucket's
//              a_max x a_max moment Hankel matrix, pooled per signal
//              (cutoff = 2B-th largest, floor = max(3 median, 1e-12 max))
//              (sfft/reconstruct.py:245-267)
//   per bucket with counts > 0 and mean|m| >= floor (one thread each):
//              single-ton by phase unwrapping over the ladder rows, else
//              Prony (linear prediction by least squares + polynomial roots,
//              sfft/reconstruct.py:270-302) with escalation over a and one
//              partner-subtraction refinement, least-squares coefficients
//              over all shifts (estimate_prony, :374-409), residual test.
//
// The small dense algebra (Hankel singular values, the linear-prediction and
// Vandermonde least squares) is a one-sided complex Jacobi SVD in fp64 — the
// least-squares solution and the rank/conditioning tests numpy's lstsq (gelsd)
// makes, from singular values of the same matrices.  Polynomial roots are
// Aberth-Ehrlich iterations with Newton polishing (numpy: companion-matrix
// eigenvalues); positions are snapped to the bucket's candidates, so both
// agree wherever the reference's decision is not a rounding tie.
#include "kernels.cuh"
#include "schedule.cuh"
#include "finalize.cuh"

namespace sfft {

constexpr int kOsMaxA = 8;      // a_max
constexpr int kOsMaxRows = 64;  // measurement shifts (= read groups)
constexpr int kOsMaxLad = 16;   // phase-ladder rungs
constexpr int kOsNT = 64;

struct OsArgs {
  int64_t n, B, k;
  int S, A, nsh, nlad;
  int64_t shifts[kOsMaxRows];
  int32_t lad_row[kOsMaxLad];    // measurement row of ladder rung j (rungs ascending)
  int64_t lad[kOsMaxLad];
  const double2* meas;           // [nsh][S][B]
  const double* floor;           // [S]
  double* svals;                 // [S][B][A] Hankel singular values, descending
  double* energy;                // [S][B] mean_t |m_t|, t < 2A
  double* cut;                   // [S] pooled cutoff
  double* sfl;                   // [S] pooled floor
  int64_t* rec_pos;              // [S][cap]
  double2* rec_coef;
  int32_t* rec_count;            // [S]
  int cap;
};

// ------------------------------------------------------------------ small algebra

__device__ __forceinline__ double cnorm2(double2 z) { return z.x * z.x + z.y * z.y; }

// One-sided (Hestenes) Jacobi SVD of the m x nc column-major matrix a
// (leading dimension ld), in place: on return column j of a is sigma_j u_j
// and sv[j] = sigma_j.  v (nc x nc, column-major, leading dimension kOsMaxA)
// accumulates the right singular vectors when non-null.
__device__ void jacobi_svd(double2* a, int ld, int m, int nc, double* sv, double2* v) {
  if (v)
    for (int j = 0; j < nc; ++j)
      for (int i = 0; i < nc; ++i) v[j * kOsMaxA + i] = cmk(i == j ? 1.0 : 0.0, 0.0);
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rot = false;
    for (int p = 0; p + 1 < nc; ++p)
      for (int q = p + 1; q < nc; ++q) {
        double al = 0.0, be = 0.0;
        double2 g = cmk(0.0, 0.0);
        for (int r = 0; r < m; ++r) {
          const double2 x = a[p * ld + r], y = a[q * ld + r];
          al += cnorm2(x);
          be += cnorm2(y);
          g = cadd(g, cmul(cconj(x), y));
        }
        const double ga = hypot(g.x, g.y);
        if (ga == 0.0 || ga <= 1e-15 * sqrt(al * be)) continue;
        rot = true;
        const double2 ph = cmk(g.x / ga, -g.y / ga);  // conj(g / |g|)
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int r = 0; r < m; ++r) {
          const double2 x = a[p * ld + r], y = cmul(ph, a[q * ld + r]);
          a[p * ld + r] = cmk(c * x.x - s * y.x, c * x.y - s * y.y);
          a[q * ld + r] = cmk(s * x.x + c * y.x, s * x.y + c * y.y);
        }
        if (v)
          for (int r = 0; r < nc; ++r) {
            const double2 x = v[p * kOsMaxA + r], y = cmul(ph, v[q * kOsMaxA + r]);
            v[p * kOsMaxA + r] = cmk(c * x.x - s * y.x, c * x.y - s * y.y);
            v[q * kOsMaxA + r] = cmk(s * x.x + c * y.x, s * x.y + c * y.y);
          }
      }
    if (!rot) break;
  }
  for (int j = 0; j < nc; ++j) {
    double z = 0.0;
    for (int r = 0; r < m; ++r) z += cnorm2(a[j * ld + r]);
    sv[j] = sqrt(z);
  }
}

// Least squares min |A x - b| from the Jacobi factors (numpy lstsq, rcond =
// eps * max(m, nc)): x = sum_{sigma_j > rcond sigma_max} v_j (a_j^H b) / sigma_j^2.
// Returns the numerical rank; smin/smax receive the extreme singular values.
__device__ int svd_lstsq(double2* a, int ld, int m, int nc, const double2* b, double2* x,
                         double* smax, double* smin) {
  double sv[kOsMaxA];
  double2 v[kOsMaxA * kOsMaxA];
  jacobi_svd(a, ld, m, nc, sv, v);
  double hi = 0.0, lo = CUDART_INF;
  for (int j = 0; j < nc; ++j) {
    hi = fmax(hi, sv[j]);
    lo = fmin(lo, sv[j]);
  }
  const double rc = 2.220446049250313e-16 * (double)(m > nc ? m : nc) * hi;
  int rank = 0;
  for (int i = 0; i < nc; ++i) x[i] = cmk(0.0, 0.0);
  for (int j = 0; j < nc; ++j) {
    if (!(sv[j] > rc)) continue;
    ++rank;
    double2 d = cmk(0.0, 0.0);
    for (int r = 0; r < m; ++r) d = cadd(d, cmul(cconj(a[j * ld + r]), b[r]));
    d = cdivr(d, sv[j] * sv[j]);
    for (int i = 0; i < nc; ++i) x[i] = cadd(x[i], cmul(v[j * kOsMaxA + i], d));
  }
  *smax = hi;
  *smin = lo;
  return rank;
}

// Roots of z^a + c[a-1] z^{a-1} + ... + c[0] (Aberth-Ehrlich, Newton polish).
__device__ void poly_roots(const double2* c, int a, double2* z) {
  if (a == 1) {
    z[0] = cmk(-c[0].x, -c[0].y);
    return;
  }
  auto eval = [&](double2 w, double2* p, double2* dp) {
    double2 pv = cmk(1.0, 0.0), dv = cmk(0.0, 0.0);
    for (int j = a - 1; j >= 0; --j) {
      dv = cadd(cmul(dv, w), pv);
      pv = cadd(cmul(pv, w), c[j]);
    }
    *p = pv;
    *dp = dv;
  };
  const double c0 = hypot(c[0].x, c[0].y);
  const double r = c0 > 0.0 ? pow(c0, 1.0 / a) : 1.0;
  for (int k = 0; k < a; ++k) {
    double sn, cs;
    sincos(6.283185307179586 * k / a + 0.4, &sn, &cs);
    z[k] = cmk(r * cs, r * sn);
  }
  for (int it = 0; it < 500; ++it) {
    double big = 0.0;
    for (int k = 0; k < a; ++k) {
      double2 p, dp;
      eval(z[k], &p, &dp);
      if (p.x == 0.0 && p.y == 0.0) continue;
      const double2 ratio = cdiv(p, dp);
      double2 sum = cmk(0.0, 0.0);
      for (int j = 0; j < a; ++j)
        if (j != k) sum = cadd(sum, cdiv(cmk(1.0, 0.0), csub(z[k], z[j])));
      const double2 w = cdiv(ratio, csub(cmk(1.0, 0.0), cmul(ratio, sum)));
      z[k] = csub(z[k], w);
      big = fmax(big, hypot(w.x, w.y) / fmax(hypot(z[k].x, z[k].y), 1e-300));
    }
    if (big < 1e-16) break;
  }
  for (int k = 0; k < a; ++k)
    for (int it = 0; it < 3; ++it) {
      double2 p, dp;
      eval(z[k], &p, &dp);
      if ((p.x == 0.0 && p.y == 0.0) || (dp.x == 0.0 && dp.y == 0.0)) break;
      z[k] = csub(z[k], cdiv(p, dp));
    }
}

__device__ __forceinline__ double fmodpos(double v, double m) {
  double r = fmod(v, m);
  if (r != 0.0 && r < 0.0) r += m;
  if (r == 0.0) r = 0.0;
  return r;
}

// _nearest_candidate (sfft/reconstruct.py:136-140) over {b + B i}: the nearest
// of the evenly spaced candidates is among the four around (raw - b)/B.
__device__ int64_t nearest_cand(double raw, int64_t b, int64_t B, int64_t n) {
  const double nd = (double)n;
  const int64_t L = n / B;
  const int64_t i0 = (int64_t)floor((raw - (double)b) / (double)B);
  double bd = CUDART_INF;
  int64_t bc = 0x7fffffffffffffffll;
  for (int64_t di = -1; di <= 2; ++di) {
    const int64_t cnd = pmod(b + B * pmod(i0 + di, L), n);
    double d = fmodpos(((double)cnd - raw) + nd / 2.0, nd);
    d = fabs(d - nd / 2.0);
    if (d < bd || (d == bd && cnd < bc)) {
      bd = d;
      bc = cnd;
    }
  }
  return bc;
}

// _unwrap_position (sfft/frameworks.py:179-196) over the ladder rungs
// (ascending, rung 0 == 1); -1 for None.
__device__ int64_t os_unwrap(const OsArgs& a, double2 y0, const double2* ys) {
  if (cabs_scalar(y0) == 0.0) return -1;
  if (a.nlad < 1 || a.lad[0] != 1) return -1;
  const double nd = (double)a.n;
  const double scl = -nd / (2.0 * 3.141592653589793);
  const double2 r1 = cdiv(ys[0], y0);
  double q = fmodpos(atan2(r1.y, r1.x) * scl, nd);
  for (int j = 1; j < a.nlad; ++j) {
    const double2 rj = cdiv(ys[j], y0);
    const double phi = fmodpos(atan2(rj.y, rj.x) * scl, nd);
    const double d = (double)a.lad[j];
    const double period = nd / d;
    const double base = phi / d;
    q = base + rint((q - base) / period) * period;
  }
  return pmod((int64_t)rint(q), a.n);
}

// int(i + round((q - i) / b) * b) % n  (_snap_to_candidates)
__device__ __forceinline__ int64_t os_snap(int64_t q, int64_t i, int64_t B, int64_t n) {
  const double r = rint((double)(q - i) / (double)B);
  return pmod(i + (int64_t)r * B, n);
}

__device__ __forceinline__ int sort_unique(int64_t* p, int np) {
  for (int i = 1; i < np; ++i) {
    const int64_t v = p[i];
    int j = i - 1;
    while (j >= 0 && p[j] > v) {
      p[j + 1] = p[j];
      --j;
    }
    p[j + 1] = v;
  }
  int k = 0;
  for (int i = 0; i < np; ++i)
    if (k == 0 || p[i] != p[k - 1]) p[k++] = p[i];
  return k;
}

// locate_prony (sfft/reconstruct.py:270-302): linear prediction by least
// squares on the 2A moments, companion roots on the unit circle, nearest
// admissible positions (sorted, deduplicated).  false: SingularMomentMatrix.
__device__ bool os_prony_positions(const OsArgs& a, const double2* m, int na, int64_t bucket,
                                   int64_t* pos, int* np) {
  const int rows = 2 * a.A - na;
  double2 mat[2 * kOsMaxA * kOsMaxA];
  double2 rhs[2 * kOsMaxA], co[kOsMaxA];
  for (int c = 0; c < na; ++c)
    for (int r = 0; r < rows; ++r) mat[c * (2 * kOsMaxA) + r] = m[r + c];
  for (int r = 0; r < rows; ++r) rhs[r] = cmk(-m[na + r].x, -m[na + r].y);
  double smax, smin;
  const int rank = svd_lstsq(mat, 2 * kOsMaxA, rows, na, rhs, co, &smax, &smin);
  if (rank < na || smax <= 0.0 || smin < 1e-10 * smax) return false;
  double2 z[kOsMaxA];
  poly_roots(co, na, z);
  const double nd = (double)a.n;
  for (int j = 0; j < na; ++j)
    if (cabs_(z[j]) < 1e-12) return false;
  for (int j = 0; j < na; ++j) {
    const double2 u = cdiv(z[j], cmk(cabs_(z[j]), 0.0));
    const double raw = fmodpos(-atan2(u.y, u.x) * nd / (2.0 * 3.141592653589793), nd);
    pos[j] = nearest_cand(raw, bucket, a.B, a.n);
  }
  *np = sort_unique(pos, na);
  return true;
}

// estimate_prony (sfft/reconstruct.py:374-409): least squares of the bucket's
// measurements on the Vandermonde columns w^{shift_t f_j}.  false: RankDeficient.
__device__ bool os_coeffs(const OsArgs& a, const int64_t* pos, int np, const double2* y,
                          double2* c) {
  if (np == 0) return true;
  if (a.nsh < np) return false;
  double2 vm[kOsMaxRows * kOsMaxA];
  for (int j = 0; j < np; ++j)
    for (int t = 0; t < a.nsh; ++t) vm[j * kOsMaxRows + t] = unit_root(a.n, a.shifts[t] * pos[j]);
  double smax, smin;
  return svd_lstsq(vm, kOsMaxRows, a.nsh, np, y, c, &smax, &smin) >= np;
}

// solve_positions: coefficients and max |meas - model| over all shifts.
__device__ bool os_solve(const OsArgs& a, const int64_t* pos, int np, const double2* y,
                         double2* c, double* resid) {
  if (!os_coeffs(a, pos, np, y, c)) return false;
  double r = 0.0;
  for (int t = 0; t < a.nsh; ++t) {
    double2 mod = cmk(0.0, 0.0);
    for (int j = 0; j < np; ++j) mod = cadd(mod, cmul(unit_root(a.n, a.shifts[t] * pos[j]), c[j]));
    r = fmax(r, cabs_(csub(y[t], mod)));
  }
  *resid = r;
  return true;
}

// refine_positions: re-locate each position by phase unwrapping after the
// other positions' contributions are removed from y0 and the ladder rows.
__device__ int os_refine(const OsArgs& a, int64_t bucket, int64_t* pos, int np, const double2* c,
                         const double2* y) {
  int64_t out[kOsMaxA];
  double2 ys[kOsMaxLad];
  for (int j = 0; j < np; ++j) {
    double2 tot = cmk(0.0, 0.0);
    for (int l = 0; l < np; ++l)
      if (l != j) tot = cadd_rn(tot, c[l]);
    const double2 y0 = csub_rn(y[0], tot);
    for (int d = 0; d < a.nlad; ++d) {
      double2 sd = cmk(0.0, 0.0);
      for (int l = 0; l < np; ++l)
        if (l != j) sd = cadd_rn(sd, cmul_rn(c[l], unit_root(a.n, a.lad[d] * pos[l])));
      ys[d] = csub_rn(y[a.lad_row[d]], sd);
    }
    const int64_t q = os_unwrap(a, y0, ys);
    out[j] = q >= 0 ? os_snap(q, bucket, a.B, a.n) : pos[j];
  }
  for (int j = 0; j < np; ++j) pos[j] = out[j];
  return sort_unique(pos, np);
}

// ------------------------------------------------------------------ kernels

// Hankel singular values and mean moment magnitude of every bucket.
__global__ void __launch_bounds__(kOsNT) k_os_svals(OsArgs a) {
  const int s = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * kOsNT + threadIdx.x;
  if (i >= a.B) return;
  const int A = a.A;
  double2 m[2 * kOsMaxA];
  double en = 0.0;
  for (int t = 0; t < 2 * A; ++t) {
    m[t] = a.meas[((int64_t)t * a.S + s) * a.B + i];
    en += cabs_(m[t]);
  }
  a.energy[(int64_t)s * a.B + i] = en / (double)(2 * A);
  double2 h[kOsMaxA * kOsMaxA];
  for (int c = 0; c < A; ++c)
    for (int r = 0; r < A; ++r) h[c * kOsMaxA + r] = m[r + c];
  double sv[kOsMaxA];
  jacobi_svd(h, kOsMaxA, A, A, sv, nullptr);
  for (int j = 1; j < A; ++j) {  // descending
    const double v = sv[j];
    int q = j - 1;
    while (q >= 0 && sv[q] < v) {
      sv[q + 1] = sv[q];
      --q;
    }
    sv[q + 1] = v;
  }
  double* o = a.svals + ((int64_t)s * a.B + i) * A;
  for (int j = 0; j < A; ++j) o[j] = sv[j];
}

struct SvKey {
  const double* v;
  __device__ __forceinline__ unsigned long long operator()(int64_t i) const { return dbits(v[i]); }
};

// Pooled singular values of one signal: cutoff = the min(2B, B A)-th largest,
// floor = max(3 median, 1e-12 max) (inf when every value is 0).
constexpr int kOsPoolNT = 1024;
__global__ void __launch_bounds__(kOsPoolNT) k_os_pool(OsArgs a) {
  __shared__ unsigned hist[256];
  __shared__ long long sh[4];
  __shared__ double redd[32];
  __shared__ unsigned long long redu[32];
  const int s = blockIdx.x;
  const int64_t M = a.B * a.A;
  SvKey key{a.svals + (int64_t)s * M};
  double med, peak;
  median_and_peak_k<kOsPoolNT>(key, M, &med, &peak, hist, sh, redd, redu);
  const int64_t kk = (2 * a.B < M ? 2 * a.B : M);
  long long below, equal;
  const unsigned long long u =
      block_radix_select<kOsPoolNT>(key, M, 0ull, M - kk, hist, sh, &below, &equal);
  if (threadIdx.x == 0) {
    a.cut[s] = __longlong_as_double((long long)u);
    a.sfl[s] = peak > 0.0 ? fmax(3.0 * med, 1e-12 * peak) : CUDART_INF;
  }
}

// The per-bucket decision of run_oneshot (frameworks.py:266-310), one thread.
__global__ void __launch_bounds__(kOsNT) k_os_solve(OsArgs a) {
  const int s = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * kOsNT + threadIdx.x;
  if (i >= a.B) return;
  const int A = a.A;
  const double* sv = a.svals + ((int64_t)s * a.B + i) * A;
  const double cut = a.cut[s], sfl = a.sfl[s];
  int cnt = 0;
  for (int j = 0; j < A; ++j) cnt += (sv[j] >= cut) && (sv[j] >= 0.1 * sv[0]) && (sv[j] > sfl);
  const double en = a.energy[(int64_t)s * a.B + i], fl = a.floor[s];
  if (cnt == 0 || en < fl) return;
  double2 y[kOsMaxRows];
  for (int t = 0; t < a.nsh; ++t) y[t] = a.meas[((int64_t)t * a.S + s) * a.B + i];
  const double tol = fmax(fl, 0.05 * en);
  bool have = false;
  double best_r = 0.0;
  int best_np = 0;
  int64_t best_pos[kOsMaxA];
  double2 best_c[kOsMaxA];
  int64_t pos[kOsMaxA];
  double2 c[kOsMaxA];
  int np;
  double r;
  if (cnt == 1) {
    double2 ys[kOsMaxLad];
    for (int d = 0; d < a.nlad; ++d) ys[d] = y[a.lad_row[d]];
    const int64_t q = os_unwrap(a, y[0], ys);
    if (q >= 0) {
      pos[0] = os_snap(q, i, a.B, a.n);
      if (os_solve(a, pos, 1, y, c, &r)) {
        have = true;
        best_r = r;
        best_np = 1;
        best_pos[0] = pos[0];
        best_c[0] = c[0];
      }
    }
  }
  if (!have || best_r >= tol) {
    for (int na = (cnt > 2 ? cnt : 2); na <= A; ++na) {
      if (!os_prony_positions(a, y, na, i, pos, &np)) continue;
      double2 c0[kOsMaxA];
      if (!os_coeffs(a, pos, np, y, c0)) continue;
      np = os_refine(a, i, pos, np, c0, y);
      if (!os_solve(a, pos, np, y, c, &r)) continue;
      if (!have || r < best_r) {
        have = true;
        best_r = r;
        best_np = np;
        for (int j = 0; j < np; ++j) {
          best_pos[j] = pos[j];
          best_c[j] = c[j];
        }
      }
      if (r < tol) break;
    }
  }
  if (!have) {
    if (!os_prony_positions(a, y, 1, i, pos, &np)) return;
    if (!os_solve(a, pos, np, y, c, &r)) return;
    have = true;
    best_np = np;
    for (int j = 0; j < np; ++j) {
      best_pos[j] = pos[j];
      best_c[j] = c[j];
    }
  }
  const int o = atomicAdd(a.rec_count + s, best_np);
  for (int j = 0; j < best_np && o + j < a.cap; ++j) {
    a.rec_pos[(int64_t)s * a.cap + o + j] = best_pos[j];
    a.rec_coef[(int64_t)s * a.cap + o + j] = best_c[j];
  }
}

__global__ void k_os_items(int S, int nsh, const int64_t* shifts, int32_t* item_sig,
                           int64_t* item_tau) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)S * nsh) return;
  // signal-major: a signal's shifts are neighbouring items (shifts 0, 1, 2, ...
  // read neighbouring samples: shared 32-byte sectors)
  item_sig[i] = (int32_t)(i / nsh);
  item_tau[i] = shifts[i % nsh];
}

__global__ void k_os_groups(int S, int nsh, int64_t n, int64_t B, const int64_t* shifts,
                            Group* groups, int32_t* ngroups, int32_t* iters, int32_t* conv) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  for (int t = 0; t < nsh; ++t) {
    Group& g = groups[(int64_t)s * kMaxGroups + t];
    g.kind = 1;
    g.a = n / B;
    g.tau = shifts[t];
    g.cnt = B;
    g.nsh = 1;
    g.sh[0] = 0;
  }
  ngroups[s] = nsh;
  iters[s] = 1;
  conv[s] = 1;
}

// ------------------------------------------------------------------ host

struct OsLayout {
  size_t off[16];
  size_t total;
};

static OsLayout os_layout(int64_t B, int S, int A, int nsh) {
  OsLayout L{};
  const int64_t cap = B * A;
  size_t sizes[] = {
      sizeof(double2) * (size_t)nsh * S * B,   // 0 meas
      sizeof(double) * (size_t)S,              // 1 floor
      sizeof(double) * (size_t)S * B * A,      // 2 svals
      sizeof(double) * (size_t)S * B,          // 3 energy
      sizeof(double) * (size_t)S,              // 4 cut
      sizeof(double) * (size_t)S,              // 5 sfl
      sizeof(int64_t) * (size_t)S * cap,       // 6 rec_pos
      sizeof(double2) * (size_t)S * cap,       // 7 rec_coef
      sizeof(int32_t) * (size_t)S,             // 8 rec_count
      sizeof(Group) * (size_t)S * kMaxGroups,  // 9 groups
      sizeof(int32_t) * (size_t)S,             // 10 ngroups
      sizeof(int32_t) * (size_t)S * nsh,       // 11 item_sig
      sizeof(int64_t) * (size_t)S * nsh,       // 12 item_tau
      sizeof(int64_t) * (size_t)nsh,           // 13 shifts (device)
  };
  size_t o = 0;
  const int cnt = sizeof(sizes) / sizeof(sizes[0]);
  for (int i = 0; i < cnt; ++i) {
    L.off[i] = o;
    o += (sizes[i] + 255) & ~size_t(255);
  }
  L.total = o;
  return L;
}

size_t oneshot_ws_bytes(int64_t n, int S, int64_t B, int A, int nsh) {
  (void)n;
  return os_layout(B, S, A, nsh).total + bucketize_ws_bytes(B, (int64_t)S * nsh);
}

int run_oneshot(int dtype, const void* x, int64_t n, int64_t xstride, int S, int64_t B, int A,
                const int64_t* shifts_host, int nsh, const int64_t* ladder_host, int nlad,
                const double2* W, int64_t k, int64_t* out_pos, double2* out_coef,
                int32_t* out_n, int32_t* out_iters, int32_t* out_conv, int64_t* out_samples,
                int64_t* out_sched, void* ws, size_t ws_bytes, cudaStream_t st) {
  SFFT_REQUIRE(A >= 1 && A <= kOsMaxA, "one_shot: a_max must be in [1, 8] on the device");
  SFFT_REQUIRE(nsh >= 2 * A && nsh <= kOsMaxRows, "one_shot: at most 64 measurement shifts");
  SFFT_REQUIRE(nlad >= 1 && nlad <= kOsMaxLad, "one_shot: 1..16 ladder rungs");
  SFFT_REQUIRE(k >= 1 && k <= kFusedMaxB, "one_shot: k must be in [1, 8192]");
  SFFT_REQUIRE(ws_bytes >= oneshot_ws_bytes(n, S, B, A, nsh), "one_shot: workspace too small");
  OsArgs a{};
  a.n = n;
  a.B = B;
  a.k = k;
  a.S = S;
  a.A = A;
  a.nsh = nsh;
  a.nlad = nlad;
  for (int t = 0; t < nsh; ++t) a.shifts[t] = pmod(shifts_host[t], n);
  // ladder rung d -> its measurement row (the first shift equal to d)
  for (int j = 0; j < nlad; ++j) {
    a.lad[j] = ladder_host[j];
    a.lad_row[j] = -1;
    for (int t = 0; t < nsh && a.lad_row[j] < 0; ++t)
      if (a.shifts[t] == pmod(ladder_host[j], n)) a.lad_row[j] = t;
    SFFT_REQUIRE(a.lad_row[j] >= 0, "one_shot: every ladder rung must be a measurement shift");
    SFFT_REQUIRE(j == 0 || ladder_host[j] > ladder_host[j - 1], "one_shot: ladder must ascend");
  }
  const OsLayout Lo = os_layout(B, S, A, nsh);
  char* w = (char*)ws;
  a.meas = (double2*)(w + Lo.off[0]);
  double* floor = (double*)(w + Lo.off[1]);
  a.floor = floor;
  a.svals = (double*)(w + Lo.off[2]);
  a.energy = (double*)(w + Lo.off[3]);
  a.cut = (double*)(w + Lo.off[4]);
  a.sfl = (double*)(w + Lo.off[5]);
  a.rec_pos = (int64_t*)(w + Lo.off[6]);
  a.rec_coef = (double2*)(w + Lo.off[7]);
  a.rec_count = (int32_t*)(w + Lo.off[8]);
  a.cap = (int)std::min<int64_t>(B * A, (int64_t)1 << 30);
  Group* groups = (Group*)(w + Lo.off[9]);
  int32_t* ngroups = (int32_t*)(w + Lo.off[10]);
  int32_t* item_sig = (int32_t*)(w + Lo.off[11]);
  int64_t* item_tau = (int64_t*)(w + Lo.off[12]);
  int64_t* dshifts = (int64_t*)(w + Lo.off[13]);
  void* bws = w + Lo.total;
  const int64_t nitems = (int64_t)S * nsh;

  SFFT_CUDA(cudaMemcpyAsync(dshifts, a.shifts, sizeof(int64_t) * nsh, cudaMemcpyHostToDevice, st));
  SFFT_CUDA(cudaMemsetAsync(a.rec_count, 0, sizeof(int32_t) * S, st));
  k_os_items<<<(unsigned)cdiv_up(nitems, 256), 256, 0, st>>>(S, nsh, dshifts, item_sig, item_tau);
  SFFT_CHECK_LAUNCH("k_os_items");
  Prod p{};
  p.x = x;
  p.xstride = xstride;
  p.n = n;
  p.B = B;
  p.item_sig = item_sig;
  p.item_a = item_tau;
  p.out_M = nsh;  // item s*nsh + t writes row t*S + s
  p.out_S = S;
  int rc = run_bucketize(dtype, PROD_SPIKE, p, nitems, W, (double2*)a.meas, bws,
                         bucketize_ws_bytes(B, nitems), st);
  if (rc) return rc;
  rc = run_floor(a.meas, S, B, 3.0, nullptr, nullptr, floor, nullptr, st);
  if (rc) return rc;
  const dim3 gb((unsigned)cdiv_up(B, kOsNT), S);
  k_os_svals<<<gb, kOsNT, 0, st>>>(a);
  SFFT_CHECK_LAUNCH("k_os_svals");
  k_os_pool<<<S, kOsPoolNT, 0, st>>>(a);
  SFFT_CHECK_LAUNCH("k_os_pool");
  k_os_solve<<<gb, kOsNT, 0, st>>>(a);
  SFFT_CHECK_LAUNCH("k_os_solve");
  const size_t dsm = (size_t)kFusedMaxB * (8 + 8 + 4);
  SFFT_CUDA(cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  k_finalize<<<S, kFinNT, dsm, st>>>(a.rec_pos, a.rec_coef, a.rec_count, a.cap, k, out_pos,
                                      out_coef, out_n);
  SFFT_CHECK_LAUNCH("k_finalize");
  k_os_groups<<<(unsigned)cdiv_up(S, 128), 128, 0, st>>>(S, nsh, n, B, dshifts, groups, ngroups,
                                                         out_iters, out_conv);
  SFFT_CHECK_LAUNCH("k_os_groups");
  rc = run_union_count(groups, ngroups, S, n, out_samples, nullptr, nullptr, st);
  if (rc) return rc;
  if (out_sched) {
    k_export_groups<<<S, 64, 0, st>>>(groups, ngroups, S, out_sched);
    SFFT_CHECK_LAUNCH("k_export_groups");
  }
  return 0;
}

}  // namespace sfft
