// Batched FFAST-style peeling (sfft/frameworks.py:614-699), device-resident.
//
//   stage j: B_j = n/p_j buckets, shifts t < s_j (3 when p_j > 3, else
//            max(p_j-1, 1)); meas_j[t] = bucketize_spike(x, B_j, t)     (A7)
//   floor_j  = robust_noise_floor(meas_j[0])                             (A8)
//   classify every bucket with mean_t|m_t| >= floor_j (a_max = 1):
//            zero / single (phase location + carrier check) / multi      (A17)
//   queues   = singles in (stage, bucket) order, verified stages (3 shifts)
//              first; then one warp per signal peels sequentially: pop a
//              still-single entry, recovered[f] += c, subtract c w^{t f} from
//              bucket f mod B_j of every stage, reclassify, push new singles
//   stuck    = any bucket's latest class is multi
#include "kernels.cuh"
#include "schedule.cuh"
#include "finalize.cuh"

namespace sfft {

constexpr int kMaxPeelStages = 16;

struct PeelArgs {
  int64_t n, k;
  int S, nst;
  int64_t p[kMaxPeelStages], Bs[kMaxPeelStages], sh[kMaxPeelStages];
  int64_t moff[kMaxPeelStages];      // meas offset of stage j (elements), layout [s_j][S][B_j]
  int64_t boff[kMaxPeelStages + 1];  // bucket offset of stage j in the per-signal class arrays
  int64_t sumB;
  double2* meas;
  double* floor;                 // [nst][S]
  int32_t* kind;                 // [S][sumB] 0 none/zero, 1 single, 2 multi
  int64_t* cf;                   // [S][sumB] single position
  double2* cc;                   // [S][sumB] single coefficient
  int64_t* q[2];                 // [S][qcap] tier 0 = verified (3 shifts), 1 = others
  int32_t* qtail[2];             // [S]
  int64_t qcap;
  int64_t* rec_pos;              // [S][cap]
  double2* rec_coef;             // [S][cap]
  int32_t* rec_count;            // [S]
  int cap;
  int64_t* ht_key;               // [S][HT]
  int32_t* ht_val;
  int HT;
  int32_t* peels;                // [S]
  int32_t* err;                  // [S] 1: a 1-shift stage had an active bucket
};

__device__ __forceinline__ int stage_of(const PeelArgs& a, int64_t g) {
  int j = 0;
  while (j + 1 < a.nst && g >= a.boff[j + 1]) ++j;
  return j;
}

__device__ __forceinline__ double2 moment(const PeelArgs& a, int j, int s, int t, int64_t b) {
  return a.meas[a.moff[j] + ((int64_t)t * a.S + s) * a.Bs[j] + b];
}

struct Verdict {
  int kind;
  int64_t f;
  double2 c;
};

// Exact stand-ins for the 64-bit '%' and fmod of the classification, which sit
// on the peel loop's critical path (one warp runs a dependent chain; a 64-bit
// modulo is ~130 instructions): their arguments are within one or two periods
// here, so conditional adds give the same values.
//   w^{t f} for t < 3, 0 <= f < n
__device__ __forceinline__ double2 unit_root_tf(int64_t n, int t, int64_t f) {
  int64_t e = (int64_t)t * f;  // < 3 n
  e -= (e >= n) ? n : 0;
  e -= (e >= n) ? n : 0;
  const double th = (-6.283185307179586 * (double)e) / (double)n;  // as unit_root
  double s, c;
  sincos(th, &s, &c);
  return cmk(c, s);
}
//   fmod(x, nd) for |x| < 2 nd (x - nd is exact there: Sterbenz)
__device__ __forceinline__ double fmod_near(double x, double nd) {
  if (fabs(x) >= 2.0 * nd) return fmod(x, nd);
  if (x >= nd) return x - nd;
  if (x <= -nd) return x + nd;
  return x;
}

// classify_bucket with a_max = 1 (sfft/reconstruct.py:412-440) after the
// peeling pre-check (sfft/frameworks.py:653-658), one thread.  The
// candidates {b + B i} are evenly spaced, so the nearest one under circular
// distance (_nearest_candidate, reconstruct.py:136-140) is among the four
// around (raw - b)/B; the reference distance formula and its tie rule (smaller
// candidate) are applied to those.
// m_in (optional): the bucket's moments already in registers (the peel loop
// just updated them), saving a dependent re-read.
__device__ Verdict classify_one(const PeelArgs& a, int s, int j, int64_t b, int32_t* err,
                                const double2* m_in = nullptr) {
  Verdict v{0, 0, cmk(0.0, 0.0)};
  const int ns = (int)a.sh[j];
  const int64_t n = a.n, B = a.Bs[j], L = a.p[j];
  const double fl = a.floor[(int64_t)j * a.S + s];
  double2 m[3];
  double sabs = 0.0;
  for (int t = 0; t < ns; ++t) {
    m[t] = m_in ? m_in[t] : moment(a, j, s, t, b);
    sabs += cabs_(m[t]);
  }
  if (sabs / ns < fl) return v;  // zero
  if (ns < 2) {                  // MomentSequence raises InvalidParameter
    atomicExch(err, 1);
    v.kind = 2;
    return v;
  }
  if (cabs_scalar(m[0]) < fl) {
    v.kind = 2;
    return v;
  }
  const double nd = (double)n;
  const double2 r = cdiv(m[1], m[0]);
  double raw = fmod_near(atan2(r.y, r.x) * (-nd / (2.0 * 3.141592653589793)), nd);
  if (raw != 0.0 && raw < 0.0) raw += nd;
  if (raw == 0.0) raw = 0.0;
  const int64_t i0 = (int64_t)floor((raw - (double)b) / (double)B);
  double bd = CUDART_INF;
  int64_t bc = 0x7fffffffffffffffll;
  for (int64_t di = -1; di <= 2; ++di) {
    int64_t iw = i0 + di;  // in [-2, L + 2]: one wrap at most when L >= 8
    if (L < 8) {
      iw = pmod(iw, L);
    } else {
      iw += (iw < 0) ? L : 0;
      iw -= (iw >= L) ? L : 0;
    }
    const int64_t cnd = b + B * iw;  // <= (B - 1) + B (L - 1) = n - 1
    double d = fmod_near(((double)cnd - raw) + nd / 2.0, nd);
    if (d != 0.0 && d < 0.0) d += nd;
    d = fabs(d - nd / 2.0);
    if (d < bd || (d == bd && cnd < bc)) {
      bd = d;
      bc = cnd;
    }
  }
  const int64_t f = bc;
  const double tol = fmax(fl, 0.05 * cabs_scalar(m[0]));
  double mx = 0.0;
  double2 sum = cmk(0.0, 0.0);
  for (int t = 0; t < ns; ++t) {
    const double2 car = unit_root_tf(n, t, f);
    mx = fmax(mx, cabs_(csub(m[t], cmul(m[0], car))));
    sum = cadd(sum, cmul(m[t], cconj(car)));
  }
  if (mx < tol) {
    v.kind = 1;
    v.f = f;
    v.c = cdivr(sum, (double)ns);
  } else {
    v.kind = 2;
  }
  return v;
}

// Initial classification of every bucket of every stage (thread per bucket).
__global__ void k_pe_classify_all(PeelArgs a) {
  const int s = blockIdx.y;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= a.sumB) return;
  const int j = stage_of(a, g);
  const int64_t b = g - a.boff[j];
  const Verdict v = classify_one(a, s, j, b, a.err + s);
  const int64_t i = (int64_t)s * a.sumB + g;
  a.kind[i] = v.kind;
  a.cf[i] = v.f;
  a.cc[i] = v.c;
}

// Singles in (stage, bucket) order into the two tier queues.
__global__ void __launch_bounds__(1024) k_pe_queue_init(PeelArgs a) {
  __shared__ int red[32];
  const int s = blockIdx.x;
  const int64_t per = (a.sumB + 1023) / 1024;
  const int64_t g0 = threadIdx.x * per, g1 = min(a.sumB, g0 + per);
  int c[2] = {0, 0};
  for (int64_t g = g0; g < g1; ++g)
    if (a.kind[(int64_t)s * a.sumB + g] == 1) ++c[a.sh[stage_of(a, g)] >= 3 ? 0 : 1];
  int tot[2];
  int off[2];
  off[0] = block_exscan<1024>(c[0], red, &tot[0]);
  off[1] = block_exscan<1024>(c[1], red, &tot[1]);
  for (int64_t g = g0; g < g1; ++g) {
    if (a.kind[(int64_t)s * a.sumB + g] != 1) continue;
    const int tier = a.sh[stage_of(a, g)] >= 3 ? 0 : 1;
    a.q[tier][(int64_t)s * a.qcap + off[tier]++] = g;
  }
  if (threadIdx.x == 0) {
    a.qtail[0][s] = tot[0];
    a.qtail[1][s] = tot[1];
  }
}

__device__ __forceinline__ uint32_t pe_slot(int64_t f, int HT) {
  return (uint32_t)(((unsigned long long)(f + 1) * 0x9E3779B97F4A7C15ull) >> 40) & (HT - 1);
}

// Bitwise equality of two post-peel bucket states (moments of the stage's
// shifts, class, and the single-ton's position / coefficient).
struct PeelState {
  double2 m[3];
  Verdict v;
};

__device__ __forceinline__ bool same_bits(double2 x, double2 y) {
  return __double_as_longlong(x.x) == __double_as_longlong(y.x) &&
         __double_as_longlong(x.y) == __double_as_longlong(y.y);
}

__device__ __forceinline__ bool same_state(const PeelState& x, const PeelState& y, int sh) {
  bool eq = x.v.kind == y.v.kind;
  for (int t = 0; t < 3; ++t)
    if (t < sh) eq = eq && same_bits(x.m[t], y.m[t]);
  if (eq && x.v.kind == 1) eq = x.v.f == y.v.f && same_bits(x.v.c, y.v.c);
  return eq;
}

constexpr int kPeelOldCap = 256;    // queued entries of the cycle's buckets kept for the replay
constexpr int kPeelSimSteps = 4096; // pops replayed before the attempt is given up

// The sequential peel of one signal, one warp (frameworks.py:669-695).
//
// Exact fast-forward of a two-state cycle.  A signal that exhausts the budget
// k + sum B_j does so in a loop of period <= 2: the same position f is peeled
// again and again (a rounding-level residual in one stage's bucket is a
// "single-ton" c; removing it leaves -c in the other stages' buckets, peeling
// that restores the first state), 77,479 times for C4's seed 213.  The next
// state of the buckets of f is a pure function of their moments and of the
// coefficient of whichever of them is popped, so once
//   * three consecutive peels had the same f,
//   * the buckets' state after this peel equals, bit for bit, the state two
//     peels ago (moments, class, single-ton position and coefficient),
//   * the queue holds no single-ton entry of any other bucket, and the replay
//     of its pops (integers only: which stage's entry is taken next, stale
//     entries skipped as the loop would) always takes an entry whose class is
//     exactly (f, the coefficient the last two peels used in that state) and
//     reaches a repeating pattern that never runs dry,
// every remaining peel is known: the states alternate, recovered[f] receives
// the two coefficients alternately (the additions are carried out, stopping
// early once they too repeat), and the budget is reached.  Results, peel
// count and final classes are bit-identical to running the loop.
//
// Windows of independent peels.  The loop is sequential by definition, but a
// peel only reads and writes the buckets of its own position (one per stage)
// and its own recovered entry, so consecutive pops whose bucket sets are
// disjoint — and disjoint from every queue entry passed over on the way —
// give the same moments, classes, queue order and sums whether they run one
// after the other or side by side.  Each step the warp walks the verified
// queue in order, drops stale entries, and accepts up to 32/stages single-tons
// until an entry or a position touches a bucket of an already accepted peel
// (that entry stays queued: its class may change); lane p*stages + j then
// peels stage j of the p-th accepted position, and the pushes are compacted in
// lane order = the loop's order.  Unverified (two-shift) stages are drawn on
// one peel at a time, as their pushes to the verified queue take precedence.
__device__ __forceinline__ int64_t bucket_mod(int64_t f, int64_t B, double invB) {
  int64_t r = f - __double2ll_rz((double)f * invB) * B;  // f < 2^53
  if (r < 0) r += B;
  if (r >= B) r -= B;
  return r;
}

__global__ void k_pe_peel(PeelArgs a, int64_t budget, int fast_forward) {
  __shared__ int8_t s_old[kPeelOldCap];
  const int s = blockIdx.x;
  const int lane = threadIdx.x;
  const int nst = a.nst;
  const int G = 32 / nst;             // peels side by side
  const int jL = lane % nst;          // this lane's stage
  const int pL = lane / nst;          // ... and window slot
  const int64_t BL = a.Bs[jL], boffL = a.boff[jL];
  const double invBL = 1.0 / (double)BL;
  const int shL = (int)a.sh[jL];
  const int tierL = shL >= 3 ? 0 : 1;
  int64_t head[2] = {0, 0};
  int32_t tail[2] = {a.qtail[0][s], a.qtail[1][s]};
  int64_t* q[2] = {a.q[0] + (int64_t)s * a.qcap, a.q[1] + (int64_t)s * a.qcap};
  int32_t* kind = a.kind + (int64_t)s * a.sumB;
  int64_t* cfs = a.cf + (int64_t)s * a.sumB;
  double2* ccs = a.cc + (int64_t)s * a.sumB;
  int64_t* rp = a.rec_pos + (int64_t)s * a.cap;
  double2* rc = a.rec_coef + (int64_t)s * a.cap;
  int64_t* hk = a.ht_key + (int64_t)s * a.HT;
  int32_t* hv = a.ht_val + (int64_t)s * a.HT;
  int nrec = 0;
  int64_t peels = 0;
  // all stages in one tier (the replay below handles a single live queue)
  int live_tier = a.sh[0] >= 3 ? 0 : 1;
  if (!fast_forward) live_tier = -1;
  for (int j = 1; j < nst; ++j)
    if ((a.sh[j] >= 3 ? 0 : 1) != live_tier) live_tier = -1;
  const int window = fast_forward == 1 ? G : 1;  // 0 / 2: one peel per step
  PeelState h1{}, h2{};  // this lane's bucket after the previous peel / the one before
  int64_t f1 = -1, f2 = -1;
  double2 cprev = cmk(0.0, 0.0);  // coefficient of the previous peel
  int64_t next_try = 0;
  while (peels < budget) {
    // ---- the window: accepted peel p lives in lanes p*nst .. p*nst + nst-1
    int m = 0;
    int64_t my_gid = -1, my_f = 0;
    double2 my_c = cmk(0.0, 0.0);
    for (int tr = 0; tr < 2 && m == 0; ++tr) {
      const int cap_m = tr == 0 ? window : 1;
      bool stop = false;
      while (!stop && head[tr] < tail[tr]) {
        const int64_t at = head[tr] + lane;
        const int64_t e = at < tail[tr] ? q[tr][at] : -1;
        const int kd = e >= 0 ? kind[e] : 0;
        int64_t fe = 0;  // requested with the class, not after it: one round trip less
        double2 ce = cmk(0.0, 0.0);
        if (e >= 0) {
          fe = cfs[e];
          ce = ccs[e];
        }
        const int64_t left = tail[tr] - head[tr];
        const int cnt = left < 32 ? (int)left : 32;
        int used = 0;
        for (int i = 0; i < cnt; ++i) {
          const int64_t ei = __shfl_sync(0xffffffffu, e, i);
          const int kdi = __shfl_sync(0xffffffffu, kd, i);
          bool clash = my_gid == ei;
          int64_t fi = 0, gnew = -1;
          if (kdi == 1) {
            fi = __shfl_sync(0xffffffffu, fe, i);
            gnew = boffL + bucket_mod(fi, BL, invBL);
            clash = clash || my_gid == gnew;
          }
          if (__any_sync(0xffffffffu, my_gid >= 0 && clash)) {
            stop = true;  // it meets an accepted peel's bucket: decided after this step
            break;
          }
          used = i + 1;
          if (kdi == 1) {
            const double cx = __shfl_sync(0xffffffffu, ce.x, i);
            const double cy = __shfl_sync(0xffffffffu, ce.y, i);
            if (pL == m && pL < G) {
              my_gid = gnew;
              my_f = fi;
              my_c = cmk(cx, cy);
            }
            ++m;
            if (m >= cap_m || peels + m >= budget) {
              stop = true;
              break;
            }
          }
        }
        head[tr] += used;
      }
    }
    if (m == 0) break;
    const bool active = pL < m && pL < G;
    // the buckets' moments are requested before the recovered-table look-up
    // below, so the two round trips overlap
    double2 mold[3] = {cmk(0.0, 0.0), cmk(0.0, 0.0), cmk(0.0, 0.0)};
    double2* mp0 = a.meas + a.moff[jL] + (int64_t)s * BL + (my_gid - boffL);
    if (active) {
#pragma unroll
      for (int t = 0; t < 3; ++t)
        if (t < shL) mold[t] = mp0[(int64_t)t * a.S * BL];
    }
    // ---- recovered[f] += c: the positions of a window differ, so look-ups
    // are independent; new ones take consecutive indices in window order
    const bool lead = active && jL == 0;
    int where = -1;
    uint32_t hslot = 0;
    if (lead) {
      hslot = pe_slot(my_f, a.HT);
      for (int pr = 0; pr < a.HT; ++pr) {
        const int64_t key = __ldcg(hk + hslot);
        if (key == my_f + 1) { where = __ldcg(hv + hslot); break; }
        if (key == 0) break;
        hslot = (hslot + 1) & (a.HT - 1);
      }
    }
    const unsigned fresh = __ballot_sync(0xffffffffu, lead && where < 0);
    if (lead) {
      if (where >= 0) {
        rc[where] = cadd(rc[where], my_c);
      } else {
        const int idx = nrec + __popc(fresh & ((1u << lane) - 1));
        if (idx < a.cap) {
          while (atomicCAS((unsigned long long*)(hk + hslot), 0ull,
                           (unsigned long long)(my_f + 1)) != 0ull)
            hslot = (hslot + 1) & (a.HT - 1);
          hv[hslot] = idx;
          rp[idx] = my_f;
          rc[idx] = my_c;
        }
      }
    }
    {
      const int grown = nrec + __popc(fresh);
      nrec = grown < a.cap ? grown : a.cap;
    }
    peels += m;
    // ---- every (peel, stage) in its own lane: subtract c w^{t f} from bucket
    // f mod B_j, reclassify; new single-tons are queued in (peel, stage) order
    PeelState cur{};
    const int64_t gi = my_gid;
    if (active) {
      const int j = jL;
      const int64_t b = gi - boffL;
#pragma unroll
      for (int t = 0; t < 3; ++t) {
        if (t < shL) {
          cur.m[t] = csub(mold[t], cmul(my_c, unit_root_tf(a.n, t, my_f)));
          mp0[(int64_t)t * a.S * BL] = cur.m[t];
        }
      }
      cur.v = classify_one(a, s, j, b, a.err + s, cur.m);
      kind[gi] = cur.v.kind;
      cfs[gi] = cur.v.f;
      ccs[gi] = cur.v.c;
    }
    const bool is_single = active && cur.v.kind == 1;
    for (int tr = 0; tr < 2; ++tr) {
      const unsigned push = __ballot_sync(0xffffffffu, is_single && tierL == tr);
      if (is_single && tierL == tr) {
        const int64_t pos = tail[tr] + __popc(push & ((1u << lane) - 1));
        if (pos < a.qcap) q[tr][pos] = gi;
      }
      const int64_t nt = (int64_t)tail[tr] + __popc(push);
      tail[tr] = (int32_t)(nt < a.qcap ? nt : a.qcap);
    }
    __syncwarp();
    if (m > 1) {  // the cycle test below follows single peels only
      f1 = f2 = -1;
      continue;
    }
    const int64_t f = __shfl_sync(0xffffffffu, my_f, 0);
    const double2 c = cmk(__shfl_sync(0xffffffffu, my_c.x, 0), __shfl_sync(0xffffffffu, my_c.y, 0));

    // ---- two-state cycle: detect, verify, fast-forward (see the header) ----
    const bool rep = f == f1 && f == f2;
    bool ok = rep && live_tier >= 0 && peels >= next_try && peels < budget;
    if (ok) {
      const bool mine = lane >= a.nst || same_state(cur, h2, (int)a.sh[lane < a.nst ? lane : 0]);
      ok = __all_sync(0xffffffffu, mine);
    }
    // single-ton buckets of the two states; those whose class is exactly the
    // pair (f, coefficient) the last two peels used may be popped in the replay
    // (c0: applied to the state two peels ago = this one; c1: to the previous)
    unsigned pm0 = 0, pm1 = 0, gm0 = 0, gm1 = 0;
    const double2 c0 = cprev, c1 = c;
    if (ok) {
      const bool s1 = lane < a.nst && h1.v.kind == 1;
      pm0 = __ballot_sync(0xffffffffu, is_single);
      pm1 = __ballot_sync(0xffffffffu, s1);
      gm0 = __ballot_sync(0xffffffffu, is_single && cur.v.f == f && same_bits(cur.v.c, c0));
      gm1 = __ballot_sync(0xffffffffu, s1 && h1.v.f == f && same_bits(h1.v.c, c1));
      ok = gm0 != 0 && gm1 != 0;
    }
    if (ok) {
      next_try = peels + 32;  // a failed attempt is retried after the queue has moved on
      // queued entries: the live tier may hold entries of the cycle's buckets
      // (kept, as stage ids) and stale entries of others (dropped: their class
      // cannot change any more); a single-ton elsewhere ends the attempt
      ok = head[1 - live_tier] >= tail[1 - live_tier];
      int L0 = 0;
      for (int64_t base = head[live_tier]; ok && base < tail[live_tier]; base += 32) {
        const int64_t at = base + lane;
        const int64_t e = at < tail[live_tier] ? q[live_tier][at] : -1;
        int stage = -1;
        for (int j = 0; j < a.nst; ++j)
          if (e == __shfl_sync(0xffffffffu, gi, j)) stage = j;
        const bool breaker = e >= 0 && stage < 0 && kind[e] == 1;
        const unsigned keep = __ballot_sync(0xffffffffu, stage >= 0);
        if (__any_sync(0xffffffffu, breaker) || L0 + __popc(keep) > kPeelOldCap) {
          ok = false;
          break;
        }
        if (stage >= 0) s_old[L0 + __popc(keep & ((1u << lane) - 1))] = (int8_t)stage;
        L0 += __popc(keep);
      }
      __syncwarp();
      if (ok) {
        // integer replay of the pops (warp-uniform): after the kept entries the
        // queue is the groups pushed by the alternating states, pm1 first
        const int n0 = __popc(pm0), n1 = __popc(pm1), W = n0 + n1;
        int64_t ptr = 0, end = L0, lag_prev = -1, off_prev = -1;
        int qpar = 0;  // parity of the state the next pop sees (0: this peel's)
        bool steady = false;
        int64_t simmed = 0;
        for (int step = 0; step < kPeelSimSteps && peels + simmed < budget; ++step) {
          const unsigned pm = qpar ? pm1 : pm0;
          bool found = false;
          while (ptr < end) {
            int stage;
            if (ptr < L0) {
              stage = s_old[ptr];
            } else {
              const int r = (int)((ptr - L0) % W);
              stage = r < n1 ? __fns(pm1, 0, r + 1) : __fns(pm0, 0, r - n1 + 1);
            }
            ++ptr;
            if ((pm >> stage) & 1u) {
              found = ((qpar ? gm1 : gm0) >> stage) & 1u;  // another class: not this cycle
              break;
            }
          }
          if (!found) break;  // dry queue or another single-ton: leave it to the loop
          ++simmed;
          qpar ^= 1;
          end += qpar ? n1 : n0;
          if (qpar == 0 && ptr >= L0) {
            const int64_t off = (ptr - L0) % W, lag = end - ptr;
            if (off == off_prev && lag >= lag_prev) { steady = true; break; }
            off_prev = off;
            lag_prev = lag;
          }
        }
        ok = steady || peels + simmed >= budget;
      }
      if (ok) {
        const int64_t R = budget - peels;
        if (lane == 0) {
          uint32_t h = pe_slot(f, a.HT);
          int where = -1;
          for (int pr = 0; pr < a.HT; ++pr) {
            const int64_t key = __ldcg(hk + h);
            if (key == f + 1) { where = __ldcg(hv + h); break; }
            if (key == 0) break;
            h = (h + 1) & (a.HT - 1);
          }
          if (where >= 0) {
            double2 r = rc[where];
            int64_t i = 0;
            while (i + 2 <= R) {
              const double2 r1 = cadd(r, c0);
              const double2 r2 = cadd(r1, c1);
              if (same_bits(r2, r)) {  // the additions repeat as well
                i = R - ((R - i) & 1);
                break;
              }
              r = r2;
              i += 2;
            }
            if (i < R) r = cadd(r, c0);
            rc[where] = r;
          }
          // (f was recorded by the earlier peels; with the table full it never was,
          // and the loop would not record it either)
        }
        if ((R & 1) && lane < a.nst) {  // an odd remainder ends in the other state
          const int j = lane;
          const int64_t b = f % a.Bs[j];
          for (int t = 0; t < a.sh[j]; ++t)
            a.meas[a.moff[j] + ((int64_t)t * a.S + s) * a.Bs[j] + b] = h1.m[t];
          kind[gi] = h1.v.kind;
          cfs[gi] = h1.v.f;
          ccs[gi] = h1.v.c;
        }
        peels = budget;
        break;
      }
    }
    h2 = h1;
    h1 = cur;
    f2 = f1;
    f1 = f;
    cprev = c;
  }
  if (lane == 0) {
    a.rec_count[s] = nrec;
    a.peels[s] = (int32_t)peels;
  }
}

__global__ void k_pe_stuck(PeelArgs a, int32_t* conv, int32_t* iters) {
  __shared__ int any;
  const int s = blockIdx.x;
  if (threadIdx.x == 0) any = 0;
  __syncthreads();
  int mine = 0;
  for (int64_t g = threadIdx.x; g < a.sumB; g += blockDim.x)
    mine |= a.kind[(int64_t)s * a.sumB + g] == 2;
  if (mine) atomicOr(&any, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    conv[s] = !any;
    iters[s] = a.peels[s];
  }
}

__global__ void k_pe_items(int S, int ns, int32_t* item_sig, int64_t* tau) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S * ns) return;
  // signal-major: the shifts 0..ns-1 of a signal are neighbouring items, so
  // they run together and share the 32-byte sectors their samples sit in
  item_sig[i] = i / ns;
  tau[i] = i % ns;
}

__global__ void k_pe_groups(PeelArgs a, Group* groups, int32_t* ngroups) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  int ng = 0;
  for (int j = 0; j < a.nst; ++j)
    for (int t = 0; t < a.sh[j] && ng < kMaxGroups; ++t, ++ng) {
      Group& g = groups[(int64_t)s * kMaxGroups + ng];
      g.kind = 1;
      g.a = a.p[j];
      g.tau = t;
      g.cnt = a.Bs[j];
      g.nsh = 1;
      g.sh[0] = 0;
    }
  ngroups[s] = ng;
}

__global__ void k_pe_samples(int64_t* samples, int S) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s > 0 && s < S) samples[s] = samples[0];
}

struct PeelLayout {
  size_t off[24];
  size_t total;
};

static size_t alp(size_t x) { return (x + 255) & ~size_t(255); }

static int pe_ht(int cap) {
  int h = 1;
  while (h < 2 * cap) h <<= 1;
  return h;
}

static PeelLayout peel_layout(int S, int64_t msize, int64_t sumB, int64_t qcap, int cap,
                              int nst, int64_t maxitems) {
  PeelLayout L{};
  const size_t HT = (size_t)pe_ht(cap);
  size_t sizes[] = {
      sizeof(double2) * (size_t)msize,            // 0 meas
      sizeof(double) * (size_t)nst * S,           // 1 floor
      sizeof(int32_t) * (size_t)S * sumB,         // 2 kind
      sizeof(int64_t) * (size_t)S * sumB,         // 3 cf
      sizeof(double2) * (size_t)S * sumB,         // 4 cc
      sizeof(int64_t) * (size_t)S * qcap,         // 5 q0
      sizeof(int64_t) * (size_t)S * qcap,         // 6 q1
      sizeof(int32_t) * (size_t)S * 2,            // 7 qtail
      sizeof(int64_t) * (size_t)S * cap,          // 8 rec_pos
      sizeof(double2) * (size_t)S * cap,          // 9 rec_coef
      sizeof(int32_t) * (size_t)S,                // 10 rec_count
      sizeof(int64_t) * (size_t)S * HT,           // 11 ht_key
      sizeof(int32_t) * (size_t)S * HT,           // 12 ht_val
      sizeof(int32_t) * (size_t)S,                // 13 peels
      sizeof(int32_t) * (size_t)S,                // 14 err
      sizeof(Group) * (size_t)S * kMaxGroups,     // 15 groups
      sizeof(int32_t) * (size_t)S,                // 16 ngroups
      sizeof(int32_t) * (size_t)maxitems,         // 17 item_sig
      sizeof(int64_t) * (size_t)maxitems,         // 18 item tau
  };
  size_t o = 0;
  const int cnt = sizeof(sizes) / sizeof(sizes[0]);
  for (int i = 0; i < cnt; ++i) {
    L.off[i] = o;
    o += alp(sizes[i]);
  }
  L.total = o;
  return L;
}

struct PeelDims {
  int64_t msize, sumB, qcap, maxitems, budget, bws;
  int cap;
};

static PeelDims peel_dims(int64_t n, int S, const int64_t* factors, int nst, int64_t k) {
  PeelDims d{};
  for (int j = 0; j < nst; ++j) {
    const int64_t p = factors[j], B = n / p;
    const int64_t sh = p > 3 ? 3 : (p - 1 > 1 ? p - 1 : 1);
    d.msize += sh * S * B;
    d.sumB += B;
    d.maxitems = std::max<int64_t>(d.maxitems, sh * S);
    d.bws = std::max<int64_t>(d.bws, (int64_t)bucketize_ws_bytes(B, sh * S));
  }
  d.budget = k + d.sumB;
  d.qcap = d.sumB + d.budget * nst;
  d.cap = (int)std::min<int64_t>(d.budget, (int64_t)1 << 30);
  return d;
}

size_t peeling_ws_bytes(int64_t n, int S, const int64_t* factors, int nst, int64_t k) {
  const PeelDims d = peel_dims(n, S, factors, nst, k);
  return peel_layout(S, d.msize, d.sumB, d.qcap, d.cap, nst, d.maxitems).total + d.bws;
}

int run_peeling(int dtype, const void* x, int64_t n, int64_t xstride, int S,
                const int64_t* factors, int nst, const double2* const* Wst, int64_t k,
                int64_t* out_pos, double2* out_coef, int32_t* out_n, int32_t* out_iters,
                int32_t* out_conv, int32_t* out_err, int64_t* out_samples, int64_t* out_sched,
                void* ws, size_t ws_bytes, cudaStream_t st) {
  SFFT_REQUIRE(nst >= 1 && nst <= kMaxPeelStages, "peeling: 1..16 co-prime factors");
  SFFT_REQUIRE(k <= kFusedMaxB, "peeling: k must be <= 8192");
  SFFT_REQUIRE(ws_bytes >= peeling_ws_bytes(n, S, factors, nst, k), "peeling: workspace too small");
  const PeelDims d = peel_dims(n, S, factors, nst, k);
  const PeelLayout Lo = peel_layout(S, d.msize, d.sumB, d.qcap, d.cap, nst, d.maxitems);
  char* w = (char*)ws;
  PeelArgs a{};
  a.n = n;
  a.k = k;
  a.S = S;
  a.nst = nst;
  int64_t mo = 0, bo = 0;
  for (int j = 0; j < nst; ++j) {
    a.p[j] = factors[j];
    a.Bs[j] = n / factors[j];
    a.sh[j] = factors[j] > 3 ? 3 : std::max<int64_t>(factors[j] - 1, 1);
    a.moff[j] = mo;
    a.boff[j] = bo;
    mo += a.sh[j] * S * a.Bs[j];
    bo += a.Bs[j];
  }
  a.boff[nst] = bo;
  a.sumB = d.sumB;
  a.meas = (double2*)(w + Lo.off[0]);
  a.floor = (double*)(w + Lo.off[1]);
  a.kind = (int32_t*)(w + Lo.off[2]);
  a.cf = (int64_t*)(w + Lo.off[3]);
  a.cc = (double2*)(w + Lo.off[4]);
  a.q[0] = (int64_t*)(w + Lo.off[5]);
  a.q[1] = (int64_t*)(w + Lo.off[6]);
  a.qtail[0] = (int32_t*)(w + Lo.off[7]);
  a.qtail[1] = a.qtail[0] + S;
  a.qcap = d.qcap;
  a.rec_pos = (int64_t*)(w + Lo.off[8]);
  a.rec_coef = (double2*)(w + Lo.off[9]);
  a.rec_count = (int32_t*)(w + Lo.off[10]);
  a.cap = d.cap;
  a.HT = pe_ht(d.cap);
  a.ht_key = (int64_t*)(w + Lo.off[11]);
  a.ht_val = (int32_t*)(w + Lo.off[12]);
  a.peels = (int32_t*)(w + Lo.off[13]);
  a.err = (int32_t*)(w + Lo.off[14]);
  Group* groups = (Group*)(w + Lo.off[15]);
  int32_t* ngroups = (int32_t*)(w + Lo.off[16]);
  int32_t* item_sig = (int32_t*)(w + Lo.off[17]);
  int64_t* item_tau = (int64_t*)(w + Lo.off[18]);
  void* bws = w + Lo.total;

  SFFT_CUDA(cudaMemsetAsync(a.ht_key, 0, sizeof(int64_t) * (size_t)S * a.HT, st));
  SFFT_CUDA(cudaMemsetAsync(a.err, 0, sizeof(int32_t) * S, st));
  for (int j = 0; j < nst; ++j) {
    const int ns = (int)a.sh[j];
    k_pe_items<<<(unsigned)cdiv_up((int64_t)S * ns, 256), 256, 0, st>>>(S, ns, item_sig, item_tau);
    SFFT_CHECK_LAUNCH("k_pe_items");
    Prod p{};
    p.x = x;
    p.xstride = xstride;
    p.n = n;
    p.B = a.Bs[j];
    p.item_sig = item_sig;
    p.item_a = item_tau;
    p.out_M = ns;  // item s*ns + t writes row t*S + s of meas_j [ns][S][B_j]
    p.out_S = S;
    int rc = run_bucketize(dtype, PROD_SPIKE, p, (int64_t)S * ns, Wst[j], a.meas + a.moff[j], bws,
                           (size_t)d.bws, st);
    if (rc) return rc;
    rc = run_floor(a.meas + a.moff[j], S, a.Bs[j], 3.0, nullptr, nullptr, a.floor + (int64_t)j * S,
                   nullptr, st);
    if (rc) return rc;
  }
  SFFT_REQUIRE(nst <= 32, "peeling: at most 32 stages");
  dim3 gc((unsigned)cdiv_up(d.sumB, 256), S);
  k_pe_classify_all<<<gc, 256, 0, st>>>(a);
  SFFT_CHECK_LAUNCH("k_pe_classify_all");
  k_pe_queue_init<<<S, 1024, 0, st>>>(a);
  SFFT_CHECK_LAUNCH("k_pe_queue_init");
  // SFFT_PEEL_NO_FF=1: the plain loop, one peel per step and every peel of a cycle
  // run; SFFT_PEEL_WINDOW=1: cycles fast-forwarded, one peel per step (A/B
  // measurement and the parity test)
  k_pe_peel<<<S, 32, 0, st>>>(a, d.budget, getenv("SFFT_PEEL_NO_FF") ? 0 : (getenv("SFFT_PEEL_WINDOW") ? 2 : 1));
  SFFT_CHECK_LAUNCH("k_pe_peel");
  k_pe_stuck<<<S, 256, 0, st>>>(a, out_conv, out_iters);
  SFFT_CHECK_LAUNCH("k_pe_stuck");
  SFFT_CUDA(cudaMemcpyAsync(out_err, a.err, sizeof(int32_t) * S, cudaMemcpyDeviceToDevice, st));
  const size_t dsm = (size_t)kFusedMaxB * (8 + 8 + 4);
  SFFT_CUDA(cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  k_finalize<<<S, kFinNT, dsm, st>>>(a.rec_pos, a.rec_coef, a.rec_count, a.cap, k, out_pos,
                                      out_coef, out_n);
  SFFT_CHECK_LAUNCH("k_finalize");
  k_pe_groups<<<(unsigned)cdiv_up(S, 128), 128, 0, st>>>(a, groups, ngroups);
  SFFT_CHECK_LAUNCH("k_pe_groups");
  // every signal reads the same samples (the stages' strides and shifts do not
  // depend on the data): the union is counted once, by 64 CTAs, and copied
  k_zero_rows<<<1, 128, 0, st>>>(out_samples, 1, nullptr, nullptr);
  SFFT_CHECK_LAUNCH("k_zero_rows");
  k_union_excl<<<dim3(64, 1), kUxNT, 0, st>>>(groups, ngroups, kMaxGroups, n, nullptr, nullptr,
                                              (unsigned long long*)out_samples);
  SFFT_CHECK_LAUNCH("k_union_excl");
  k_pe_samples<<<(unsigned)cdiv_up(S, 256), 256, 0, st>>>(out_samples, S);
  SFFT_CHECK_LAUNCH("k_pe_samples");
  if (out_sched) {
    k_export_groups<<<S, 64, 0, st>>>(groups, ngroups, S, out_sched);
    SFFT_CHECK_LAUNCH("k_export_groups");
  }
  return 0;
}

}  // namespace sfft
