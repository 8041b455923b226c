// Batched iterative framework with phase location (sfft/frameworks.py:439-516,
// :556-570) and the residual polish (:573-608), device-resident.
//
// Continuous batching: S slots work through a queue of Q signals.  Every
// round advances each busy slot by one step of its own state machine — a
// loop iteration (LOOP) or a polish pass (POLISH) — and a slot whose signal
// finishes is refilled from the queue by the device at the start of the next
// round, so signals that need many iterations never leave the GPU idle.
// Every decision (convergence, heavy set, ladder unwrapping, consistency,
// merge, residual test, polish corrections, admission) is taken on the
// device; the host only issues the rounds and reads one counter per round.
//
// Per loop iteration of a slot (perm = perms[sig][it-1]):
//   y[j] = bucketize(x, sigma, tau + d_j), d = {0} U ladder       (one launch)
//   y0  -= model(recovered)                   all B buckets      (k_subtract)
//   floor, convergence, heavy list (-|y0|, b)                    (k_it_decide)
//   y[j>0] - model(recovered) at heavy buckets; unwrap; checks   (k_it_locate)
//   merge found into recovered (insertion order = heavy order)   (k_it_merge)
//   |y0 - model(found)| < 1.3 floor ?                            (k_subtract, k_it_resid)
//
// Binary / multiscale location (sfft/frameworks.py:517-554) replaces the
// ladder by the class-split measurements: the loop items of a slot are the
// L = N/B shifts d*B (d < L, every d*(n/step) the split search can ask for)
// plus the alias-check shifts 1 and 3; k_sp_model subtracts the recovered
// model from them at the heavy buckets, k_sp_search runs the digit-by-digit
// split per heavy bucket (one warp each), k_sp_prefix forms the shifts the
// reference would have cached by then (a prefix over the heavy order) and
// k_sp_verify applies the consistency checks, the weight check and the
// estimate.
#include "kernels.cuh"
#include "schedule.cuh"
#include "finalize.cuh"

#ifndef SFFT_SPEC_POLISH
#define SFFT_SPEC_POLISH 5
#endif

namespace sfft {

enum SlotPhase { PH_FREE = 0, PH_LOOP = 1, PH_POLISH = 2, PH_FINISH = 3, PH_IDLE = 4 };

struct IterState {
  int32_t sig;         // queue index of the signal in this slot
  int32_t phase;
  int32_t it;          // loop iterations entered so far
  int32_t pidx;        // permutation index of this round's measurement
  int32_t nsh;         // measurements this round (M loop, 3 polish, 0 idle)
  int32_t epoch, pass; // polish position
  int32_t newslot;     // admitted this round: hash table needs clearing
  double scale_ref;
  double floor;
  double final_resid;
  int32_t iterations;
  int32_t converged;
  int32_t entries;     // loop entries = permutations consumed by the loop
  int32_t n_rec;
  int32_t nheavy;
  int32_t nfound;
  int32_t polish;
  int32_t pending;
  int32_t cursor;      // next permutation index (polish)
  int32_t ngroups;
};

struct IterArgs {
  int64_t n, B, L, omega, k;
  int S, P, M, max_it, cap;      // S slots; cap = recovered capacity per slot
  int Q;                         // signals in the queue
  const int32_t* avail;          // optional: signals [0, *avail) have arrived in HBM
  int64_t pstride;               // perms row stride per signal (0: shared stream)
  int32_t* item_active;          // [S*M] items of the per-item flat bucketization
  int32_t* item_fold;            // [S*M] split loop items d*B of the row-correlation path
  int use_fold;                  // split location folds its loop shifts d*B as a row correlation
  RealTab rt;                    // real form of the response table (rt.at null: complex)
  int32_t* pgate;                // [S] polish pass this round
  int64_t ladder[kMaxShifts];    // d_1..d_{M-1} (phase location)
  const int64_t* shifts;         // [M] shift of loop item j (device)
  int loc;                       // 0 phase, 1 class-split (binary / multiscale)
  int branching, digits;         // split search: L = branching^digits
  int32_t* sp_r;                 // [S][B] split offset per heavy rank
  int32_t* sp_ok;                // [S][B] 1 located, 0 ambiguous
  int32_t* sp_depth;             // [S][B] largest step the search measured
  const int64_t* psig;           // [S][P]
  const int64_t* ptau;           // [S][P]
  const double2* gt;             // [L][B]
  const double* gmax;
  // workspace
  IterState* st;
  int32_t* active;               // [S] main loop gate
  int32_t* gate;                 // [S] secondary gate (residual / polish)
  int32_t* n_active;             // device counter
  int32_t* item_sig;             // [S*M] items signal-major (s*M + j)
  int64_t* item_sigma_it;        // [S*M] per item
  int64_t* item_tau_it;          // [S*M] per item
  int64_t* item_sigma;           // [S] shift-0 sigma of each signal's current measurement
  int64_t* item_tau;             // [S] shift-0 tau
  double2* y;                    // [M][S][B]
  double2* resid;                // [S][B]
  int64_t* rec_pos;              // [S][cap]
  double2* rec_coef;             // [S][cap]
  int32_t* rec_count;            // [S]
  int32_t* heavy;                // [S][B] heavy buckets in (-|y0|, b) order (merge order)
  int32_t* heavy_b;              // [S][B] heavy buckets in bucket order (coalesced table reads)
  int32_t* hrank;                // [S][B] position of bucket b in the (-|y0|, b) order
  int64_t* f_pos;                // [S][B] per heavy index
  double2* f_coef;               // [S][B]
  int32_t* f_ok;                 // [S][B]
  int64_t* fc_pos;               // [S][B] compacted found (heavy order)
  double2* fc_coef;              // [S][B]
  int32_t* fc_count;             // [S]
  int32_t* pend;                 // [S][cap] polish pending flags
  double2* delta;                // [S][cap] polish corrections
  Group* groups;                 // [S][kMaxGroups]
  int32_t* stats;                // [8]: -, max recovered, max heavy, done, next
  int64_t* ht_key;               // [S][HT] recovered-position hash (key f+1, 0 empty)
  int32_t* ht_val;               // [S][HT] index into rec_*
  int HT;                        // power of two >= 2*cap
  double2* part;                 // tone-split partial sums (subtract / ladder)
  // measurement row cache (phase location): C rows per slot after the M*S
  // working rows of y; entry c of slot s holds the bucketization of
  // (perm dir_p[s][c], shift dir_d[s][c]) in row M*S + s*C + c
  int C;
  int32_t* dir_p;                // [S][C] permutation index (-1 empty)
  int64_t* dir_d;                // [S][C] shift
  int32_t* role_src;             // [S][M] cache entry feeding working row j this round (-1: measure)
  int32_t* cnt;                  // [S + 1] items per slot, then exclusive offsets; [S] = total
  int32_t* it2_sig;              // [S*(M+C)] compacted items: signal, sigma, tau_tot, output row
  int64_t* it2_sigma;
  int64_t* it2_tau;
  int32_t* it2_row;
  // permutation runs of the compacted list (consecutive items of one signal
  // and sigma): run_first/run_cnt, rcnt = runs per slot then their offsets
  int32_t* rcnt;                 // [S + 1]
  int32_t* act_list;             // [S] the round's loop slots (compacted in the prologue)
  int32_t* run_first;            // [S*(M+C)]
  int32_t* run_cnt;
  // streamed slots: a slot whose round reads a large part of its signal (the
  // first loop round with its speculative rows) is folded by k_stream_fold
  // from sequential 64-byte granules instead of per-sample gathers
  int stream;                    // 1: the stream fold can take this problem
  int32_t* dcnt;                 // [S + 1] 1 per streamed slot, then exclusive offsets
  int32_t* dense;                // [S][4] the round's streamed slots: slot, first item, items, signal
};

// samples_read memo: every signal draws the same seeded permutation stream, so
// signals that ran the same schedule (the same read groups: most converging
// signals) read the same index set.  A finishing slot hashes its group list
// (two independent 64-bit mixes); the first slot with a key computes the
// exclusion count, the rest take it.  Entries live for one engine call.
constexpr int kMemo = 8192;  // power of two
struct SchedMemo {
  unsigned long long k1[kMemo], k2[kMemo];
  long long count[kMemo];
  int32_t ready[kMemo];
};

__device__ __forceinline__ uint32_t ht_slot(int64_t f, int HT) {
  return (uint32_t)(((unsigned long long)(f + 1) * 0x9E3779B97F4A7C15ull) >> 40) & (HT - 1);
}

// index of f in the recovered list of signal s, or -1
__device__ __forceinline__ int ht_find(const IterArgs& a, int s, int64_t f) {
  const int64_t* keys = a.ht_key + (int64_t)s * a.HT;
  const int32_t* vals = a.ht_val + (int64_t)s * a.HT;
  uint32_t h = ht_slot(f, a.HT);
  for (int probe = 0; probe < a.HT; ++probe) {
    const int64_t k = keys[h];
    if (k == f + 1) return vals[h];
    if (k == 0) return -1;
    h = (h + 1) & (a.HT - 1);
  }
  return -1;
}

__device__ __forceinline__ void ht_insert(const IterArgs& a, int s, int64_t f, int idx) {
  unsigned long long* keys = (unsigned long long*)(a.ht_key + (int64_t)s * a.HT);
  int32_t* vals = a.ht_val + (int64_t)s * a.HT;
  uint32_t h = ht_slot(f, a.HT);
  for (int probe = 0; probe < a.HT; ++probe) {
    const unsigned long long old = atomicCAS(&keys[h], 0ull, (unsigned long long)(f + 1));
    if (old == 0ull || old == (unsigned long long)(f + 1)) {
      vals[h] = idx;
      return;
    }
    h = (h + 1) & (a.HT - 1);
  }
}

// ------------------------------------------------------------------ rounds
// Admission: free slots take the next queued signals, in slot order.  One
// CTA owns the queue head: it reads the streaming limit once, ranks the free
// slots with a block scan and hands out [head, min(head + free, limit)) --
// no atomics, so a concurrently raised limit can never make two slots take
// the same signal or skip one.
constexpr int kAdmNT = 1024;
__global__ void __launch_bounds__(kAdmNT) k_cb_admit(IterArgs a) {
  __shared__ int red[32];
  __shared__ int s_head, s_lim;
  // signals still being copied in (streaming admission) are not taken yet;
  // the limit is read once for the whole launch
  if (threadIdx.x == 0) {
    s_head = a.stats[4];
    s_lim = a.avail ? min(a.Q, *(volatile const int32_t*)a.avail) : a.Q;
  }
  __syncthreads();
  const int lim = s_lim;
  for (int base = 0; base < a.S; base += kAdmNT) {
    const int s = base + threadIdx.x;
    const bool fr = s < a.S && a.st[s].phase == PH_FREE;
    int tot;
    const int rank = block_exscan<kAdmNT>(fr ? 1 : 0, red, &tot);
    const int head = s_head;
    if (fr) {
      IterState& S = a.st[s];
      const int idx = head + rank;
      if (idx < lim) {
        S = IterState{};
        S.sig = idx;
        S.phase = PH_LOOP;
        S.newslot = 1;
        a.rec_count[s] = 0;
      } else if (lim >= a.Q) {
        S.phase = PH_IDLE;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_head = min(head + tot, max(lim, head));
    __syncthreads();
  }
  if (threadIdx.x == 0) a.stats[4] = s_head;
}

__global__ void k_cb_clear(IterArgs a) {
  const int s = blockIdx.y;
  if (!a.st[s].newslot) return;
  int64_t* keys = a.ht_key + (int64_t)s * a.HT;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.HT;
       i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = 0;
}

// This round's step of every slot: a loop iteration or a polish pass.
__global__ void k_cb_step(IterArgs a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  IterState& S = a.st[s];
  S.newslot = 0;
  a.active[s] = 0;
  a.pgate[s] = 0;
  a.gate[s] = 0;
  S.nsh = 0;
  if (S.phase == PH_LOOP) {
    S.it += 1;
    S.entries = S.it;
    S.pidx = S.it - 1;
    S.nsh = a.M;
    a.active[s] = 1;
  } else if (S.phase == PH_POLISH) {
    if (S.pass == 0) S.pending = S.n_rec;  // epoch start: every tone pending
    S.pidx = S.cursor;
    S.cursor += 1;
    S.nsh = 3;
    a.pgate[s] = 1;
  } else {
    return;
  }
  const int pp = S.pidx < a.P ? S.pidx : a.P - 1;
  const int64_t sg = a.psig[(int64_t)S.sig * a.pstride + pp];
  const int64_t t0 = pmod(a.ptau[(int64_t)S.sig * a.pstride + pp], a.n);
  a.item_sigma[s] = sg;
  a.item_tau[s] = t0;
  if (S.phase == PH_POLISH) {
    const int g = S.ngroups;
    if (g < kMaxGroups) {
      Group& G = a.groups[(int64_t)s * kMaxGroups + g];
      G.kind = 0;
      G.a = sg;
      G.tau = t0;
      G.cnt = a.omega;
      G.nsh = 3;
      G.sh[0] = 0;
      G.sh[1] = 1;
      G.sh[2] = 2;
      S.ngroups = g + 1;
    }
  }
}

// The round's loop slots, compacted (one CTA, slot order): the per-slot
// kernels of the loop (subtractions, ladder, location) run over this list
// instead of every slot, so the late rounds -- a few non-converging signals --
// do not launch hundreds of thousands of empty CTAs.  Count in stats[7].
__global__ void __launch_bounds__(kAdmNT) k_act_list(IterArgs a) {
  __shared__ int red[32];
  __shared__ int s_base;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int base = 0; base < a.S; base += kAdmNT) {
    const int s = base + threadIdx.x;
    const bool on = s < a.S && a.active[s];
    int tot;
    const int r = block_exscan<kAdmNT>(on ? 1 : 0, red, &tot);
    if (on) a.act_list[s_base + r] = s;
    __syncthreads();
    if (threadIdx.x == 0) s_base += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.stats[7] = s_base;
}

// Items are slot-major (i = s*M + j) so that the shifted measurements of one
// signal, which re-read most of the same samples, run side by side and share
// L2 lines; outputs land shift-major (row j*S + s, see Prod::out_M).
__global__ void k_cb_items(IterArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.M * a.S) return;
  const int s = i / a.M, j = i - s * a.M;
  const IterState& S = a.st[s];
  const bool on = j < S.nsh;
  // split location: the loop shifts d*B (d < L) are folded as a row correlation
  const bool fold = on && a.use_fold && S.phase == PH_LOOP && j < a.L;
  a.item_active[i] = on && !fold;
  a.item_fold[i] = fold;
  a.item_sig[i] = S.sig > 0 ? S.sig : 0;
  if (!on) return;
  const int64_t d = (S.phase == PH_LOOP) ? a.shifts[j] : j;
  a.item_sigma_it[i] = a.item_sigma[s];
  a.item_tau_it[i] = pmod(a.item_tau[s] + d, a.n);
}

// Measurement planning with a row cache (phase location).  A slot's first
// loop round also measures, speculatively and side by side with its own 8
// loop items, the next loop permutation's M shifts and the 3 shifts of the 6
// permutations after it (the polish passes of a signal that converges in two
// iterations); every later round copies the rows it finds in the cache and
// measures only the rest.  A transform's bucketizations then share their L2
// lines across permutations (one launch instead of eight; measured 18 % less
// gather time per transform), and the results are identical: the same
// (sigma, tau_tot) item gives the same bucket values whenever it runs.
__device__ __forceinline__ int64_t role_shift(const IterArgs& a, const IterState& S, int j) {
  return (S.phase == PH_LOOP) ? a.shifts[j] : (int64_t)j;
}

// Greedy packing of a slot's permutation chunks (the items of one
// permutation, in emission order) into groups of at most kGfItems items: a
// chunk that does not fit the open group starts a new one; chunks longer than
// a group are split.  Counting (plan) and emission (fill) share it.
struct GroupPack {
  int cur = 0;  // items in the open group
  int go = 0;   // next group index
  int32_t* gf = nullptr;
  int32_t* gc = nullptr;
  __device__ void chunk(int first_item, int z) {
    if (cur > 0 && cur + z > kGfItems) cur = 0;
    while (z > 0) {
      if (cur == 0) {
        if (gf) {
          gf[go] = first_item;
          gc[go] = 0;
        }
        ++go;
      }
      const int take = min(z, kGfItems - cur);
      if (gc) gc[go - 1] += take;
      cur += take;
      z -= take;
      first_item += take;
      if (cur == kGfItems) cur = 0;
    }
  }
};

__global__ void k_cb_plan(IterArgs a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  const IterState& S = a.st[s];
  int32_t* dp = a.dir_p + (int64_t)s * a.C;
  int64_t* dd = a.dir_d + (int64_t)s * a.C;
  const bool first = S.phase == PH_LOOP && S.it == 1;
  if (first)
    for (int c = 0; c < a.C; ++c) dp[c] = -1;
  int nm = 0;
  for (int j = 0; j < a.M; ++j) {
    int src = -1;
    if (j < S.nsh) {
      const int64_t d = role_shift(a, S, j);
      for (int c = 0; c < a.C && src < 0; ++c)
        if (dp[c] == S.pidx && dd[c] == d) src = c;
      nm += src < 0;
    }
    a.role_src[(int64_t)s * a.M + j] = src;
  }
  int spec = 0;
  GroupPack gp;
  if (nm > 0) gp.chunk(0, nm);
  if (first) {
    for (int c = 0; c < a.C; ++c) {
      const int pp = S.pidx + 1 + (c < a.M ? 0 : 1 + (c - a.M) / 3);
      spec += pp < a.P;
    }
    if (S.pidx + 1 < a.P) gp.chunk(0, a.M);  // the next loop permutation's ladder
    for (int c = a.M; c < a.C; c += 3)        // polish permutations, 3 shifts each
      if (S.pidx + 2 + (c - a.M) / 3 < a.P) gp.chunk(0, 3);
  }
  a.cnt[s] = nm + spec;
  // streamed when the round's windows add up to a quarter of the signal (by
  // then most 64-byte granules are touched: reading every granule once,
  // sequentially, is cheaper than the gathers)
  const bool dense = a.stream && first && nm == a.M && (int64_t)(nm + spec) * a.omega * 4 >= a.n;
  a.dcnt[s] = dense;
  a.rcnt[s] = dense ? 0 : gp.go;
}

// exclusive scan of cnt[0..S) in place, total in cnt[S] (one CTA)
__device__ void cb_scan_one(int32_t* v, int S, int* red, int* carry, int32_t* total) {
  if (threadIdx.x == 0) *carry = 0;
  __syncthreads();
  for (int base = 0; base < S; base += 1024) {
    const int i = base + threadIdx.x;
    const int x = i < S ? v[i] : 0;
    int tot;
    const int ex = block_exscan<1024>(x, red, &tot);
    if (i < S) v[i] = *carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) *carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    v[S] = *carry;
    *total = *carry;  // read by the host with the round status
  }
  __syncthreads();
}

// exclusive scans of the per-slot item and run counts (one CTA)
__global__ void __launch_bounds__(1024) k_cb_scan(IterArgs a) {
  __shared__ int red[32];
  __shared__ int carry;
  cb_scan_one(a.cnt, a.S, red, &carry, a.stats + 5);
  cb_scan_one(a.rcnt, a.S, red, &carry, a.stats + 6);
  cb_scan_one(a.dcnt, a.S, red, &carry, a.stats + 0);
}

__global__ void k_cb_fill(IterArgs a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  const IterState& S = a.st[s];
  int o = a.cnt[s];
  GroupPack gp;
  gp.go = a.rcnt[s];
  const bool dense = a.dcnt[s + 1] > a.dcnt[s];
  if (dense) {
    // no groups: the slot's items go to the stream fold
    reinterpret_cast<int4*>(a.dense)[a.dcnt[s]] =
        make_int4(s, a.cnt[s], a.cnt[s + 1] - a.cnt[s], S.sig > 0 ? S.sig : 0);
  } else {
    gp.gf = a.run_first;
    gp.gc = a.run_cnt;
  }
  const int sig = S.sig > 0 ? S.sig : 0;
  const int o_own = o;
  for (int j = 0; j < S.nsh && j < a.M; ++j) {
    if (a.role_src[(int64_t)s * a.M + j] >= 0) continue;
    a.it2_sig[o] = sig;
    a.it2_sigma[o] = a.item_sigma[s];
    a.it2_tau[o] = pmod(a.item_tau[s] + role_shift(a, S, j), a.n);
    a.it2_row[o] = j * a.S + s;
    ++o;
  }
  if (o > o_own) gp.chunk(o_own, o - o_own);
  if (!(S.phase == PH_LOOP && S.it == 1)) return;
  int32_t* dp = a.dir_p + (int64_t)s * a.C;
  int64_t* dd = a.dir_d + (int64_t)s * a.C;
  for (int c = 0; c < a.C; ++c) {
    const int pp = S.pidx + 1 + (c < a.M ? 0 : 1 + (c - a.M) / 3);
    if (pp >= a.P) continue;
    const int64_t d = c < a.M ? a.shifts[c] : (int64_t)((c - a.M) % 3);
    const int64_t row = (int64_t)sig * a.pstride + pp;
    if (c == 0) gp.chunk(o, a.M);                              // ladder permutation
    else if (c >= a.M && (c - a.M) % 3 == 0) gp.chunk(o, 3);  // polish permutation
    a.it2_sig[o] = sig;
    a.it2_sigma[o] = a.psig[row];
    a.it2_tau[o] = pmod(pmod(a.ptau[row], a.n) + d, a.n);
    a.it2_row[o] = (int32_t)((int64_t)a.M * a.S + (int64_t)s * a.C + c);
    dp[c] = pp;
    dd[c] = d;
    ++o;
  }
}

// working row j of slot s <- its cache entry
__global__ void k_cb_copy(IterArgs a) {
  const int s = blockIdx.x / a.M, j = blockIdx.x - s * a.M;
  const int c = a.role_src[(int64_t)s * a.M + j];
  if (c < 0) return;
  const double2* src = a.y + ((int64_t)a.M * a.S + (int64_t)s * a.C + c) * a.B;
  double2* dst = a.y + ((int64_t)j * a.S + s) * a.B;
  for (int64_t b = threadIdx.x; b < a.B; b += blockDim.x) dst[b] = src[b];
}

// End of a slot's loop: polish when converged well below the scale, else done
// (frameworks.py:566-569).
__device__ __forceinline__ void loop_end(const IterArgs& a, IterState& S, int s) {
  a.active[s] = 0;
  const bool pol = S.converged && S.n_rec > 0 && S.final_resid < 0.01 * S.scale_ref;
  if (pol) {
    S.phase = PH_POLISH;
    S.epoch = 0;
    S.pass = 0;
    S.cursor = S.entries;
  } else {
    S.phase = PH_FINISH;
  }
}

// ------------------------------------------------------------------ decide
constexpr int kDecNT = 512;

// Floor / convergence / heavy list of y0 (sfft/frameworks.py:478-490).
__global__ void __launch_bounds__(kDecNT) k_it_decide(IterArgs a) {
  extern __shared__ unsigned char dsm[];
  __shared__ unsigned hist[256];
  __shared__ long long sh[4];
  __shared__ double redd[32];
  __shared__ unsigned long long redu[32];
  __shared__ int redi[32];
  const int s = blockIdx.x;
  if (!a.active[s]) return;
  IterState& S = a.st[s];
  const int it = S.it;
  const int64_t B = a.B;
  const double2* y0 = a.y + (int64_t)s * B;  // slot 0
  unsigned long long* k1 = (unsigned long long*)dsm;
  long long* k2 = (long long*)(k1 + kFusedMaxB);
  int* pay = (int*)(k2 + kFusedMaxB);
  const bool cached = B <= kFusedMaxB;
  // |y0| bits cached in shared memory (k2) for the radix passes
  unsigned long long* mg = (unsigned long long*)k2;
  double med, peak;
  if (cached) {
    for (int64_t i = threadIdx.x; i < B; i += kDecNT) mg[i] = dbits(cabs_(y0[i]));
    __syncthreads();
    median_and_peak_k<kDecNT>(SmemKey{mg}, B, &med, &peak, hist, sh, redd, redu);
  } else {
    median_and_peak<kDecNT>(y0, B, &med, &peak, hist, sh, redd, redu);
  }
  const double robust = fmax(fmax(fmin(3.0 * med, 0.25 * peak), 1e-9 * peak), 1e-300);
  const double sref = fmax(S.scale_ref, peak);
  const double fl = fmax(robust, 1e-9 * sref);
  const bool conv = peak < 1.3 * fl;
  // log the measurement group (the ladder only counts when it was used)
  if (threadIdx.x == 0) {
    S.scale_ref = sref;
    S.floor = fl;
    const int g = S.ngroups;
    // split location logs its (data-dependent) shifts in k_sp_check
    if (g < kMaxGroups && (conv || a.loc == 0)) {
      Group& G = a.groups[(int64_t)s * kMaxGroups + g];
      G.kind = 0;
      G.a = a.item_sigma[s];
      G.tau = a.item_tau[s];
      G.cnt = a.omega;
      G.nsh = conv ? 1 : a.M;
      G.sh[0] = 0;
      if (!conv)
        for (int j = 1; j < a.M; ++j) G.sh[j] = a.ladder[j - 1];
      S.ngroups = g + 1;
    }
    if (conv) {
      S.converged = 1;
      S.final_resid = peak;
      S.iterations = it - 1;
      loop_end(a, S, s);
    }
  }
  if (conv) return;
  // heavy = {b : |y0[b]| >= floor} in (-|y0|, b) order
  const unsigned long long ufl = dbits(fl);
  constexpr int kPer = kFusedMaxB / kDecNT;
  const int64_t per = (B + kDecNT - 1) / kDecNT;
  const int64_t i0 = threadIdx.x * per, i1 = min(B, i0 + per);
  unsigned long long mine_u[kPer];
  int mine = 0;
  for (int64_t i = i0; i < i1; ++i) {
    const unsigned long long u = cached ? mg[i] : dbits(cabs_(y0[i]));
    if (cached) mine_u[i - i0] = u;
    mine += u >= ufl;
  }
  int total;
  int off = block_exscan<kDecNT>(mine, redi, &total);  // also orders the mg reads before reuse
  int32_t* hv = a.heavy + (int64_t)s * B;
  int32_t* hb = a.heavy_b + (int64_t)s * B;
  for (int64_t i = i0; i < i1; ++i) {
    const unsigned long long u = cached ? mine_u[i - i0] : dbits(cabs_(y0[i]));
    if (u >= ufl) {
      hb[off] = (int)i;
      if (cached) {
        k1[off] = ~u;
        k2[off] = i;
        pay[off] = (int)i;
      } else {
        hv[off] = (int)i;
      }
      ++off;
    }
  }
  __syncthreads();
  if (cached) {
    int cap = 1;
    while (cap < total) cap <<= 1;
    block_bitonic<kDecNT>(k1, k2, pay, total, cap);
    for (int i = threadIdx.x; i < total; i += kDecNT) {
      hv[i] = pay[i];
      a.hrank[(int64_t)s * B + pay[i]] = i;
    }
  } else {
    for (int i = threadIdx.x; i < total; i += kDecNT) a.hrank[(int64_t)s * B + hv[i]] = i;
  }
  if (threadIdx.x == 0) {
    S.nheavy = total;
    atomicMax(a.stats + 2, total);
  }
}

// ------------------------------------------------------------------ locate
constexpr int kLocNT = 128;
constexpr int kLocChunk = 64;

// Sum of the recovered model over tones [tb, te) at heavy bucket b for the
// ladder shifts j = 1..M-1, subtracted from ys[] (running, in tone order).
template <int M>
__device__ __forceinline__ void ladder_model(const IterArgs& a, int s, int b, bool live,
                                             int64_t tb, int64_t te, double2* ys,
                                             int64_t (*t_row), int64_t (*t_q), double2* t_c,
                                             double2 (*t_ph)[M]) {
  const int64_t n = a.n, B = a.B, L = a.L;
  const int64_t sigma = a.item_sigma[s];
  const int64_t tau = a.item_tau[s];
  const int64_t* rp = a.rec_pos + (int64_t)s * a.cap;
  const double2* rc = a.rec_coef + (int64_t)s * a.cap;
  for (int64_t t0 = tb; t0 < te; t0 += kLocChunk) {
    __syncthreads();
    for (int q = threadIdx.x; q < kLocChunk * M; q += kLocNT) {
      const int tt = q / M, j = q - tt * M;
      if (t0 + tt >= te || j == 0) continue;
      const int64_t m = mulmod(sigma, pmod(rp[t0 + tt], n), n);
      const int64_t tj = pmod(tau + a.ladder[j - 1], n);
      t_ph[tt][j] = unit_root(n, mulmod(tj, m, n));
      if (j == 1) {
        t_row[tt] = (L - m % L) % L;
        t_q[tt] = (m + L - 1) / L;
        t_c[tt] = rc[t0 + tt];
      }
    }
    __syncthreads();
    if (live) {
      const int tn = (int)((te - t0 < kLocChunk) ? te - t0 : kLocChunk);
      int tt = 0;
      for (; tt + 4 <= tn; tt += 4) {
        double2 w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int64_t col = b - t_q[tt + u];
          col += (col < 0) ? B : 0;
          w[u] = ld_table(a.gt + t_row[tt + u] * B + col);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double2 cw = cmul(t_c[tt + u], w[u]);
#pragma unroll
          for (int j = 1; j < M; ++j) ys[j] = csub(ys[j], cmul(cw, t_ph[tt + u][j]));
        }
      }
      for (; tt < tn; ++tt) {
        int64_t col = b - t_q[tt];
        col += (col < 0) ? B : 0;
        const double2 cw = cmul(t_c[tt], ld_table(a.gt + t_row[tt] * B + col));
#pragma unroll
        for (int j = 1; j < M; ++j) ys[j] = csub(ys[j], cmul(cw, t_ph[tt][j]));
      }
    }
  }
}

// Real-table form of ladder_model (RealTab): per tone and shift
// beta_tj = c w^{(tau+d_j) m} w^{-m h} / B and alpha_tj = c w^{(tau+d_j) m} t0 / B;
// ys[j] -= sum_t alpha_tj + w^{b L h} sum_t beta_tj A_{bL-m}.  The alpha sums
// do not depend on the bucket: thread j of the block forms them (in tone order).
template <int M>
__device__ __forceinline__ void ladder_model_real(const IterArgs& a, int s, int b, bool live,
                                                  int64_t tb, int64_t te, double2* ys,
                                                  int64_t* t_row, int64_t* t_q,
                                                  double2 (*t_be)[M],
                                                  double2 (*t_al)[M], double2* s_al) {
  const int64_t n = a.n, B = a.B, L = a.L;
  const int64_t sigma = a.item_sigma[s];
  const int64_t tau = a.item_tau[s];
  const int64_t* rp = a.rec_pos + (int64_t)s * a.cap;
  const double2* rc = a.rec_coef + (int64_t)s * a.cap;
  const double t0v = a.rt.taps[0];
  const double invB = 1.0 / (double)B;
  const int64_t hh = a.rt.h % n;
  double2 S[M];
#pragma unroll
  for (int j = 0; j < M; ++j) S[j] = cmk(0.0, 0.0);
  if (threadIdx.x < M) s_al[threadIdx.x] = cmk(0.0, 0.0);
  // per-tone quantities once per tone (m, w^{-m h}, table row), then the
  // per-(tone, shift) factors from them: the same values as forming each
  // (tone, shift) entry from scratch, with one sincos per tone fewer per shift
  __shared__ int64_t u_m[kLocChunk];
  __shared__ double2 u_wmh[kLocChunk], u_c[kLocChunk];
  for (int64_t t0 = tb; t0 < te; t0 += kLocChunk) {
    __syncthreads();
    for (int tt = threadIdx.x; tt < kLocChunk; tt += kLocNT) {
      if (t0 + tt >= te) continue;
      const int64_t m = mulmod(sigma, pmod(rp[t0 + tt], n), n);
      u_m[tt] = m;
      u_wmh[tt] = unit_root(n, pmod(-mulmod(m, hh, n), n));
      u_c[tt] = rc[t0 + tt];
      t_row[tt] = (L - m % L) % L;
      t_q[tt] = (m + L - 1) / L;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < kLocChunk * M; q += kLocNT) {
      const int tt = q / M, j = q - tt * M;
      if (t0 + tt >= te || j == 0) continue;
      const int64_t tj = pmod(tau + a.ladder[j - 1], n);
      const double2 cp = cmul(u_c[tt], unit_root(n, mulmod(tj, u_m[tt], n)));
      t_be[tt][j] = cscale(cmul(cp, u_wmh[tt]), invB);
      t_al[tt][j] = cscale(cp, t0v * invB);
    }
    __syncthreads();
    const int tn = (int)((te - t0 < kLocChunk) ? te - t0 : kLocChunk);
    if (threadIdx.x > 0 && threadIdx.x < M)
      for (int tt = 0; tt < tn; ++tt) s_al[threadIdx.x] = cadd(s_al[threadIdx.x], t_al[tt][threadIdx.x]);
    if (live) {
      int tt = 0;
      for (; tt + 4 <= tn; tt += 4) {
        double w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int64_t col = b - t_q[tt + u];
          col += (col < 0) ? B : 0;
          SFFT_DASSERT(col >= 0 && col < B && t_row[tt + u] >= 0 && t_row[tt + u] < L);
          w[u] = __ldg(a.rt.at + t_row[tt + u] * B + col);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 1; j < M; ++j) {
            S[j].x = fma(t_be[tt + u][j].x, w[u], S[j].x);
            S[j].y = fma(t_be[tt + u][j].y, w[u], S[j].y);
          }
      }
      for (; tt < tn; ++tt) {
        int64_t col = b - t_q[tt];
        col += (col < 0) ? B : 0;
        const double w = __ldg(a.rt.at + t_row[tt] * B + col);
#pragma unroll
        for (int j = 1; j < M; ++j) {
          S[j].x = fma(t_be[tt][j].x, w, S[j].x);
          S[j].y = fma(t_be[tt][j].y, w, S[j].y);
        }
      }
    }
  }
  __syncthreads();
  if (live && te > tb) {
    const double2 pb = unit_root(n, mulmod(mulmod(b, L, n), hh, n));
#pragma unroll
    for (int j = 1; j < M; ++j) ys[j] = csub(ys[j], cadd(s_al[j], cmul(pb, S[j])));
  }
}

constexpr int kLadPerSplit = 256;  // tones per split

// splits of a slot's ladder model (0: small list, subtracted inline)
__device__ __forceinline__ int lad_splits(int64_t T, int maxTS) {
  if (T <= kLadPerSplit || maxTS <= 0) return 0;
  const int64_t z = (T + kLadPerSplit - 1) / kLadPerSplit;
  return (int)(z > maxTS ? maxTS : z);
}

// Tone-split partial ladder sums for large recovered lists:
// part[s][z][h][j-1] = -sum_{tones of split z} c w ph_j.
#ifndef SFFT_LAD_MINB
#define SFFT_LAD_MINB 4   // 4, 5, 6 CTAs per SM measured equal (128, 96, 80 registers); 8 spills and is 6 % slower
#endif
template <int M>
__global__ void __launch_bounds__(kLocNT, SFFT_LAD_MINB) k_it_ladder_part(IterArgs a) {
  __shared__ int64_t t_row[kLocChunk], t_q[kLocChunk];
  __shared__ double2 t_c[kLocChunk];
  __shared__ double2 t_ph[kLocChunk][M];  // per (tone, shift): sized by the ladder, not kMaxShifts
  __shared__ double2 t_al[kLocChunk][M];
  __shared__ double2 s_al[kMaxShifts];
  const int s = a.act_list[blockIdx.y];  // grid over the loop slots of the round
  if (!a.active[s]) return;
  const int nh = a.st[s].nheavy;
  const int h0 = blockIdx.x * kLocNT;
  if (h0 >= nh) return;
  const int h = h0 + threadIdx.x;
  const bool live = h < nh;
  const int64_t T = a.rec_count[s];
  const int TS = lad_splits(T, gridDim.z);
  if ((int)blockIdx.z >= TS) return;  // TS == 0: k_it_locate subtracts inline
  const int64_t per = (T + TS - 1) / TS;
  const int64_t tb = (int64_t)blockIdx.z * per;
  const int64_t te = (tb + per < T) ? tb + per : T;
  const int b = live ? a.heavy_b[(int64_t)s * a.B + h] : 0;
  double2 ys[M];
#pragma unroll
  for (int j = 0; j < M; ++j) ys[j] = cmk(0.0, 0.0);
  if (a.rt.at)
    ladder_model_real<M>(a, s, b, live, tb, te, ys, t_row, t_q, t_ph, t_al, s_al);
  else
    ladder_model<M>(a, s, b, live, tb, te, ys, t_row, t_q, t_c, t_ph);
  if (!live) return;
  double2* o = a.part + (((int64_t)s * gridDim.z + blockIdx.z) * a.B + h) * (M - 1);
#pragma unroll
  for (int j = 1; j < M; ++j) o[j - 1] = ys[j];
}

// Ladder values at heavy buckets minus the recovered model, phase unwrap,
// passband / consistency / weight checks, coefficient (frameworks.py:493-516).
// TS == 0: the model is subtracted here in tone order; TS > 0: summed from
// k_it_ladder_part's splits.
template <int M>
__global__ void __launch_bounds__(kLocNT) k_it_locate(IterArgs a, int maxTS) {
  __shared__ int64_t t_row[kLocChunk], t_q[kLocChunk];
  __shared__ double2 t_c[kLocChunk];
  __shared__ double2 t_ph[kLocChunk][M];  // per (tone, shift): sized by the ladder, not kMaxShifts
  __shared__ double2 t_al[kLocChunk][M];
  __shared__ double2 s_al[kMaxShifts];
  const int s = a.act_list[blockIdx.y];  // grid over the loop slots of the round
  if (!a.active[s]) return;
  const IterState& S = a.st[s];
  const int nh = S.nheavy;
  const int h0 = blockIdx.x * kLocNT;
  if (h0 >= nh) return;
  const int h = h0 + threadIdx.x;
  const bool live = h < nh;
  const int64_t n = a.n, B = a.B, L = a.L;
  const int64_t sigma = a.item_sigma[s];
  const int64_t tau = a.item_tau[s];  // shift 0 item
  // heavy buckets are visited in bucket order (coalesced table rows); the
  // result goes to the bucket's rank in the (-|y0|, b) order used by merge
  const int b = live ? a.heavy_b[(int64_t)s * B + h] : 0;
  double2 ys[M];
#pragma unroll
  for (int j = 0; j < M; ++j) ys[j] = a.y[((int64_t)j * a.S + s) * B + b];
  const int TS = lad_splits(a.rec_count[s], maxTS);
  if (TS == 0) {
    if (a.rt.at)
      ladder_model_real<M>(a, s, b, live, 0, a.rec_count[s], ys, t_row, t_q, t_ph, t_al, s_al);
    else
      ladder_model<M>(a, s, b, live, 0, a.rec_count[s], ys, t_row, t_q, t_c, t_ph);
  } else if (live) {
    for (int z = 0; z < TS; ++z) {
      const double2* p = a.part + (((int64_t)s * maxTS + z) * B + h) * (M - 1);
#pragma unroll
      for (int j = 1; j < M; ++j) ys[j] = cadd(ys[j], p[j - 1]);
    }
  }
  if (!live) return;
  const int64_t fi = (int64_t)s * B + a.hrank[(int64_t)s * B + b];
  a.f_ok[fi] = 0;
  const double2 y0 = ys[0];
  // _unwrap_position (frameworks.py:179-196): ladder[0] == 1
  if (cabs_scalar(y0) == 0.0) return;
  const double nd = (double)n;
  const double scl = -nd / (2.0 * 3.141592653589793);
  auto fmodpos = [&](double v, double m) {
    double r = fmod(v, m);
    if (r != 0.0 && r < 0.0) r += m;
    if (r == 0.0) r = 0.0;
    return r;
  };
  double2 r1 = cdiv(ys[1], y0);
  double q = fmodpos(atan2(r1.y, r1.x) * scl, nd);
#pragma unroll
  for (int j = 2; j < M; ++j) {
    const double2 rj = cdiv(ys[j], y0);
    const double phi = fmodpos(atan2(rj.y, rj.x) * scl, nd);
    const double d = (double)a.ladder[j - 1];
    const double period = nd / d;
    const double base = phi / d;
    q = base + rint((q - base) / period) * period;
  }
  const int64_t qi = pmod((int64_t)rint(q), n);
  // passband of bucket b
  const int64_t lo = pmod((int64_t)b * L - L / 2, n);
  if (pmod(qi - lo, n) >= L) return;
  // ladder consistency
  const double tol = fmax(3.0 * S.floor, 0.15 * cabs_scalar(y0));
#pragma unroll
  for (int j = 1; j < M; ++j) {
    const double2 pred = cmul(y0, unit_root(n, mulmod(a.ladder[j - 1] % n, qi, n)));
    if (cabs_scalar(csub(ys[j], pred)) > tol) return;
  }
  const int64_t e = pmod((int64_t)b * L - qi, n);
  const double2 w = a.gt[(e % L) * B + e / L];
  if (cabs_scalar(w) < 0.05 * a.gmax[0]) return;
  // mean of the dephased ladder values / w
  double2 sum = cmk(0.0, 0.0);
#pragma unroll
  for (int j = 0; j < M; ++j) {
    const int64_t sh = (j == 0) ? 0 : a.ladder[j - 1];
    const int64_t ex = pmod(-mulmod(pmod(tau + sh, n), qi, n), n);
    sum = cadd(sum, cmul(ys[j], unit_root(n, ex)));
  }
  const double2 coeff = cdiv(cdivr(sum, (double)M), w);
  const int64_t f = mulmod(modinv(sigma, n), qi, n);
  a.f_pos[fi] = f;
  a.f_coef[fi] = coeff;
  a.f_ok[fi] = 1;
}


// ------------------------------------------------------------------ split location
// y[j][s][b] -= sum_t (c_t * G[(bL - m_t) mod N]) * w^{(tau + d_j) m_t} for
// the loop items j >= 1 at the heavy buckets, tones in order (the running
// subtraction of _subtract_flat, frameworks.py:423-436).  Tile: 32 heavy
// buckets (lanes) x 32 shifts (8 warps x 4), tones staged 16 at a time.
constexpr int kSpNT = 256;
constexpr int kSpH = 32, kSpJ = 32, kSpT = 16;

__global__ void __launch_bounds__(kSpNT) k_sp_model(IterArgs a) {
  __shared__ double2 cw[kSpT][kSpH];
  __shared__ double2 ph[kSpT][kSpJ];
  __shared__ int64_t tm[kSpT], trow[kSpT], tq[kSpT];
  __shared__ double2 tc[kSpT];
  const int s = blockIdx.z;
  if (!a.active[s]) return;
  const int nh = a.st[s].nheavy;
  const int h0 = blockIdx.x * kSpH;
  const int j0 = 1 + blockIdx.y * kSpJ;
  if (h0 >= nh || j0 >= a.M) return;
  const int64_t n = a.n, B = a.B, L = a.L;
  const int64_t sigma = a.item_sigma[s], tau = a.item_tau[s];
  const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
  const int h = h0 + lane;
  const bool hl = h < nh;
  const int b = hl ? a.heavy_b[(int64_t)s * B + h] : 0;
  double2 acc[4];
  bool jl[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = j0 + wq * 4 + u;
    jl[u] = hl && j < a.M;
    acc[u] = jl[u] ? a.y[((int64_t)j * a.S + s) * B + b] : cmk(0.0, 0.0);
  }
  const int T = a.rec_count[s];
  const int64_t* rp = a.rec_pos + (int64_t)s * a.cap;
  const double2* rc = a.rec_coef + (int64_t)s * a.cap;
  for (int t0 = 0; t0 < T; t0 += kSpT) {
    const int tn = min(kSpT, T - t0);
    __syncthreads();
    if (threadIdx.x < tn) {
      const int64_t m = mulmod(sigma, pmod(rp[t0 + threadIdx.x], n), n);
      tm[threadIdx.x] = m;
      trow[threadIdx.x] = (L - m % L) % L;
      tq[threadIdx.x] = (m + L - 1) / L;
      tc[threadIdx.x] = rc[t0 + threadIdx.x];
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kSpT * kSpH; e += kSpNT) {
      const int t = e / kSpH, hh = e - t * kSpH;
      if (t >= tn || h0 + hh >= nh) continue;
      const int bb = a.heavy_b[(int64_t)s * B + h0 + hh];
      int64_t col = bb - tq[t];
      col += (col < 0) ? B : 0;
      cw[t][hh] = cmul(tc[t], ld_table(a.gt + trow[t] * B + col));
    }
    for (int e = threadIdx.x; e < kSpT * kSpJ; e += kSpNT) {
      const int t = e / kSpJ, jj = e - t * kSpJ;
      if (t >= tn || j0 + jj >= a.M) continue;
      ph[t][jj] = unit_root(n, mulmod(pmod(tau + a.shifts[j0 + jj], n), tm[t], n));
    }
    __syncthreads();
    for (int t = 0; t < tn; ++t) {
      const double2 c = cw[t][lane];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = csub(acc[u], cmul(c, ph[t][wq * 4 + u]));
    }
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = j0 + wq * 4 + u;
    if (jl[u]) a.y[((int64_t)j * a.S + s) * B + b] = acc[u];
  }
}

// measurement of loop shift d*B (d < L) at bucket b (d = 0: y0)
__device__ __forceinline__ double2 sp_val(const IterArgs& a, int s, int64_t d, int b) {
  return a.y[(d * a.S + s) * a.B + b];
}

// _split_search (sfft/reconstruct.py:197-215) with the class sums of
// sub_bucketizer (frameworks.py:524-529): one warp per heavy bucket.
constexpr int kSrNT = 128;
__global__ void __launch_bounds__(kSrNT) k_sp_search(IterArgs a) {
  const int s = blockIdx.y;
  if (!a.active[s]) return;
  const IterState& S = a.st[s];
  const int h = blockIdx.x * (kSrNT / 32) + (threadIdx.x >> 5);
  if (h >= S.nheavy) return;
  const int lane = threadIdx.x & 31;
  const int64_t n = a.n, L = a.L;
  const int b = a.heavy[(int64_t)s * a.B + h];
  const int64_t base = pmod((int64_t)b * L - L / 2, n);
  const double noise = S.floor / 2.0;
  const double twopi = 6.283185307179586;
  int64_t r = 0, scale = 1, depth = 1;
  int ok = 1;
  for (int dg = 0; dg < a.digits; ++dg) {
    const int64_t step = scale * a.branching;
    depth = step;
    const int64_t jstep = L / step;
    const double inv = 1.0 / (double)step;
    double m1 = -1.0, m2 = -1.0;
    int64_t i1 = 0;
    for (int64_t dd = 0; dd < a.branching; ++dd) {
      const int64_t qc = (base + r + dd * scale) % step;
      double2 acc = cmk(0.0, 0.0);
      for (int64_t d = lane; d < step; d += 32) {
        // exp(2j*pi*d*qc/step) formed as numpy forms it
        const double th = ((twopi * (double)d) * (double)qc) * inv;
        double sn, cs;
        sincos(th, &sn, &cs);
        acc = cadd(acc, cmul(sp_val(a, s, d * jstep, b), cmk(cs, sn)));
      }
      for (int o = 16; o; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      const double mg = cabs_scalar(cmk(acc.x * inv, acc.y * inv));
      if (mg > m1) {
        m2 = m1;
        m1 = mg;
        i1 = dd;
      } else if (mg > m2) {
        m2 = mg;
      }
    }
    if (m1 - m2 < noise) {
      ok = 0;
      break;
    }
    r += scale * i1;
    scale = step;
  }
  if (lane == 0) {
    const int64_t i = (int64_t)s * a.B + h;
    a.sp_r[i] = (int32_t)r;
    a.sp_ok[i] = ok;
    a.sp_depth[i] = (int32_t)depth;
  }
}


// ------------------------------------------------------------------ split fold
// The split loop measures shifts d*B for every d < L with one sigma: sample i
// of item d is U[i - d*B], U[u] = x[sigma (u - tau)], so in the fold matrix
// (rows of B) item d reads the same columns d rows higher:
//   folded_d[c] = sum_{r < R_c} taps[c + rB] * U[c + (r - d)B]   (rows in order)
// One CTA owns 32 columns x kFdJ shifts: it gathers the (kFdJ + R - 1) rows of
// its columns once (instead of kFdJ x R gathers), forms the sums from shared
// memory in the reference's row order, and writes the folded slots into y;
// the B-point FFTs then run in place (PROD_LOAD).  The values equal the
// per-item fold bit for bit.
constexpr int kFdNT = 256, kFdC = 32, kFdJ = 64, kFdRmax = 64;

template <typename Tin>
__global__ void __launch_bounds__(kFdNT) k_sp_fold(IterArgs a, const void* __restrict__ xv,
                                                   int64_t xstride,
                                                   const double* __restrict__ taps, int R) {
  extern __shared__ __align__(16) unsigned char fsm[];
  const int s = blockIdx.z;
  if (!a.active[s]) return;
  const int64_t n = a.n, B = a.B, L = a.L, omega = a.omega;
  const int64_t c0 = (int64_t)blockIdx.x * kFdC;
  const int64_t j0 = (int64_t)blockIdx.y * kFdJ;
  if (j0 >= L) return;
  const int64_t j1 = min(L, j0 + kFdJ);
  const int64_t wlo = -(j1 - 1), whi = R - j0;  // rows [wlo, whi)
  const int nrow = (int)(whi - wlo);
  Tin* V = (Tin*)fsm;                                        // [nrow][kFdC]
  double* G = (double*)(fsm + (size_t)(kFdRmax + kFdJ) * kFdC * sizeof(Tin));  // [R][kFdC]
  const int64_t sigma = a.item_sigma[s], tau = a.item_tau[s];
  const Tin* xs = (const Tin*)xv + (int64_t)a.st[s].sig * xstride;
  const int c = threadIdx.x & (kFdC - 1), g = threadIdx.x / kFdC;
  constexpr int NG = kFdNT / kFdC;
  {
    // column c, rows wlo + g, wlo + g + NG, ...: u advances by NG*B
    int64_t u = c0 + c + (wlo + g) * B;
    int64_t idx = mulmod(sigma, pmod(u - tau, n), n);
    const int64_t step = mulmod(sigma, (NG * B) % n, n);
    for (int w = g; w < nrow; w += NG) {
      if (u < omega) V[w * kFdC + c] = __ldcg(xs + idx);
      u += NG * B;
      idx += step;
      idx -= (idx >= n) ? n : 0;
    }
    for (int r = g; r < R; r += NG) {
      const int64_t i = c0 + c + (int64_t)r * B;
      G[r * kFdC + c] = i < omega ? __ldg(taps + i) : 0.0;
    }
  }
  __syncthreads();
  const int64_t col = c0 + c;
  const int Rc = (int)((omega - col + B - 1) / B);  // rows of slot col
  for (int64_t j = j0 + g; j < j1; j += NG) {
    // u row of (r, j) is r - j; shared row index r - j - wlo
    const Tin* v = V + (int)(-j - wlo) * kFdC + c;
    double2 acc = cmk(0.0, 0.0);
    for (int r = 0; r < Rc; ++r) {
      const double gg = G[r * kFdC + c];
      const double2 x = to_d2_(v[r * kFdC]);
      acc = cadd_rn(acc, cmk(__dmul_rn(gg, x.x), __dmul_rn(gg, x.y)));
    }
    a.y[(j * a.S + s) * B + col] = acc;
  }
}

template <typename Tin>
static size_t sp_fold_smem() {
  return (size_t)(kFdRmax + kFdJ) * kFdC * sizeof(Tin) + (size_t)kFdRmax * kFdC * sizeof(double);
}

// Prefix over the heavy order of the shifts measured so far (the reference's
// lazy cache, frameworks.py:470-476 / :538-541): sp_depth[h] becomes the
// largest step any bucket up to h measured.  Logs the iteration's reads.
constexpr int kSckNT = 256;
__global__ void __launch_bounds__(kSckNT) k_sp_prefix(IterArgs a) {
  __shared__ int red[32];
  __shared__ int smax_tot;
  const int s = blockIdx.x;
  if (!a.active[s]) return;
  IterState& S = a.st[s];
  const int nh = S.nheavy;
  const int64_t n = a.n, B = a.B;
  const int per = (nh + kSckNT - 1) / kSckNT;
  const int hb = threadIdx.x * per, he = min(nh, hb + per);
  int32_t* dep = a.sp_depth + (int64_t)s * B;
  const int32_t* okv = a.sp_ok + (int64_t)s * B;
  int lm = 0, lc = 0;
  for (int h = hb; h < he; ++h) {
    lm = max(lm, (int)dep[h]);
    lc += okv[h];
  }
  // exclusive max-scan of the per-thread maxima
  int xm = lm;
  const int ln = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, xm, o);
    if (ln >= o) xm = max(xm, t);
  }
  const int prev = __shfl_up_sync(0xffffffffu, xm, 1);
  if (ln == 31) red[w] = xm;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int i = 0; i < kSckNT / 32; ++i) {
      const int v = red[i];
      red[i] = run;
      run = max(run, v);
    }
    smax_tot = run;
  }
  __syncthreads();
  int pm = ln == 0 ? red[w] : max(red[w], prev);
  for (int h = hb; h < he; ++h) {
    pm = max(pm, (int)dep[h]);
    dep[h] = pm;
  }
  int tot;
  block_exscan<kSckNT>(lc, red, &tot);
  if (threadIdx.x == 0) {
    // reads of this iteration: shifts k*(n/Smax), k < Smax, then 1 and 3
    const int64_t sigma = a.item_sigma[s], tau = a.item_tau[s];
    const int smax = max(1, smax_tot);
    int g = S.ngroups;
    if (g < kMaxGroups) {
      Group& G = a.groups[(int64_t)s * kMaxGroups + g];
      G.kind = 2;
      G.a = sigma;
      G.tau = tau;
      G.cnt = a.omega;
      G.nsh = smax;
      G.sh[0] = n / smax;
      S.ngroups = ++g;
    }
    if (tot > 0 && g < kMaxGroups) {
      Group& G = a.groups[(int64_t)s * kMaxGroups + g];
      G.kind = 0;
      G.a = sigma;
      G.tau = tau;
      G.cnt = a.omega;
      G.nsh = 2;
      G.sh[0] = 1;
      G.sh[1] = 3;
      S.ngroups = ++g;
    }
  }
}

// Consistency checks against the cached shifts k*(n/pm), 1 <= k < pm, and
// 1, 3 (lanes split the shifts, one warp per located bucket), the weight
// check and the estimate y0 * w^{-tau q} / G (frameworks.py:538-554).
constexpr int kVfNT = 128;
__global__ void __launch_bounds__(kVfNT) k_sp_verify(IterArgs a) {
  const int s = blockIdx.y;
  if (!a.active[s]) return;
  const IterState& S = a.st[s];
  const int h = blockIdx.x * (kVfNT / 32) + (threadIdx.x >> 5);
  if (h >= S.nheavy) return;
  const int lane = threadIdx.x & 31;
  const int64_t n = a.n, B = a.B, L = a.L;
  const int64_t fi = (int64_t)s * B + h;
  if (!a.sp_ok[fi]) {
    if (lane == 0) a.f_ok[fi] = 0;
    return;
  }
  const int b = a.heavy[fi];
  const int64_t q = pmod((int64_t)b * L - L / 2 + a.sp_r[fi], n);
  const double2 y0 = sp_val(a, s, 0, b);
  const double tol = fmax(3.0 * S.floor, 0.15 * cabs_scalar(y0));
  const int64_t pm = a.sp_depth[fi];
  const int64_t jst = L / pm, tst = n / pm;
  bool bad = false;
  // shifts k*(n/pm) for 1 <= k < pm (item k*jst), then 1 and 3 (items L, L+1)
  for (int64_t kk = 1 + lane; kk < pm + 2 && !bad; kk += 32) {
    int64_t t, item;
    if (kk < pm) {
      t = kk * tst;
      item = kk * jst;
    } else {
      t = kk == pm ? 1 : 3;
      item = L + (kk - pm);
    }
    const double2 pred = cmul(y0, unit_root(n, mulmod(t % n, q, n)));
    bad = cabs_scalar(csub(sp_val(a, s, item, b), pred)) > tol;
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane != 0) return;
  a.f_ok[fi] = 0;
  if (bad) return;
  const int64_t e = pmod((int64_t)b * L - q, n);
  const double2 gw = a.gt[(e % L) * B + e / L];
  if (cabs_scalar(gw) < 0.05 * a.gmax[0]) return;
  const double2 coeff =
      cdiv(cmul(y0, unit_root(n, pmod(-mulmod(a.item_tau[s], q, n), n))), gw);
  a.f_pos[fi] = mulmod(modinv(a.item_sigma[s], n), q, n);
  a.f_coef[fi] = coeff;
  a.f_ok[fi] = 1;
}

// ------------------------------------------------------------------ merge
constexpr int kMrgNT = 512;

// recovered[f] += c for every tone found now, new positions appended in
// heavy order (dict insertion order, frameworks.py:556-557); lookups through a
// per-signal open-addressing hash of the recovered positions.
__global__ void __launch_bounds__(kMrgNT) k_it_merge(IterArgs a) {
  __shared__ int redi[32];
  const int s = blockIdx.x;
  if (!a.active[s]) return;
  IterState& S = a.st[s];
  const int nh = S.nheavy;
  const int64_t B = a.B;
  const int n_old = a.rec_count[s];
  int64_t* rp = a.rec_pos + (int64_t)s * a.cap;
  double2* rc = a.rec_coef + (int64_t)s * a.cap;
  const int64_t* fp = a.f_pos + (int64_t)s * B;
  const double2* fcf = a.f_coef + (int64_t)s * B;
  const int32_t* fok = a.f_ok + (int64_t)s * B;
  const int per = (nh + kMrgNT - 1) / kMrgNT;
  const int h0 = threadIdx.x * per, h1 = min(nh, h0 + per);
  int nnew = 0, nok = 0;
  for (int h = h0; h < h1; ++h) {
    if (!fok[h]) continue;
    ++nok;
    nnew += ht_find(a, s, fp[h]) < 0;
  }
  int tot_new, tot_ok;
  int off_new = block_exscan<kMrgNT>(nnew, redi, &tot_new);
  int off_ok = block_exscan<kMrgNT>(nok, redi, &tot_ok);
  int64_t* cp = a.fc_pos + (int64_t)s * B;
  double2* cc = a.fc_coef + (int64_t)s * B;
  for (int h = h0; h < h1; ++h) {
    if (!fok[h]) continue;
    cp[off_ok] = fp[h];
    cc[off_ok] = fcf[h];
    ++off_ok;
    const int where = ht_find(a, s, fp[h]);
    if (where >= 0) {
      rc[where] = cadd(rc[where], fcf[h]);
    } else if (n_old + off_new < a.cap) {
      rp[n_old + off_new] = fp[h];
      rc[n_old + off_new] = fcf[h];
      ++off_new;
    }
  }
  __syncthreads();  // all lookups of this iteration precede the inserts
  {
    // insert the appended positions
    const int nrec = min(a.cap, n_old + tot_new);
    for (int t = n_old + threadIdx.x; t < nrec; t += kMrgNT) ht_insert(a, s, rp[t], t);
  }
  if (threadIdx.x == 0) {
    const int nrec = min(a.cap, n_old + tot_new);
    a.rec_count[s] = nrec;
    S.n_rec = nrec;
    S.nfound = tot_ok;
    a.fc_count[s] = tot_ok;
    a.gate[s] = (nrec >= a.k && tot_ok > 0) ? 1 : 0;
    atomicMax(a.stats + 1, nrec);
  }
}

// ------------------------------------------------------------------ residual test
// Residual convergence test, early out (frameworks.py:562-565): the test is
// max_b |y0 - model(found)| < 1.3 floor, so one bucket at or above the bound
// decides "not converged".  The residual at the first kResPre heavy buckets is
// formed exactly as the full pass forms it (the candidate-restricted
// subtraction is bitwise equal at those buckets); a witness clears the slot's
// gate and skips its full-B pass (non-converging signals find a witness at
// once).  Padded entries use bucket 0, whose residual is as valid a witness.
constexpr int kResPre = 32;

__global__ void k_resid_list(IterArgs a, int32_t* plist) {
  const int s = blockIdx.x, i = threadIdx.x;
  if (!a.gate[s] || i >= kResPre) return;
  plist[(int64_t)s * kResPre + i] = i < a.st[s].nheavy ? a.heavy[(int64_t)s * a.B + i] : 0;
}

__global__ void k_resid_pre(IterArgs a, const double2* rpre) {
  const int s = blockIdx.x, i = threadIdx.x;
  if (!a.gate[s]) return;
  const bool witness = i < kResPre &&
                       cabs_(rpre[(int64_t)s * kResPre + i]) >= 1.3 * a.st[s].floor;
  if (__any_sync(0xffffffffu, witness) && i == 0) a.gate[s] = 0;
}

__global__ void __launch_bounds__(kDecNT) k_it_resid(IterArgs a) {
  __shared__ double redd[32];
  const int s = blockIdx.x;
  if (!a.active[s]) return;
  IterState& S = a.st[s];
  const int it = S.it;
  bool conv = false;
  double mx = 0.0;
  if (a.gate[s]) {
    const double2* r = a.resid + (int64_t)s * a.B;
    double m = 0.0;
    for (int64_t i = threadIdx.x; i < a.B; i += kDecNT) m = fmax(m, cabs_(r[i]));
    mx = block_max<kDecNT>(m, redd);
    conv = mx < 1.3 * S.floor;
  }
  if (threadIdx.x == 0) {
    if (conv) {
      S.converged = 1;
      S.final_resid = mx;
      S.iterations = it;
      loop_end(a, S, s);
    } else if (it == a.max_it) {
      S.iterations = it;
      loop_end(a, S, s);
    }
  }
}

// ------------------------------------------------------------------ polish
// Epoch start: every recovered tone pending again (frameworks.py:586).
__global__ void k_po_epoch(IterArgs a) {
  const int s = blockIdx.y;
  const IterState& S = a.st[s];
  if (!a.pgate[s] || S.pass != 0) return;
  const int T = S.n_rec;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x)
    a.pend[(int64_t)s * a.cap + t] = 1;
}

// After a pass: at most 3 passes per epoch, an epoch ends when nothing is
// pending, 2 epochs (frameworks.py:585-589).
__global__ void k_po_after(IterArgs a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S || !a.pgate[s]) return;
  IterState& S = a.st[s];
  S.pass += 1;
  if (S.pending <= 0 || S.pass == 3) {
    S.epoch += 1;
    S.pass = 0;
    if (S.epoch == 2) S.phase = PH_FINISH;
  }
}

constexpr int kPoNT = 128;
constexpr int kPoChunk = 128;

// Occupancy of the buckets of every recovered tone under this pass's
// permutation (frameworks.py:596-598).  occ zeroed by the caller.
__global__ void k_po_occ(IterArgs a, int32_t* occ) {
  const int s = blockIdx.y;
  if (!a.pgate[s]) return;
  const int T = a.rec_count[s];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int64_t n = a.n, L = a.L;
  const int64_t m = mulmod(a.item_sigma[s], pmod(a.rec_pos[(int64_t)s * a.cap + t], n), n);
  atomicAdd(&occ[(int64_t)s * a.B + pmod(m + L / 2, n) / L], 1);
}

// Correction of every pending, non-collided tone with a usable weight:
// mean_t(resid_t[b] * w^{-(tau+t)m}) / w, resid_t = y_t - model(all recovered)
// at the tone's own bucket, with the pre-pass coefficients (frameworks.py:599-608).
__global__ void __launch_bounds__(kPoNT) k_po_delta(IterArgs a, const int32_t* occ,
                                                    int32_t* corr) {
  __shared__ int64_t u_row[kPoChunk], u_q[kPoChunk];
  __shared__ double2 u_c[kPoChunk];
  __shared__ double2 u_ph[kPoChunk][3];
  const int s = blockIdx.y;
  if (!a.pgate[s]) return;
  const int64_t n = a.n, B = a.B, L = a.L;
  const int T = a.rec_count[s];
  const int t = blockIdx.x * kPoNT + threadIdx.x;
  if (blockIdx.x * kPoNT >= T) return;
  const int64_t* rp = a.rec_pos + (int64_t)s * a.cap;
  const double2* rc = a.rec_coef + (int64_t)s * a.cap;
  const int64_t sigma = a.item_sigma[s];
  const int64_t tau = a.item_tau[s];
  bool mine = false;
  int64_t m = 0, bi = 0;
  double2 w = cmk(0.0, 0.0);
  if (t < T && a.pend[(int64_t)s * a.cap + t]) {
    m = mulmod(sigma, pmod(rp[t], n), n);
    bi = pmod(m + L / 2, n) / L;
    if (occ[(int64_t)s * B + bi] == 1) {
      const int64_t e = pmod(bi * L - m, n);
      w = a.gt[(e % L) * B + e / L];
      mine = cabs_scalar(w) >= 0.05 * a.gmax[0];
    }
  }
  if (t < T) corr[(int64_t)s * a.cap + t] = mine;
  double2 r[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) r[d] = mine ? a.y[((int64_t)d * a.S + s) * B + bi] : cmk(0, 0);
  if (a.rt.at) {
    // real form of the response (see k_subtract): c G ph = alpha + w^{b L h} beta A,
    // alpha = c ph t0 / B, beta = c ph w^{-m h} / B; the alpha sums do not
    // depend on the bucket (one warp forms them per chunk), the inner loop
    // reads 8 bytes and does 6 FMA per tone pair
    __shared__ double2 u_be[kPoChunk][3];
    __shared__ double2 u_al[kPoChunk][3];
    __shared__ double2 s_al[3];
    const double t0v = a.rt.taps[0];
    const double invB = 1.0 / (double)B;
    const int64_t hh = a.rt.h % n;
    double2 S3[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) S3[d] = cmk(0.0, 0.0);
    if (threadIdx.x < 3) s_al[threadIdx.x] = cmk(0.0, 0.0);
    for (int u0 = 0; u0 < T; u0 += kPoChunk) {
      __syncthreads();
      for (int q = threadIdx.x; q < kPoChunk; q += kPoNT) {
        if (u0 + q >= T) continue;
        const int64_t mu = mulmod(sigma, pmod(rp[u0 + q], n), n);
        u_row[q] = (L - mu % L) % L;
        u_q[q] = (mu + L - 1) / L;
        const double2 cu = rc[u0 + q];
        const double2 wmh = unit_root(n, pmod(-mulmod(mu, hh, n), n));
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double2 cp = cmul(cu, unit_root(n, mulmod(pmod(tau + d, n), mu, n)));
          u_be[q][d] = cscale(cmul(cp, wmh), invB);
          u_al[q][d] = cscale(cp, t0v * invB);
        }
      }
      __syncthreads();
      const int un = min(kPoChunk, T - u0);
      if (threadIdx.x < 3) {
        double2 z = s_al[threadIdx.x];
        for (int q = 0; q < un; ++q) z = cadd(z, u_al[q][threadIdx.x]);
        s_al[threadIdx.x] = z;
      }
      if (mine) {
        int q = 0;
        for (; q + 8 <= un; q += 8) {
          double w[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            int64_t col = bi - u_q[q + u];
            col += (col < 0) ? B : 0;
            w[u] = __ldg(a.rt.at + u_row[q + u] * B + col);
          }
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
              S3[d].x = fma(u_be[q + u][d].x, w[u], S3[d].x);
              S3[d].y = fma(u_be[q + u][d].y, w[u], S3[d].y);
            }
        }
        for (; q < un; ++q) {
          int64_t col = bi - u_q[q];
          col += (col < 0) ? B : 0;
          const double w1 = __ldg(a.rt.at + u_row[q] * B + col);
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            S3[d].x = fma(u_be[q][d].x, w1, S3[d].x);
            S3[d].y = fma(u_be[q][d].y, w1, S3[d].y);
          }
        }
      }
    }
    __syncthreads();
    if (mine) {
      const double2 pb = unit_root(n, mulmod(mulmod(bi, L, n), hh, n));
#pragma unroll
      for (int d = 0; d < 3; ++d) r[d] = csub(csub(r[d], s_al[d]), cmul(pb, S3[d]));
    }
  } else {
  for (int u0 = 0; u0 < T; u0 += kPoChunk) {
    __syncthreads();
    for (int q = threadIdx.x; q < kPoChunk; q += kPoNT) {
      if (u0 + q >= T) continue;
      const int64_t mu = mulmod(sigma, pmod(rp[u0 + q], n), n);
      u_row[q] = (L - mu % L) % L;
      u_q[q] = (mu + L - 1) / L;
      u_c[q] = rc[u0 + q];
      for (int d = 0; d < 3; ++d) u_ph[q][d] = unit_root(n, mulmod(pmod(tau + d, n), mu, n));
    }
    __syncthreads();
    if (mine) {
      const int un = min(kPoChunk, T - u0);
      int q = 0;
      for (; q + 8 <= un; q += 8) {
        double2 w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          int64_t col = bi - u_q[q + u];
          col += (col < 0) ? B : 0;
          w[u] = ld_table(a.gt + u_row[q + u] * B + col);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const double2 cw = cmul(u_c[q + u], w[u]);
#pragma unroll
          for (int d = 0; d < 3; ++d) r[d] = csub(r[d], cmul(cw, u_ph[q + u][d]));
        }
      }
      for (; q < un; ++q) {
        int64_t col = bi - u_q[q];
        col += (col < 0) ? B : 0;
        const double2 cw = cmul(u_c[q], ld_table(a.gt + u_row[q] * B + col));
#pragma unroll
        for (int d = 0; d < 3; ++d) r[d] = csub(r[d], cmul(cw, u_ph[q][d]));
      }
    }
  }
  }
  if (mine) {
    double2 acc = cmk(0.0, 0.0);
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int64_t ex = pmod(-mulmod(pmod(tau + d, n), m, n), n);
      acc = cadd(acc, cmul(r[d], unit_root(n, ex)));
    }
    a.delta[(int64_t)s * a.cap + t] = cdiv(cdivr(acc, 3.0), w);
  }
}

// Apply after every residual has been formed with the pre-pass coefficients.
__global__ void k_po_apply(IterArgs a, const int32_t* corr) {
  __shared__ int cnt;
  const int s = blockIdx.y;
  if (!a.pgate[s]) return;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const int T = a.rec_count[s];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T && corr[(int64_t)s * a.cap + t]) {
    const int64_t i = (int64_t)s * a.cap + t;
    a.rec_coef[i] = cadd(a.rec_coef[i], a.delta[i]);
    a.pend[i] = 0;
    atomicAdd(&cnt, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0 && cnt) atomicSub(&a.st[s].pending, cnt);
}

// ------------------------------------------------------------------ host driver

struct IterLayout {
  size_t off[64];
  size_t total;
};

static size_t al(size_t x) { return (x + 255) & ~size_t(255); }

constexpr int kMaxSubSplit = 16;   // tone splits of the full-B subtraction
constexpr int kMaxLadSplit = 8;    // tone splits of the ladder model

// cached rows per slot: the next loop permutation's M shifts and kSpecPolish x 3
// polish shifts (phase-location ladders only, M <= 13)
constexpr int kSpecPolish = SFFT_SPEC_POLISH;
static int spec_rows(int M) { return M <= 13 ? M + 3 * kSpecPolish : 0; }

static int ht_size(int cap) {
  int h = 1;
  while (h < 2 * cap) h <<= 1;
  return h;
}

static IterLayout iter_layout(int64_t n, int64_t B, int S, int M, int cap) {
  IterLayout L{};
  size_t o = 0;
  const size_t HT = (size_t)ht_size(cap);
  const size_t part = std::max((size_t)kMaxSubSplit * B, (size_t)kMaxLadSplit * B * (M - 1));
  size_t sizes[] = {
      sizeof(IterState) * S,                 // 0 st
      sizeof(int32_t) * S,                   // 1 active
      sizeof(int32_t) * S,                   // 2 gate
      sizeof(int32_t) * 8,                   // 3 stats
      sizeof(int32_t) * M * S,               // 4 item_sig
      sizeof(int64_t) * M * S * 2,           // 5 item_sigma_it + item_sigma
      sizeof(int64_t) * M * S * 2,           // 6 item_tau_it + item_tau
      sizeof(double2) * (size_t)(M + spec_rows(M)) * S * B,  // 7 y (working rows + row cache)
      sizeof(double2) * (size_t)S * B,       // 8 resid
      sizeof(int64_t) * (size_t)S * cap,     // 9 rec_pos
      sizeof(double2) * (size_t)S * cap,     // 10 rec_coef
      sizeof(int32_t) * S,                   // 11 rec_count
      sizeof(int32_t) * (size_t)S * B,       // 12 heavy
      sizeof(int64_t) * (size_t)S * B,       // 13 f_pos
      sizeof(double2) * (size_t)S * B,       // 14 f_coef
      sizeof(int32_t) * (size_t)S * B,       // 15 f_ok
      sizeof(int64_t) * (size_t)S * B,       // 16 fc_pos
      sizeof(double2) * (size_t)S * B,       // 17 fc_coef
      sizeof(int32_t) * S,                   // 18 fc_count
      sizeof(int32_t) * (size_t)S * cap,     // 19 pend
      sizeof(double2) * (size_t)S * cap,     // 20 delta
      sizeof(Group) * (size_t)S * kMaxGroups,// 21 groups
      sizeof(int32_t) * 2 * S,               // 22 fin + rows
      sizeof(int32_t) * S,                   // 23 ngroups copy
      sizeof(int64_t) * (size_t)S * HT,      // 24 ht_key
      sizeof(int32_t) * (size_t)S * HT,      // 25 ht_val
      sizeof(double2) * (size_t)S * part,    // 26 part
      sizeof(int32_t) * (size_t)S * B,       // 27 occ (polish)
      sizeof(int32_t) * (size_t)S * cap,     // 28 corr (polish)
      sizeof(int32_t) * (size_t)S * M,       // 29 item_active
      sizeof(int32_t) * (size_t)S,           // 30 pgate
      sizeof(int32_t) * 2 * (size_t)S,       // 31 union-count fallback gate
      sizeof(int32_t) * (size_t)S * B,       // 32 heavy_b
      sizeof(int32_t) * (size_t)S * B,       // 33 hrank
      sizeof(int64_t) * (size_t)M,           // 34 loop shift of each item
      sizeof(int32_t) * (size_t)S * B * 3,   // 35 split search r / ok / depth
      sizeof(int32_t) * (size_t)S * M,       // 36 item_fold
      sizeof(double) * (size_t)n,            // 37 real response table
      sizeof(int32_t) * (size_t)S * spec_rows(M),               // 38 dir_p
      sizeof(int64_t) * (size_t)S * spec_rows(M),               // 39 dir_d
      sizeof(int32_t) * (size_t)S * M,                          // 40 role_src
      sizeof(int32_t) * (size_t)(S + 1),                        // 41 cnt
      sizeof(int32_t) * (size_t)S * (M + spec_rows(M)) * 2,     // 42 it2_sig + it2_row
      sizeof(int64_t) * (size_t)S * (M + spec_rows(M)) * 2,     // 43 it2_sigma + it2_tau
      sizeof(double2) * (size_t)S * kResPre,                    // 44 residual pre-check values
      sizeof(int32_t) * (size_t)S * kResPre,                    // 45 residual pre-check buckets
      sizeof(int32_t) * (size_t)(S + 1),                        // 46 rcnt
      sizeof(int32_t) * (size_t)S * (M + spec_rows(M)) * 2,     // 47 run_first + run_cnt
      flat_groups_desc_bytes((int64_t)S * (M + spec_rows(M))),  // 48 group descriptors
      sizeof(int32_t) * (size_t)S,                              // 49 act_list
      sizeof(SchedMemo) + sizeof(int32_t) * 2 * (size_t)S,       // 50 samples_read memo, own/ent
      sizeof(int32_t) * (5 * (size_t)S + 8),                     // 51 dcnt + dense (streamed slots)
      stream_fold_taps_bytes(B, M + spec_rows(M)),               // 52 stream fold tap table
  };
  const int cnt = sizeof(sizes) / sizeof(sizes[0]);
  static_assert(sizeof(sizes) / sizeof(sizes[0]) <= sizeof(L.off) / sizeof(L.off[0]),
                "IterLayout::off too small");
  for (int i = 0; i < cnt; ++i) {
    L.off[i] = o;
    o += al(sizes[i]);
  }
  L.total = o;
  return L;
}

size_t iterative_ws_bytes(int64_t n, int64_t B, int S, int M, int cap) {
  return iter_layout(n, B, S, M, cap).total +
         bucketize_ws_bytes(B, (int64_t)(M + spec_rows(M)) * S);
}

template <int M>
static int launch_locate_t(const IterArgs& a, int64_t B, int S, int lts, cudaStream_t st) {
  if (S <= 0) return 0;  // no loop slot this round
  if (lts) {
    dim3 gp((unsigned)cdiv_up(B, kLocNT), S, lts);
    k_it_ladder_part<M><<<gp, kLocNT, 0, st>>>(a);
    SFFT_CHECK_LAUNCH("k_it_ladder_part");
  }
  dim3 gl((unsigned)cdiv_up(B, kLocNT), S);
  k_it_locate<M><<<gl, kLocNT, 0, st>>>(a, lts);
  SFFT_CHECK_LAUNCH("k_it_locate");
  return 0;
}

// ladder lengths 1..12 (M = 2..13); _phase_ladder(N) has ~log8(N/16)+1 rungs
static int launch_locate(const IterArgs& a, int M, int64_t B, int S, int lts, cudaStream_t st) {
  switch (M) {
    case 2: return launch_locate_t<2>(a, B, S, lts, st);
    case 3: return launch_locate_t<3>(a, B, S, lts, st);
    case 4: return launch_locate_t<4>(a, B, S, lts, st);
    case 5: return launch_locate_t<5>(a, B, S, lts, st);
    case 6: return launch_locate_t<6>(a, B, S, lts, st);
    case 7: return launch_locate_t<7>(a, B, S, lts, st);
    case 8: return launch_locate_t<8>(a, B, S, lts, st);
    case 9: return launch_locate_t<9>(a, B, S, lts, st);
    case 10: return launch_locate_t<10>(a, B, S, lts, st);
    case 11: return launch_locate_t<11>(a, B, S, lts, st);
    case 12: return launch_locate_t<12>(a, B, S, lts, st);
    case 13: return launch_locate_t<13>(a, B, S, lts, st);
    default: set_error("iterative: phase ladder length outside 1..12"); return -2;
  }
}

static int splits(int T, int per, int mx) {
  const int z = (T + per - 1) / per;
  return z < 1 ? 1 : (z > mx ? mx : z);
}

__global__ void k_cb_finish(IterArgs a, int32_t* fin, int32_t* rows, int32_t* ngroups,
                            int32_t* out_iters, int32_t* out_conv) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  const IterState& S = a.st[s];
  const bool f = S.phase == PH_FINISH;
  fin[s] = f;
  rows[s] = S.sig;
  ngroups[s] = S.ngroups;
  if (f) {
    out_iters[S.sig] = S.iterations;
    out_conv[S.sig] = S.converged;
  }
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long h, unsigned long long v,
                                                    unsigned long long m) {
  h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  h *= m;
  return h ^ (h >> 31);
}

// own[s]: 1 = compute, 0 = not finishing / memo hit; ent[s]: memo entry (-1 none)
__global__ void k_memo_lookup(const Group* __restrict__ groups, const int32_t* ngroups,
                              const int32_t* fin, const int32_t* rows, SchedMemo* memo,
                              int64_t* samples, int32_t* own, int32_t* ent, int S) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  own[s] = 0;
  ent[s] = -1;
  if (!fin[s]) return;
  const int G = min(ngroups[s], kMaxGroups);
  const Group* gs = groups + (int64_t)s * kMaxGroups;
  unsigned long long h1 = 0x243F6A8885A308D3ull ^ (unsigned long long)G;
  unsigned long long h2 = 0x13198A2E03707344ull + (unsigned long long)G;
  for (int g = 0; g < G; ++g) {
    const Group& q = gs[g];
    const unsigned long long f[5] = {(unsigned long long)q.a, (unsigned long long)q.tau,
                                     (unsigned long long)q.cnt, (unsigned long long)q.kind,
                                     (unsigned long long)q.nsh};
    for (int i = 0; i < 5; ++i) {
      h1 = mix64(h1, f[i], 0xBF58476D1CE4E5B9ull);
      h2 = mix64(h2, f[i], 0x94D049BB133111EBull);
    }
    const int ns = q.kind == 2 ? 1 : min(q.nsh, kMaxShifts);
    for (int i = 0; i < ns; ++i) {
      h1 = mix64(h1, (unsigned long long)q.sh[i], 0xBF58476D1CE4E5B9ull);
      h2 = mix64(h2, (unsigned long long)q.sh[i], 0x94D049BB133111EBull);
    }
  }
  if (h1 == 0) h1 = 1;
  uint32_t e = (uint32_t)(h1 >> 17) & (kMemo - 1);
  for (int probe = 0; probe < kMemo; ++probe, e = (e + 1) & (kMemo - 1)) {
    const unsigned long long old = atomicCAS(&memo->k1[e], 0ull, h1);
    if (old == 0ull) {  // new key: this slot computes
      memo->k2[e] = h2;
      own[s] = 1;
      ent[s] = (int)e;
      return;
    }
    if (old == h1) {
      // the same schedule (k2 is written right after the claim of k1; a slot
      // that cannot confirm it this round computes on its own)
      const unsigned long long o2 = *(volatile unsigned long long*)&memo->k2[e];
      if (o2 != h2) break;
      if (*(volatile int32_t*)&memo->ready[e]) {
        samples[rows[s]] = memo->count[e];
      } else {
        ent[s] = (int)e;  // same round as its owner: copied after the count
      }
      return;
    }
  }
  own[s] = 1;  // table full or unconfirmed key: compute without the memo
}

// after the exclusion count: owners publish, then same-round followers copy
__global__ void k_memo_publish(const int32_t* own, const int32_t* ent, const int32_t* rows,
                               SchedMemo* memo, const int64_t* samples, int S) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S || !own[s] || ent[s] < 0) return;
  memo->count[ent[s]] = samples[rows[s]];
  __threadfence();
  memo->ready[ent[s]] = 1;
}

__global__ void k_memo_copy(const int32_t* fin, const int32_t* own, const int32_t* ent,
                            const int32_t* rows, const SchedMemo* memo, int64_t* samples, int S) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S || !fin[s] || own[s] || ent[s] < 0) return;
  samples[rows[s]] = memo->count[ent[s]];
}

__global__ void k_cb_release(IterArgs a) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= a.S) return;
  IterState& S = a.st[s];
  if (S.phase != PH_FINISH) return;
  S.phase = PH_FREE;
  atomicAdd(a.stats + 3, 1);
}

int run_iterative(int dtype, const void* x, int64_t n, int64_t xstride, int Q, int S,
                  const double* taps, int64_t omega, int64_t B, const double2* gt,
                  const double* gmax, const double2* W, const int64_t* psig, const int64_t* ptau,
                  int P, int64_t pstride, int64_t k, int max_it, const int64_t* ladder, int nlad,
                  int loc, int branching, int cap, int64_t* out_pos, double2* out_coef,
                  int32_t* out_n, int32_t* out_iters, int32_t* out_conv, int64_t* out_samples,
                  int64_t* out_sched, const int32_t* avail, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  SFFT_REQUIRE(loc == 0 || loc == 1, "iterative: location must be 0 (phase) or 1 (split)");
  const int64_t Lw = B > 0 ? n / B : 0;
  int digits = 0;
  if (loc == 1) {
    SFFT_REQUIRE(B >= 4 && n % B == 0, "iterative: split location needs 4 <= B, B | n");
    SFFT_REQUIRE(branching >= 2, "iterative: branching must be >= 2");
    int64_t p = 1;
    while (p < Lw) {
      p *= branching;
      ++digits;
    }
    SFFT_REQUIRE(p == Lw, "iterative: bucket width is not a power of the branching factor");
    SFFT_REQUIRE(2 * max_it + 7 <= kMaxGroups, "iterative: max_iterations too large");
  }
  const int M = loc == 1 ? (int)Lw + 2 : 1 + nlad;
  SFFT_REQUIRE(loc == 1 || M <= kMaxShifts, "iterative: ladder too long");
  SFFT_REQUIRE(max_it + 7 <= kMaxGroups, "iterative: max_iterations too large");
  SFFT_REQUIRE(P >= max_it + 6, "iterative: need max_iterations + 6 permutations");
  SFFT_REQUIRE(k <= kFusedMaxB, "iterative: k must be <= 8192");
  SFFT_REQUIRE(S >= 1 && Q >= 1, "iterative: need slots and signals");
  SFFT_REQUIRE(ws_bytes >= iterative_ws_bytes(n, B, S, M, cap), "iterative: workspace too small");
  const IterLayout Lo = iter_layout(n, B, S, M, cap);
  char* w = (char*)ws;
  IterArgs a{};
  a.n = n;
  a.B = B;
  a.L = n / B;
  a.omega = omega;
  a.k = k;
  a.S = S;
  a.Q = Q;
  a.avail = avail;
  a.P = P;
  a.pstride = pstride;
  a.M = M;
  a.max_it = max_it;
  a.cap = cap;
  a.loc = loc;
  a.branching = branching;
  a.digits = digits;
  if (loc == 0)
    for (int j = 0; j < nlad; ++j) a.ladder[j] = ladder[j];
  a.psig = psig;
  a.ptau = ptau;
  a.gt = gt;
  a.gmax = gmax;
  a.st = (IterState*)(w + Lo.off[0]);
  a.active = (int32_t*)(w + Lo.off[1]);
  a.gate = (int32_t*)(w + Lo.off[2]);
  a.stats = (int32_t*)(w + Lo.off[3]);
  a.n_active = a.stats;
  a.item_sig = (int32_t*)(w + Lo.off[4]);
  a.item_sigma_it = (int64_t*)(w + Lo.off[5]);
  a.item_sigma = a.item_sigma_it + (size_t)M * S;
  a.item_tau_it = (int64_t*)(w + Lo.off[6]);
  a.item_tau = a.item_tau_it + (size_t)M * S;
  a.y = (double2*)(w + Lo.off[7]);
  a.resid = (double2*)(w + Lo.off[8]);
  a.rec_pos = (int64_t*)(w + Lo.off[9]);
  a.rec_coef = (double2*)(w + Lo.off[10]);
  a.rec_count = (int32_t*)(w + Lo.off[11]);
  a.heavy = (int32_t*)(w + Lo.off[12]);
  a.f_pos = (int64_t*)(w + Lo.off[13]);
  a.f_coef = (double2*)(w + Lo.off[14]);
  a.f_ok = (int32_t*)(w + Lo.off[15]);
  a.fc_pos = (int64_t*)(w + Lo.off[16]);
  a.fc_coef = (double2*)(w + Lo.off[17]);
  a.fc_count = (int32_t*)(w + Lo.off[18]);
  a.pend = (int32_t*)(w + Lo.off[19]);
  a.delta = (double2*)(w + Lo.off[20]);
  a.groups = (Group*)(w + Lo.off[21]);
  int32_t* fin = (int32_t*)(w + Lo.off[22]);
  int32_t* rows = fin + S;
  int32_t* ngroups = (int32_t*)(w + Lo.off[23]);
  a.HT = ht_size(cap);
  a.ht_key = (int64_t*)(w + Lo.off[24]);
  a.ht_val = (int32_t*)(w + Lo.off[25]);
  a.part = (double2*)(w + Lo.off[26]);
  int32_t* occ = (int32_t*)(w + Lo.off[27]);
  int32_t* corr = (int32_t*)(w + Lo.off[28]);
  a.item_active = (int32_t*)(w + Lo.off[29]);
  a.pgate = (int32_t*)(w + Lo.off[30]);
  a.heavy_b = (int32_t*)(w + Lo.off[32]);
  a.hrank = (int32_t*)(w + Lo.off[33]);
  int64_t* shifts = (int64_t*)(w + Lo.off[34]);
  a.shifts = shifts;
  a.sp_r = (int32_t*)(w + Lo.off[35]);
  a.sp_ok = a.sp_r + (size_t)S * B;
  a.sp_depth = a.sp_ok + (size_t)S * B;
  a.item_fold = (int32_t*)(w + Lo.off[36]);
  // the row cache pays where the gathers dominate (C3: Omega = 76,848) and
  // enough slots fill the GPU; small windows and small batches are latency-
  // bound and keep the per-round items
  // (SFFT_ROW_CACHE=1 forces it on, SFFT_NO_ROW_CACHE=1 off: parity tests run both)
  const bool rc_on = getenv("SFFT_ROW_CACHE") ? atoi(getenv("SFFT_ROW_CACHE")) != 0
                                              : (omega >= 32768 && S >= 512);
  a.C = (loc == 0 && rc_on && !getenv("SFFT_NO_ROW_CACHE")) ? spec_rows(M) : 0;
  a.dir_p = (int32_t*)(w + Lo.off[38]);
  a.dir_d = (int64_t*)(w + Lo.off[39]);
  a.role_src = (int32_t*)(w + Lo.off[40]);
  a.cnt = (int32_t*)(w + Lo.off[41]);
  a.it2_sig = (int32_t*)(w + Lo.off[42]);
  a.it2_row = a.it2_sig + (size_t)S * (M + spec_rows(M));
  a.it2_sigma = (int64_t*)(w + Lo.off[43]);
  a.it2_tau = a.it2_sigma + (size_t)S * (M + spec_rows(M));
  a.rcnt = (int32_t*)(w + Lo.off[46]);
  a.act_list = (int32_t*)(w + Lo.off[49]);
  a.dcnt = (int32_t*)(w + Lo.off[51]);
  a.dense = a.dcnt + ((S + 1 + 3) / 4) * 4;  // 16-byte aligned descriptors
  // SFFT_STREAM_FOLD=1: first-round slots on the stream fold (measured slower
  // than the group fold, so opt-in; the parity tests run both)
  a.stream = (getenv("SFFT_STREAM_FOLD") && atoi(getenv("SFFT_STREAM_FOLD"))) &&
             !(getenv("SFFT_RUN_FOLD") && !atoi(getenv("SFFT_RUN_FOLD"))) &&
             pstride == 0 &&  // one shared permutation stream: first-round slots run the same items
             stream_fold_ok(dtype, x, xstride, n, B, omega);
  SchedMemo* memo = (SchedMemo*)(w + Lo.off[50]);
  int32_t* m_own = (int32_t*)(memo + 1);
  int32_t* m_ent = m_own + S;
  const bool memo_off = getenv("SFFT_NO_SCHED_MEMO") && atoi(getenv("SFFT_NO_SCHED_MEMO"));
  a.run_first = (int32_t*)(w + Lo.off[47]);
  a.run_cnt = a.run_first + (size_t)S * (M + spec_rows(M));
  double2* rpre = (double2*)(w + Lo.off[44]);
  int32_t* rlist = (int32_t*)(w + Lo.off[45]);
  RealTab rt{};
  if (real_table_ok(omega)) {
    rt.at = (const double*)(w + Lo.off[37]);
    rt.taps = taps;
    rt.h = omega / 2;
    int rc0 = build_real_table(gt, taps, n, B, omega, (double*)(w + Lo.off[37]), st);
    if (rc0) return rc0;
  }
  a.rt = rt;
  void* bws = w + Lo.total;
  {
    // loop shifts: phase {0} + ladder; split {d*B : d < L} + {1, 3}
    std::vector<int64_t> sh(M);
    if (loc == 0) {
      sh[0] = 0;
      for (int j = 1; j < M; ++j) sh[j] = ladder[j - 1];
    } else {
      for (int64_t d = 0; d < Lw; ++d) sh[d] = d * B;
      sh[Lw] = 1;
      sh[Lw + 1] = 3;
    }
    SFFT_CUDA(cudaMemcpyAsync(shifts, sh.data(), sizeof(int64_t) * M, cudaMemcpyHostToDevice, st));
    SFFT_CUDA(cudaStreamSynchronize(st));  // sh is a host temporary
  }
  const size_t bws_bytes = bucketize_ws_bytes(B, (int64_t)(M + spec_rows(M)) * S);

  // all slots free; queue counter 0
  SFFT_CUDA(cudaMemsetAsync(a.st, 0, sizeof(IterState) * S, st));
  SFFT_CUDA(cudaMemsetAsync(a.stats, 0, sizeof(int32_t) * 8, st));
  SFFT_CUDA(cudaMemsetAsync(a.rec_count, 0, sizeof(int32_t) * S, st));
  SFFT_CUDA(cudaMemsetAsync(memo, 0, sizeof(SchedMemo), st));

  Prod p{};
  p.x = x;
  p.xstride = xstride;
  p.n = n;
  p.taps = taps;
  p.omega = omega;
  p.B = B;
  p.item_sig = a.item_sig;
  p.item_a = a.item_sigma_it;
  p.item_b = a.item_tau_it;
  p.item_active = a.item_active;
  p.out_M = M;
  p.out_S = S;

  // split location: row-correlation fold when a CTA can hold its rows
  const int fold_R = (loc == 1 && B % kFdC == 0 && cdiv_up(omega, B) <= kFdRmax &&
                      !getenv("SFFT_NO_SPLIT_FOLD"))
                         ? (int)cdiv_up(omega, B)
                         : 0;
  a.use_fold = fold_R > 0;
  // compacted item list of the row-cache planner (k_cb_fill)
  Prod pc = p;
  pc.item_sig = a.it2_sig;
  pc.item_a = a.it2_sigma;
  pc.item_b = a.it2_tau;
  pc.item_active = nullptr;
  pc.item_row = a.it2_row;
  pc.out_M = 0;
  Prod pl = p;
  pl.z = a.y;
  pl.item_active = a.item_fold;
  if (fold_R > 0) {
    SFFT_CUDA(cudaFuncSetAttribute(k_sp_fold<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sp_fold_smem<float2>()));
    SFFT_CUDA(cudaFuncSetAttribute(k_sp_fold<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sp_fold_smem<double2>()));
  }

  const size_t dsm = (size_t)kFusedMaxB * (8 + 8 + 4);
  SFFT_CUDA(cudaFuncSetAttribute(k_it_decide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
  SFFT_CUDA(cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));

  const unsigned sb = (unsigned)cdiv_up(S, 128);
  int t_max = 0;  // largest recovered list seen (host copy, refreshed every round)
  int h_max = 0;  // largest heavy list seen
  // streaming admission may spend rounds waiting for data: no round cap then
  const int max_rounds = avail ? (1 << 30) : (Q / S + 2) * (max_it + 8) + 16;
  int round = 0;
  // Round prologue (admission, the step of every slot's state machine, item
  // planning).  It runs at the end of the previous round, so that the host
  // reads the next round's item count with the round's one status read.
  auto prologue = [&]() -> int {
    k_cb_admit<<<1, kAdmNT, 0, st>>>(a);
    SFFT_CHECK_LAUNCH("k_cb_admit");
    k_cb_clear<<<dim3(16, S), 256, 0, st>>>(a);
    SFFT_CHECK_LAUNCH("k_cb_clear");
    k_cb_step<<<sb, 128, 0, st>>>(a);
    SFFT_CHECK_LAUNCH("k_cb_step");
    k_act_list<<<1, kAdmNT, 0, st>>>(a);
    SFFT_CHECK_LAUNCH("k_act_list");
    k_po_epoch<<<dim3(4, S), 256, 0, st>>>(a);
    SFFT_CHECK_LAUNCH("k_po_epoch");
    if (a.C > 0) {
      k_cb_plan<<<sb, 128, 0, st>>>(a);
      SFFT_CHECK_LAUNCH("k_cb_plan");
      k_cb_scan<<<1, 1024, 0, st>>>(a);
      SFFT_CHECK_LAUNCH("k_cb_scan");
      k_cb_fill<<<sb, 128, 0, st>>>(a);
      SFFT_CHECK_LAUNCH("k_cb_fill");
    } else {
      k_cb_items<<<(unsigned)cdiv_up((int64_t)M * S, 256), 256, 0, st>>>(a);
      SFFT_CHECK_LAUNCH("k_cb_items");
    }
    return 0;
  };
  int nit = 0;  // planned items of the coming round (row-cache path)
  int nrun = 0;  // their permutation runs (slots on the group fold)
  int ndense = 0;  // slots on the stream fold
  int n_act = S;  // loop slots of the coming round (k_act_list)
  // item-group fold (one gather per sample of a permutation window, the
  // measurements of a slot's permutations folded from shared memory, then the
  // row FFTs): c64/c128 flat items with b' = 0 on the row-cache path.
  // SFFT_RUN_FOLD=0 keeps the per-item cluster kernel (A/B measurements;
  // the parity tests run both)
  const bool run_fold_off = getenv("SFFT_RUN_FOLD") && !atoi(getenv("SFFT_RUN_FOLD"));
  {
    int rc0 = prologue();
    if (rc0) return rc0;
    if (a.C > 0) {
    }
    {
      int32_t h8[8];
      SFFT_CUDA(cudaMemcpyAsync(h8, a.stats, sizeof(h8), cudaMemcpyDeviceToHost, st));
      SFFT_CUDA(cudaStreamSynchronize(st));
      if (a.C > 0) {
        nit = h8[5];
        nrun = h8[6];
        ndense = h8[0];
      }
      n_act = h8[7];
    }
  }
  for (; round < max_rounds; ++round) {
    int rc = 0;
    if (a.C > 0) {
      k_cb_copy<<<(unsigned)(S * M), 256, 0, st>>>(a);
      SFFT_CHECK_LAUNCH("k_cb_copy");
      if (nit > 0 && !run_fold_off)
        rc = run_flat_groups(dtype, pc, a.run_first, a.run_cnt, nrun, nit, W, a.y, bws,
                             bws_bytes, w + Lo.off[48], st, a.dense, ndense, w + Lo.off[52],
                             M + spec_rows(M));
      else if (nit > 0)
        rc = run_bucketize(dtype, PROD_FLAT, pc, nit, W, a.y, bws, bws_bytes, st);
    } else {
      rc = run_bucketize(dtype, PROD_FLAT, p, (int64_t)M * S, W, a.y, bws, bws_bytes, st);
    }
    if (rc) return rc;
    if (fold_R > 0) {
      // split loop shifts d*B: row-correlation fold, then the FFTs in place
      dim3 gf((unsigned)(B / kFdC), (unsigned)cdiv_up(Lw, kFdJ), S);
      if (dtype == 0)
        k_sp_fold<float2><<<gf, kFdNT, sp_fold_smem<float2>(), st>>>(a, x, xstride, taps, fold_R);
      else
        k_sp_fold<double2><<<gf, kFdNT, sp_fold_smem<double2>(), st>>>(a, x, xstride, taps, fold_R);
      SFFT_CHECK_LAUNCH("k_sp_fold");
      rc = run_bucketize(dtype, PROD_LOAD, pl, (int64_t)M * S, W, a.y, bws, bws_bytes, st);
      if (rc) return rc;
    }
    // ---- loop slots
    rc = run_subtract_gated(a.y, a.y, B, B, nullptr, S, gt, n, nullptr, a.item_sigma,
                            a.item_tau, a.rec_pos, a.rec_coef, a.rec_count, cap, a.active, st,
                            splits(t_max, 128, kMaxSubSplit), a.part, &rt, a.act_list, n_act);
    if (rc) return rc;
    k_it_decide<<<S, kDecNT, dsm, st>>>(a);
    SFFT_CHECK_LAUNCH("k_it_decide");
    if (loc == 0) {
      const int lts = t_max > 256 ? splits(t_max, 256, kMaxLadSplit) : 0;
      rc = launch_locate(a, M, B, n_act, lts, st);
      if (rc) return rc;
    } else {
      const unsigned hb = (unsigned)cdiv_up(B, kSpH);
      k_sp_model<<<dim3(hb, (unsigned)cdiv_up(M - 1, kSpJ), S), kSpNT, 0, st>>>(a);
      SFFT_CHECK_LAUNCH("k_sp_model");
      k_sp_search<<<dim3((unsigned)cdiv_up(B, kSrNT / 32), S), kSrNT, 0, st>>>(a);
      SFFT_CHECK_LAUNCH("k_sp_search");
      k_sp_prefix<<<S, kSckNT, 0, st>>>(a);
      SFFT_CHECK_LAUNCH("k_sp_prefix");
      k_sp_verify<<<dim3((unsigned)cdiv_up(B, kVfNT / 32), S), kVfNT, 0, st>>>(a);
      SFFT_CHECK_LAUNCH("k_sp_verify");
    }
    k_it_merge<<<S, kMrgNT, 0, st>>>(a);
    SFFT_CHECK_LAUNCH("k_it_merge");
    if (loc == 0) {
      k_resid_list<<<S, 32, 0, st>>>(a, rlist);
      SFFT_CHECK_LAUNCH("k_resid_list");
      rc = run_subtract_gated(a.y, rpre, B, kResPre, rlist, S, gt, n, nullptr, a.item_sigma,
                              a.item_tau, a.fc_pos, a.fc_coef, a.fc_count, B, a.gate, st,
                              splits(h_max, 128, kMaxSubSplit), a.part, &rt, a.act_list, n_act);
      if (rc) return rc;
      k_resid_pre<<<S, 32, 0, st>>>(a, rpre);
      SFFT_CHECK_LAUNCH("k_resid_pre");
    }
    rc = run_subtract_gated(a.y, a.resid, B, B, nullptr, S, gt, n, nullptr, a.item_sigma,
                            a.item_tau, a.fc_pos, a.fc_coef, a.fc_count, B, a.gate, st,
                            splits(h_max, 128, kMaxSubSplit), a.part, &rt, a.act_list, n_act);
    if (rc) return rc;
    k_it_resid<<<S, kDecNT, 0, st>>>(a);
    SFFT_CHECK_LAUNCH("k_it_resid");
    // ---- polish slots
    SFFT_CUDA(cudaMemsetAsync(occ, 0, sizeof(int32_t) * (size_t)S * B, st));
    const unsigned tb = (unsigned)std::max<int64_t>(1, cdiv_up(t_max, 256));
    k_po_occ<<<dim3(tb, S), 256, 0, st>>>(a, occ);
    SFFT_CHECK_LAUNCH("k_po_occ");
    const unsigned td = (unsigned)std::max<int64_t>(1, cdiv_up(t_max, kPoNT));
    k_po_delta<<<dim3(td, S), kPoNT, 0, st>>>(a, occ, corr);
    SFFT_CHECK_LAUNCH("k_po_delta");
    k_po_apply<<<dim3(tb, S), 256, 0, st>>>(a, corr);
    SFFT_CHECK_LAUNCH("k_po_apply");
    k_po_after<<<sb, 128, 0, st>>>(a);
    SFFT_CHECK_LAUNCH("k_po_after");
    // ---- finished slots: results to their signal's row, then free the slot
    k_cb_finish<<<sb, 128, 0, st>>>(a, fin, rows, ngroups, out_iters, out_conv);
    SFFT_CHECK_LAUNCH("k_cb_finish");
    k_finalize<<<S, kFinNT, dsm, st>>>(a.rec_pos, a.rec_coef, a.rec_count, cap, k, out_pos,
                                        out_coef, out_n, fin, rows);
    SFFT_CHECK_LAUNCH("k_finalize");
    // samples_read: memo hits take the count of an identical schedule; the
    // first slot of each schedule computes it (SFFT_NO_SCHED_MEMO=1: all compute)
    if (!memo_off) {
      k_memo_lookup<<<sb, 128, 0, st>>>(a.groups, ngroups, fin, rows, memo, out_samples, m_own,
                                        m_ent, S);
      SFFT_CHECK_LAUNCH("k_memo_lookup");
    }
    rc = run_union_count(a.groups, ngroups, S, n, out_samples, memo_off ? fin : m_own, rows, st,
                         (int32_t*)(w + Lo.off[31]));
    if (rc) return rc;
    if (!memo_off) {
      k_memo_publish<<<sb, 128, 0, st>>>(m_own, m_ent, rows, memo, out_samples, S);
      SFFT_CHECK_LAUNCH("k_memo_publish");
      k_memo_copy<<<sb, 128, 0, st>>>(fin, m_own, m_ent, rows, memo, out_samples, S);
      SFFT_CHECK_LAUNCH("k_memo_copy");
    }
    if (out_sched) {
      k_export_groups<<<S, 64, 0, st>>>(a.groups, ngroups, S, out_sched, fin, rows);
      SFFT_CHECK_LAUNCH("k_export_groups");
    }
    k_cb_release<<<sb, 128, 0, st>>>(a);
    SFFT_CHECK_LAUNCH("k_cb_release");
    rc = prologue();
    if (rc) return rc;
    int32_t hs[8];
    SFFT_CUDA(cudaMemcpyAsync(hs, a.stats, sizeof(hs), cudaMemcpyDeviceToHost, st));
    SFFT_CUDA(cudaStreamSynchronize(st));
    t_max = hs[1];
    h_max = hs[2];
    nit = hs[5];
    nrun = hs[6];
    ndense = hs[0];
    n_act = hs[7];
    if (hs[3] >= Q) break;
  }
  SFFT_REQUIRE(round < max_rounds, "iterative: round limit reached (internal error)");
  return 0;
}

}  // namespace sfft
