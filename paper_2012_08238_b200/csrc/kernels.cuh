// Host-side launchers shared by the .cu translation units.
#pragma once

#include <algorithm>
#include <mutex>
#include <vector>

#include "fft.cuh"

namespace sfft {

enum ProdMode { PROD_FLAT = 0, PROD_SPIKE = 1, PROD_GTAB = 2, PROD_LOAD = 3, PROD_DIRICHLET = 4 };

struct Prod {
  const void* x;             // [nsig][xstride] float2 (c64) or double2 (c128)
  int64_t xstride;
  int64_t n;
  const double* taps;        // real taps [omega]
  int64_t omega;
  int64_t B;
  const int32_t* item_sig;   // item -> signal (null: item == signal)
  const int64_t* item_a;     // flat: sigma | spike: tau | gtab: rho
  const int64_t* item_b;     // flat: tau_tot
  const int64_t* item_c;     // flat: b'*sigma mod n (null: 0)
  const int32_t* active;     // per-signal gate (null: all active)
  const int32_t* item_active;  // per-item gate (null: all)
  const double2* z;          // PROD_LOAD source [nitems][B]
  unsigned long long* prof_items;  // profiling: count of non-skipped items (null: off)
  const double2* ctaps;      // Dirichlet: complex box taps [omega] (omega = L)
  int half_offset;           // Dirichlet: 1 = rounding boundaries (no half-bucket modulation)
  int out_M;                 // > 0: item i writes output row (i % out_M) * out_S + i / out_M
  int64_t out_S;             //      (items ordered signal-major, rows shift-major)
  const int32_t* item_row;   // non-null: item i writes output row item_row[i] (takes precedence)
};

__host__ __device__ __forceinline__ int64_t out_row(const Prod& p, int64_t item) {
  if (p.item_row) return p.item_row[item];
  return p.out_M > 0 ? (item % p.out_M) * p.out_S + item / p.out_M : item;
}

// Profiling of the bucketization (gather-fold-FFT) launches: CUDA events on
// the launching stream around every launch, items counted on the device.
struct BucketProf {
  bool on = false;
  unsigned long long* d_items = nullptr;  // device counter
  double ms = 0.0;
  long long launches = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;  // read at prof_collect
  std::mutex mu;
};
BucketProf& bucket_prof();
int prof_collect();
int prof_begin(cudaStream_t st, cudaEvent_t* ev0);
int prof_end(cudaStream_t st, cudaEvent_t ev0);


size_t bucketize_ws_bytes(int64_t B, int64_t nitems);
int run_bucketize(int dtype, int mode, const Prod& p, int64_t nitems, const double2* W,
                  double2* out, void* ws, size_t ws_bytes, cudaStream_t st);
int run_twiddle(double2* W, int64_t B, cudaStream_t st);
constexpr int kGfItems = 8;  // items per group of the group fold (one warp each per column half)

// item groups of flat items (iterative ladder / polish permutations of one
// slot): one gather per sample of a window, then the FFTs in place (bucketize.cu)
size_t flat_groups_desc_bytes(int64_t ngroups);  // scratch for the per-group descriptors
// dense/ndense: slots folded by the stream fold instead (descriptor i =
// {slot, first item, items, signal}, 16 bytes each; none of their items is in
// a group); stream_fold_ok says whether a problem qualifies
int run_flat_groups(int dtype, const Prod& p, const int32_t* gfirst, const int32_t* gcnt,
                    int64_t ngroups, int64_t nitems, const double2* W, double2* out, void* ws,
                    size_t ws_bytes, void* desc_ws, cudaStream_t st,
                    const int32_t* dense = nullptr, int64_t ndense = 0,
                    void* taps_ws = nullptr, int max_items = 0);
// scratch for the stream fold's permuted tap table (max_items items per slot)
size_t stream_fold_taps_bytes(int64_t B, int64_t nitems);
bool stream_fold_ok(int dtype, const void* x, int64_t xstride, int64_t n, int64_t B,
                    int64_t omega);
// Dirichlet bank (sfft/bucketize.py:181-211): per-offset transforms y [noff][B]
// (forward FFT of the conjugated fold / B) combined into out [B]
int run_dirichlet_combine(const double2* y, int64_t noff, const int64_t* offsets, int64_t n,
                          int64_t L, int64_t B, int half_offset, int64_t center_offset,
                          double2* out, cudaStream_t st);
int run_freqshift(int dtype, const void* x, int64_t n, const int64_t* idx, int64_t count,
                  int64_t f, double2* partial, double2* out, cudaStream_t st);
int run_flat_taps(double* taps, int64_t omega, int64_t B, double gsig, cudaStream_t st);
int run_absmax(const double2* v, int64_t count, double* out, cudaStream_t st);

int run_mark(uint8_t* map, int64_t n, int kind, int64_t a, int64_t b, int64_t c,
             const int64_t* idx, cudaStream_t st);
int run_count_nonzero(const uint8_t* map, int64_t n, int64_t* out, cudaStream_t st);

// decode.cu
int run_floor(const double2* values, int64_t nsets, int64_t B, double mult,
              const int32_t* item_sig, const int32_t* active, double* floor_out, double* peak_out,
              cudaStream_t st);
// floor + heavy bitmap of each set in one kernel (|v| bits cached in shared memory)
int run_floor_heavy(const double2* values, int64_t nsets, int64_t B, double mult, int64_t hc,
                    double* floor_out, uint32_t* bits, int32_t* nheavy, cudaStream_t st);
int run_heavy_bitmap(const double2* values, int64_t nsets, int64_t B, const double* thr,
                     int64_t hc, const int32_t* item_sig, const int32_t* active, uint32_t* bits,
                     int32_t* nheavy, cudaStream_t st);
// Most rounds a vote count covers (scores are stored in 8 bits per position).
constexpr int kMaxVoteRounds = 255;

struct VoteRounds {
  const uint32_t* bits;   // [S][R][words]
  const int64_t* sigma;   // [S*R]
  const int64_t* bprime;  // [S*R] (null: 0)
  int64_t n, B, L, words, cs;
  int R;
  int bits_global;        // 1: the bitmaps are read from global memory (too big for
                          // shared memory); set by the launchers
};
// Runner fast path: candidates (score >= need) of every signal in (-score, pos)
// order, first keep, without materialising per-position scores.  Returns 1 in
// *overflow_host when a signal has more than the sort capacity of candidates
// (the caller then uses run_votes).
size_t votes_fast_ws_bytes(int S, int R, int64_t hc);
int run_votes_fast(const VoteRounds& vr, int S, int need, int keep, int64_t hc, int64_t* cand,
                   int32_t* ncand, void* ws, size_t ws_bytes, int* overflow_host,
                   cudaStream_t st);
int run_votes(const VoteRounds& vr, int S, const int64_t* counts_in, int64_t* counts_out,
              int need, int keep, int64_t* cand, int32_t* ncand, int* chist, bool emit,
              cudaStream_t st);
size_t votes_ws_bytes(int64_t n, int S, int R);
// vote_tally over bucket sets of any kind / width / centre shift (stage API)
int run_vote_tally(int64_t n, int R, const int64_t* Bs, const int64_t* boff, const uint32_t* bits,
                   const int64_t* sigma, const int64_t* bprime, const int32_t* kind,
                   const int64_t* cs, int64_t* counts, cudaStream_t st);
int run_trimmed_mean(const double2* est, int R, int64_t C, double2* out, cudaStream_t st);
int run_energy_est(const double2* y, int64_t B, const double2* gt, const double* gmax, int64_t n,
                   int R, const int64_t* sigma, const int64_t* tau, const int64_t* cand,
                   int64_t C, double2* est, cudaStream_t st);
int run_subtract(const double2* y, double2* out, int64_t B, int64_t nb, const int32_t* blist,
                 int64_t nitems, const double2* gt, int64_t n, const int32_t* item_sig,
                 const int64_t* sigma, const int64_t* tau_tot, const int64_t* tpos,
                 const double2* tcoef, const int32_t* tcount, int64_t tstride, cudaStream_t st);

// Real-table form of the flat response (even support Omega, taps symmetric
// about h = Omega/2): G_f = (t0 + w^{f h} A_f) / B with A real, so a tone's
// model at bucket b is (c ph)(t0/B) + w^{b L h} [(c ph w^{-m h} / B) A_{bL-m}]:
// half the table bytes and half the multiplies of the complex form.
struct RealTab {
  const double* at;   // [L][B] A in the transposed layout of the complex table
  const double* taps; // taps[0] = t0
  int64_t h;          // Omega / 2
};
int build_real_table(const double2* gt, const double* taps, int64_t n, int64_t B, int64_t omega,
                     double* at, cudaStream_t st);
bool real_table_ok(int64_t omega);

int run_subtract_gated(const double2* y, double2* out, int64_t B, int64_t nb,
                       const int32_t* blist, int64_t nitems, const double2* gt, int64_t n,
                       const int32_t* item_sig, const int64_t* sigma, const int64_t* tau_tot,
                       const int64_t* tpos, const double2* tcoef, const int32_t* tcount,
                       int64_t tstride, const int32_t* gate, cudaStream_t st, int TS = 1,
                       double2* part = nullptr, const RealTab* rt = nullptr,
                       const int32_t* list = nullptr, int64_t nlist = -1);

// voting.cu
size_t voting_ws_bytes(int64_t n, int64_t B, int S, int R, int C, int64_t Bpre);
int run_voting(int dtype, const void* x, int64_t n, int64_t xstride, int S, const double* taps,
               int64_t omega, int64_t B, const double2* gt, const double* gmax, const double2* W,
               const int64_t* psig, const int64_t* ptau, int R, int64_t k, int need,
               int64_t Bpre, const double2* Wpre, int64_t* out_pos, double2* out_coef,
               int32_t* out_n, int64_t* out_samples, int64_t* out_sched, void* ws,
               size_t ws_bytes, cudaStream_t st);

// peeling.cu
size_t peeling_ws_bytes(int64_t n, int S, const int64_t* factors, int nst, int64_t k);
int run_peeling(int dtype, const void* x, int64_t n, int64_t xstride, int S,
                const int64_t* factors, int nst, const double2* const* Wst, int64_t k,
                int64_t* out_pos, double2* out_coef, int32_t* out_n, int32_t* out_iters,
                int32_t* out_conv, int32_t* out_err, int64_t* out_samples, int64_t* out_sched,
                void* ws, size_t ws_bytes, cudaStream_t st);

// oneshot.cu
size_t oneshot_ws_bytes(int64_t n, int S, int64_t B, int A, int nsh);
int run_oneshot(int dtype, const void* x, int64_t n, int64_t xstride, int S, int64_t B, int A,
                const int64_t* shifts_host, int nsh, const int64_t* ladder_host, int nlad,
                const double2* W, int64_t k, int64_t* out_pos, double2* out_coef,
                int32_t* out_n, int32_t* out_iters, int32_t* out_conv, int64_t* out_samples,
                int64_t* out_sched, void* ws, size_t ws_bytes, cudaStream_t st);

// iterative.cu
size_t iterative_ws_bytes(int64_t n, int64_t B, int S, int M, int cap);
int run_iterative(int dtype, const void* x, int64_t n, int64_t xstride, int Q, int S,
                  const double* taps, int64_t omega, int64_t B, const double2* gt,
                  const double* gmax, const double2* W, const int64_t* psig, const int64_t* ptau,
                  int P, int64_t pstride, int64_t k, int max_it, const int64_t* ladder, int nlad,
                  int loc, int branching, int cap, int64_t* out_pos, double2* out_coef,
                  int32_t* out_n, int32_t* out_iters, int32_t* out_conv, int64_t* out_samples,
                  int64_t* out_sched, const int32_t* avail, void* ws, size_t ws_bytes,
                  cudaStream_t st);

}  // namespace sfft
