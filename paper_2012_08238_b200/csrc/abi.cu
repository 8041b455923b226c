// extern "C" boundary of libsfft_b200.so (declared in include/sfft_b200.h).
//
// Plain pointers and sizes only; every device buffer is caller-owned; every
// call is asynchronous on the given stream and returns 0 or a negative code
// (-1 bad argument, -2 unsupported / workspace too small, -3 CUDA error) with
// the message in sfft_last_error().
#include <string>

#include "kernels.cuh"
#include "schedule.cuh"

#include <atomic>

namespace sfft {
static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace sfft

using namespace sfft;

#define SFFT_API extern "C" __attribute__((visibility("default")))

SFFT_API int sfft_version(void) { return 1; }

// Number of kernels this library has launched in this process.
SFFT_API int64_t sfft_launch_count(void) { return g_launches.load(); }

// Bucketization profiling: CUDA events recorded on the launching stream around
// every flat/spike bucketization launch (no synchronisation; the events are
// read by sfft_prof_read) and a device count of the items each launch
// actually processed.
SFFT_API int sfft_prof_enable(int on) {
  BucketProf& p = bucket_prof();
  if (on && !p.d_items) SFFT_CUDA(cudaMalloc(&p.d_items, sizeof(unsigned long long)));
  if (p.d_items) SFFT_CUDA(cudaMemset(p.d_items, 0, sizeof(unsigned long long)));
  if (int rc = prof_collect()) return rc;
  p.on = on != 0;
  p.ms = 0.0;
  p.launches = 0;
  return 0;
}

SFFT_API int sfft_prof_read(double* ms, int64_t* launches, int64_t* items) {
  BucketProf& p = bucket_prof();
  if (int rc = prof_collect()) return rc;
  unsigned long long it = 0;
  if (p.d_items) SFFT_CUDA(cudaMemcpy(&it, p.d_items, sizeof(it), cudaMemcpyDeviceToHost));
  *ms = p.ms;
  *launches = p.launches;
  *items = (int64_t)it;
  return 0;
}

// Layout of the optional read-schedule export of the runners.
SFFT_API int sfft_schedule_layout(int32_t* max_groups, int32_t* words_per_group) {
  *max_groups = kMaxGroups;
  *words_per_group = kSchedWords;
  return 0;
}

SFFT_API const char* sfft_last_error(void) { return last_error(); }

SFFT_API int sfft_twiddles(void* W, int64_t B, void* stream) {
  SFFT_REQUIRE(W && B > 0, "sfft_twiddles: bad argument");
  return run_twiddle((double2*)W, B, (cudaStream_t)stream);
}

SFFT_API int sfft_flat_taps(double* taps, int64_t omega, int64_t B, double gauss_sigma,
                            void* stream) {
  SFFT_REQUIRE(taps && omega > 0 && B > 0 && gauss_sigma > 0, "sfft_flat_taps: bad argument");
  return run_flat_taps(taps, omega, B, gauss_sigma, (cudaStream_t)stream);
}

SFFT_API size_t sfft_bucketize_ws_bytes(int64_t B, int64_t nitems) {
  return bucketize_ws_bytes(B, nitems);
}

// Response table T[rho][j] = G[rho + j*L] (L = n/B rows of B) and max|G|.
SFFT_API int sfft_build_gtable(const double* taps, int64_t omega, int64_t n, int64_t B,
                               const void* W, void* gtable, double* gmax, const int64_t* rows,
                               void* ws, size_t ws_bytes, void* stream) {
  SFFT_REQUIRE(taps && gtable && W && rows && n > 0 && B > 0 && n % B == 0,
               "sfft_build_gtable: bad argument");
  Prod p{};
  p.n = n;
  p.taps = taps;
  p.omega = omega;
  p.B = B;
  p.item_a = rows;  // rho = rows[item] (0..L-1)
  const int64_t L = n / B;
  int rc = run_bucketize(1, PROD_GTAB, p, L, (const double2*)W, (double2*)gtable, ws, ws_bytes,
                         (cudaStream_t)stream);
  if (rc) return rc;
  if (gmax) return run_absmax((const double2*)gtable, n, gmax, (cudaStream_t)stream);
  return 0;
}

// Batched flat bucketization: item i reads signal item_sig[i] (row of x with
// stride xstride elements) under (sigma[i], tau_tot[i], bsig[i]).
SFFT_API int sfft_flat_bucketize(int dtype, const void* x, int64_t n, int64_t xstride,
                                 const double* taps, int64_t omega, int64_t B, int64_t nitems,
                                 const int32_t* item_sig, const int64_t* sigma,
                                 const int64_t* tau_tot, const int64_t* bsig,
                                 const int32_t* active, const void* W, void* out, void* ws,
                                 size_t ws_bytes, void* stream) {
  SFFT_REQUIRE(dtype == 0 || dtype == 1, "sfft_flat_bucketize: dtype must be 0 (c64) or 1 (c128)");
  SFFT_REQUIRE(x && taps && sigma && tau_tot && W && out, "sfft_flat_bucketize: null pointer");
  SFFT_REQUIRE(n > 0 && B > 0 && n % B == 0 && omega > 0 && omega <= n && nitems >= 0,
               "sfft_flat_bucketize: bad sizes");
  SFFT_REQUIRE(n < (int64_t(1) << 31), "sfft_flat_bucketize: n must be < 2^31");
  Prod p{};
  p.x = x;
  p.xstride = xstride;
  p.n = n;
  p.taps = taps;
  p.omega = omega;
  p.B = B;
  p.item_sig = item_sig;
  p.item_a = sigma;
  p.item_b = tau_tot;
  p.item_c = bsig;
  p.active = active;
  return run_bucketize(dtype, PROD_FLAT, p, nitems, (const double2*)W, (double2*)out, ws,
                       ws_bytes, (cudaStream_t)stream);
}

// Batched spike-train bucketization: item i reads x[(n/B)*j - tau[i] mod n].
SFFT_API int sfft_spike_bucketize(int dtype, const void* x, int64_t n, int64_t xstride,
                                  int64_t B, int64_t nitems, const int32_t* item_sig,
                                  const int64_t* tau, const int32_t* active, const void* W,
                                  void* out, void* ws, size_t ws_bytes, void* stream) {
  SFFT_REQUIRE(dtype == 0 || dtype == 1, "sfft_spike_bucketize: dtype must be 0 or 1");
  SFFT_REQUIRE(x && tau && W && out, "sfft_spike_bucketize: null pointer");
  SFFT_REQUIRE(n > 0 && B > 0 && n % B == 0 && nitems >= 0, "sfft_spike_bucketize: bad sizes");
  SFFT_REQUIRE(n < (int64_t(1) << 31), "sfft_spike_bucketize: n must be < 2^31");
  Prod p{};
  p.x = x;
  p.xstride = xstride;
  p.n = n;
  p.B = B;
  p.item_sig = item_sig;
  p.item_a = tau;
  p.active = active;
  return run_bucketize(dtype, PROD_SPIKE, p, nitems, (const double2*)W, (double2*)out, ws,
                       ws_bytes, (cudaStream_t)stream);
}

// Dirichlet bank bucketization (sfft/bucketize.py:181-211).
SFFT_API size_t sfft_dirichlet_ws_bytes(int64_t B, int64_t noffsets) {
  return (size_t)noffsets * (size_t)B * sizeof(double2) + bucketize_ws_bytes(B, noffsets) + 256;
}

SFFT_API int sfft_dirichlet_bucketize(int dtype, const void* x, int64_t n, const void* taps,
                                      int64_t L, int64_t B, int32_t half_offset,
                                      int64_t center_offset, int64_t noffsets,
                                      const int64_t* offsets, const void* W, void* out, void* ws,
                                      size_t ws_bytes, void* stream) {
  SFFT_REQUIRE(dtype == 0 || dtype == 1, "sfft_dirichlet_bucketize: dtype must be 0 or 1");
  SFFT_REQUIRE(x && taps && offsets && W && out && ws, "sfft_dirichlet_bucketize: null pointer");
  SFFT_REQUIRE(n > 0 && B > 0 && L > 0 && L * B == n && noffsets >= 1,
               "sfft_dirichlet_bucketize: need L*B == n and at least one offset");
  SFFT_REQUIRE(n < (int64_t(1) << 31), "sfft_dirichlet_bucketize: n must be < 2^31");
  SFFT_REQUIRE(ws_bytes >= sfft_dirichlet_ws_bytes(B, noffsets),
               "sfft_dirichlet_bucketize: workspace too small");
  double2* y = (double2*)ws;
  char* bws = (char*)ws + (((size_t)noffsets * B * sizeof(double2) + 255) & ~size_t(255));
  Prod p{};
  p.x = x;
  p.xstride = 0;  // every item (offset) reads the one signal
  p.n = n;
  p.B = B;
  p.omega = L;
  p.ctaps = (const double2*)taps;
  p.half_offset = half_offset ? 1 : 0;
  p.item_a = offsets;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = run_bucketize(dtype, PROD_DIRICHLET, p, noffsets, (const double2*)W, y, bws,
                         bucketize_ws_bytes(B, noffsets), st);
  if (rc) return rc;
  return run_dirichlet_combine(y, noffsets, offsets, n, L, B, half_offset ? 1 : 0,
                               center_offset, (double2*)out, st);
}

// estimate_freqshift (sfft/reconstruct.py:356-371): mean of x[idx] w^{f idx}.
SFFT_API int sfft_freqshift_estimate(int dtype, const void* x, int64_t n, const int64_t* idx,
                                     int64_t count, int64_t f, void* out, void* ws,
                                     size_t ws_bytes, void* stream) {
  SFFT_REQUIRE(dtype == 0 || dtype == 1, "sfft_freqshift_estimate: dtype must be 0 or 1");
  SFFT_REQUIRE(x && idx && out && ws, "sfft_freqshift_estimate: null pointer");
  SFFT_REQUIRE(n > 0 && count >= 1, "sfft_freqshift_estimate: need n > 0 and count >= 1");
  SFFT_REQUIRE(ws_bytes >= 256 * sizeof(double2), "sfft_freqshift_estimate: workspace too small");
  return run_freqshift(dtype, x, n, idx, count, f, (double2*)ws, (double2*)out,
                       (cudaStream_t)stream);
}

// Mark one read schedule into a byte map (kind 0 flat: a=sigma b=tau_tot
// c=omega; 1 spike: a=stride b=tau c=count; 2 all; 3 list: idx[c]).
SFFT_API int sfft_access_mark(uint8_t* map, int64_t n, int kind, int64_t a, int64_t b,
                              int64_t c, const int64_t* idx, void* stream) {
  SFFT_REQUIRE(map && n > 0 && kind >= 0 && kind <= 3, "sfft_access_mark: bad argument");
  SFFT_REQUIRE(kind != 3 || idx, "sfft_access_mark: list kind needs indices");
  return run_mark(map, n, kind, a, b, c, idx, (cudaStream_t)stream);
}

SFFT_API int sfft_count_nonzero(const uint8_t* map, int64_t n, int64_t* out, void* stream) {
  SFFT_REQUIRE(map && out && n >= 0, "sfft_count_nonzero: bad argument");
  return run_count_nonzero(map, n, out, (cudaStream_t)stream);
}

// ---- decode stages --------------------------------------------------------

SFFT_API int sfft_noise_floor(const void* values, int64_t nsets, int64_t B, double median_mult,
                              double* floor_out, double* peak_out, void* stream) {
  SFFT_REQUIRE(values && floor_out && B > 0 && nsets >= 0, "sfft_noise_floor: bad argument");
  return run_floor((const double2*)values, nsets, B, median_mult, nullptr, nullptr, floor_out,
                   peak_out, (cudaStream_t)stream);
}

SFFT_API int sfft_heavy_bitmap(const void* values, int64_t nsets, int64_t B, const double* thr,
                               int64_t heavy_count, uint32_t* bits, int32_t* nheavy,
                               void* stream) {
  SFFT_REQUIRE(values && thr && bits && B > 0 && nsets >= 0 && heavy_count >= 0,
               "sfft_heavy_bitmap: bad argument");
  return run_heavy_bitmap((const double2*)values, nsets, B, thr, heavy_count, nullptr, nullptr,
                          bits, nheavy, (cudaStream_t)stream);
}

SFFT_API size_t sfft_votes_ws_bytes(int64_t n, int64_t nsig, int64_t rounds) {
  return votes_ws_bytes(n, (int)nsig, (int)rounds);
}

SFFT_API int sfft_vote_select(int64_t n, int64_t B, int64_t rounds, int64_t nsig,
                              const uint32_t* bits, const int64_t* sigma, const int64_t* bprime,
                              int64_t center_shift, const int64_t* counts_in, int64_t* counts_out,
                              int64_t need, int64_t keep, int64_t* cand, int32_t* ncand,
                              void* ws, size_t ws_bytes, void* stream) {
  SFFT_REQUIRE(n > 0 && B > 0 && n % B == 0 && rounds >= 0 && rounds <= kMaxVoteRounds && nsig >= 1,
               "sfft_vote_select: bad sizes");
  SFFT_REQUIRE(counts_in || (bits && sigma), "sfft_vote_select: need counts or bitmaps");
  SFFT_REQUIRE(need >= 1, "sfft_vote_select: need >= 1");
  SFFT_REQUIRE(!cand || (ncand && keep > 0), "sfft_vote_select: cand needs ncand and keep > 0");
  SFFT_REQUIRE(ws && ws_bytes >= votes_ws_bytes(n, (int)nsig, (int)rounds),
               "sfft_vote_select: workspace too small");
  VoteRounds vr{};
  vr.bits = bits;
  vr.sigma = sigma;
  vr.bprime = bprime;
  vr.n = n;
  vr.B = B;
  vr.L = n / B;
  vr.words = (B + 31) / 32;
  vr.cs = center_shift;
  vr.R = (int)rounds;
  return run_votes(vr, (int)nsig, counts_in, counts_out, (int)need, (int)keep, cand, ncand,
                   (int*)ws, cand != nullptr, (cudaStream_t)stream);
}

SFFT_API int sfft_vote_tally(int64_t n, int64_t rounds, const int64_t* nbuckets,
                             const int64_t* bit_offset, const uint32_t* bits,
                             const int64_t* sigma, const int64_t* bprime, const int32_t* kind,
                             const int64_t* center_shift, int64_t* counts, void* stream) {
  SFFT_REQUIRE(n > 0 && rounds >= 0 && rounds <= (1 << 30), "sfft_vote_tally: bad sizes");
  SFFT_REQUIRE(counts && (rounds == 0 || (nbuckets && bit_offset && bits && sigma)),
               "sfft_vote_tally: null pointer");
  return run_vote_tally(n, (int)rounds, nbuckets, bit_offset, bits, sigma, bprime, kind,
                        center_shift, counts, (cudaStream_t)stream);
}

SFFT_API int sfft_energy_estimates(const void* y, int64_t B, const void* gtable,
                                   const double* gmax, int64_t n, int64_t rounds,
                                   const int64_t* sigma, const int64_t* tau, const int64_t* cand,
                                   int64_t ncand, void* est, void* stream) {
  SFFT_REQUIRE(y && gtable && gmax && sigma && tau && est && n % B == 0,
               "sfft_energy_estimates: bad argument");
  SFFT_REQUIRE(ncand == 0 || cand, "sfft_energy_estimates: null candidates");
  return run_energy_est((const double2*)y, B, (const double2*)gtable, gmax, n, (int)rounds,
                        sigma, tau, cand, ncand, (double2*)est, (cudaStream_t)stream);
}

SFFT_API int sfft_trimmed_mean(const void* est, int64_t rounds, int64_t ncand, void* out,
                               void* stream) {
  SFFT_REQUIRE(est && out, "sfft_trimmed_mean: null pointer");
  return run_trimmed_mean((const double2*)est, (int)rounds, ncand, (double2*)out,
                          (cudaStream_t)stream);
}

SFFT_API int sfft_subtract_flat(const void* y, void* out, int64_t B, int64_t nb,
                                const int32_t* blist, int64_t nitems, const void* gtable,
                                int64_t n, const int32_t* item_sig, const int64_t* sigma,
                                const int64_t* tau_tot, const int64_t* tone_pos,
                                const void* tone_coef, const int32_t* tone_count,
                                int64_t tone_stride, void* stream) {
  SFFT_REQUIRE(y && out && gtable && sigma && tau_tot && tone_count && n % B == 0,
               "sfft_subtract_flat: bad argument");
  SFFT_REQUIRE(nb == B || blist, "sfft_subtract_flat: partial bucket lists need blist");
  return run_subtract((const double2*)y, (double2*)out, B, nb, blist, nitems,
                      (const double2*)gtable, n, item_sig, sigma, tau_tot, tone_pos,
                      (const double2*)tone_coef, tone_count, tone_stride, (cudaStream_t)stream);
}

// ---- runners ---------------------------------------------------------------

SFFT_API size_t sfft_iterative_ws_bytes(int64_t n, int64_t B, int64_t nsig, int64_t nshifts,
                                        int64_t cap) {
  return iterative_ws_bytes(n, B, (int)nsig, (int)nshifts, (int)cap);
}

SFFT_API int sfft_run_iterative(int dtype, const void* x, int64_t n, int64_t xstride,
                                int64_t nsig, int64_t nslots, const double* taps, int64_t omega,
                                int64_t B, const void* gtable, const double* gmax, const void* W,
                                const int64_t* perm_sigma, const int64_t* perm_tau, int64_t nperm,
                                int64_t perm_stride, int64_t k, int64_t max_iterations,
                                const int64_t* ladder_host, int64_t nladder, int32_t location,
                                int32_t branching, int64_t cap,
                                int64_t* out_pos, void* out_coef, int32_t* out_count,
                                int32_t* out_iterations, int32_t* out_converged,
                                int64_t* out_samples, int64_t* out_sched,
                                const int32_t* avail, void* ws, size_t ws_bytes, void* stream) {
  SFFT_REQUIRE(dtype == 0 || dtype == 1, "sfft_run_iterative: dtype must be 0 or 1");
  SFFT_REQUIRE(x && taps && gtable && gmax && W && perm_sigma && perm_tau &&
                   (ladder_host || location == 1),
               "sfft_run_iterative: null pointer");
  SFFT_REQUIRE(n > 0 && B > 0 && n % B == 0 && nsig >= 1 && nslots >= 1 && k >= 1 &&
                   max_iterations >= 1, "sfft_run_iterative: bad sizes");
  SFFT_REQUIRE(n < (int64_t(1) << 31), "sfft_run_iterative: n must be < 2^31");
  SFFT_REQUIRE(out_pos && out_coef && out_count && out_iterations && out_converged && out_samples,
               "sfft_run_iterative: null output");
  return run_iterative(dtype, x, n, xstride, (int)nsig, (int)std::min(nslots, nsig), taps, omega,
                       B, (const double2*)gtable, gmax, (const double2*)W, perm_sigma, perm_tau,
                       (int)nperm, perm_stride, k, (int)max_iterations, ladder_host,
                       (int)nladder, (int)location, (int)branching, (int)cap, out_pos,
                       (double2*)out_coef, out_count,
                       out_iterations, out_converged, out_samples, out_sched, avail, ws,
                       ws_bytes, (cudaStream_t)stream);
}

SFFT_API size_t sfft_voting_ws_bytes(int64_t n, int64_t B, int64_t nsig, int64_t rounds,
                                     int64_t k, int64_t prestage_buckets) {
  return voting_ws_bytes(n, B, (int)nsig, (int)rounds, (int)(2 * k), prestage_buckets);
}

SFFT_API int sfft_run_voting(int dtype, const void* x, int64_t n, int64_t xstride, int64_t nsig,
                             const double* taps, int64_t omega, int64_t B, const void* gtable,
                             const double* gmax, const void* W, const int64_t* perm_sigma,
                             const int64_t* perm_tau, int64_t rounds, int64_t k,
                             int64_t need_votes, int64_t prestage_buckets, const void* W_pre,
                             int64_t* out_pos, void* out_coef, int32_t* out_count,
                             int64_t* out_samples, int64_t* out_sched, void* ws, size_t ws_bytes,
                             void* stream) {
  SFFT_REQUIRE(dtype == 0 || dtype == 1, "sfft_run_voting: dtype must be 0 or 1");
  SFFT_REQUIRE(x && taps && gtable && gmax && W && perm_sigma && perm_tau,
               "sfft_run_voting: null pointer");
  SFFT_REQUIRE(n > 0 && B > 0 && n % B == 0 && nsig >= 1 && k >= 1 && need_votes >= 1,
               "sfft_run_voting: bad sizes");
  SFFT_REQUIRE(n < (int64_t(1) << 31), "sfft_run_voting: n must be < 2^31");
  SFFT_REQUIRE(prestage_buckets == 0 || (n % prestage_buckets == 0 && W_pre),
               "sfft_run_voting: pre-stage buckets must divide n (and need twiddles)");
  SFFT_REQUIRE(out_pos && out_coef && out_count && out_samples, "sfft_run_voting: null output");
  return run_voting(dtype, x, n, xstride, (int)nsig, taps, omega, B, (const double2*)gtable,
                    gmax, (const double2*)W, perm_sigma, perm_tau, (int)rounds, k,
                    (int)need_votes, prestage_buckets, (const double2*)W_pre, out_pos,
                    (double2*)out_coef, out_count, out_samples, out_sched, ws, ws_bytes,
                    (cudaStream_t)stream);
}

SFFT_API size_t sfft_peeling_ws_bytes(int64_t n, int64_t nsig, const int64_t* factors_host,
                                      int64_t nfactors, int64_t k) {
  return peeling_ws_bytes(n, (int)nsig, factors_host, (int)nfactors, k);
}

SFFT_API int sfft_run_peeling(int dtype, const void* x, int64_t n, int64_t xstride, int64_t nsig,
                              const int64_t* factors_host, int64_t nfactors,
                              const void* const* W_stages_host, int64_t k, int64_t* out_pos,
                              void* out_coef, int32_t* out_count, int32_t* out_iterations,
                              int32_t* out_converged, int32_t* out_error, int64_t* out_samples,
                              int64_t* out_sched, void* ws, size_t ws_bytes, void* stream) {
  SFFT_REQUIRE(dtype == 0 || dtype == 1, "sfft_run_peeling: dtype must be 0 or 1");
  SFFT_REQUIRE(x && factors_host && W_stages_host && nfactors >= 1 && k >= 1 && nsig >= 1,
               "sfft_run_peeling: bad argument");
  SFFT_REQUIRE(n > 0 && n < (int64_t(1) << 31), "sfft_run_peeling: n must be in (0, 2^31)");
  int64_t prod = 1;
  for (int64_t j = 0; j < nfactors; ++j) {
    SFFT_REQUIRE(factors_host[j] > 1 && n % factors_host[j] == 0,
                 "sfft_run_peeling: factors must be > 1 and divide n");
    prod *= factors_host[j];
  }
  SFFT_REQUIRE(prod == n, "sfft_run_peeling: factors must multiply to n");
  SFFT_REQUIRE(out_pos && out_coef && out_count && out_iterations && out_converged && out_error &&
               out_samples, "sfft_run_peeling: null output");
  return run_peeling(dtype, x, n, xstride, (int)nsig, factors_host, (int)nfactors,
                     (const double2* const*)W_stages_host, k, out_pos, (double2*)out_coef,
                     out_count, out_iterations, out_converged, out_error, out_samples, out_sched,
                     ws, ws_bytes, (cudaStream_t)stream);
}

SFFT_API size_t sfft_oneshot_ws_bytes(int64_t n, int64_t nsig, int64_t B, int64_t a_max,
                                      int64_t nshifts) {
  return oneshot_ws_bytes(n, (int)nsig, B, (int)a_max, (int)nshifts);
}

SFFT_API int sfft_run_oneshot(int dtype, const void* x, int64_t n, int64_t xstride, int64_t nsig,
                              int64_t B, int64_t a_max, const int64_t* shifts_host,
                              int64_t nshifts, const int64_t* ladder_host, int64_t nladder,
                              const void* W, int64_t k, int64_t* out_pos, void* out_coef,
                              int32_t* out_count, int32_t* out_iterations,
                              int32_t* out_converged, int64_t* out_samples, int64_t* out_sched,
                              void* ws, size_t ws_bytes, void* stream) {
  SFFT_REQUIRE(dtype == 0 || dtype == 1, "sfft_run_oneshot: dtype must be 0 or 1");
  SFFT_REQUIRE(x && shifts_host && ladder_host && W && nsig >= 1 && k >= 1,
               "sfft_run_oneshot: bad argument");
  SFFT_REQUIRE(n > 0 && n < (int64_t(1) << 31), "sfft_run_oneshot: n must be in (0, 2^31)");
  SFFT_REQUIRE(B > 0 && n % B == 0, "sfft_run_oneshot: B must divide n");
  SFFT_REQUIRE(out_pos && out_coef && out_count && out_iterations && out_converged && out_samples,
               "sfft_run_oneshot: null output");
  return run_oneshot(dtype, x, n, xstride, (int)nsig, B, (int)a_max, shifts_host, (int)nshifts,
                     ladder_host, (int)nladder, (const double2*)W, k, out_pos,
                     (double2*)out_coef, out_count, out_iterations, out_converged, out_samples,
                     out_sched, ws, ws_bytes, (cudaStream_t)stream);
}

// Publish "signals [0, value) have arrived" for streaming admission (run on
// the copy stream after each chunk's host-to-device copy).
__global__ void k_set_avail(int32_t* avail, int32_t value) { *avail = value; }

SFFT_API int sfft_set_avail(int32_t* avail, int32_t value, void* stream) {
  SFFT_REQUIRE(avail, "sfft_set_avail: null pointer");
  k_set_avail<<<1, 1, 0, (cudaStream_t)stream>>>(avail, value);
  SFFT_CHECK_LAUNCH("k_set_avail");
  return 0;
}
