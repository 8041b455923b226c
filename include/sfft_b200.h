/*
 * libsfft_b200 — C ABI of the B200-native (sm_100a) sparse-FFT bucketization
 * hot path.  Reference: the Python package `sparsefft` (arXiv 2012.08238
 * toolkit) at /root/reference/pkg/src/sparsefft ("sfft/" below).  The
 * reference has no FFI; each entry point replaces the numpy body of the
 * Python function cited beside it, and the package paper_2012_08238_b200
 * wraps them behind the reference's own signatures.
 *
 * Conventions
 *   - every pointer argument is DEVICE memory owned by the caller, except
 *     where a comment says "host";
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on it and never synchronises unless stated;
 *   - dtype: 0 = complex64 input (float2; rounded once, all accumulation
 *     and every decision in fp64), 1 = complex128 input (double2);
 *   - bucket values are always complex128 (double2);
 *   - return 0 on success, -1/-2 on argument or workspace errors, -3 on a
 *     CUDA launch error; sfft_last_error() returns the message (per thread).
 */
#ifndef SFFT_B200_H
#define SFFT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int sfft_version(void);
const char* sfft_last_error(void);

/* Read-schedule export of the runners: per signal max_groups records of
 * words_per_group int64 = {kind (0 flat, 1 spike, -1 unused), a (sigma or
 * stride), tau, cnt (Omega or samples), nshift, shift[0..]}.  Host pointers. */
int sfft_schedule_layout(int32_t* max_groups, int32_t* words_per_group);

/* Number of kernels this library has launched in this process. */
int64_t sfft_launch_count(void);

/* Measurement aid: with profiling on, every flat/spike bucketization launch
 * is bracketed by CUDA events recorded on its stream (no synchronisation;
 * read back by sfft_prof_read), and the items it processed are counted on
 * the device.  sfft_prof_read returns the
 * summed kernel milliseconds, launch count and item count since enable. */
int sfft_prof_enable(int on);
int sfft_prof_read(double* ms, int64_t* launches, int64_t* items);

/* ---- setup ------------------------------------------------------------ */

/* W[e] = exp(-2*pi*i*e/B), e < B (complex128).  FFT twiddle table. */
int sfft_twiddles(void* W, int64_t B, void* stream);

/* Flat-window taps g[i], i < omega (sfft/filters.py:125-151 taps). */
int sfft_flat_taps(double* taps, int64_t omega, int64_t B, double gauss_sigma, void* stream);

/* Bytes of workspace the bucketizers need for B buckets x nitems (0 when
 * B <= 8192 and B factors into 2,3,5,7,11,13). */
size_t sfft_bucketize_ws_bytes(int64_t B, int64_t nitems);

/* Flat response table gtable[rho][j] = G[rho + j*L], L = n/B, and
 * *gmax = max|G| — replaces the N-point FFT of make_flat_filter
 * (sfft/filters.py:146-149).  rows = 0..L-1 (int64, device). */
int sfft_build_gtable(const double* taps, int64_t omega, int64_t n, int64_t B, const void* W,
                      void* gtable, double* gmax, const int64_t* rows, void* ws,
                      size_t ws_bytes, void* stream);

/* ---- encode: bucketization (A5, A6, A7) --------------------------------- */

/* Flat bucketization of nitems items — replaces bucketize_flat
 * (sfft/bucketize.py:142-161).  Item i reads row item_sig[i] of x (row
 * stride xstride elements; item_sig NULL => item i reads row i) with
 * index sigma[i]*(j - tau_tot[i]) mod n, j < omega, window taps[j], phase
 * w_n^{bsig[i]*j} (bsig NULL => b' = 0), folds mod B and writes
 * out[i][0..B) = FFT_B(fold)/B.  active (per row, NULL => all) skips rows. */
int sfft_flat_bucketize(int dtype, const void* x, int64_t n, int64_t xstride,
                        const double* taps, int64_t omega, int64_t B, int64_t nitems,
                        const int32_t* item_sig, const int64_t* sigma, const int64_t* tau_tot,
                        const int64_t* bsig, const int32_t* active, const void* W, void* out,
                        void* ws, size_t ws_bytes, void* stream);

/* Spike-train bucketization — replaces bucketize_spike
 * (sfft/bucketize.py:164-178): out[i][k] = FFT_B(x[(n/B)*j - tau[i] mod n])[k]/B. */
int sfft_spike_bucketize(int dtype, const void* x, int64_t n, int64_t xstride, int64_t B,
                         int64_t nitems, const int32_t* item_sig, const int64_t* tau,
                         const int32_t* active, const void* W, void* out, void* ws,
                         size_t ws_bytes, void* stream);

/* ---- sampling accounting (A2: TimeSignal.access_count, sfft/signal.py:82-94) */

/* Mark one read schedule into a byte map: kind 0 flat (a=sigma, b=tau_tot,
 * c=omega), 1 spike (a=stride, b=tau, c=count), 2 all, 3 list (idx[c]). */
int sfft_access_mark(uint8_t* map, int64_t n, int kind, int64_t a, int64_t b, int64_t c,
                     const int64_t* idx, void* stream);
/* *out (device int64) = number of non-zero bytes of map[0..n). */
int sfft_count_nonzero(const uint8_t* map, int64_t n, int64_t* out, void* stream);

/* ---- decode stages ------------------------------------------------------- */

/* A8 robust_noise_floor (sfft/reconstruct.py:119-133), one value per set:
 * floor = max(min(mult*median|v|, peak/4), 1e-9*peak, 1e-300); peak = max|v|
 * (peak_out may be NULL).  values: complex128 [nsets][B]. */
int sfft_noise_floor(const void* values, int64_t nsets, int64_t B, double median_mult,
                     double* floor_out, double* peak_out, void* stream);

/* A9 heavy buckets of vote_tally (sfft/reconstruct.py:171-177): bit b of
 * bits[set][B/32] is set iff bucket b is among the first heavy_count buckets
 * with |v| >= max(thr[set], 0) in (-|v|, index) order.  nheavy may be NULL. */
int sfft_heavy_bitmap(const void* values, int64_t nsets, int64_t B, const double* thr,
                      int64_t heavy_count, uint32_t* bits, int32_t* nheavy, void* stream);

/* Workspace bytes for sfft_vote_select. */
size_t sfft_votes_ws_bytes(int64_t n, int64_t nsig, int64_t rounds);

/* A10 vote_tally + A11 select_by_votes (sfft/reconstruct.py:158-194), for
 * nsig independent signals of `rounds` rounds each (rounds <= 255).
 * Position f of signal s scores one per round r whose heavy bitmap
 * bits[s][r] holds f's flat bucket (((sigma*(f-b') mod n) - cs + L/2) mod n)/L.
 * counts_out [nsig][n] (optional) receives the scores (or counts_in supplies
 * them).  If cand != NULL, cand[s][0..keep) receives the positions with
 * score >= need ordered by (-score, position) and ncand[s] their number. */
int sfft_vote_select(int64_t n, int64_t B, int64_t rounds, int64_t nsig, const uint32_t* bits,
                     const int64_t* sigma, const int64_t* bprime, int64_t center_shift,
                     const int64_t* counts_in, int64_t* counts_out, int64_t need, int64_t keep,
                     int64_t* cand, int32_t* ncand, void* ws, size_t ws_bytes, void* stream);

/* A10 vote_tally for bucket sets of any kind (sfft/reconstruct.py:158-179,
 * preimages sfft/bucketize.py:108-118): counts[f] (int64 [n]) = number of
 * rounds r whose heavy bitmap bits[bit_offset[r] ..] (B_r = nbuckets[r] bits,
 * as sfft_heavy_bitmap writes it) holds f's bucket under round r's hash view:
 * m = sigma[r]*(f - bprime[r]) mod n, L = n/B_r, and by kind[r]:
 *   0 flat / Dirichlet with half offset: ((m - cs[r] + L/2) mod n)/L mod B_r,
 *   1 spike: m mod B_r,  2 Dirichlet without half offset: ((m - cs[r]) mod n)/L mod B_r.
 * bprime, kind, center_shift may be NULL (0).  Any number of rounds. */
int sfft_vote_tally(int64_t n, int64_t rounds, const int64_t* nbuckets, const int64_t* bit_offset,
                    const uint32_t* bits, const int64_t* sigma, const int64_t* bprime,
                    const int32_t* kind, const int64_t* center_shift, int64_t* counts,
                    void* stream);

/* A12 _energy_estimates (sfft/frameworks.py:321-332) for `rounds` bucket sets
 * y[r][B]: est[r][c] = y[r][b]/(G[bL-m]*w^{tau[r] m}), m = sigma[r]*cand[c],
 * (NaN, 0) where |G| < 0.05*(*gmax). */
int sfft_energy_estimates(const void* y, int64_t B, const void* gtable, const double* gmax,
                          int64_t n, int64_t rounds, const int64_t* sigma, const int64_t* tau,
                          const int64_t* cand, int64_t ncand, void* est, void* stream);

/* A13 _trimmed_mean (sfft/frameworks.py:335-351) over the rows of est
 * [rounds][ncand] (rounds <= 255). */
int sfft_trimmed_mean(const void* est, int64_t rounds, int64_t ncand, void* out, void* stream);

/* A14 _subtract_flat (sfft/frameworks.py:423-436):
 * out[i][j] = y[i][b] - sum_t coef_t * G[(b*L - sigma[i]*pos_t) mod n] *
 *             w^{(tau_tot[i]*sigma[i]*pos_t) mod n},
 * b = j (nb == B, blist NULL) or blist[i*nb + j]; the tones of item i are
 * tone_pos/tone_coef[item_sig[i]*tone_stride + t], t < tone_count[item_sig[i]],
 * summed in order.  out may alias y when blist is NULL. */
int sfft_subtract_flat(const void* y, void* out, int64_t B, int64_t nb, const int32_t* blist,
                       int64_t nitems, const void* gtable, int64_t n, const int32_t* item_sig,
                       const int64_t* sigma, const int64_t* tau_tot, const int64_t* tone_pos,
                       const void* tone_coef, const int32_t* tone_count, int64_t tone_stride,
                       void* stream);

/* ---- runners (device-resident frameworks) ---------------------------------- */

/* ---- Dirichlet bank and freq-shift estimate -------------- */

/* Workspace bytes of sfft_dirichlet_bucketize for B buckets and noffsets offsets. */
size_t sfft_dirichlet_ws_bytes(int64_t B, int64_t noffsets);

/* bucketize_dirichlet (sfft/bucketize.py:181-211) for a bank of B boxes of
 * width L (L*B == n, make_dirichlet_bank sfft/filters.py:168-187, possibly
 * freq-shifted by filter_freq_shift :190-200): taps complex128[L];
 * half_offset / center_offset as WindowFilter; offsets device int64[noffsets]
 * (the sample offsets, any integers).  out complex128[B] = the averaged,
 * de-rotated bucket values.  Reads L samples per offset. */
int sfft_dirichlet_bucketize(int dtype, const void* x, int64_t n, const void* taps, int64_t L,
                             int64_t B, int32_t half_offset, int64_t center_offset,
                             int64_t noffsets, const int64_t* offsets, const void* W, void* out,
                             void* ws, size_t ws_bytes, void* stream);

/* estimate_freqshift (sfft/reconstruct.py:356-371): out = mean over the count
 * positions idx (device int64, drawn by the caller exactly as the reference
 * draws them) of x[i] * w^{f i}.  ws >= 4096 bytes. */
int sfft_freqshift_estimate(int dtype, const void* x, int64_t n, const int64_t* idx,
                            int64_t count, int64_t f, void* out, void* ws, size_t ws_bytes,
                            void* stream);

/* Workspace bytes of sfft_run_iterative for nslots slots (nshifts = 1 +
 * ladder length for phase location, n/B + 2 for split location; cap =
 * recovered-tone capacity per slot, max_iterations * B suffices). */
size_t sfft_iterative_ws_bytes(int64_t n, int64_t B, int64_t nslots, int64_t nshifts, int64_t cap);

/* A16 run_iterative + _polish_flat_estimates (sfft/frameworks.py:439-608)
 * with phase location (location 0, :493-516) or binary / multiscale
 * class-split location (location 1, :517-554; branching 2 for binary,
 * AlgorithmConfig.branching for multiscale; n/B must be a power of it) for
 * nsig signals (rows of x), continuously
 * batched over nslots device slots: a slot whose signal finishes takes the
 * next queued signal.  perm_sigma/perm_tau hold each signal's permutation
 * stream (PermutationParams.random draws in order; nperm >= max_iterations
 * + 6) at row stride perm_stride (0: one stream shared by all signals).
 * ladder_host (HOST int64[nladder]) is _phase_ladder(n) (unused, may be NULL,
 * for split location).  Outputs per signal:
 * out_pos/out_coef [nsig][k] the top-k entries in (-|c|, f) order,
 * out_count, out_iterations, out_converged, out_samples (samples_read);
 * out_sched (optional) receives the read schedule, see sfft_schedule_layout;
 * avail (optional) enables streaming admission, see sfft_set_avail.
 * Synchronises the stream once per round (one step of every busy slot). */
int sfft_run_iterative(int dtype, const void* x, int64_t n, int64_t xstride, int64_t nsig,
                       int64_t nslots, const double* taps, int64_t omega, int64_t B,
                       const void* gtable, const double* gmax, const void* W,
                       const int64_t* perm_sigma, const int64_t* perm_tau, int64_t nperm,
                       int64_t perm_stride, int64_t k, int64_t max_iterations,
                       const int64_t* ladder_host, int64_t nladder, int32_t location,
                       int32_t branching, int64_t cap, int64_t* out_pos,
                       void* out_coef, int32_t* out_count, int32_t* out_iterations,
                       int32_t* out_converged, int64_t* out_samples, int64_t* out_sched,
                       const int32_t* avail, void* ws, size_t ws_bytes, void* stream);

/* Streaming admission for sfft_run_iterative: with avail != NULL the engine
 * only admits signals [0, *avail); a copy stream publishes progress with
 * sfft_set_avail after each chunk's host-to-device copy, so transfers overlap
 * the compute of earlier signals. */
int sfft_set_avail(int32_t* avail, int32_t value, void* stream);

/* Workspace bytes of sfft_run_voting. */
size_t sfft_voting_ws_bytes(int64_t n, int64_t B, int64_t nsig, int64_t rounds, int64_t k,
                            int64_t prestage_buckets);

/* A15 run_voting (sfft/frameworks.py:354-417) for nsig signals: rounds
 * bucketizations each (perm_sigma/perm_tau [nsig][rounds]), floors, top-2k
 * heavy sets, votes, candidates with >= need_votes votes ((-votes, pos),
 * first 2k), optional spike pre-stage filter (prestage_buckets > 0, with its
 * twiddle table W_pre), energy estimates, trimmed mean and two
 * model-refinement passes.  Outputs as sfft_run_iterative (iterations =
 * rounds, converged = 1 are implied).  Never synchronises. */
int sfft_run_voting(int dtype, const void* x, int64_t n, int64_t xstride, int64_t nsig,
                    const double* taps, int64_t omega, int64_t B, const void* gtable,
                    const double* gmax, const void* W, const int64_t* perm_sigma,
                    const int64_t* perm_tau, int64_t rounds, int64_t k, int64_t need_votes,
                    int64_t prestage_buckets, const void* W_pre, int64_t* out_pos,
                    void* out_coef, int32_t* out_count, int64_t* out_samples, int64_t* out_sched,
                    void* ws, size_t ws_bytes, void* stream);

/* Workspace bytes of sfft_run_peeling (factors_host: HOST int64[nfactors]). */
size_t sfft_peeling_ws_bytes(int64_t n, int64_t nsig, const int64_t* factors_host,
                             int64_t nfactors, int64_t k);

/* A17 run_peeling (sfft/frameworks.py:614-699) for nsig signals: one spike
 * stage per co-prime factor p (B = n/p buckets, 3 shifts when p > 3 else
 * max(p-1, 1)), floors, a_max = 1 classification of every active bucket,
 * two-tier FIFO single-ton queues and the sequential peel (one warp per
 * signal).  W_stages_host: HOST array of device twiddle tables, one per
 * stage (size n/p).  out_error[s] = 1 where the reference would raise
 * InvalidParameter (an active bucket in a one-shift stage).  out_iterations
 * = peels, out_converged = no multi-ton left.  Never synchronises. */
int sfft_run_peeling(int dtype, const void* x, int64_t n, int64_t xstride, int64_t nsig,
                     const int64_t* factors_host, int64_t nfactors,
                     const void* const* W_stages_host, int64_t k, int64_t* out_pos,
                     void* out_coef, int32_t* out_count, int32_t* out_iterations,
                     int32_t* out_converged, int32_t* out_error, int64_t* out_samples,
                     int64_t* out_sched, void* ws, size_t ws_bytes, void* stream);

/* Workspace bytes of sfft_run_oneshot. */
size_t sfft_oneshot_ws_bytes(int64_t n, int64_t nsig, int64_t B, int64_t a_max, int64_t nshifts);

/* run_oneshot (sfft/frameworks.py:216-311) for nsig signals: spike
 * bucketizations at the HOST shift list (0..2a_max-1, the ladder rungs not
 * among them, the seeded pursuit shifts; at most 64), the robust floor of
 * |meas[0]|, count_collisions over the a_max x a_max moment Hankel matrices
 * (sfft/reconstruct.py:245-267), then per active bucket the single-ton
 * unwrap / Prony escalation / refinement / least-squares decision of the
 * reference (locate_prony :270-302, estimate_prony :374-409).  ladder_host:
 * HOST int64[nladder] phase-ladder rungs (ascending, each a shift).  a_max
 * <= 8 on the device.  out_iterations = 1, out_converged = 1.  Never
 * synchronises. */
int sfft_run_oneshot(int dtype, const void* x, int64_t n, int64_t xstride, int64_t nsig,
                     int64_t B, int64_t a_max, const int64_t* shifts_host, int64_t nshifts,
                     const int64_t* ladder_host, int64_t nladder, const void* W, int64_t k,
                     int64_t* out_pos, void* out_coef, int32_t* out_count,
                     int32_t* out_iterations, int32_t* out_converged, int64_t* out_samples,
                     int64_t* out_sched, void* ws, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SFFT_B200_H */
