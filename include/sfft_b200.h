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

#ifdef __cplusplus
}
#endif

#endif /* SFFT_B200_H */
