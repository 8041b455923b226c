// extern "C" boundary of libsfft_b200.so (declared in include/sfft_b200.h).
//
// Plain pointers and sizes only; every device buffer is caller-owned; every
// call is asynchronous on the given stream and returns 0 or a negative code
// (-1 bad argument, -2 unsupported / workspace too small, -3 CUDA error) with
// the message in sfft_last_error().
#include <string>

#include "kernels.cuh"

namespace sfft {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
const char* last_error() { return g_err.c_str(); }
}  // namespace sfft

using namespace sfft;

#define SFFT_API extern "C" __attribute__((visibility("default")))

SFFT_API int sfft_version(void) { return 1; }

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
