// Host-side launchers shared by the .cu translation units.
#pragma once

#include "fft.cuh"

namespace sfft {

enum ProdMode { PROD_FLAT = 0, PROD_SPIKE = 1, PROD_GTAB = 2, PROD_LOAD = 3 };

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
  const double2* z;          // PROD_LOAD source [nitems][B]
};


size_t bucketize_ws_bytes(int64_t B, int64_t nitems);
int run_bucketize(int dtype, int mode, const Prod& p, int64_t nitems, const double2* W,
                  double2* out, void* ws, size_t ws_bytes, cudaStream_t st);
int run_twiddle(double2* W, int64_t B, cudaStream_t st);
int run_flat_taps(double* taps, int64_t omega, int64_t B, double gsig, cudaStream_t st);
int run_absmax(const double2* v, int64_t count, double* out, cudaStream_t st);

int run_mark(uint8_t* map, int64_t n, int kind, int64_t a, int64_t b, int64_t c,
             const int64_t* idx, cudaStream_t st);
int run_count_nonzero(const uint8_t* map, int64_t n, int64_t* out, cudaStream_t st);

}  // namespace sfft
