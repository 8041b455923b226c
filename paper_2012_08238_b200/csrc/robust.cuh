// Trimmed mean over rounds (sfft/frameworks.py:335-351) with numpy's NaN
// rules: nanmedian per component, |est - med| (array abs), the linear
// 0.25-quantile of the finite distances, keep dev <= max(4*spread,
// 1e-8*(|med|+1e-300)), nanmean of the kept values; a + 1j*b joins as numpy.
#pragma once

#include "common.cuh"

namespace sfft {

// numpy linear quantile interpolation (_lerp in numpy/lib/_function_base_impl.py)
__device__ __forceinline__ double np_lerp(double a, double b, double t) {
  const double d = b - a;
  return (t >= 0.5) ? (b - d * (1.0 - t)) : (a + d * t);
}

__device__ __forceinline__ void isort(double* v, int m) {
  for (int i = 1; i < m; ++i) {
    const double x = v[i];
    int j = i - 1;
    while (j >= 0 && v[j] > x) {
      v[j + 1] = v[j];
      --j;
    }
    v[j + 1] = x;
  }
}

// nanmedian over m values (mean of the two middle values for even counts)
__device__ __forceinline__ double nanmedian(const double* src, int R, double* tmp) {
  int m = 0;
  for (int i = 0; i < R; ++i)
    if (!isnan(src[i])) tmp[m++] = src[i];
  if (m == 0) return CUDART_NAN;
  isort(tmp, m);
  const int h = m / 2;
  return (m % 2) ? (tmp[h] + tmp[h]) / 2.0 : (tmp[h - 1] + tmp[h]) / 2.0;
}

// a + 1j*b as numpy forms it (NaN/inf in b poisons the real part)
__device__ __forceinline__ double2 np_join(double a, double b) {
  return cmk(a + (0.0 * b - 0.0), 0.0 + b);
}

constexpr int kMaxRounds = 255;  // = kMaxVoteRounds

// Trimmed mean over the R <= MAXR rows of est (row stride ld) for one column.
template <int MAXR = 64>
__device__ inline double2 trimmed_mean_col_t(const double2* est, int64_t ld, int R) {
  double re[MAXR], im[MAXR], tmp[MAXR], dev[MAXR];
  for (int r = 0; r < R; ++r) {
    const double2 v = est[(int64_t)r * ld];
    re[r] = v.x;
    im[r] = v.y;
  }
  const double mr = nanmedian(re, R, tmp);
  const double mi = nanmedian(im, R, tmp);
  const double2 med = np_join(mr, mi);
  int m = 0;
  for (int r = 0; r < R; ++r) {
    dev[r] = cabs_(cmk(re[r] - med.x, im[r] - med.y));
    if (!isnan(dev[r])) tmp[m++] = dev[r];
  }
  double spread = CUDART_NAN;
  if (m > 0) {
    isort(tmp, m);
    const double vi = (double)m * 0.25 + (1.0 + 0.25 * (1.0 - 1.0 - 1.0)) - 1.0;
    double prev = floor(vi);
    const double gamma = vi - prev;
    int lo = (int)prev;
    lo = lo < 0 ? 0 : (lo > m - 1 ? m - 1 : lo);
    const int hi = lo + 1 > m - 1 ? m - 1 : lo + 1;
    spread = np_lerp(tmp[lo], tmp[hi], gamma);
  }
  const double a4 = 4.0 * spread;
  const double b8 = 1e-8 * (cabs_(med) + 1e-300);
  const double tol = (isnan(a4) || isnan(b8)) ? CUDART_NAN : fmax(a4, b8);
  double sr = 0.0, si = 0.0;
  int cr = 0, ci = 0;
  for (int r = 0; r < R; ++r) {
    const bool keep = dev[r] <= tol;
    const bool bad = !keep || isnan(re[r]) || isnan(im[r]);
    if (!bad) {
      sr += re[r];
      si += im[r];
      ++cr;
      ++ci;
    }
  }
  const double mre = cr ? sr / cr : CUDART_NAN;
  const double mim = ci ? si / ci : CUDART_NAN;
  return np_join(mre, mim);
}

// small per-thread arrays for the usual round counts, the large ones otherwise
__device__ inline double2 trimmed_mean_col(const double2* est, int64_t ld, int R) {
  return R <= 64 ? trimmed_mean_col_t<64>(est, ld, R) : trimmed_mean_col_t<kMaxRounds>(est, ld, R);
}


}  // namespace sfft
