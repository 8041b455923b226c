// Sampling accounting (sfft/signal.py:82-94: samples_read = |union of read
// indices|) evaluated from read schedules instead of a bool map written by
// the gather.
//
// mark/count: explicit byte map, used by the stage-level TimeSignal API and as
// the cross-check for the runners' map-free union count (runners.cu).
#include "kernels.cuh"

namespace sfft {

__global__ void k_mark(uint8_t* __restrict__ map, int64_t n, int kind, int64_t a, int64_t b,
                       int64_t c, const int64_t* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (kind == 0) {          // flat: sigma=a, tau=b, omega=c
    if (i < c) map[mulmod(a, pmod(i - b, n), n)] = 1;
  } else if (kind == 1) {   // spike: step=a, tau=b, count=c
    if (i < c) map[pmod(a * i - b, n)] = 1;
  } else if (kind == 2) {   // all
    if (i < n) map[i] = 1;
  } else {                  // explicit list of c indices (already reduced)
    if (i < c) map[pmod(idx[i], n)] = 1;
  }
}

__global__ void k_count_nonzero(const uint8_t* __restrict__ map, int64_t n,
                                unsigned long long* out) {
  unsigned long long cnt = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    cnt += map[i] != 0;
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(out, cnt);
}

int run_mark(uint8_t* map, int64_t n, int kind, int64_t a, int64_t b, int64_t c,
             const int64_t* idx, cudaStream_t st) {
  const int64_t work = (kind == 2) ? n : c;
  if (work <= 0) return 0;
  k_mark<<<(unsigned)cdiv_up(work, 256), 256, 0, st>>>(map, n, kind, a, b, c, idx);
  SFFT_CHECK_LAUNCH("k_mark");
  return 0;
}

int run_count_nonzero(const uint8_t* map, int64_t n, int64_t* out, cudaStream_t st) {
  SFFT_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), st));
  const int blocks = (int)std::min<int64_t>(1184, cdiv_up(n, 256));
  k_count_nonzero<<<blocks, 256, 0, st>>>(map, n, (unsigned long long*)out);
  SFFT_CHECK_LAUNCH("k_count_nonzero");
  return 0;
}

}  // namespace sfft
