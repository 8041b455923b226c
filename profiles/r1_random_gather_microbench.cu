// Micro-benchmark: DRAM bytes per random 8-byte gather under various load flavours.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void g_cg(const float2* __restrict__ x, long long n, long long cnt, unsigned seed, double* out) {
  double acc = 0;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned long long st = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
  for (long long k = 0; k < cnt; ++k) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    long long idx = (st >> 20) % n;
    float2 v = __ldcg(x + idx);
    acc += v.x;
  }
  if (acc == 12345.678) out[0] = acc;
}
__global__ void g_ldg(const float2* __restrict__ x, long long n, long long cnt, unsigned seed, double* out) {
  double acc = 0;
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  unsigned long long st = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
  for (long long k = 0; k < cnt; ++k) {
    st = st * 6364136223846793005ull + 1442695040888963407ull;
    long long idx = (st >> 20) % n;
    float2 v = __ldg(x + idx);
    acc += v.x;
  }
  if (acc == 12345.678) out[0] = acc;
}
int main(int argc, char** argv) {
  int gran = argc > 1 ? atoi(argv[1]) : 0;
  if (gran > 0) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran);
    size_t v = 0; cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("set granularity %d -> %s, now %zu\n", gran, cudaGetErrorString(e), v);
  } else {
    size_t v = 0; cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
    printf("default granularity %zu\n", v);
  }
  long long n = 1LL << 29;  // 4 GB of float2
  float2* x; double* out;
  cudaMalloc(&x, n * sizeof(float2)); cudaMalloc(&out, 8);
  cudaMemset(x, 0, n * sizeof(float2));
  int threads = 256, blocks = 148 * 8; long long cnt = 256;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    g_cg<<<blocks, threads>>>(x, n, cnt, 1 + rep, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double gathers = (double)blocks * threads * cnt;
    printf("cg : %.3f ms  %.1f Ggathers/s  %.1f GB/s of 8B\n", ms, gathers / ms / 1e6, gathers * 8 / ms / 1e6);
    cudaEventRecord(a);
    g_ldg<<<blocks, threads>>>(x, n, cnt, 7 + rep, out);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("ldg: %.3f ms  %.1f Ggathers/s  %.1f GB/s of 8B\n", ms, gathers / ms / 1e6, gathers * 8 / ms / 1e6);
  }
  return 0;
}
