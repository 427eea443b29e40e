// Microbenchmark: throughput of random 16-byte gathers on B200 (the access pattern of the
// column-wise best-shift evaluation: one row-state load per nonzero). Not part of the library.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <stdint.h>

template <int K>
__global__ void __launch_bounds__(256) k_gather(const double2* __restrict__ A, const int* __restrict__ idx,
                                                long long M, double* out) {
  long long base = ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  const long long stride = (long long)gridDim.x * blockDim.x;
  double acc = 0.0;
  for (long long s = base; s * K < M; s += stride) {
    int id[K];
#pragma unroll
    for (int q = 0; q < K; ++q) id[q] = __ldcs(idx + s * K + q);
    double2 v[K];
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] = __ldg(A + id[q]);
#pragma unroll
    for (int q = 0; q < K; ++q) acc += v[q].x;
  }
  if (acc == 12345.0) out[0] = acc;
}

// coalesced-index variant: lane-strided index loads (like the warp tiles)
template <int K>
__global__ void __launch_bounds__(256) k_gather_strided(const double2* __restrict__ A, const int* __restrict__ idx,
                                                        long long M, double* out) {
  const int lane = threadIdx.x & 31;
  long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  for (; w * 32 * K < M; w += nw) {
    int id[K];
#pragma unroll
    for (int q = 0; q < K; ++q) id[q] = __ldcs(idx + w * 32 * K + lane + 32 * q);
    double2 v[K];
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] = __ldg(A + id[q]);
#pragma unroll
    for (int q = 0; q < K; ++q) acc += v[q].x;
  }
  if (acc == 12345.0) out[0] = acc;
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < 10; ++r) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 10;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const long long M = 13 << 20;
  int* idx;
  double2* A;
  double* out;
  cudaMalloc(&idx, M * sizeof(int));
  cudaMalloc(&out, 8);
  const long long Nbig = 1 << 24;
  cudaMalloc(&A, Nbig * sizeof(double2));
  cudaMemset(A, 0, Nbig * sizeof(double2));
  int* h = (int*)malloc(M * sizeof(int));
  long long Ns[] = {1 << 12, 230000, 1 << 20, Nbig};
  printf("SMs %d clock %d kHz\n", sms, clk);
  for (long long N : Ns) {
    srand(1);
    for (long long i = 0; i < M; ++i) h[i] = (int)(((unsigned long long)rand() * 2654435761ull) % N);
    cudaMemcpy(idx, h, M * sizeof(int), cudaMemcpyHostToDevice);
    for (int occ : {4, 8}) {
      const int grid = sms * occ;
      float t4 = timeit([&] { k_gather<4><<<grid, 256>>>(A, idx, M, out); });
      float t8 = timeit([&] { k_gather<8><<<grid, 256>>>(A, idx, M, out); });
      float t16 = timeit([&] { k_gather<16><<<grid, 256>>>(A, idx, M, out); });
      float s8 = timeit([&] { k_gather_strided<8><<<grid, 256>>>(A, idx, M, out); });
      auto rate = [&](float ms) { return M / (ms * 1e-3) / sms / (clk * 1e3); };
      printf("N=%9lld (%6.1f MB) grid=%d: K4 %.3f ms (%.3f/SM-cyc)  K8 %.3f (%.3f)  K16 %.3f (%.3f)  strided8 %.3f (%.3f)\n",
             N, N * 16 / 1e6, grid, t4, rate(t4), t8, rate(t8), t16, rate(t16), s8, rate(s8));
    }
  }
  return 0;
}
