// Microbenchmark: random fp64 atomic adds (RED) into a score array, as a row-wise binary flip
// kernel would issue them, versus random 16-byte gathers. Not part of the library.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

__global__ void k_red(const int* __restrict__ idx, const double* __restrict__ val, long long M, double* score) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < M; e += (long long)gridDim.x * blockDim.x)
    atomicAdd(score + __ldcs(idx + e), __ldcs(val + e));
}
__global__ void k_gather(const int* __restrict__ idx, const double2* __restrict__ A, long long M, double* out) {
  double acc = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < M; e += (long long)gridDim.x * blockDim.x) {
    const double2 v = __ldg(A + __ldcs(idx + e));
    acc += v.x;
  }
  if (acc == 1234.5) out[0] = acc;
}
int main() {
  const long long M = 7100000;
  const int N = 700000, R = 200000;
  std::vector<int> hi(M), hr(M);
  srand(1);
  for (long long e = 0; e < M; ++e) { hi[e] = rand() % N; hr[e] = rand() % R; }
  int *di, *dr; double *dv, *ds; double2* dA;
  cudaMalloc(&di, M * 4); cudaMalloc(&dr, M * 4); cudaMalloc(&dv, M * 8); cudaMalloc(&ds, N * 8); cudaMalloc(&dA, R * 16);
  cudaMemcpy(di, hi.data(), M * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, hr.data(), M * 4, cudaMemcpyHostToDevice);
  cudaMemset(dv, 0, M * 8); cudaMemset(ds, 0, N * 8); cudaMemset(dA, 0, R * 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bps = 4; bps <= 16; bps *= 2) {
    const int grid = 148 * bps;
    for (int it = 0; it < 3; ++it) k_red<<<grid, 256>>>(di, dv, M, ds);
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) k_red<<<grid, 256>>>(di, dv, M, ds);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("RED f64  grid %5d: %.1f us per 7.1M  (%.0f G/s)\n", grid, ms * 1000 / 20, M / (ms / 20 * 1e-3) / 1e9);
    for (int it = 0; it < 3; ++it) k_gather<<<grid, 256>>>(dr, dA, M, ds);
    cudaEventRecord(a);
    for (int it = 0; it < 20; ++it) k_gather<<<grid, 256>>>(dr, dA, M, ds);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("gather16 grid %5d: %.1f us per 7.1M  (%.0f G/s)\n", grid, ms * 1000 / 20, M / (ms / 20 * 1e-3) / 1e9);
  }
  return 0;
}
