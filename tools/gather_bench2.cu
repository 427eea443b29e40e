// Microbenchmark 2: random 16-byte gathers (row state) while a 12 B/element stream (row index +
// coefficient, like the CSC) flows through L2. Variants: plain / evict-first stream / L2
// persisting access-policy window on the gathered array. Not part of the library.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ unsigned long long pol_ef() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double ld_ef(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol_ef()));
  return v;
}
__device__ __forceinline__ int ld_ef(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol_ef()));
  return v;
}

template <int MODE>   // 0: __ldg stream, 1: __ldcs stream, 2: evict_first stream
__global__ void __launch_bounds__(256) k(const double2* __restrict__ A, const int* __restrict__ idx,
                                         const double* __restrict__ val, long long M, double* out) {
  const int lane = threadIdx.x & 31;
  long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  constexpr int K = 8;
  double acc = 0.0;
  for (; w * 32 * K < M; w += nw) {
    int id[K];
    double a[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const long long e = w * 32 * K + lane + 32 * q;
      if (MODE == 0) { id[q] = __ldg(idx + e); a[q] = __ldg(val + e); }
      else if (MODE == 1) { id[q] = __ldcs(idx + e); a[q] = __ldcs(val + e); }
      else { id[q] = ld_ef(idx + e); a[q] = ld_ef(val + e); }
    }
    double2 v[K];
#pragma unroll
    for (int q = 0; q < K; ++q) v[q] = __ldg(A + id[q]);
#pragma unroll
    for (int q = 0; q < K; ++q) acc += v[q].x * a[q];
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
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  int l2;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  int maxpersist;
  cudaDeviceGetAttribute(&maxpersist, cudaDevAttrMaxPersistingL2CacheSize, 0);
  printf("SMs %d clock %d kHz L2 %d B, max persisting %d B\n", sms, clk, l2, maxpersist);
  const long long N = 230000;
  double2* A;
  cudaMalloc(&A, N * sizeof(double2));
  cudaMemset(A, 0, N * sizeof(double2));
  double* out;
  cudaMalloc(&out, 8);
  for (long long M : {1ll << 20, 4ll << 20, 13ll << 20}) {
    int* idx;
    double* val;
    cudaMalloc(&idx, M * sizeof(int));
    cudaMalloc(&val, M * sizeof(double));
    cudaMemset(val, 0, M * sizeof(double));
    int* h = (int*)malloc(M * sizeof(int));
    srand(1);
    for (long long i = 0; i < M; ++i) h[i] = (int)(((unsigned long long)rand() * 2654435761ull) % N);
    cudaMemcpy(idx, h, M * sizeof(int), cudaMemcpyHostToDevice);
    free(h);
    cudaStream_t s;
    cudaStreamCreate(&s);
    const int grid = sms * 8;
    auto rate = [&](float ms) { return M / (ms * 1e-3) / sms / (clk * 1e3); };
    float t0 = timeit([&] { k<0><<<grid, 256, 0, s>>>(A, idx, val, M, out); });
    float t1 = timeit([&] { k<1><<<grid, 256, 0, s>>>(A, idx, val, M, out); });
    float t2 = timeit([&] { k<2><<<grid, 256, 0, s>>>(A, idx, val, M, out); });
    // persisting window on A
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 16 << 20);
    cudaStreamAttrValue attr = {};
    attr.accessPolicyWindow.base_ptr = A;
    attr.accessPolicyWindow.num_bytes = N * sizeof(double2);
    attr.accessPolicyWindow.hitRatio = 1.0f;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &attr);
    float t3 = timeit([&] { k<2><<<grid, 256, 0, s>>>(A, idx, val, M, out); });
    float t4 = timeit([&] { k<0><<<grid, 256, 0, s>>>(A, idx, val, M, out); });
    attr.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &attr);
    cudaCtxResetPersistingL2Cache();
    printf("M=%6.1fM stream %5.0f MB: ldg %.3f ms (%.3f/SM-cyc) ldcs %.3f (%.3f) evict_first %.3f (%.3f) "
           "persist+ef %.3f (%.3f) persist+ldg %.3f (%.3f)  | stream GB/s at ef: %.0f\n",
           M / 1e6, M * 12 / 1e6, t0, rate(t0), t1, rate(t1), t2, rate(t2), t3, rate(t3), t4, rate(t4),
           M * 12 / (t2 * 1e-3) / 1e9);
    cudaFree(idx);
    cudaFree(val);
  }
  return 0;
}
