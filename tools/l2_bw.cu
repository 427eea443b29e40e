// L2 read bandwidth of the B200 (the roofline of L2-resident workloads such as config P): a 48 MB
// buffer (< 126 MB L2) read repeatedly with coalesced 16-byte loads after a warm-up pass.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_bw tools/l2_bw.cu && /tmp/l2_bw
#include <cstdio>
#include <cuda_runtime.h>
__global__ void rd(const float4* __restrict__ a, size_t n, int reps, float* out) {
  float acc = 0.f;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const float4 v = __ldcg(a + i);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 1.2345f) *out = acc;
}
int main() {
  const size_t bytes = 48ull << 20, n = bytes / 16;
  float4* a;
  float* o;
  cudaMalloc(&a, bytes);
  cudaMalloc(&o, 4);
  cudaMemset(a, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  rd<<<sms * 8, 256>>>(a, n, 1, o);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 50;
  cudaEventRecord(e0);
  rd<<<sms * 8, 256>>>(a, n, reps, o);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"l2_read_gbs\": %.1f, \"bytes\": %zu, \"reps\": %d, \"ms\": %.3f}\n", bytes * (double)reps / (ms * 1e6), bytes, reps, ms);
  return 0;
}
