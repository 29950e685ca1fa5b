// icache_bench.cu — cost of executing straight-line code the SM has not run recently: a k_compress-shaped
// grid (148 x 3 CTAs of 256 threads) runs a KB-sized block of code twice per launch (pass 0 cold,
// pass 1 warm); between launches a 300 MB stream (or another kernel) runs.  %globaltimer per pass.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/icache_bench tools/icache_bench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <vector>

__device__ uint64_t g_t[2][4096];
__device__ uint32_t g_sink;

template <int K>
__global__ void __launch_bounds__(256, 3) blob() {
  uint32_t x = threadIdx.x;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    __syncthreads();
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
#pragma unroll
    for (int i = 0; i < K; ++i) asm volatile("mad.lo.u32 %0, %0, 1664525, %1;" : "+r"(x) : "r"(1013904223u + (uint32_t)i));
    __syncthreads();
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) g_t[pass][blockIdx.x] = t1 - t0;
  }
  if (x == 0x12345678u) g_sink = x;
}

__global__ void stream(const float4* __restrict__ a, float4* b, uint64_t n4) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

template <int K>
void run(int sms, float4* a, float4* b, uint64_t n4, bool flush) {
  std::vector<double> c0, c1;
  for (int it = 0; it < 12; ++it) {
    if (flush) stream<<<sms * 8, 256>>>(a, b, n4);
    blob<K><<<sms * 3, 256>>>();
    cudaDeviceSynchronize();
    static uint64_t h[2][4096];
    cudaMemcpyFromSymbol(h, g_t, sizeof(h));
    std::vector<uint64_t> p0(h[0], h[0] + sms * 3), p1(h[1], h[1] + sms * 3);
    std::sort(p0.begin(), p0.end());
    std::sort(p1.begin(), p1.end());
    if (it >= 2) { c0.push_back(p0[p0.size() / 2] / 1e3); c1.push_back(p1[p1.size() / 2] / 1e3); }
  }
  std::sort(c0.begin(), c0.end());
  std::sort(c1.begin(), c1.end());
  printf("%6d B of SASS, %s: pass 0 (cold) %6.2f us, pass 1 (warm) %6.2f us (median CTA, median launch)\n", K * 16,
         flush ? "300 MB stream between launches" : "back-to-back launches        ", c0[c0.size() / 2], c1[c1.size() / 2]);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t n4 = (150ull << 20) / 16;
  float4 *a, *b;
  cudaMalloc(&a, n4 * 16);
  cudaMalloc(&b, n4 * 16);
  cudaMemset(a, 0, n4 * 16);
  for (int fl = 0; fl < 2; ++fl) {
    run<512>(sms, a, b, n4, fl);
    run<2048>(sms, a, b, n4, fl);
    run<8192>(sms, a, b, n4, fl);
  }
  return 0;
}
