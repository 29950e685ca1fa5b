// writebench.cu — pure-store bandwidth for the decompression's output pattern (102 MB / 440 MB fp32).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void w(float4* __restrict__ o, uint64_t n4) {
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    if (MODE == 0) o[i] = z;
    else if (MODE == 1) __stcs(o + i, z);
    else __stcg(o + i, z);
  }
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (uint64_t n : {25600000ull, 110000000ull}) {
    float4* o;
    cudaMalloc(&o, n * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode)
      for (int occ : {4, 8, 16}) {
        float best = 1e9;
        for (int it = 0; it < 10; ++it) {
          cudaEventRecord(a);
          if (mode == 0) w<0><<<sms * occ, 256>>>(o, n / 4);
          else if (mode == 1) w<1><<<sms * occ, 256>>>(o, n / 4);
          else w<2><<<sms * occ, 256>>>(o, n / 4);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (it >= 2 && ms < best) best = ms;
        }
        printf("n=%llu mode %d occ %2d: %7.2f us  %6.0f GB/s\n", (unsigned long long)n, mode, occ, best * 1e3,
               n * 4 / (best * 1e-3) / 1e9);
      }
    cudaFree(o);
  }
}
