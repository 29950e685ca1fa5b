// barrier_bench.cu — cost of a grid-wide barrier in a cooperative persistent kernel on B200.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void grid_sync_flat(uint32_t* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile uint32_t* gen = bar + 1;
    const uint32_t g0 = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}
// two-level: groups of GS CTAs arrive on their own counter; the last of each group arrives on the top
template <int GS>
__device__ __forceinline__ void grid_sync_2l(uint32_t* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile uint32_t* gen = bar + 1;
    const uint32_t g0 = *gen;
    const uint32_t ngroups = (gridDim.x + GS - 1) / GS;
    const uint32_t grp = blockIdx.x / GS;
    const uint32_t gsize = min((uint32_t)GS, gridDim.x - grp * GS);
    __threadfence();
    bool last = false;
    if (atomicAdd(bar + 32 + grp * 32, 1u) == gsize - 1) {
      atomicExch(bar + 32 + grp * 32, 0u);
      if (atomicAdd(bar, 1u) == ngroups - 1) {
        atomicExch(bar, 0u);
        last = true;
      }
    }
    if (last) {
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g0) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}
template <int MODE>
__global__ void k(uint32_t* bar, int iters) {
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) grid_sync_flat(bar);
    else if (MODE == 1) grid_sync_2l<16>(bar);
    else grid_sync_2l<32>(bar);
  }
}
int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* bar;
  cudaMalloc(&bar, 1 << 20);
  cudaMemset(bar, 0, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int occ : {1, 2, 3}) {
    for (int mode = 0; mode < 3; ++mode) {
      int iters = 200;
      void* args[] = {&bar, &iters};
      const void* fn = mode == 0 ? (const void*)k<0> : mode == 1 ? (const void*)k<1> : (const void*)k<2>;
      cudaLaunchCooperativeKernel(fn, sms * occ, 256, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel(fn, sms * occ, 256, args, 0, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %4d mode %d: %.2f us per barrier (%s)\n", sms * occ, mode, ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
}
