// barrier_bench2.cu — grid-barrier variants for the persistent cooperative k_compress (B200).
//   V0 generation word + arrival counter (round-1 grid_sync), __threadfence + volatile poll
//   V3 monotonic arrival counter only: red.release.gpu add, ld.acquire.gpu poll until epoch*G
//   V4 V0 with acq_rel atomics / acquire polls instead of full fences
//   V5 per-CTA arrival flags (st.release), CTA 0 gathers them (all threads poll) and releases a
//      generation word the others poll (ld.acquire)
// Also: an empty cooperative launch (launch overhead) and a 1-block launch.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t atom_add_acqrel(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void v0(uint32_t* bar) {
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

__device__ __forceinline__ void v3(uint32_t* bar, uint32_t epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    red_add_release(bar + 64, 1u);
    const uint32_t target = epoch * gridDim.x;
    while ((int32_t)(ld_acquire(bar + 64) - target) < 0) {
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void v4(uint32_t* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t g0 = ld_acquire(bar + 129);
    if (atom_add_acqrel(bar + 128, 1u) == gridDim.x - 1) {
      atomicExch(bar + 128, 0u);
      red_add_release(bar + 129, 1u);
    } else {
      while (ld_acquire(bar + 129) == g0) {
      }
    }
  }
  __syncthreads();
}

// flags at bar[256 + b], generation at bar[255]
__device__ __forceinline__ void v5(uint32_t* bar, uint32_t epoch) {
  __syncthreads();
  if (blockIdx.x == 0) {
    for (uint32_t b = threadIdx.x + 1; b < gridDim.x; b += blockDim.x)
      while (ld_acquire(bar + 256 + b) != epoch) {
      }
    __syncthreads();
    if (threadIdx.x == 0) st_release(bar + 255, epoch);
  } else {
    if (threadIdx.x == 0) {
      st_release(bar + 256 + blockIdx.x, epoch);
      while (ld_acquire(bar + 255) != epoch) {
      }
    }
  }
  __syncthreads();
}

template <int MODE>
__global__ void k(uint32_t* bar, int iters, uint32_t base) {
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) v0(bar);
    else if (MODE == 3) v3(bar, base + i + 1);
    else if (MODE == 4) v4(bar);
    else if (MODE == 5) v5(bar, base + i + 1);
  }
}
__global__ void empty_k() {}
__global__ void empty_smem(uint32_t* p) {
  __shared__ uint32_t big[9000];
  big[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (big[(threadIdx.x + 1) % blockDim.x] == 12345678u) p[0] = 1;
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
  uint32_t base3 = 0, base5 = 0;
  for (int occ : {1, 3}) {
    for (int mode : {0, 3, 4, 5}) {
      int iters = 400;
      const void* fn = mode == 0 ? (const void*)k<0> : mode == 3 ? (const void*)k<3> : mode == 4 ? (const void*)k<4>
                                                                                                  : (const void*)k<5>;
      float best = 1e9f;
      cudaMemset(bar, 0, 1 << 20);
      base3 = 0;
      base5 = 0;
      for (int rep = 0; rep < 3; ++rep) {
        uint32_t base = mode == 3 ? base3 : base5;
        void* args[] = {&bar, &iters, &base};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel(fn, sms * occ, 256, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (mode == 3) base3 += iters;
        if (mode == 5) base5 += iters;
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("grid %4d V%d: %.3f us per barrier (%s)\n", sms * occ, mode, best * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  // launch overhead of an empty kernel vs grid shape (CTA count, threads, static smem)
  {
    struct Cfg { int ctas, threads; bool smem; };
    const Cfg cfgs[] = {{sms, 256, false}, {sms, 768, false}, {2 * sms, 256, false}, {3 * sms, 256, false},
                        {3 * sms, 256, true}, {sms, 768, true}, {sms, 1024, false}};
    for (const Cfg& c : cfgs) {
      const int n = 200;
      for (int w = 0; w < 2; ++w) {
        cudaEventRecord(a);
        for (int i = 0; i < n; ++i) {
          if (c.smem) empty_smem<<<c.ctas, c.threads>>>(bar);
          else empty_k<<<c.ctas, c.threads>>>();
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("empty launch %4d x %4d%s: %.2f us each\n", c.ctas, c.threads, c.smem ? " (36 KB smem)" : "", ms * 1e3 / n);
    }
  }
  // launch overhead: back-to-back empty cooperative launches of the full grid, and a plain launch
  for (int coop : {1, 0}) {
    const int n = 200;
    cudaEventRecord(a);
    for (int i = 0; i < n; ++i) {
      if (coop) cudaLaunchCooperativeKernel((const void*)empty_k, sms * 3, 256, nullptr, 0, 0);
      else empty_k<<<sms * 3, 256>>>();
    }
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s empty launch of %d CTAs: %.2f us each\n", coop ? "cooperative" : "plain", sms * 3, ms * 1e3 / n);
  }
  return 0;
}
