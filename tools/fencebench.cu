// Micro-benchmark: cost of publishing a small per-CTA run of pairs to a peer GPU over NVLink
// (remote coalesced stores + fence + remote arrival counter), as the fused all-gather does at
// the end of k_compress.  One process, two GPUs, peer access enabled.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fencebench tools/fencebench.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// mode bit 0: remote stores; bit 1: fence.sys by writers (else fence.gpu); bit 2: remote atomic;
// bit 3: heavy local write traffic before (simulates the residual/out writes); bit 4: no fence
__global__ void k(uint32_t* remote, uint32_t* local, uint32_t* flag, uint32_t per_cta, int mode, uint64_t* tns,
                  float* big, size_t big_n) {
  const uint32_t tid = threadIdx.x;
  if (mode & 8) {
    for (size_t i = blockIdx.x * blockDim.x + tid; i < big_n; i += (size_t)gridDim.x * blockDim.x) big[i] = 0.f;
  }
  __syncthreads();
  const uint64_t t0 = gtime();
  const uint32_t base = blockIdx.x * per_cta;
  for (uint32_t p = tid; p < per_cta; p += blockDim.x) {
    local[base + p] = p;
    if (mode & 1) remote[base + p] = p;
  }
  if (!(mode & (16 | 32 | 128))) {
    if (tid < per_cta) {
      if (mode & 2) __threadfence_system(); else __threadfence();
    }
  }
  __syncthreads();
  if (tid == 0) {
    if (mode & 32) {
      if (mode & 64) asm volatile("fence.acq_rel.sys;" ::: "memory");
      else __threadfence_system();
    }
    if (mode & 128) asm volatile("red.release.sys.global.add.u32 [%0], %1;" :: "l"(flag), "r"(1u) : "memory");
    else if (mode & 4) atomicAdd_system(flag, 1u); else atomicAdd(flag + 1, 1u);
    const uint64_t t1 = gtime();
    tns[blockIdx.x] = t1 - t0;
  }
}

int main() {
  int n = 0;
  cudaGetDeviceCount(&n);
  if (n < 2) { printf("need 2 GPUs\n"); return 0; }
  int can = 0;
  cudaDeviceCanAccessPeer(&can, 0, 1);
  printf("peer access 0->1: %d\n", can);
  cudaSetDevice(1);
  uint32_t* remote;
  cudaMalloc(&remote, 64 << 20);
  uint32_t* rflag;
  cudaMalloc(&rflag, 64);
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  uint32_t *local, *lflag;
  uint64_t* tns;
  float* big;
  const size_t big_n = 100u << 20;
  cudaMalloc(&local, 64 << 20);
  cudaMalloc(&lflag, 64);
  cudaMalloc(&tns, 8 * 4096);
  cudaMalloc(&big, big_n * 4);
  const int grid = 444, threads = 256;
  const uint32_t per = 58;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int modes[] = {0, 2, 3, 7, 5, 21, 37, 101, 133, 15, 29, 45, 109, 141};
  for (int mode : modes) {
    uint32_t* fl = (mode & 4) ? rflag : lflag;
    for (int w = 0; w < 3; ++w) k<<<grid, threads>>>(remote, local, fl, per, mode, tns, big, big_n);
    const int it = 20;
    float ms_tot = 0;
    double avg = 0, mx = 0;
    for (int i = 0; i < it; ++i) {
      cudaEventRecord(e0);
      k<<<grid, threads>>>(remote, local, fl, per, mode, tns, big, big_n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ms_tot += ms;
      uint64_t h[grid];
      cudaMemcpy(h, tns, 8 * grid, cudaMemcpyDeviceToHost);
      for (int b = 0; b < grid; ++b) { avg += h[b]; mx = mx > h[b] ? mx : h[b]; }
    }
    printf("mode %2d [remote=%d fence=%s atomic=%s bigwrite=%d]: kernel %.2f us, per-CTA publish avg %.2f us max %.2f us\n",
           mode, mode & 1, (mode & 128) ? "red.release.sys" : (mode & 32) ? ((mode & 64) ? "1thr acq_rel.sys" : "1thr sc.sys") : (mode & 16) ? "none" : ((mode & 2) ? "sys" : "gpu"), (mode & 4) ? "remote" : "local",
           (mode >> 3) & 1, 1e3 * ms_tot / it, avg / it / grid / 1e3, mx / 1e3);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
