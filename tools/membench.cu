// membench.cu — read-bandwidth probes for the access patterns the hot-path kernels use.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench tools/membench.cu
// Run:   tools/membench [n_floats]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ uint32_t g_sink;

// V1: grid-stride, each thread 4 x 128-bit loads per iteration (block-contiguous 16 KB tiles)
__global__ void v_gridstride(const uint4* __restrict__ a, uint64_t n4) {
  uint32_t acc = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x * 4 + threadIdx.x; i < n4; i += stride) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (i + k * blockDim.x < n4) ? a[i + k * blockDim.x] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < 4; ++k) acc += v[k].x ^ v[k].y ^ v[k].z ^ v[k].w;
  }
  if (acc == 0x12345678u) g_sink = acc;
}

// V2: per-warp contiguous slabs, rounds of 4 x 128-bit loads per lane, DEPTH rounds in flight
template <int DEPTH>
__global__ void v_warpslab(const uint4* __restrict__ a, uint64_t n4, uint64_t slab4) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const uint64_t lo = w * slab4, hi = min(n4, lo + slab4);
  uint32_t acc = 0;
  uint4 v[DEPTH][4];
  const uint64_t nr = hi > lo ? (hi - lo) / 128 : 0;
#pragma unroll
  for (int d = 0; d < DEPTH; ++d)
    if (d < (int)nr)
#pragma unroll
      for (int k = 0; k < 4; ++k) v[d][k] = a[lo + d * 128 + k * 32 + lane];
  for (uint64_t r = 0; r < nr; r += DEPTH) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      if (r + d < nr) {
#pragma unroll
        for (int k = 0; k < 4; ++k) acc += v[d][k].x ^ v[d][k].y ^ v[d][k].z ^ v[d][k].w;
        if (r + d + DEPTH < nr)
#pragma unroll
          for (int k = 0; k < 4; ++k) v[d][k] = a[lo + (r + d + DEPTH) * 128 + k * 32 + lane];
      }
    }
  }
  if (acc == 0x12345678u) g_sink = acc;
}

// V4: per-warp TMA bulk ring: lane 0 streams 2 KB chunks of its slab into a STAGES-deep smem ring
template <int STAGES>
__global__ void v_tma(const uint4* __restrict__ a, uint64_t n4, uint64_t slab4) {
  extern __shared__ __align__(128) uint4 smem[];
  __shared__ __align__(8) uint64_t bars[8][STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + warp;
  const uint64_t lo = w * slab4, hi = min(n4, lo + slab4);
  const uint64_t nr = hi > lo ? (hi - lo) / 128 : 0;
  uint4* ring = smem + (size_t)warp * STAGES * 128;
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  auto issue = [&](uint64_t r, int s) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
    uint32_t d = (uint32_t)__cvta_generic_to_shared(ring + s * 128);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(2048));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(d), "l"(a + lo + r * 128), "r"(2048), "r"(b) : "memory");
  };
  if (lane == 0)
    for (int s = 0; s < STAGES && s < (int)nr; ++s) issue(s, s);
  uint32_t acc = 0;
  uint32_t phase[STAGES];
  for (int s = 0; s < STAGES; ++s) phase[s] = 0;
  for (uint64_t r = 0; r < nr; ++r) {
    const int s = (int)(r % STAGES);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(b), "r"(phase[s]));
    }
    phase[s] ^= 1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint4 v = ring[s * 128 + k * 32 + lane];
      acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    __syncwarp();
    if (lane == 0 && r + STAGES < nr) issue(r + STAGES, s);
  }
  if (acc == 0x12345678u) g_sink = acc;
}

int main(int argc, char** argv) {
  uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 25600000ull;
  uint64_t n4 = n / 4;
  uint4* a;
  CK(cudaMalloc(&a, n4 * 16));
  CK(cudaMemset(a, 1, n4 * 16));
  char* flush;
  const size_t FL = 512ull << 20;
  CK(cudaMalloc(&flush, FL));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch, bool cold) {
    float best = 1e9, sum = 0;
    for (int it = 0; it < 12; ++it) {
      if (cold) cudaMemsetAsync(flush, it, FL);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) { best = std::min(best, ms); sum += ms; }
    }
    cudaError_t e = cudaGetLastError();
    printf("%-34s %s  best %7.2f us  %7.0f GB/s   mean %7.2f us  %s\n", name, cold ? "cold" : "warm", best * 1e3,
           n4 * 16 / (best * 1e-3) / 1e9, sum / 10 * 1e3, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  for (int cold = 0; cold < 2; ++cold) {
    for (int occ : {4, 8, 16}) {
      char nm[64];
      snprintf(nm, 64, "gridstride %dx%d", sms, occ);
      timeit(nm, [&] { v_gridstride<<<sms * occ, 256>>>(a, n4); }, cold);
    }
    for (int occ : {4, 6, 8}) {
      const uint64_t W = (uint64_t)sms * occ * 8;
      uint64_t slab4 = ((n4 + W - 1) / W + 127) / 128 * 128;
      char nm[64];
      snprintf(nm, 64, "warpslab d1 %dx%d", sms, occ);
      timeit(nm, [&] { v_warpslab<1><<<sms * occ, 256>>>(a, n4, slab4); }, cold);
      snprintf(nm, 64, "warpslab d2 %dx%d", sms, occ);
      timeit(nm, [&] { v_warpslab<2><<<sms * occ, 256>>>(a, n4, slab4); }, cold);
      snprintf(nm, 64, "warpslab d3 %dx%d", sms, occ);
      timeit(nm, [&] { v_warpslab<3><<<sms * occ, 256>>>(a, n4, slab4); }, cold);
    }
    for (int occ : {2, 3, 4}) {
      const uint64_t W = (uint64_t)sms * occ * 8;
      uint64_t slab4 = ((n4 + W - 1) / W + 127) / 128 * 128;
      char nm[64];
      snprintf(nm, 64, "tma ring4 %dx%d", sms, occ);
      cudaFuncSetAttribute(v_tma<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * 2048);
      timeit(nm, [&] { v_tma<4><<<sms * occ, 256, 8 * 4 * 2048>>>(a, n4, slab4); }, cold);
      snprintf(nm, 64, "tma ring6 %dx%d", sms, occ);
      cudaFuncSetAttribute(v_tma<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 6 * 2048);
      timeit(nm, [&] { v_tma<6><<<sms * occ, 256, 8 * 6 * 2048>>>(a, n4, slab4); }, cold);
    }
  }
  return 0;
}
