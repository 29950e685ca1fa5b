// nvlbench.cu — HiTopKComm step 1's access pattern over NVLink (one process, all visible GPUs, P2P):
// GPU i sums segment i of every GPU's gradient (n sources: its own + n-1 peers), 4 B/element per
// source, and writes the sum once (the EF pass also reads / writes the residual; left out here).
// Variants: SM loads (the k_compress EF-pass layout: 512-element units, one 128-bit load per chunk
// per source) with DEPTH units in flight, TMA bulk copies of the peer segments into shared memory,
// and the copy engines (cudaMemcpyPeerAsync of the n-1 remote segments) for reference.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/nvlbench tools/nvlbench.cu
// Run:   tools/nvlbench [d]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Src { const float* p[8]; };

template <int NS, int DEPTH>
__global__ void __launch_bounds__(256) k_sum(Src s, float* out, uint64_t n, uint32_t upw) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const uint64_t u0 = w * upw, nu = n / 512;
  const uint32_t nun = u0 >= nu ? 0u : (uint32_t)min((uint64_t)upw, nu - u0);
  float4 v[DEPTH][NS][4];
  auto load = [&](uint32_t i, int d) {
    const uint64_t base = (u0 + i) * 512 + 4 * lane;
#pragma unroll
    for (int q = 0; q < NS; ++q)
#pragma unroll
      for (int c = 0; c < 4; ++c) v[d][q][c] = __ldcs(reinterpret_cast<const float4*>(s.p[q] + base + c * 128));
  };
#pragma unroll
  for (int d = 0; d < DEPTH; ++d)
    if (d < (int)nun) load(d, d);
  for (uint32_t i = 0; i < nun; i += DEPTH) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      if (i + d < nun) {
        float4 a[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          a[c] = v[d][0][c];
#pragma unroll
          for (int q = 1; q < NS; ++q)
            a[c] = make_float4(a[c].x + v[d][q][c].x, a[c].y + v[d][q][c].y, a[c].z + v[d][q][c].z, a[c].w + v[d][q][c].w);
        }
        if (i + d + DEPTH < nun) load(i + d + DEPTH, d);
        const uint64_t base = (u0 + i + d) * 512 + 4 * lane;
#pragma unroll
        for (int c = 0; c < 4; ++c) __stcs(reinterpret_cast<float4*>(out + base + c * 128), a[c]);
      }
    }
  }
}

// TMA: per warp, STAGES-deep ring of (NS sources x 2 KB) bulk copies per unit
template <int NS, int STAGES>
__global__ void __launch_bounds__(256) k_sum_tma(Src s, float* out, uint64_t n, uint32_t upw) {
  extern __shared__ __align__(128) float4 smem[];
  __shared__ __align__(8) uint64_t bars[8][STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t w = (uint64_t)blockIdx.x * 8 + warp;
  const uint64_t u0 = w * upw, nu = n / 512;
  const uint32_t nun = u0 >= nu ? 0u : (uint32_t)min((uint64_t)upw, nu - u0);
  float4* ring = smem + (size_t)warp * STAGES * NS * 128;
  if (lane == 0) {
    for (int st = 0; st < STAGES; ++st) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][st]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  auto issue = [&](uint32_t i, int st) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][st]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2048 * NS));
    for (int q = 0; q < NS; ++q) {
      uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + (st * NS + q) * 128);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "l"(s.p[q] + (u0 + i) * 512), "r"(2048), "r"(b) : "memory");
    }
  };
  if (lane == 0)
    for (int st = 0; st < STAGES && st < (int)nun; ++st) issue(st, st);
  uint32_t phase = 0;
  for (uint32_t i = 0; i < nun; ++i) {
    const int st = (int)(i % STAGES);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][st]);
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(b), "r"((phase >> st) & 1u));
    phase ^= 1u << st;
    float4 a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      a[c] = ring[(st * NS) * 128 + c * 32 + lane];
#pragma unroll
      for (int q = 1; q < NS; ++q) {
        const float4 x = ring[(st * NS + q) * 128 + c * 32 + lane];
        a[c] = make_float4(a[c].x + x.x, a[c].y + x.y, a[c].z + x.z, a[c].w + x.w);
      }
    }
    __syncwarp();
    if (lane == 0 && i + STAGES < nun) issue(i + STAGES, st);
    const uint64_t base = (u0 + i) * 512 + 4 * lane;
#pragma unroll
    for (int c = 0; c < 4; ++c) __stcs(reinterpret_cast<float4*>(out + base + c * 128), a[c]);
  }
}

int main(int argc, char** argv) {
  const uint64_t d = argc > 1 ? strtoull(argv[1], 0, 10) : 25600000ull;
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  ng = std::min(ng, 8);
  if (ng < 2) { printf("needs >= 2 GPUs\n"); return 0; }
  const int n = ng;
  const uint64_t seg = d / n;
  std::vector<float*> g(n), out(n);
  std::vector<cudaStream_t> st(n);
  std::vector<cudaEvent_t> e0(n), e1(n);
  int sms = 0;
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(i));
    for (int j = 0; j < n; ++j)
      if (j != i) { cudaError_t e = cudaDeviceEnablePeerAccess(j, 0); if (e != cudaSuccess) (void)cudaGetLastError(); }
    CK(cudaMalloc(&g[i], d * 4));
    CK(cudaMalloc(&out[i], seg * 4));
    CK(cudaMemset(g[i], 0, d * 4));
    CK(cudaStreamCreate(&st[i]));
    CK(cudaEventCreate(&e0[i]));
    CK(cudaEventCreate(&e1[i]));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, i);
  }
  const double remote = (double)(n - 1) * seg * 4;  // bytes each GPU pulls over NVLink
  auto timeit = [&](const char* name, auto launch) -> int {
    std::vector<float> best(n, 1e9);
    for (int it = 0; it < 12; ++it) {
      for (int i = 0; i < n; ++i) { cudaSetDevice(i); cudaDeviceSynchronize(); }
      for (int i = 0; i < n; ++i) {
        cudaSetDevice(i);
        cudaEventRecord(e0[i], st[i]);
        launch(i);
        cudaEventRecord(e1[i], st[i]);
      }
      for (int i = 0; i < n; ++i) {
        cudaSetDevice(i);
        cudaEventSynchronize(e1[i]);
        float ms;
        cudaEventElapsedTime(&ms, e0[i], e1[i]);
        if (it >= 2) best[i] = std::min(best[i], ms);
      }
    }
    const float worst = *std::max_element(best.begin(), best.end());
    cudaError_t e = cudaGetLastError();
    printf("n=%d %-34s %8.1f us  remote ingress %6.0f GB/s per GPU %s\n", n, name, worst * 1e3, remote / (worst * 1e-3) / 1e9,
           e == cudaSuccess ? "" : cudaGetErrorString(e));
    return 0;
  };
  auto srcs = [&](int i) { Src s; for (int q = 0; q < n; ++q) s.p[q] = g[q] + (size_t)i * seg; return s; };
  char nm[64];
  for (int occ : {3, 4, 6}) {
    const uint64_t W = (uint64_t)sms * occ * 8;
    const uint32_t upw = (uint32_t)((seg / 512 + W - 1) / W);
#define RUN(NS, D)                                                                                                 \
    if (n == NS) {                                                                                                 \
      snprintf(nm, 64, "SM loads depth %d, %dx%d", D, sms, occ);                                                   \
      timeit(nm, [&](int i) { k_sum<NS, D><<<sms * occ, 256, 0, st[i]>>>(srcs(i), out[i], seg, upw); });          \
    }
    RUN(2, 1) RUN(2, 2) RUN(4, 1) RUN(4, 2) RUN(8, 1)
  }
  for (int occ : {1, 2, 3}) {
    const uint64_t W = (uint64_t)sms * occ * 8;
    const uint32_t upw = (uint32_t)((seg / 512 + W - 1) / W);
#define RUNT(NS, S)                                                                                                \
    if (n == NS) {                                                                                                 \
      const int sm = 8 * S * NS * 2048;                                                                            \
      if (sm <= 200 * 1024) {                                                                                      \
        for (int i = 0; i < n; ++i) { cudaSetDevice(i); cudaFuncSetAttribute(k_sum_tma<NS, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm); } \
        snprintf(nm, 64, "TMA ring %d, %dx%d", S, sms, occ);                                                       \
        timeit(nm, [&](int i) { k_sum_tma<NS, S><<<sms * occ, 256, sm, st[i]>>>(srcs(i), out[i], seg, upw); });   \
      }                                                                                                            \
    }
    RUNT(2, 2) RUNT(2, 4) RUNT(4, 2) RUNT(4, 3) RUNT(8, 1)
  }
  // copy engines: the n-1 remote segments into a local staging buffer
  std::vector<float*> stage(n);
  for (int i = 0; i < n; ++i) { cudaSetDevice(i); CK(cudaMalloc(&stage[i], (size_t)n * seg * 4)); }
  timeit("copy engines (cudaMemcpyPeerAsync)", [&](int i) {
    for (int q = 0; q < n; ++q)
      if (q != i) cudaMemcpyPeerAsync(stage[i] + (size_t)q * seg, i, g[q] + (size_t)i * seg, q, seg * 4, st[i]);
  });
  return 0;
}
