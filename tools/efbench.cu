// efbench.cu — ceiling of the EF pass's access pattern (read g, read r, write r := g + r in place;
// 12 B/element) at C2 size, for the launch shapes and pipelining depths k_compress could use.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/efbench tools/efbench.cu
// Run:   tools/efbench [n_floats]
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <algorithm>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ double g_sink;

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z), __fadd_rn(a.w, b.w));
}

// A: one float4 per thread, one-shot grid (n/4 threads)
__global__ void a_flat(const float4* __restrict__ g, float4* r, uint64_t n4) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n4) __stcs(r + i, add4(__ldcs(g + i), __ldcs(r + i)));
}

// B: persistent warp slabs of 512-element units (4 coalesced 128-element chunks, as k_compress),
// DEPTH units loaded ahead; TREE adds the fp64 xor-shuffle tree of |acc| per chunk
template <int DEPTH, bool TREE>
__global__ void b_slab(const float* __restrict__ g, float* r, uint64_t n, uint32_t upw) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const uint64_t u0 = w * upw;
  const uint64_t nu = n / 512;
  const uint32_t nun = u0 >= nu ? 0u : (uint32_t)min((uint64_t)upw, nu - u0);
  float4 gv[DEPTH][4], rv[DEPTH][4];
  auto load = [&](uint32_t i, int d) {
    const uint64_t base = (u0 + i) * 512 + 4 * lane;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      gv[d][c] = __ldcs(reinterpret_cast<const float4*>(g + base + c * 128));
      rv[d][c] = __ldcs(reinterpret_cast<const float4*>(r + base + c * 128));
    }
  };
#pragma unroll
  for (int d = 0; d < DEPTH; ++d)
    if (d < (int)nun) load(d, d);
  double tot = 0.0;
  for (uint32_t i = 0; i < nun; i += DEPTH) {
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      if (i + d < nun) {
        const uint64_t base = (u0 + i + d) * 512 + 4 * lane;
        float4 a[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) a[c] = add4(gv[d][c], rv[d][c]);
        if (i + d + DEPTH < nun) load(i + d + DEPTH, d);
#pragma unroll
        for (int c = 0; c < 4; ++c) __stcs(reinterpret_cast<float4*>(r + base + c * 128), a[c]);
        if (TREE) {
          double cs[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            double s = __dadd_rn(__dadd_rn((double)fabsf(a[c].x), (double)fabsf(a[c].y)),
                                 __dadd_rn((double)fabsf(a[c].z), (double)fabsf(a[c].w)));
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
            cs[c] = s;
          }
          tot = __dadd_rn(tot, __dadd_rn(__dadd_rn(cs[0], cs[1]), __dadd_rn(cs[2], cs[3])));
        }
      }
    }
  }
  if (tot == 1.2345) g_sink = tot;
}

// C: per-warp TMA bulk ring for g and r (2 KB each per unit), STAGES deep; sum from smem,
// write with per-lane streaming stores
template <int STAGES, bool TREE>
__global__ void c_tma(const float* __restrict__ g, float* r, uint64_t n, uint32_t upw) {
  extern __shared__ __align__(128) float4 smem[];
  __shared__ __align__(8) uint64_t bars[8][STAGES];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + warp;
  const uint64_t u0 = w * upw;
  const uint64_t nu = n / 512;
  const uint32_t nun = u0 >= nu ? 0u : (uint32_t)min((uint64_t)upw, nu - u0);
  float4* ring = smem + (size_t)warp * STAGES * 256;  // per stage: 128 float4 of g, 128 of r
  if (lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  auto issue = [&](uint32_t i, int s) {
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
    uint32_t dg = (uint32_t)__cvta_generic_to_shared(ring + s * 256);
    uint32_t dr = (uint32_t)__cvta_generic_to_shared(ring + s * 256 + 128);
    const uint64_t base = (u0 + i) * 512;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(4096));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dg),
                 "l"(g + base), "r"(2048), "r"(b) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dr),
                 "l"(r + base), "r"(2048), "r"(b) : "memory");
  };
  if (lane == 0)
    for (int s = 0; s < STAGES && s < (int)nun; ++s) issue(s, s);
  uint32_t phase = 0;
  double tot = 0.0;
  for (uint32_t i = 0; i < nun; ++i) {
    const int s = (int)(i % STAGES);
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bars[warp][s]);
    uint32_t done = 0;
    while (!done) {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(b), "r"((phase >> s) & 1u));
    }
    phase ^= 1u << s;
    float4 a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = add4(ring[s * 256 + c * 32 + lane], ring[s * 256 + 128 + c * 32 + lane]);
    __syncwarp();
    if (lane == 0 && i + STAGES < nun) issue(i + STAGES, s);
    const uint64_t base = (u0 + i) * 512 + 4 * lane;
#pragma unroll
    for (int c = 0; c < 4; ++c) __stcs(reinterpret_cast<float4*>(r + base + c * 128), a[c]);
    if (TREE) {
      double cs[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double sm = __dadd_rn(__dadd_rn((double)fabsf(a[c].x), (double)fabsf(a[c].y)),
                              __dadd_rn((double)fabsf(a[c].z), (double)fabsf(a[c].w)));
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) sm = __dadd_rn(sm, __shfl_xor_sync(0xffffffffu, sm, off));
        cs[c] = sm;
      }
      tot = __dadd_rn(tot, __dadd_rn(__dadd_rn(cs[0], cs[1]), __dadd_rn(cs[2], cs[3])));
    }
  }
  if (tot == 1.2345) g_sink = tot;
}


// D: persistent, CTA-contiguous runs, warps interleaved by unit inside the CTA's run (MODE 0), or
// grid-interleaved units: unit u -> warp u mod W (MODE 1)
template <int MODE>
__global__ void d_inter(const float* __restrict__ g, float* r, uint64_t n, uint32_t upc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t nu = n / 512;
  uint64_t u, stride, end;
  if (MODE == 0) {
    const uint64_t c0 = (uint64_t)blockIdx.x * upc;
    u = c0 + warp; stride = 8; end = min(nu, c0 + upc);
  } else {
    u = (uint64_t)blockIdx.x * 8 + warp; stride = (uint64_t)gridDim.x * 8; end = nu;
  }
  double tot = 0.0;
  for (; u < end; u += stride) {
    const uint64_t base = u * 512 + 4 * lane;
    float4 gv[4], rv[4], a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      gv[c] = __ldcs(reinterpret_cast<const float4*>(g + base + c * 128));
      rv[c] = __ldcs(reinterpret_cast<const float4*>(r + base + c * 128));
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = add4(gv[c], rv[c]);
#pragma unroll
    for (int c = 0; c < 4; ++c) __stcs(reinterpret_cast<float4*>(r + base + c * 128), a[c]);
    double cs[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double s = __dadd_rn(__dadd_rn((double)fabsf(a[c].x), (double)fabsf(a[c].y)),
                           __dadd_rn((double)fabsf(a[c].z), (double)fabsf(a[c].w)));
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
      cs[c] = s;
    }
    tot = __dadd_rn(tot, __dadd_rn(__dadd_rn(cs[0], cs[1]), __dadd_rn(cs[2], cs[3])));
  }
  if (tot == 1.2345) g_sink = tot;
}

// E: the persistent warp-slab layout with the fp64 tree (as k_compress's EF pass) plus a TMA bulk
// prefetch into L2 of the units PF ahead (g and r, 2 KB each, issued by lane 0; no registers held)
template <int PF>
__global__ void e_slab_pf(const float* __restrict__ g, float* r, uint64_t n, uint32_t upw) {
  const int lane = threadIdx.x & 31;
  const uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const uint64_t u0 = w * upw;
  const uint64_t nu = n / 512;
  const uint32_t nun = u0 >= nu ? 0u : (uint32_t)min((uint64_t)upw, nu - u0);
  auto pf = [&](uint32_t i) {
    if (lane == 0 && i < nun) {
      const uint64_t b = (u0 + i) * 512;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g + b), "r"(2048) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(r + b), "r"(2048) : "memory");
    }
  };
  for (int q = 1; q <= PF; ++q) pf(q);
  double tot = 0.0;
  for (uint32_t i = 0; i < nun; ++i) {
    pf(i + PF + 1);
    const uint64_t base = (u0 + i) * 512 + 4 * lane;
    float4 gv[4], rv[4], a[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      gv[c] = __ldcs(reinterpret_cast<const float4*>(g + base + c * 128));
      rv[c] = __ldcs(reinterpret_cast<const float4*>(r + base + c * 128));
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) a[c] = add4(gv[c], rv[c]);
#pragma unroll
    for (int c = 0; c < 4; ++c) __stcs(reinterpret_cast<float4*>(r + base + c * 128), a[c]);
    double cs[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double sm = __dadd_rn(__dadd_rn((double)fabsf(a[c].x), (double)fabsf(a[c].y)),
                            __dadd_rn((double)fabsf(a[c].z), (double)fabsf(a[c].w)));
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) sm = __dadd_rn(sm, __shfl_xor_sync(0xffffffffu, sm, off));
      cs[c] = sm;
    }
    tot = __dadd_rn(tot, __dadd_rn(__dadd_rn(cs[0], cs[1]), __dadd_rn(cs[2], cs[3])));
  }
  if (tot == 1.2345) g_sink = tot;
}

int main(int argc, char** argv) {
  uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 25600000ull;
  const int NB = 6;  // rotate through fresh (g, r) pairs: 6 x 205 MB, beyond L2
  float *g[NB], *r[NB];
  for (int b = 0; b < NB; ++b) {
    CK(cudaMalloc(&g[b], n * 4));
    CK(cudaMalloc(&r[b], n * 4));
    CK(cudaMemset(g[b], 0, n * 4));
    CK(cudaMemset(r[b], 0, n * 4));
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = 12.0 * n;
  auto timeit = [&](const char* name, auto launch) {
    float best = 1e9, sum = 0;
    const int IT = 30;
    for (int it = 0; it < IT; ++it) {
      const int b = it % NB;
      cudaEventRecord(e0);
      launch(g[b], r[b]);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 6) { best = std::min(best, ms); sum += ms; }
    }
    cudaError_t e = cudaGetLastError();
    const float mean = sum / (IT - 6);
    printf("%-30s best %7.2f us %6.0f GB/s   mean %7.2f us %6.0f GB/s %s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9,
           mean * 1e3, bytes / (mean * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
  };
  const uint64_t n4 = n / 4;
  timeit("flat 1xfloat4/thread", [&](float* gg, float* rr) {
    a_flat<<<(unsigned)((n4 + 255) / 256), 256>>>(reinterpret_cast<float4*>(gg), reinterpret_cast<float4*>(rr), n4);
  });
  const uint64_t nu = n / 512;
  char nm[96];
  for (int occ : {2, 3, 4, 6, 8}) {
    const uint64_t W = (uint64_t)sms * occ * 8;
    const uint32_t upw = (uint32_t)((nu + W - 1) / W);
    snprintf(nm, 96, "slab d1 %dx%d", sms, occ);
    timeit(nm, [&](float* gg, float* rr) { b_slab<1, false><<<sms * occ, 256>>>(gg, rr, n, upw); });
    snprintf(nm, 96, "slab d1 tree %dx%d", sms, occ);
    timeit(nm, [&](float* gg, float* rr) { b_slab<1, true><<<sms * occ, 256>>>(gg, rr, n, upw); });
    snprintf(nm, 96, "slab d2 %dx%d", sms, occ);
    timeit(nm, [&](float* gg, float* rr) { b_slab<2, false><<<sms * occ, 256>>>(gg, rr, n, upw); });
    snprintf(nm, 96, "slab d2 tree %dx%d", sms, occ);
    timeit(nm, [&](float* gg, float* rr) { b_slab<2, true><<<sms * occ, 256>>>(gg, rr, n, upw); });
  }
  for (int occ : {3, 4, 6, 8}) {
    const uint32_t G = sms * occ;
    const uint32_t upc = (uint32_t)((nu + G - 1) / G);
    snprintf(nm, 96, "cta-interleaved tree %dx%d", sms, occ);
    timeit(nm, [&](float* gg, float* rr) { d_inter<0><<<G, 256>>>(gg, rr, n, upc); });
    snprintf(nm, 96, "grid-interleaved tree %dx%d", sms, occ);
    timeit(nm, [&](float* gg, float* rr) { d_inter<1><<<G, 256>>>(gg, rr, n, upc); });
  }
  for (int occ : {1, 2, 3}) {
    const uint64_t W = (uint64_t)sms * occ * 8;
    const uint32_t upw = (uint32_t)((nu + W - 1) / W);
    snprintf(nm, 96, "tma s4 tree %dx%d", sms, occ);
    cudaFuncSetAttribute(c_tma<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 4 * 4096);
    timeit(nm, [&](float* gg, float* rr) { c_tma<4, true><<<sms * occ, 256, 8 * 4 * 4096>>>(gg, rr, n, upw); });
    if (occ <= 2) {
      snprintf(nm, 96, "tma s6 tree %dx%d", sms, occ);
      cudaFuncSetAttribute(c_tma<6, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 6 * 4096);
      timeit(nm, [&](float* gg, float* rr) { c_tma<6, true><<<sms * occ, 256, 8 * 6 * 4096>>>(gg, rr, n, upw); });
    }
  }
  for (int occ : {3}) {
    const uint64_t W = (uint64_t)sms * occ * 8;
    const uint32_t upw = (uint32_t)((nu + W - 1) / W);
    snprintf(nm, 96, "slab d1 tree %dx%d (again)", sms, occ);
    timeit(nm, [&](float* gg, float* rr) { b_slab<1, true><<<sms * occ, 256>>>(gg, rr, n, upw); });
    snprintf(nm, 96, "slab tree + L2 prefetch +1 %dx%d", sms, occ);
    timeit(nm, [&](float* gg, float* rr) { e_slab_pf<0><<<sms * occ, 256>>>(gg, rr, n, upw); });
    snprintf(nm, 96, "slab tree + L2 prefetch +2 %dx%d", sms, occ);
    timeit(nm, [&](float* gg, float* rr) { e_slab_pf<1><<<sms * occ, 256>>>(gg, rr, n, upw); });
    snprintf(nm, 96, "slab tree + L2 prefetch +4 %dx%d", sms, occ);
    timeit(nm, [&](float* gg, float* rr) { e_slab_pf<3><<<sms * occ, 256>>>(gg, rr, n, upw); });
  }
  return 0;
}
