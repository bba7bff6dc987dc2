// Streaming micro-benchmark (design input, not product code): how fast can persistent CTAs
// pull a 512 MiB u32 + 256 MiB u16 stream through shared memory with 1-D bulk async copies
// (double-buffered tiles), versus plain vector loads; and shared atomics on 64 counters.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
typedef uint32_t u32; typedef uint64_t u64;
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(b) : "memory"); }
__device__ __forceinline__ void bulk_g2s(void* d, const void* s, u32 b, u64* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(d)), "l"(s), "r"(b), "r"(smem_u32(bar)) : "memory"); }
__device__ __forceinline__ void mbar_wait(u64* bar, u32 ph) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}" ::"r"(smem_u32(bar)), "r"(ph) : "memory"); }

// MODE 0: TMA tiles, no work;  MODE 1: TMA tiles + read smem into regs + sum;  MODE 2: plain uint4 loads, 4 in flight
template <int MODE, int STAGES>
__global__ void __launch_bounds__(512) kstream(const u32* a, const uint16_t* b, u32 n, u32 tile, u32* out) {
  extern __shared__ __align__(16) char sm[];
  u64* bar = (u64*)sm;
  char* buf = sm + 128;
  const u32 per = tile * 6;
  u32 acc = 0;
  const u32 ntiles = n / tile;
  if (MODE == 2) {
    const uint4* a4 = (const uint4*)a;
    for (u32 v = blockIdx.x * 512 * 4 + threadIdx.x; v < n / 4; v += gridDim.x * 512 * 4) {
      uint4 r[4];
      #pragma unroll
      for (int u = 0; u < 4; ++u) if (v + u * 512 < n / 4) r[u] = __ldcs(a4 + v + u * 512); else r[u] = make_uint4(0,0,0,0);
      #pragma unroll
      for (int u = 0; u < 4; ++u) acc += r[u].x ^ r[u].y ^ r[u].z ^ r[u].w;
    }
    if (acc == 0x12345) out[0] = acc;
    return;
  }
  if (threadIdx.x == 0) { for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  __syncthreads();
  auto issue = [&](u32 t, u32 s) {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bar[s], tile * 6);
    bulk_g2s(buf + s * per, a + (size_t)t * tile, tile * 4, &bar[s]);
    bulk_g2s(buf + s * per + tile * 4, b + (size_t)t * tile, tile * 2, &bar[s]);
  };
  u32 it = 0;
  if (threadIdx.x == 0) for (int s = 0; s < STAGES - 1; ++s) { u32 t = blockIdx.x + s * gridDim.x; if (t < ntiles) issue(t, s); }
  for (u32 t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const u32 s = it % STAGES;
    u32 tn = t + (STAGES - 1) * gridDim.x;
    if (threadIdx.x == 0 && tn < ntiles) issue(tn, (it + STAGES - 1) % STAGES);
    mbar_wait(&bar[s], (it / STAGES) & 1);
    if (MODE == 1) {
      const u32* k = (const u32*)(buf + s * per);
      const uint16_t* id = (const uint16_t*)(buf + s * per + tile * 4);
      for (u32 o = threadIdx.x; o < tile; o += 512) acc += k[o] ^ id[o];
    }
    __syncthreads();
  }
  if (acc == 0x12345) out[0] = acc;
}

// shared atomics on NG counters (random groups), 16 per thread per round
__global__ void __launch_bounds__(512) katom(u32 ng, u32 rounds, u32* out) {
  __shared__ u32 c[1024];
  for (u32 i = threadIdx.x; i < 1024; i += 512) c[i] = 0;
  __syncthreads();
  u32 x = threadIdx.x * 2654435761u + blockIdx.x, acc = 0;
  for (u32 r = 0; r < rounds; ++r) {
    u32 g[16];
    #pragma unroll
    for (int j = 0; j < 16; ++j) { x = x * 1664525u + 1013904223u; g[j] = (x >> 10) % ng; }
    #pragma unroll
    for (int j = 0; j < 16; ++j) acc += atomicAdd(&c[g[j]], 1u);
  }
  if (acc == 0x12345) out[0] = acc;
}

int main() {
  const u32 n = 1u << 27;
  u32 *a, *out; uint16_t* b;
  cudaMalloc(&a, 4ull * n); cudaMalloc(&b, 2ull * n); cudaMalloc(&out, 64);
  cudaMemset(a, 1, 4ull * n); cudaMemset(b, 2, 2ull * n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](const char* nm, auto kern, int grid, size_t smem, u32 tile) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 512, smem>>>(a, b, n, tile, out);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) kern<<<grid, 512, smem>>>(a, b, n, tile, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-44s grid %4d tile %6u: %.3f ms  %.0f GB/s (%s)\n", nm, grid, tile, ms, 6.0 * n / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  for (u32 tile : {4096u, 8192u, 16384u}) {
    run("TMA 2 stages, no work, 1 CTA/SM", kstream<0, 2>, 148, 128 + 2 * 6 * tile, tile);
    run("TMA 2 stages, no work, 2 CTA/SM", kstream<0, 2>, 296, 128 + 2 * 6 * tile, tile);
    run("TMA 3 stages, no work, 1 CTA/SM", kstream<0, 3>, 148, 128 + 3 * 6 * tile, tile);
    run("TMA 2 stages, read smem, 1 CTA/SM", kstream<1, 2>, 148, 128 + 2 * 6 * tile, tile);
    run("TMA 2 stages, read smem, 2 CTA/SM", kstream<1, 2>, 296, 128 + 2 * 6 * tile, tile);
  }
  run("plain uint4 x4 loads (u32 stream only)", kstream<2, 2>, 148 * 4, 0, 8192);
  for (u32 ng : {64u, 128u, 1024u}) {
    cudaEventRecord(e0);
    katom<<<296, 512>>>(ng, 100, out);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double lanes = 296.0 * 512 * 16 * 100;
    printf("shared atomics, %4u counters: %.3f ms  %.2f lanes/clk/SM\n", ng, ms, lanes / (ms * 1e-3 * 1.965e9 * 148));
  }
  return 0;
}
