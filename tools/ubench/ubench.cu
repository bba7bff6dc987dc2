// Micro-benchmarks of the SMEM / warp primitives the classifier, histogram and scatter
// kernels are built from (design input, not product code).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) { x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }

template <int MODE>
__global__ void kern(uint32_t* out, int iters, uint32_t mask) {
  extern __shared__ uint32_t sm[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = i * 7;
  __syncthreads();
  uint32_t acc = 0, x = hsh(threadIdx.x + blockIdx.x * 1024);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
    x = x * 1664525u + 1013904223u;
    uint32_t b = (x >> 8) & mask;
    if (MODE == 0) {            // SMEM atomicAdd, random address
      atomicAdd(&sm[b], 1u);
    } else if (MODE == 1) {     // LDS random gather
      acc += sm[b];
    } else if (MODE == 2) {     // match_any on b
      acc += __match_any_sync(0xffffffffu, b);
    } else if (MODE == 3) {     // warp-aggregated: match_any + leader RMW on warp-private counters
      uint32_t peers = __match_any_sync(0xffffffffu, b);
      int leader = __ffs(peers) - 1;
      uint32_t* h = sm + (warp & 7) * 2048;
      uint32_t base = 0;
      if (lane == leader) { base = h[b & 2047]; h[b & 2047] = base + __popc(peers); }
      base = __shfl_sync(0xffffffffu, base, leader);
      acc += base + __popc(peers & ((1u << lane) - 1));
    } else if (MODE == 4) {     // 8-bit peers via 8 ballots
      uint32_t peers = 0xffffffffu;
#pragma unroll
      for (int k = 0; k < 8; ++k) { uint32_t bb = __ballot_sync(0xffffffffu, (b >> k) & 1); peers &= ((b >> k) & 1) ? bb : ~bb; }
      acc += peers;
    } else if (MODE == 5) {     // STS random
      sm[b] = x;
    } else if (MODE == 6) {     // 2-level dependent LDS (LUT then splitter)
      uint32_t e = sm[b];
      acc += sm[(e + b) & mask];
    }
  }
  __syncthreads();
  if (MODE == 0 || MODE == 5) acc = sm[threadIdx.x];
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE>
void run(const char* name, uint32_t mask, int threads) {
  uint32_t* d; cudaMalloc(&d, 4);
  int iters = 4096; int blocks = 148 * (2048 / threads);
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  kern<MODE><<<blocks, threads, 65536>>>(d, 16, mask);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<MODE><<<blocks, threads, 65536>>>(d, iters, mask);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (double)blocks * threads * iters;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double per_clk_sm = ops / (ms * 1e-3) / 148 / 1.9e9;
  printf("%-28s mask=%5u: %8.3f ms  %7.2f Gops/s  %6.2f lane-ops/clk/SM(@1.9GHz)  err=%s\n", name, mask, ms, ops / ms / 1e6, per_clk_sm,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<1>("lds_random", 4095, 1024);
  run<1>("lds_random", 16383, 1024);
  run<1>("lds_random", 31, 1024);
  run<5>("sts_random", 4095, 1024);
  run<0>("atomics_random", 4095, 1024);
  run<0>("atomics_random", 255, 1024);
  run<0>("atomics_random", 15, 1024);
  run<2>("match_any", 4095, 1024);
  run<2>("match_any", 255, 1024);
  run<3>("match+private_rmw", 4095, 1024);
  run<3>("match+private_rmw", 255, 1024);
  run<4>("ballot8_peers", 255, 1024);
  run<6>("lds_dep2", 4095, 1024);
  return 0;
}
