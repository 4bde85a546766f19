// Gather-path microbenchmarks: LDS gathers vs SHFL gathers, alone and mixed.
// Indices are precomputed per lane (registers), so only the gather path is timed.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_cycles[1024];
__device__ unsigned g_sink[1 << 16];
constexpr int ITERS = 4096;

// MODE 0: 8 LDS.32 gathers from a 64-entry fp32 table
// MODE 1: 8 SHFL gathers (single register table, 32 entries)
// MODE 2: 4 LDS + 4 SHFL
// MODE 3: 8 LDS.U16 gathers from a 64-entry half table (128 B)
// MODE 4: 8 LDS.128 broadcasts (same address for the warp)
// MODE 5: 8 LDS.32 coalesced (lane-consecutive words, like bucket loads)
template <int MODE>
__global__ void k(const uint32_t* __restrict__ seed) {
  __shared__ __align__(16) uint32_t tab[64 * 4 + 1024];
  for (int i = threadIdx.x; i < 64 * 4 + 1024; i += blockDim.x) tab[i] = seed[i & 255];
  __syncthreads();
  uint32_t idx[8];
  for (int i = 0; i < 8; ++i) idx[i] = (seed[(threadIdx.x * 8 + i) & 255] * 2654435761u) >> 26;  // 0..63
  uint32_t reg = seed[threadIdx.x & 255];
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t j = idx[i];
      uint32_t v;
      if (MODE == 0) v = tab[j + (i & 3) * 64];
      else if (MODE == 1) v = __shfl_sync(0xffffffffu, reg, j);
      else if (MODE == 2) v = (i & 1) ? __shfl_sync(0xffffffffu, reg, j) : tab[j + (i & 3) * 64];
      else if (MODE == 3) v = reinterpret_cast<const uint16_t*>(tab)[j + (i & 3) * 64];
      else if (MODE == 4) { uint4 q = reinterpret_cast<const uint4*>(tab)[(i + it) & 63]; v = q.x ^ q.w; }
      else v = tab[256 + ((threadIdx.x & 31) + 32 * ((i + it) & 31))];
      acc += v;
      idx[i] = (j + v) & 63;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x12345) g_sink[threadIdx.x] = acc;
}

template <int MODE>
int run(const char* name, const uint32_t* seed, int sms, int threads) {
  k<MODE><<<sms, threads>>>(seed);
  CK(cudaDeviceSynchronize());
  unsigned long long cyc[1024];
  CK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * sms));
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += cyc[i];
  mean /= sms;
  double warp_ops = 8.0 * ITERS * (threads / 32);
  printf("%-34s threads=%4d  cycles per warp-op per SM = %.3f\n", name, threads, mean / warp_ops);
  return 0;
}

int main() {
  int sms = 148;
  uint32_t* seed;
  CK(cudaMalloc(&seed, 256 * 4));
  uint32_t h[256];
  for (int i = 0; i < 256; ++i) h[i] = i * 7919u + 13u;
  CK(cudaMemcpy(seed, h, sizeof(h), cudaMemcpyHostToDevice));
  for (int threads : {256, 512, 1024}) {
    run<0>("LDS.32 gather (64 x fp32)", seed, sms, threads);
    run<1>("SHFL.IDX gather", seed, sms, threads);
    run<2>("LDS + SHFL mixed 1:1", seed, sms, threads);
    run<3>("LDS.U16 gather (64 x fp16)", seed, sms, threads);
    run<4>("LDS.128 broadcast", seed, sms, threads);
    run<5>("LDS.32 coalesced", seed, sms, threads);
  }
  return 0;
}
