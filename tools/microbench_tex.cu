// Can texture fetches run beside shared-memory loads?  Random 64-entry-table gathers via
// LDS (shared) and via TEX (tex1Dfetch on an L1-resident global table), alone and
// interleaved.  1 CTA per SM; reports gathers (warp instructions) per SM per clock.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_tex tools/microbench_tex.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_cycles[1024];
__device__ float g_sink[4096];
constexpr int ITERS = 1024;

// MODE 0: LDS gathers; 1: TEX gathers; 2: one of each per step.  8 independent chains.
template <int MODE>
__global__ void k_bench(cudaTextureObject_t tex, const float* __restrict__ table_g) {
  __shared__ float table[64 * 16];
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) table[i] = table_g[i & 63];
  __syncthreads();
  uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
  float acc = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x = x * 1664525u + 1013904223u;
      const uint32_t idx = (x >> 20) & 63u;
      if (MODE != 1) acc += table[idx + 64 * (i & 7)];
      if (MODE != 0) acc += tex1Dfetch<float>(tex, (int)(idx + 64 * ((i + 3) & 7)));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (acc == 42.f) g_sink[threadIdx.x] = acc;
}

template <int MODE>
int run(const char* name, int sms, int threads, cudaTextureObject_t tex, const float* d) {
  k_bench<MODE><<<sms, threads>>>(tex, d);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  k_bench<MODE><<<sms, threads>>>(tex, d);
  CK(cudaDeviceSynchronize());
  unsigned long long cyc[1024];
  CK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * sms));
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += (double)cyc[i];
  mean /= sms;
  const double per = threads / 32.0 * ITERS * 8;  // warp-gathers of each kind
  printf("%-14s threads=%4d cycles=%9.0f  lds/clk/SM=%5.2f  tex/clk/SM=%5.2f\n", name, threads, mean,
         MODE != 1 ? per / mean : 0.0, MODE != 0 ? per / mean : 0.0);
  return 0;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  float h[64 * 8];
  for (int i = 0; i < 64 * 8; ++i) h[i] = (float)i * 0.5f;
  float* d;
  CK(cudaMalloc(&d, sizeof(h)));
  CK(cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice));
  cudaResourceDesc rd{};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = d;
  rd.res.linear.desc = cudaCreateChannelDesc<float>();
  rd.res.linear.sizeInBytes = sizeof(h);
  cudaTextureDesc td{};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex;
  CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  printf("device %s SMs=%d\n", prop.name, sms);
  for (int t : {256, 512, 1024}) {
    run<0>("lds", sms, t, tex, d);
    run<1>("tex", sms, t, tex, d);
    run<2>("lds + tex", sms, t, tex, d);
  }
  return 0;
}
