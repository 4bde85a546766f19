// Does SHFL compete with LDS for the shared-memory pipe?  Throughput per SM of
// dynamic-index SHFL, conflict-free LDS.32 and the two interleaved (1 CTA per SM).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_shfl tools/microbench_shfl.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_cycles[1024];
__device__ unsigned long long g_sink[4096];
constexpr int ITERS = 2048;

// MODE 0: SHFL only; 1: LDS only; 2: one of each per step.  8 independent chains.
template <int MODE>
__global__ void k_bench() {
  __shared__ __align__(16) uint32_t table[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) table[i] = i * 2654435761u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(table)) + 4 * lane;
  uint32_t v[8], a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { v[i] = lane * 7 + i; a[i] = 128u * i; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE != 1) v[i] = __shfl_sync(0xffffffffu, v[i], v[i] & 31) + 1;
      if (MODE != 0) {
        uint32_t s;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(s) : "r"(base + (a[i] & 0x1f80u)));
        a[i] += s & 128u;  // data-dependent next row: loads stay real and conflict-free
        a[i] += 128u;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= v[i] ^ a[i];
  if (acc == 42u) g_sink[threadIdx.x] = acc;
}

template <int MODE>
int run(const char* name, int sms, int threads) {
  k_bench<MODE><<<sms, threads>>>();
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  k_bench<MODE><<<sms, threads>>>();
  CK(cudaDeviceSynchronize());
  unsigned long long cyc[1024];
  CK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * sms));
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += (double)cyc[i];
  mean /= sms;
  const double warp_ops = threads / 32.0 * ITERS * 8;
  printf("%-18s threads=%4d cycles=%9.0f  shfl/clk/SM=%5.2f  lds/clk/SM=%5.2f\n", name, threads, mean,
         MODE != 1 ? warp_ops / mean : 0.0, MODE != 0 ? warp_ops / mean : 0.0);
  return 0;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  printf("device %s SMs=%d\n", prop.name, sms);
  for (int t : {256, 512, 1024}) {
    run<0>("shfl", sms, t);
    run<1>("lds", sms, t);
    run<2>("shfl + lds", sms, t);
  }
  return 0;
}
