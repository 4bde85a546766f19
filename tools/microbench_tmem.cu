// Can tensor memory serve the apply kernel's bucket words next to the shared-memory
// pipe?  Measures tcgen05.ld (32x32b shape: each thread reads columns of its own TMEM
// lane) throughput per SM, conflict-free LDS throughput, and the two interleaved.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_tmem tools/microbench_tmem.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_cycles[1024];
__device__ unsigned long long g_sink[4096];
constexpr int ITERS = 1024;

template <int X> __device__ __forceinline__ void tld(uint32_t taddr, uint32_t (&r)[X]);
template <> __device__ __forceinline__ void tld<1>(uint32_t a, uint32_t (&r)[1]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(a));
}
template <> __device__ __forceinline__ void tld<2>(uint32_t a, uint32_t (&r)[2]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(a));
}
template <> __device__ __forceinline__ void tld<4>(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void twait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// MODE 0: tcgen05.ld only; 1: LDS only; 2: both interleaved (B of each per batch)
template <int MODE, int X, int B>
__global__ void k_bench(int cols_per_warp_group) {
  __shared__ uint32_t tbase;
  __shared__ __align__(16) uint32_t table[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) table[i] = i * 2654435761u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * cols_per_warp_group);
  const uint32_t my = smem_u32(table) + 4 * (threadIdx.x & 1023);
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    uint32_t r[B][X];
    uint32_t s[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const uint32_t col = (uint32_t)((it * 7 + b * 5) & 31) * X;
      if (MODE != 1) tld<X>(base + col, r[b]);
      if (MODE != 0) asm volatile("ld.shared.u32 %0, [%1];" : "=r"(s[b]) : "r"(my + 512u * ((it + b) & 3)));
    }
    if (MODE != 1) twait();
#pragma unroll
    for (int b = 0; b < B; ++b) {
      if (MODE != 1)
#pragma unroll
        for (int x = 0; x < X; ++x) acc ^= r[b][x];
      if (MODE != 0) acc += s[b];
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (acc == 42u) g_sink[threadIdx.x] = acc + lane;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

template <int MODE, int X, int B>
int run(const char* name, int sms, int threads) {
  const int groups = (threads / 32 + 3) / 4;
  const int cols = 512 / groups;
  k_bench<MODE, X, B><<<sms, threads>>>(cols);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  k_bench<MODE, X, B><<<sms, threads>>>(cols);
  CK(cudaDeviceSynchronize());
  unsigned long long cyc[1024];
  CK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * sms));
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += (double)cyc[i];
  mean /= sms;
  const double warps = threads / 32.0;
  const double tmem_bytes = MODE != 1 ? warps * ITERS * B * X * 128.0 : 0;
  const double lds_bytes = MODE != 0 ? warps * ITERS * B * 128.0 : 0;
  printf("%-28s threads=%4d cycles=%9.0f  TMEM B/clk/SM=%7.1f  LDS B/clk/SM=%7.1f  insts/clk/SM=%5.2f\n", name, threads,
         mean, tmem_bytes / mean, lds_bytes / mean, warps * ITERS * B * ((MODE != 1) + (MODE != 0)) / mean);
  return 0;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  const int sms = prop.multiProcessorCount;
  printf("device %s SMs=%d\n", prop.name, sms);
  for (int t : {128, 256, 512}) {
    run<0, 1, 8>("tcgen05.ld x1 batch8", sms, t);
    run<0, 2, 8>("tcgen05.ld x2 batch8", sms, t);
    run<0, 4, 8>("tcgen05.ld x4 batch8", sms, t);
    run<0, 1, 16>("tcgen05.ld x1 batch16", sms, t);
    run<1, 1, 8>("lds.u32 batch8", sms, t);
    run<2, 1, 8>("tcgen05.ld x1 + lds batch8", sms, t);
    run<2, 1, 16>("tcgen05.ld x1 + lds batch16", sms, t);
  }
  return 0;
}
