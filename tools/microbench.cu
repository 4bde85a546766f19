// Pipe-rate microbenchmarks that shape the tree-apply kernel design.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
// Every kernel runs one CTA per SM (or as stated) and reports lane-ops per SM per cycle
// measured with clock64 inside the kernel, so the numbers are clock-independent.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_cycles[1024];
__device__ unsigned long long g_sink[1024];

constexpr int ITERS = 2048;

// F2F.F64.F32 throughput: 8 independent conversions per iteration.
__global__ void k_f2f(const float* __restrict__ seed) {
  float f[8];
  for (int i = 0; i < 8; ++i) f[i] = seed[(threadIdx.x + i) & 255];
  unsigned long long acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double d = (double)f[i];
      acc ^= (unsigned long long)__double_as_longlong(d);
      f[i] = __int_as_float(__float_as_int(f[i]) + 1);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (acc == 42) g_sink[threadIdx.x] = acc;
}

// DADD throughput: 8 independent accumulators.
__global__ void k_dadd(const float* __restrict__ seed) {
  double a[8], b[8];
  for (int i = 0; i < 8; ++i) { a[i] = seed[(threadIdx.x + i) & 255]; b[i] = seed[(threadIdx.x + 3 * i) & 255]; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __dadd_rn(a[i], b[i]);
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 42.0) g_sink[threadIdx.x] = 1;
}

// Random gather from a 64-entry table held in shared memory, element type T.
// Indices come from a per-lane LCG so they are uniformly random across lanes.
template <typename T>
__global__ void k_gather(const T* __restrict__ table_g, int entries) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* table = reinterpret_cast<T*>(smem_raw);
  for (int i = threadIdx.x; i < entries * 16; i += blockDim.x) table[i] = table_g[i % entries];
  __syncthreads();
  uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
  uint32_t acc = 0;
  const uint32_t mask = entries - 1;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x = x * 1664525u + 1013904223u;
      uint32_t idx = (x >> 20) & mask;
      T v = table[idx + (i & 3) * entries];
      if constexpr (sizeof(T) == 8) acc += (uint32_t)v ^ (uint32_t)(v >> 32);
      else acc += (uint32_t)v;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (acc == 42) g_sink[threadIdx.x] = acc;
}

// Same LCG loop with no load, to subtract the index-generation cost.
__global__ void k_gather_none(int entries) {
  uint32_t x = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
  uint32_t acc = 0;
  const uint32_t mask = entries - 1;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      x = x * 1664525u + 1013904223u;
      acc += (x >> 20) & mask;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (acc == 42) g_sink[threadIdx.x] = acc;
}

// SWAR byte-compare step of the leaf indexer: LDS.32 + IADD + SHF + LOP3 per depth.
__global__ void k_swar(int tile_words) {
  extern __shared__ __align__(16) uint32_t q[];
  for (int i = threadIdx.x; i < tile_words * 8; i += blockDim.x) q[i] = i * 0x01030507u & 0x7f7f7f7fu;
  __syncthreads();
  uint32_t idx_acc = 0;
  uint32_t f = threadIdx.x & 7;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
    uint32_t idx = 0;
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      uint32_t w = q[((f + d * 3 + it) & 7) * tile_words + threadIdx.x];
      uint32_t t = w + 0x3f3f3f3fu + d;
      idx |= (t >> (7 - d)) & (0x01010101u << d);
    }
    idx_acc += idx;
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  if (idx_acc == 42) g_sink[threadIdx.x] = idx_acc;
}

static double report(const char* name, int blocks, int threads, double lane_ops_per_thread) {
  unsigned long long cyc[1024];
  cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * blocks);
  double mean = 0; for (int i = 0; i < blocks; ++i) mean += cyc[i]; mean /= blocks;
  double per_sm_clk = lane_ops_per_thread * threads / mean;  // one CTA per SM
  printf("%-28s threads/CTA=%4d cycles=%.0f  lane-ops/SM/clk=%.2f\n", name, threads, mean, per_sm_clk);
  return per_sm_clk;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs=%d smemPerBlockOptin=%zu clock=%d kHz\n", p.name, p.multiProcessorCount,
         p.sharedMemPerBlockOptin, p.clockRate);
  int sms = p.multiProcessorCount;
  float* seed; CK(cudaMalloc(&seed, 256 * sizeof(float)));
  float hs[256]; for (int i = 0; i < 256; ++i) hs[i] = 0.001f * (i + 1);
  CK(cudaMemcpy(seed, hs, sizeof(hs), cudaMemcpyHostToDevice));
  void* tbl; CK(cudaMalloc(&tbl, 1 << 16)); CK(cudaMemset(tbl, 0x11, 1 << 16));

  for (int threads : {256, 512, 1024}) {
    k_f2f<<<sms, threads>>>(seed); CK(cudaDeviceSynchronize());
    report("F2F.F64.F32", sms, threads, 8.0 * ITERS);
    k_dadd<<<sms, threads>>>(seed); CK(cudaDeviceSynchronize());
    report("DADD", sms, threads, 8.0 * ITERS);
  }
  for (int entries : {64, 256}) {
    for (int threads : {256, 1024}) {
      printf("-- gather table of %d entries\n", entries);
      k_gather_none<<<sms, threads>>>(entries); CK(cudaDeviceSynchronize());
      report("  lcg only", sms, threads, 8.0 * ITERS);
      k_gather<uint16_t><<<sms, threads, entries * 16 * 2>>>((const uint16_t*)tbl, entries); CK(cudaDeviceSynchronize());
      report("  LDS.U16 gather", sms, threads, 8.0 * ITERS);
      k_gather<uint32_t><<<sms, threads, entries * 16 * 4>>>((const uint32_t*)tbl, entries); CK(cudaDeviceSynchronize());
      report("  LDS.32 gather", sms, threads, 8.0 * ITERS);
      k_gather<unsigned long long><<<sms, threads, entries * 16 * 8>>>((const unsigned long long*)tbl, entries); CK(cudaDeviceSynchronize());
      report("  LDS.64 gather", sms, threads, 8.0 * ITERS);
    }
  }
  for (int threads : {256, 512, 1024}) {
    k_swar<<<sms, threads, threads * 8 * 4>>>(threads); CK(cudaDeviceSynchronize());
    report("SWAR depth step (x6, 4 obj)", sms, threads, 6.0 * 4 * ITERS);
  }
  return 0;
}
