// Shared-memory cost of multi-output record gathers under the leaf indices of random-split
// oblivious trees (K5 / config 5: depth 10, C = 10 fp32 values per leaf).  Indices are
// generated BEFORE the timed loop (16 trees per lane, in registers), so the loop is loads
// and adds only; cycles per warp-wide load ~ shared-memory wavefronts per load.
//   level order: "raw" (bias per level uniform, random order) or "entropy" (the level
//   nearest p = 1/2 in bit 0: the predict path's plan_level_order)
//   layouts: A = 48-byte AoS records, three LDS.128; S = ten SoA planes, ten LDS.32;
//            L = lane = (object j of 3, output c of 10): one LDS.32 per 3 objects
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_gather2 tools/microbench_gather2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_cycles[1024];
__device__ float g_sink[65536];
constexpr int ITERS = 256;
constexpr int NT = 16;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 15; x *= 0x2c1b3c6du; x ^= x >> 12; x *= 0x297a2d39u; x ^= x >> 15;
  return x;
}

template <int LAYOUT, bool ENTROPY>
__global__ void __launch_bounds__(512, 1) k_gather() {
  extern __shared__ __align__(16) float tab[];  // 64 KB
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) tab[i] = (float)i;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  uint32_t ids[NT];
  uint32_t h = mix(threadIdx.x * 7919u + blockIdx.x * 104729u + 1u);
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    uint32_t tr = mix((uint32_t)(t + 16 * warp) * 2654435761u + blockIdx.x * 977u);
    uint32_t id = 0;
    for (int d = 0; d < 10; ++d) {
      tr = tr * 1664525u + 1013904223u;
      uint32_t pd;
      if (ENTROPY) {
        const uint32_t dist = 51u * d + ((tr >> 10) % 51u);
        pd = (tr >> 31) ? 512u + dist : 512u - dist;
      } else {
        pd = tr >> 22;
      }
      h = h * 1664525u + 1013904223u;
      id |= ((h >> 22) < pd ? 1u : 0u) << d;
    }
    if (LAYOUT == 2) id = __shfl_sync(0xffffffffu, id, lane / 10 < 3 ? 10 * (lane / 10) : 0);
    ids[t] = id;
  }
  __syncthreads();
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const uint32_t id = ids[t] ^ (uint32_t)(it & 1);  // stay data-dependent per iteration
      if constexpr (LAYOUT == 0) {
        const uint32_t rec = base + id * 48u;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          float4 v;
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(rec + 16u * r));
          acc0 += v.x; acc1 += v.y; acc2 += v.z; acc3 += v.w;
        }
      } else if constexpr (LAYOUT == 1) {
#pragma unroll
        for (int c = 0; c < 10; ++c) {
          float x;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(base + 4096u * c + 4u * id));
          acc0 += x;
        }
      } else {
        if (lane < 30) {
          float x;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(base + id * 48u + 4u * (lane % 10)));
          acc0 += x;
        }
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  g_sink[blockIdx.x * 512 + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

template <int LAYOUT, bool ENTROPY>
int run(const char* name, int sms, int instr_per_group, int records_per_group) {
  CK(cudaFuncSetAttribute(k_gather<LAYOUT, ENTROPY>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  k_gather<LAYOUT, ENTROPY><<<sms, 512, 65536>>>();
  CK(cudaDeviceSynchronize());
  k_gather<LAYOUT, ENTROPY><<<sms, 512, 65536>>>();
  CK(cudaDeviceSynchronize());
  unsigned long long c[1024];
  CK(cudaMemcpyFromSymbol(c, g_cycles, sizeof(unsigned long long) * sms));
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += (double)c[i];
  avg /= sms;
  const double groups = 16.0 * ITERS * NT;  // warp-level groups per SM
  printf("%-46s cycles/warp-load %.2f  cycles/record %.3f\n", name, avg / (groups * instr_per_group),
         avg / (groups * records_per_group));
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  run<0, false>("AoS 48 B, 3 x LDS.128, raw levels", sms, 3, 32);
  run<0, true>("AoS 48 B, 3 x LDS.128, entropy levels", sms, 3, 32);
  run<1, false>("SoA planes, 10 x LDS.32, raw levels", sms, 10, 32);
  run<1, true>("SoA planes, 10 x LDS.32, entropy levels", sms, 10, 32);
  run<2, false>("lane=(obj of 3, out), LDS.32, raw levels", sms, 1, 3);
  run<2, true>("lane=(obj of 3, out), LDS.32, entropy levels", sms, 1, 3);
  return 0;
}
