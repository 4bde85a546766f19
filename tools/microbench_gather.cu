// Shared-memory cost of random record gathers (the multi-output fold, K5): clock cycles
// per warp-wide load instruction, one CTA of 16 warps per SM, every lane a random record
// of a 1024-record table each step.  Cycles per instruction ~ wavefronts per instruction
// when the shared-memory pipe is the bound (one wavefront per clock).
//   MODE 0: 48-byte records, three LDS.128 rows per record (K5 today)
//   MODE 1: 64-byte record slots, rows visited in a lane-rotated order: step s loads row
//           (s + lane) % 4 (row 3, the padding, predicated off), four LDS.128 per record
//   MODE 2: 256-entry fp32 table, one LDS.32 per lane (the single-output fold), uniform
//   MODE 3: 64-byte slots, plain order (rows 0..2), three LDS.128
//   MODE 5: as MODE 4, rows 0-1 LDS.128 and row 2 LDS.64 (only the 40 bytes of C = 10)
//   MODE 6: 48-byte records, entropy-ordered depth-10 indices (the most uncertain level
//           in the lowest bit), three LDS.128
//   MODE 7: entropy-ordered indices, ten SoA planes of 1024 fp32 (one LDS.32 per output)
//   MODE 8: entropy-ordered indices, lane = (object j of 3, output c of 10): 30 lanes load
//           word c of record j (48-byte stride), one LDS.32 per 3 objects
//   MODE 4: 48-byte records, indices of a depth-10 oblivious tree with random splits:
//           bit d set with probability p_d, p_d uniform per "tree" (shared by the warp)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench_gather tools/microbench_gather.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ unsigned long long g_cycles[1024];
__device__ float g_sink[65536];
constexpr int ITERS = 512;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 15; x *= 0x2c1b3c6du; x ^= x >> 12; x *= 0x297a2d39u; x ^= x >> 15;
  return x;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) k_gather(int n_instr_out) {
  extern __shared__ __align__(16) float tab[];  // 64 KB
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) tab[i] = (float)i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
  uint32_t h = mix(threadIdx.x * 7919u + blockIdx.x * 104729u);
  float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      h = h * 1664525u + 1013904223u;
      const uint32_t idx = (h >> 12) & 1023u;
      float4 v;
      if constexpr (MODE == 0) {
        const uint32_t rec = base + idx * 48u;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(rec + 16u * r));
          acc0 += v.x; acc1 += v.y; acc2 += v.z; acc3 += v.w;
        }
      } else if constexpr (MODE == 1) {
        const uint32_t rec = base + idx * 64u;
#pragma unroll
        for (int s = 0; s < 4; ++s) {
          const uint32_t r = (uint32_t)(s + lane) & 3u;
          if (r != 3u) {
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(rec + 16u * r));
            acc0 += v.x; acc1 += v.y; acc2 += v.z; acc3 += v.w;
          }
        }
      } else if constexpr (MODE == 4 || MODE == 5) {
        // per-tree level biases (warp-uniform), per-lane bits
        uint32_t tr = mix((uint32_t)(it * 4 + u) * 2654435761u + blockIdx.x);
        uint32_t id = 0;
#pragma unroll
        for (int d = 0; d < 10; ++d) {
          tr = tr * 1664525u + 1013904223u;
          const uint32_t pd = tr >> 22;         // bias in 1/1024 units
          h = h * 1664525u + 1013904223u;
          id |= ((h >> 22) < pd ? 1u : 0u) << d;
        }
        const uint32_t rec = base + id * 48u;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          if (MODE == 5 && r == 2) {
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(rec + 16u * r));
            acc0 += v.x; acc1 += v.y;
          } else {
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(rec + 16u * r));
            acc0 += v.x; acc1 += v.y; acc2 += v.z; acc3 += v.w;
          }
        }
      } else if constexpr (MODE >= 6) {
        // per-tree level biases (warp-uniform) already in entropy order: |p_d - 1/2| grows
        // with d (uniform order statistics of the distance), random side
        uint32_t tr = mix((uint32_t)(it * 4 + u) * 2654435761u + blockIdx.x);
        uint32_t pd[10];
#pragma unroll
        for (int d = 0; d < 10; ++d) {
          tr = tr * 1664525u + 1013904223u;
          const uint32_t dist = 51u * d + ((tr >> 10) % 51u);  // 0..510
          pd[d] = (tr >> 31) ? 512u + dist : 512u - dist;
        }
        uint32_t id = 0;
#pragma unroll
        for (int d = 0; d < 10; ++d) {
          h = h * 1664525u + 1013904223u;
          id |= ((h >> 22) < pd[d] ? 1u : 0u) << d;
        }
        if constexpr (MODE == 6) {
          const uint32_t rec = base + id * 48u;
#pragma unroll
          for (int r = 0; r < 3; ++r) {
            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(rec + 16u * r));
            acc0 += v.x; acc1 += v.y; acc2 += v.z; acc3 += v.w;
          }
        } else if constexpr (MODE == 7) {
#pragma unroll
          for (int c = 0; c < 10; ++c) {
            float x;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(base + 4096u * c + 4u * id));
            acc0 += x;
          }
        } else {
          // lanes 10j..10j+9 take object j's record: the object's id from lane 10j
          const int j = lane / 10, c = lane % 10;
          const uint32_t idj = __shfl_sync(0xffffffffu, id, j < 3 ? 10 * j : 0);
          if (lane < 30) {
            float x;
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(base + idj * 48u + 4u * c));
            acc0 += x;
          }
        }
      } else if constexpr (MODE == 2) {
        const uint32_t a = base + (idx & 255u) * 4u;
        float x;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(a));
        acc0 += x;
      } else {
        const uint32_t rec = base + idx * 64u;
#pragma unroll
        for (int r = 0; r < 3; ++r) {
          asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(rec + 16u * r));
          acc0 += v.x; acc1 += v.y; acc2 += v.z; acc3 += v.w;
        }
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  g_sink[blockIdx.x * 512 + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

template <int MODE>
int run(const char* name, int sms, int instr_per_record) {
  CK(cudaFuncSetAttribute(k_gather<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  k_gather<MODE><<<sms, 512, 65536>>>(0);
  CK(cudaDeviceSynchronize());
  k_gather<MODE><<<sms, 512, 65536>>>(0);
  CK(cudaDeviceSynchronize());
  unsigned long long c[1024];
  CK(cudaMemcpyFromSymbol(c, g_cycles, sizeof(unsigned long long) * sms));
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += (double)c[i];
  avg /= sms;
  const double instr = 16.0 * ITERS * 4 * instr_per_record;  // warp instructions per SM
  printf("%-48s cycles/warp-instr %.2f  cycles/record %.2f\n", name, avg / instr, avg / (16.0 * ITERS * 4));
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  run<0>("48-B records, 3 x LDS.128", sms, 3);
  run<1>("64-B slots, rotated rows, 4 x LDS.128 (3 active)", sms, 4);
  run<3>("64-B slots, plain rows, 3 x LDS.128", sms, 3);
  run<2>("256 x fp32 table, LDS.32", sms, 1);
  run<4>("48-B records, depth-10 random-split indices", sms, 3);
  run<5>("  same, third row as LDS.64 (40 bytes)", sms, 3);
  run<6>("48-B records, entropy-ordered depth-10 indices", sms, 3);
  run<7>("  same indices, 10 SoA planes, 10 x LDS.32", sms, 10);
  run<8>("  same indices, lane = (object of 3, output): per 3 objects", sms, 1);
  return 0;
}
