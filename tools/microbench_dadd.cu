// Dependent-chain latency of DADD, F2F.F64.F32 + DADD and FADD on sm_100a (one warp, clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const float* in, double* out, long long* cyc, int n) {
  double acc = in[threadIdx.x];
  float facc = in[threadIdx.x];
  double w = in[32 + threadIdx.x];
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) acc = __dadd_rn(acc, w);
  long long t1 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) facc = __fadd_rn(facc, (float)w);
  long long t2 = clock64();
  // the K2f fold shape: load (L1-resident) + widen + add
  double acc2 = acc;
#pragma unroll 8
  for (int i = 0; i < n; ++i) acc2 = __dadd_rn(acc2, (double)__ldg(in + ((i * 32 + threadIdx.x) & 1023)));
  long long t3 = clock64();
  out[threadIdx.x] = acc + facc + acc2;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
  float* in; double* out; long long* cyc;
  cudaMalloc(&in, 4096 * 4); cudaMalloc(&out, 32 * 8); cudaMalloc(&cyc, 24);
  cudaMemset(in, 0, 4096 * 4);
  const int n = 4096;
  for (int r = 0; r < 2; ++r) k<<<1, 32>>>(in, out, cyc, n);
  long long h[3]; cudaMemcpy(h, cyc, 24, cudaMemcpyDeviceToHost);
  printf("dependent DADD: %.2f cycles; dependent FADD: %.2f cycles; load+F2F+DADD chain: %.2f cycles per add\n",
         (double)h[0] / n, (double)h[1] / n, (double)h[2] / n);
  return 0;
}
