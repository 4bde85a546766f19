// Host copy throughput from pageable memory into pinned memory, by thread count (the
// staging path of obt_predict_host for pageable features).
// Build: nvcc -O3 -o tools/memcpy_probe tools/memcpy_probe.cu
#include <chrono>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cuda_runtime.h>

int main() {
  const size_t bytes = (size_t)128 << 20, total = (size_t)4 << 30;
  std::vector<char> src(total);
  for (size_t i = 0; i < total; i += 4096) src[i] = (char)i;
  std::memset(src.data(), 1, total);
  void* dst = nullptr;
  cudaHostAlloc(&dst, bytes, cudaHostAllocPortable);
  printf("hardware_concurrency %u\n", std::thread::hardware_concurrency());
  for (int nt : {1, 2, 4, 8, 12, 16, 24, 32}) {
    auto t0 = std::chrono::steady_clock::now();
    for (size_t off = 0; off + bytes <= total; off += bytes) {
      const size_t per = bytes / nt;
      std::vector<std::thread> th;
      for (int t = 0; t < nt; ++t)
        th.emplace_back([&, t] { std::memcpy(static_cast<char*>(dst) + t * per, src.data() + off + t * per, per); });
      for (auto& x : th) x.join();
    }
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    printf("threads %2d: %.1f GB/s\n", nt, total / s / 1e9);
  }
  return 0;
}
