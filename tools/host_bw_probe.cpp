// host_bw_probe.cpp -- host memory bandwidth on the GPU box: memcpy and the
// library's float -> f16 quantiser (fmha_host_quantize) with 1..N threads.
//   g++ -O3 -std=c++17 -pthread tools/host_bw_probe.cpp -o build/host_bw_probe -ldl
#include <dlfcn.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

int main(int argc, char** argv) {
  const size_t n = size_t(100) << 20;  // 100 M floats = 400 MB
  std::vector<float> src(n);
  std::vector<uint16_t> dst(n);
  std::vector<float> dst32(n);
  for (size_t i = 0; i < n; ++i) src[i] = float(i % 1000) * 0.001f;
  std::memset(dst.data(), 0, n * 2);
  std::memset(dst32.data(), 0, n * 4);
  auto now = [] { return std::chrono::steady_clock::now(); };
  for (int T : {1, 4, 8, 16}) {
    double best = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      auto t0 = now();
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          const size_t a = n * t / T, b = n * (t + 1) / T;
          std::memcpy(dst32.data() + a, src.data() + a, (b - a) * 4);
        });
      for (auto& x : th) x.join();
      best = std::min(best, std::chrono::duration<double>(now() - t0).count());
    }
    printf("memcpy %2d threads: %.1f GB/s (read+write)\n", T, 2.0 * n * 4 / best / 1e9);
  }
  void* lib = dlopen(argc > 1 ? argv[1] : "paper_2312_11918_b200/libfmha_b200.so", RTLD_NOW);
  if (!lib) {
    printf("dlopen failed: %s\n", dlerror());
    return 1;
  }
  auto q = reinterpret_cast<void (*)(const float*, uint16_t*, int64_t, int)>(dlsym(lib, "fmha_host_quantize"));
  auto dq = reinterpret_cast<void (*)(const uint16_t*, float*, int64_t, int)>(dlsym(lib, "fmha_host_dequantize"));
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = now();
    q(src.data(), dst.data(), int64_t(n), 0);
    double s = std::chrono::duration<double>(now() - t0).count();
    t0 = now();
    dq(dst.data(), dst32.data(), int64_t(n), 0);
    double s2 = std::chrono::duration<double>(now() - t0).count();
    printf("fmha_host_quantize f16: %.1f GB/s of float input (%.2f ms / 400 MB); dequantize %.1f GB/s of float output\n",
           n * 4 / s / 1e9, s * 1e3, n * 4 / s2 / 1e9);
  }
  return 0;
}
