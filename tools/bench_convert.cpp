#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>
#include <atomic>
#include "host/convert.hpp"
int main(int argc, char** argv) {
  const size_t n = 16ull * 2 * (1 << 17);
  std::vector<double> src(n, 0.5);
  float* dst = static_cast<float*>(aligned_alloc(64, n * 4));
  for (int T : {1, 2, 4, 8, 12, 16}) {
    double best = 1e9;
    for (int rep = 0; rep < 20; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t) th.emplace_back([&, t] {
        size_t lo = n * t / T, hi = n * (t + 1) / T;
        mixgraph::hostconv::f64_to_f32(src.data() + lo, dst + lo, hi - lo);
      });
      for (auto& x : th) x.join();
      double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      if (ms < best) best = ms;
    }
    printf("threads %2d: %.3f ms  (%.1f GB/s read)\n", T, best, n * 8 / best / 1e6);
  }
}
