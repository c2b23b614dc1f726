// Device-resident constant tables shared by the FFT kernels.
#include <cmath>
#include <map>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "fft_smem.cuh"
#include "launch.hpp"

namespace mgb {

const float2* twiddle_table(int device) {
  static std::mutex mu;
  static std::map<int, float2*> tables;
  std::scoped_lock lock(mu);
  auto it = tables.find(device);
  if (it != tables.end()) return it->second;
  // [kTwN float2 twiddles][kCosN doubles: cos(2 pi m / 2047)] in one allocation.
  std::vector<float2> host(kTwN + kCosN);
  for (int k = 0; k < kTwN; ++k) {
    const double a = -2.0 * 3.14159265358979323846 * static_cast<double>(k) / kTwN;
    host[static_cast<std::size_t>(k)] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
  }
  auto* cosd = reinterpret_cast<double*>(host.data() + kTwN);
  for (int m = 0; m < kCosN; ++m) cosd[m] = std::cos(2.0 * 3.14159265358979323846 * m / kCosN);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  float2* d = nullptr;
  if (cudaMalloc(&d, sizeof(float2) * host.size()) != cudaSuccess ||
      cudaMemcpy(d, host.data(), sizeof(float2) * host.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaSetDevice(prev);
    throw std::runtime_error("twiddle table upload failed");
  }
  cudaSetDevice(prev);
  tables.emplace(device, d);
  return d;
}

}  // namespace mgb
