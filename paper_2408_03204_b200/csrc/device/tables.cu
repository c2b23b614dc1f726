// Device-resident constant tables shared by the FFT kernels.
#include <cmath>
#include <map>
#include <mutex>
#include <set>
#include <stdexcept>
#include <vector>

#include "fft_smem.cuh"
#include "launch.hpp"

namespace mgb {

namespace {
// fft_smem.cuh per-pass tables: block (m, k) = [k][NS] of exp(-2 pi i j 2^i / 2^m), fp64-exact
// values rounded to the element type.
template <typename C>
std::vector<C> pass_tables() {
  std::vector<C> t(static_cast<std::size_t>(kTwPassTotal));
  for (int m = 1; m <= 13; ++m) {
    for (int k = 1; k <= 4 && k <= m; ++k) {
      const int NS = 1 << (m - k), off = tw_pass_off(m, k);
      for (int i = 0; i < k; ++i) {
        for (int j = 0; j < NS; ++j) {
          const double a = -2.0 * 3.14159265358979323846 * static_cast<double>(j) * (1 << i) / static_cast<double>(1 << m);
          C& v = t[static_cast<std::size_t>(off + i * NS + j)];
          v.x = static_cast<decltype(v.x)>(std::cos(a));
          v.y = static_cast<decltype(v.y)>(std::sin(a));
        }
      }
    }
  }
  return t;
}
}  // namespace

const float2* twiddle_table(int device) {
  static std::mutex mu;
  static std::map<int, float2*> tables;
  std::scoped_lock lock(mu);
  auto it = tables.find(device);
  if (it != tables.end()) return it->second;
  // One allocation (float2 units): [per-pass tables (fft_smem.cuh tw_pass_off)][kTwN twiddles]
  // [kCosN doubles cos(2 pi m / 2047)][384 twiddles exp(-2 pi i k / 384)][192 float2: inverse
  // Hann covers for the reverb OLA]; the returned pointer is the kTwN table.
  std::vector<float2> pass = pass_tables<float2>();
  std::vector<float2> host(kConstFloat2s);
  for (int k = 0; k < kTwN; ++k) {
    const double a = -2.0 * 3.14159265358979323846 * static_cast<double>(k) / kTwN;
    host[static_cast<std::size_t>(k)] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
  }
  auto* cosd = reinterpret_cast<double*>(host.data() + kTwN);
  for (int m = 0; m < kCosN; ++m) cosd[m] = std::cos(2.0 * 3.14159265358979323846 * m / kCosN);
  for (int k = 0; k < 384; ++k) {
    const double a = -2.0 * 3.14159265358979323846 * k / 384.0;
    host[static_cast<std::size_t>(kTw384Off + k)] = make_float2(static_cast<float>(std::cos(a)), static_cast<float>(std::sin(a)));
  }
  for (int o = 0; o < 192; ++o) {
    // dsp.cpp:165-190: periodic Hann cover; out = cover > 1e-8 ? sum / cover : 0 (IFFT 1/384 folded in)
    const double w0 = 0.5 - 0.5 * std::cos(2.0 * 3.14159265358979323846 * o / 384.0);
    const double w1 = 0.5 - 0.5 * std::cos(2.0 * 3.14159265358979323846 * (o + 192) / 384.0);
    host[static_cast<std::size_t>(kCoverOff + o)] =
        make_float2(w0 > 1e-8 ? static_cast<float>(1.0 / (384.0 * w0)) : 0.f,
                    (w0 + w1) > 1e-8 ? static_cast<float>(1.0 / (384.0 * (w0 + w1))) : 0.f);
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  host.insert(host.begin(), pass.begin(), pass.end());
  float2* d = nullptr;
  if (cudaMalloc(&d, sizeof(float2) * host.size()) != cudaSuccess ||
      cudaMemcpy(d, host.data(), sizeof(float2) * host.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaSetDevice(prev);
    throw std::runtime_error("twiddle table upload failed");
  }
  cudaSetDevice(prev);
  tables.emplace(device, d + kTwPassTotal);
  return d + kTwPassTotal;
}

const double2* twiddle_table64(int device) {
  static std::mutex mu;
  static std::map<int, double2*> tables;
  std::scoped_lock lock(mu);
  auto it = tables.find(device);
  if (it != tables.end()) return it->second;
  std::vector<double2> host = pass_tables<double2>();
  for (int k = 0; k < kTwN; ++k) {
    const double a = -2.0 * 3.14159265358979323846 * static_cast<double>(k) / kTwN;
    host.push_back(make_double2(std::cos(a), std::sin(a)));
  }
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  double2* d = nullptr;
  if (cudaMalloc(&d, sizeof(double2) * host.size()) != cudaSuccess ||
      cudaMemcpy(d, host.data(), sizeof(double2) * host.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaSetDevice(prev);
    throw std::runtime_error("fp64 twiddle table upload failed");
  }
  cudaSetDevice(prev);
  tables.emplace(device, d + kTwPassTotal);
  return d + kTwPassTotal;
}

static bool g_fft_fp64 = false;
bool fft_fp64() { return g_fft_fp64; }
void set_fft_fp64(bool on) { g_fft_fp64 = on; }

namespace {
std::mutex g_prologue_mu;
std::set<const void*>& prologue_set() {
  static std::set<const void*> s;
  return s;
}
}  // namespace

void note_prologue_kernel(const void* fn) {
  std::scoped_lock lock(g_prologue_mu);
  prologue_set().insert(fn);
}

bool is_prologue_kernel(const void* fn) {
  std::scoped_lock lock(g_prologue_mu);
  return prologue_set().count(fn) != 0;
}

}  // namespace mgb
