// Host-side sample conversion for RenderPipeline's double-audio path (the reference's
// AudioBuffer is double, `audio_buffer.hpp:7-32`; the device arena is fp32). Converting on
// the host halves the PCIe bytes of every source. The f64 -> f32 direction streams into
// pinned staging that only the DMA engine reads back, so it uses non-temporal stores (no
// read-for-ownership of the staging lines, no cache pollution); AVX-512 when the CPU has
// it, a plain loop otherwise.
#include "host/convert.hpp"

#include <immintrin.h>

#include <cstdint>

namespace mixgraph::hostconv {

namespace {

__attribute__((target("avx512f"))) void f64_to_f32_avx512(const double* src, float* dst, std::size_t n) {
  std::size_t i = 0;
  // Head until dst is 32-byte aligned (streaming stores need it).
  while (i < n && (reinterpret_cast<std::uintptr_t>(dst + i) & 31u) != 0) {
    dst[i] = static_cast<float>(src[i]);
    ++i;
  }
  for (; i + 32 <= n; i += 32) {
    const __m512d a = _mm512_loadu_pd(src + i), b = _mm512_loadu_pd(src + i + 8);
    const __m512d c = _mm512_loadu_pd(src + i + 16), d = _mm512_loadu_pd(src + i + 24);
    _mm256_stream_ps(dst + i, _mm512_cvtpd_ps(a));
    _mm256_stream_ps(dst + i + 8, _mm512_cvtpd_ps(b));
    _mm256_stream_ps(dst + i + 16, _mm512_cvtpd_ps(c));
    _mm256_stream_ps(dst + i + 24, _mm512_cvtpd_ps(d));
  }
  for (; i < n; ++i) dst[i] = static_cast<float>(src[i]);
  _mm_sfence();  // the streamed lines must be globally visible before the DMA is issued
}

void f64_to_f32_plain(const double* src, float* dst, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i) dst[i] = static_cast<float>(src[i]);
}

bool has_avx512() {
  static const bool v = __builtin_cpu_supports("avx512f");
  return v;
}

}  // namespace

void f64_to_f32(const double* src, float* dst, std::size_t n) {
  if (has_avx512()) {
    f64_to_f32_avx512(src, dst, n);
  } else {
    f64_to_f32_plain(src, dst, n);
  }
}

void f32_to_f64(const float* src, double* dst, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i) dst[i] = static_cast<double>(src[i]);
}

}  // namespace mixgraph::hostconv
