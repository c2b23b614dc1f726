// FFTW3-API stand-in (test infrastructure for the reference oracle; see fftw3.h).
//
// Restates FFTW's c2c contract: X[k] = sum_n x[n] * exp(sign * 2*pi*i * n*k / N), unscaled,
// for any N >= 1. Algorithm: mixed-radix Stockham auto-sort (radix 4, 2, 3, 5 and direct
// O(R^2) butterflies for larger prime factors such as 23 and 89 in N = 2047), double
// precision, twiddles precomputed per plan with std::polar. The reference calls it from
// `proj/src/dsp.cpp:46-56` (fft_inplace) in place, from several threads once plans exist,
// so execution uses only per-call scratch.
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstring>
#include <numbers>
#include <vector>

namespace {

using cd = std::complex<double>;

struct Pass {
  int radix = 0;
  int ns = 0;                 // product of the radices of earlier passes
  std::vector<cd> twiddle;    // [ (j % ns) * (radix-1) + (r-1) ]
  std::vector<cd> roots;      // exp(sign*2*pi*i*k/radix), k < radix (generic butterflies)
};

}  // namespace

struct oracle_fftw_plan_s {
  int n = 0;
  int sign = -1;
  std::vector<Pass> passes;
};

namespace {

std::vector<int> factorize(int n) {
  std::vector<int> f;
  while (n % 4 == 0) { f.push_back(4); n /= 4; }
  while (n % 2 == 0) { f.push_back(2); n /= 2; }
  for (int p = 3; p * p <= n; p += 2) {
    while (n % p == 0) { f.push_back(p); n /= p; }
  }
  if (n > 1) f.push_back(n);
  return f;
}

inline cd cmul_g(cd a, cd b) {
  return {a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real()};
}

inline void butterfly(const Pass& pass, cd* v, int sign) {
  const int R = pass.radix;
  if (R == 2) {
    cd a = v[0], b = v[1];
    v[0] = a + b;
    v[1] = a - b;
    return;
  }
  if (R == 4) {
    cd t0 = v[0] + v[2], t1 = v[0] - v[2], t2 = v[1] + v[3];
    cd d = v[1] - v[3];
    cd t3 = sign < 0 ? cd(d.imag(), -d.real()) : cd(-d.imag(), d.real());  // d * (sign*i)
    v[0] = t0 + t2;
    v[2] = t0 - t2;
    v[1] = t1 + t3;
    v[3] = t1 - t3;
    return;
  }
  cd out[128];
  cd* tmp = R <= 128 ? out : new cd[static_cast<std::size_t>(R)];
  for (int k = 0; k < R; ++k) {
    cd acc = 0.0;
    for (int r = 0; r < R; ++r) acc += cmul_g(v[r], pass.roots[static_cast<std::size_t>((static_cast<long>(r) * k) % R)]);
    tmp[k] = acc;
  }
  for (int k = 0; k < R; ++k) v[k] = tmp[k];
  if (tmp != out) delete[] tmp;
}

}  // namespace

extern "C" fftw_plan fftw_plan_dft_1d(int n, fftw_complex*, fftw_complex*, int sign, unsigned) {
  auto* p = new oracle_fftw_plan_s;
  p->n = n;
  p->sign = sign < 0 ? -1 : 1;
  if (n <= 1) return p;
  int ns = 1;
  for (int R : factorize(n)) {
    Pass pass;
    pass.radix = R;
    pass.ns = ns;
    pass.twiddle.resize(static_cast<std::size_t>(ns) * (R - 1));
    for (int j = 0; j < ns; ++j) {
      for (int r = 1; r < R; ++r) {
        const double ang = p->sign * 2.0 * std::numbers::pi * static_cast<double>(j) * r /
                           (static_cast<double>(ns) * R);
        pass.twiddle[static_cast<std::size_t>(j) * (R - 1) + (r - 1)] = std::polar(1.0, ang);
      }
    }
    if (R != 2 && R != 4) {
      pass.roots.resize(static_cast<std::size_t>(R));
      for (int k = 0; k < R; ++k) pass.roots[static_cast<std::size_t>(k)] = std::polar(1.0, p->sign * 2.0 * std::numbers::pi * k / R);
    }
    p->passes.push_back(std::move(pass));
    ns *= R;
  }
  return p;
}

namespace {

// Complex multiply without the C99 Annex G NaN/Inf recovery path (std::complex's operator*
// compiles to a __muldc3 call at -O2/-O3 without -ffast-math); results are identical for
// finite operands.
inline cd cmul(cd a, cd b) {
  return {a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real()};
}

void radix4_pass(const Pass& pass, const cd* __restrict x, cd* __restrict y, int n, int sign) {
  const int ns = pass.ns;
  const int m = n / 4;
  const int blocks = m / ns;
  for (int blk = 0; blk < blocks; ++blk) {
    const int j0 = blk * ns;
    cd* __restrict yb = y + static_cast<long>(blk) * ns * 4;
    for (int jm = 0; jm < ns; ++jm) {
      const int j = j0 + jm;
      const cd* tw = pass.twiddle.data() + static_cast<std::size_t>(jm) * 3;
      const cd a0 = x[j];
      const cd a1 = cmul(x[j + m], tw[0]);
      const cd a2 = cmul(x[j + 2L * m], tw[1]);
      const cd a3 = cmul(x[j + 3L * m], tw[2]);
      const cd t0 = a0 + a2, t1 = a0 - a2, t2 = a1 + a3, d = a1 - a3;
      const cd t3 = sign < 0 ? cd(d.imag(), -d.real()) : cd(-d.imag(), d.real());
      yb[jm] = t0 + t2;
      yb[jm + ns] = t1 + t3;
      yb[jm + 2L * ns] = t0 - t2;
      yb[jm + 3L * ns] = t1 - t3;
    }
  }
}

}  // namespace

extern "C" void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
  const int n = p->n;
  cd* src = reinterpret_cast<cd*>(in);
  cd* dst = reinterpret_cast<cd*>(out);
  if (n <= 1) {
    if (n == 1 && dst != src) dst[0] = src[0];
    return;
  }
  thread_local std::vector<cd> a, b;
  a.assign(src, src + n);
  b.resize(static_cast<std::size_t>(n));
  cd* x = a.data();
  cd* y = b.data();
  cd v[128];
  for (const Pass& pass : p->passes) {
    const int R = pass.radix;
    if (R == 4) {
      radix4_pass(pass, x, y, n, p->sign);
      std::swap(x, y);
      continue;
    }
    const int ns = pass.ns;
    const int m = n / R;
    cd* vv = R <= 128 ? v : new cd[static_cast<std::size_t>(R)];
    for (int j = 0; j < m; ++j) {
      const int jm = j % ns;
      const cd* tw = pass.twiddle.data() + static_cast<std::size_t>(jm) * (R - 1);
      vv[0] = x[j];
      for (int r = 1; r < R; ++r) vv[r] = cmul(x[j + static_cast<long>(r) * m], tw[r - 1]);
      butterfly(pass, vv, p->sign);
      const long base = static_cast<long>(j / ns) * ns * R + jm;
      for (int r = 0; r < R; ++r) y[base + static_cast<long>(r) * ns] = vv[r];
    }
    if (vv != v) delete[] vv;
    std::swap(x, y);
  }
  std::memcpy(static_cast<void*>(dst), static_cast<const void*>(x), sizeof(cd) * static_cast<std::size_t>(n));
}

extern "C" void fftw_execute(const fftw_plan) {}

extern "C" void fftw_destroy_plan(fftw_plan p) { delete p; }
