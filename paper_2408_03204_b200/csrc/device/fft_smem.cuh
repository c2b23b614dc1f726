// Shared-memory Stockham FFT building blocks (sm_100a, fp32 complex).
//
// Replaces the reference's FFTW c2c transforms (`proj/src/dsp.cpp:46-56`) on the device.
// All sizes, radices and pass strides are compile-time so index math folds to shifts and
// the register-resident radix-R DFTs have constant twiddles. A pass reads every butterfly
// input into registers, barriers, then writes the outputs in place (Stockham auto-sort:
// natural order in, natural order out, no bit reversal). Pass twiddles
// exp(dir*2*pi*i * j*r / (Ns*R)) come from sincospif (full fp32 accuracy) for the powers
// r = 1, 2, 4 (and 8) and at most two complex products for the rest.
#pragma once

#include <cuda_runtime.h>

namespace mgb {

struct c2 {
  float x, y;
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }
// a * (dir * i)
template <int DIR>
__device__ __forceinline__ float2 cmul_i(float2 a) {
  return DIR < 0 ? make_float2(a.y, -a.x) : make_float2(-a.y, a.x);
}

// exp(i*pi*x)
__device__ __forceinline__ float2 expi_pi(float x) {
  float s, c;
  sincospif(x, &s, &c);
  return make_float2(c, s);
}

// ---- register DFTs of size R (DIT split, constant twiddles) --------------------------

template <int R, int DIR>
struct Dft;

template <int DIR>
struct Dft<2, DIR> {
  static __device__ __forceinline__ void run(float2* v) {
    const float2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <int DIR>
struct Dft<4, DIR> {
  static __device__ __forceinline__ void run(float2* v) {
    const float2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    const float2 t2 = cadd(v[1], v[3]), t3 = cmul_i<DIR>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  }
};

template <int DIR>
struct Dft<8, DIR> {
  static __device__ __forceinline__ void run(float2* v) {
    float2 e[4] = {v[0], v[2], v[4], v[6]};
    float2 o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, DIR>::run(e);
    Dft<4, DIR>::run(o);
    constexpr float h = 0.70710678118654752440f;
    // o[k] *= exp(dir*2*pi*i*k/8)
    o[1] = make_float2(h * (o[1].x - DIR * o[1].y), h * (o[1].y + DIR * o[1].x));
    o[2] = cmul_i<DIR>(o[2]);
    o[3] = make_float2(h * (-o[3].x - DIR * o[3].y), h * (-o[3].y + DIR * o[3].x));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = cadd(e[k], o[k]);
      v[k + 4] = csub(e[k], o[k]);
    }
  }
};

template <int DIR>
struct Dft<3, DIR> {
  static __device__ __forceinline__ void run(float2* v) {
    constexpr float c = -0.5f;
    constexpr float s = 0.86602540378443864676f * DIR;  // sin(dir*2*pi/3)
    const float2 a = v[0], b = v[1], d = v[2];
    const float2 sum = cadd(b, d), dif = csub(b, d);
    v[0] = cadd(a, sum);
    const float2 m = make_float2(a.x + c * sum.x, a.y + c * sum.y);
    const float2 r = make_float2(-s * dif.y, s * dif.x);  // i*s*(b-d)
    v[1] = cadd(m, r);
    v[2] = csub(m, r);
  }
};

// Twiddles w[r] = exp(dir*2*pi*i * r * x / 2), r < R, for x = 2*j/(Ns*R) (so w[1] = exp(i*pi*dir*x)).
template <int R, int DIR>
__device__ __forceinline__ void pass_twiddles(float x, float2* w) {
  const float s = DIR * x;
  w[1] = expi_pi(s);
  if constexpr (R >= 3) w[2] = expi_pi(2.f * s);
  if constexpr (R >= 4) w[3] = cmul(w[1], w[2]);
  if constexpr (R >= 8) {
    w[4] = expi_pi(4.f * s);
    w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]);
    w[7] = cmul(w[3], w[4]);
  }
}

// One Stockham pass of radix R over COUNT independent transforms of size N held in smem
// at buf[f*FSTRIDE + i]; NS = product of earlier radices; NTHR threads participate.
template <int N, int R, int NS, int COUNT, int NTHR, int DIR>
__device__ __forceinline__ void stockham_pass(float2* buf, int fstride) {
  constexpr int M = N / R;                 // butterflies per transform
  constexpr int TOTAL = COUNT * M;
  constexpr int PER = (TOTAL + NTHR - 1) / NTHR;
  const int tid = threadIdx.x;
  float2 v[PER][R];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int b = tid + q * NTHR;
    if (TOTAL % NTHR == 0 || b < TOTAL) {
      const int f = b / M, j = b - f * M;
      const float2* base = buf + f * fstride;
#pragma unroll
      for (int r = 0; r < R; ++r) v[q][r] = base[j + r * M];
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int b = tid + q * NTHR;
    if (TOTAL % NTHR == 0 || b < TOTAL) {
      const int f = b / M, j = b - f * M;
      const int jm = j % NS;
      if constexpr (NS > 1) {
        float2 w[R];
        pass_twiddles<R, DIR>(2.f * static_cast<float>(jm) / static_cast<float>(NS * R), w);
#pragma unroll
        for (int r = 1; r < R; ++r) v[q][r] = cmul(v[q][r], w[r]);
      }
      Dft<R, DIR>::run(v[q]);
      float2* base = buf + f * fstride + (j / NS) * NS * R + jm;
#pragma unroll
      for (int r = 0; r < R; ++r) base[r * NS] = v[q][r];
    }
  }
  __syncthreads();
}

// Power-of-two FFT: radix-8 passes, finishing with radix 4/2 (or 4+4 when 16 remain).
template <int LOG2N, int LOGNS, int COUNT, int NTHR, int DIR>
struct Pow2Fft {
  static __device__ __forceinline__ void run(float2* buf, int fstride) {
    constexpr int REM = LOG2N - LOGNS;
    if constexpr (REM > 0) {
      constexpr int RL = (REM == 4 || REM == 2) ? 2 : (REM == 1 ? 1 : 3);
      stockham_pass<(1 << LOG2N), (1 << RL), (1 << LOGNS), COUNT, NTHR, DIR>(buf, fstride);
      Pow2Fft<LOG2N, LOGNS + RL, COUNT, NTHR, DIR>::run(buf, fstride);
    }
  }
};

template <int LOG2N, int COUNT, int NTHR, int DIR>
__device__ __forceinline__ void fft_pow2(float2* buf, int fstride) {
  Pow2Fft<LOG2N, 0, COUNT, NTHR, DIR>::run(buf, fstride);
}

// 384 = 3 * 8 * 4 * 4 (reverb STFT frames).
template <int COUNT, int NTHR, int DIR>
__device__ __forceinline__ void fft_384(float2* buf, int fstride) {
  stockham_pass<384, 3, 1, COUNT, NTHR, DIR>(buf, fstride);
  stockham_pass<384, 8, 3, COUNT, NTHR, DIR>(buf, fstride);
  stockham_pass<384, 4, 24, COUNT, NTHR, DIR>(buf, fstride);
  stockham_pass<384, 4, 96, COUNT, NTHR, DIR>(buf, fstride);
}

}  // namespace mgb
