// Shared-memory Stockham FFT building blocks (sm_100a), generic over the complex element
// type: float2 (fp32) or double2 (fp64 arithmetic for the precision-critical convolutions).
//
// Replaces the reference's FFTW c2c transforms (`proj/src/dsp.cpp:46-56`) on the device.
// All sizes, radices and pass strides are compile-time so index math folds to shifts and
// the register-resident radix-R DFTs have constant twiddles. A pass reads every butterfly
// input into registers, barriers, then writes the outputs in place (Stockham auto-sort:
// natural order in, natural order out, no bit reversal). Pass twiddles
// exp(dir*2*pi*i * j*r / (Ns*R)) are read from a precomputed table (fp32 rounded from fp64,
// or fp64).
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

namespace mgb {

// Scalar type of a complex element and its constructor.
template <typename C> struct Cx;
template <> struct Cx<float2> {
  using Real = float;
  static __host__ __device__ __forceinline__ float2 mk(float re, float im) { return make_float2(re, im); }
};
template <> struct Cx<double2> {
  using Real = double;
  static __host__ __device__ __forceinline__ double2 mk(double re, double im) { return make_double2(re, im); }
};
template <typename C> using RealOf = typename Cx<C>::Real;

// fp32 complex arithmetic on Blackwell's packed f32x2 pipe (FADD2 / FMUL2 / FFMA2: both
// lanes of a float2 in one instruction, IEEE round-to-nearest per lane, so every value equals
// the scalar operation's). ptxas folds lane swaps, broadcasts and per-lane negations into the
// operands (R.F32x2.LO_HI, R.F32, -R.NP), so a*i +- b is one FADD2 and a complex product two
// instructions, where the scalar forms took two and four: the FFT passes are issue-bound.
__device__ __forceinline__ float2 f2_add(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 x, y, z;\n\tmov.b64 x, {%2,%3};\n\tmov.b64 y, {%4,%5};\n\tadd.rn.f32x2 z, x, y;\n\t"
      "mov.b64 {%0,%1}, z;}" : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2_sub(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 x, y, z;\n\tmov.b64 x, {%2,%3};\n\tmov.b64 y, {%4,%5};\n\tsub.rn.f32x2 z, x, y;\n\t"
      "mov.b64 {%0,%1}, z;}" : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  float2 r;
  asm("{.reg .b64 x, y, z;\n\tmov.b64 x, {%2,%3};\n\tmov.b64 y, {%4,%5};\n\tmul.rn.f32x2 z, x, y;\n\t"
      "mov.b64 {%0,%1}, z;}" : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return r;
}
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  float2 r;
  asm("{.reg .b64 x, y, z, w;\n\tmov.b64 x, {%2,%3};\n\tmov.b64 y, {%4,%5};\n\tmov.b64 z, {%6,%7};\n\t"
      "fma.rn.f32x2 w, x, y, z;\n\tmov.b64 {%0,%1}, w;}"
      : "=f"(r.x), "=f"(r.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}
// a*b = a*b.x + (-a.y, a.x)*b.y: re = fma(-a.y, b.y, a.x b.x), im = fma(a.x, b.y, a.y b.x).
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return f2_fma(make_float2(-a.y, a.x), make_float2(b.y, b.y), f2_mul(a, make_float2(b.x, b.x)));
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
template <typename C>
__device__ __forceinline__ C cadd(C a, C b) { return Cx<C>::mk(a.x + b.x, a.y + b.y); }
template <typename C>
__device__ __forceinline__ C csub(C a, C b) { return Cx<C>::mk(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return f2_add(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return f2_sub(a, b); }
template <typename C>
__device__ __forceinline__ C cconj(C a) { return Cx<C>::mk(a.x, -a.y); }
template <typename C>
__device__ __forceinline__ C cscale(C a, RealOf<C> s) { return Cx<C>::mk(a.x * s, a.y * s); }
__device__ __forceinline__ float2 cscale(float2 a, float s) { return f2_mul(a, make_float2(s, s)); }
// a * s + b (one rounding per component)
template <typename C>
__device__ __forceinline__ C caxpy(C a, RealOf<C> s, C b) { return Cx<C>::mk(fma(a.x, s, b.x), fma(a.y, s, b.y)); }
__device__ __forceinline__ float2 caxpy(float2 a, float s, float2 b) { return f2_fma(a, make_float2(s, s), b); }
// a * (dir * i)
template <int DIR, typename C>
__device__ __forceinline__ C cmul_i(C a) {
  return DIR < 0 ? Cx<C>::mk(a.y, -a.x) : Cx<C>::mk(-a.y, a.x);
}

// exp(i*pi*x)
__device__ __forceinline__ float2 expi_pi(float x) {
  float s, c;
  sincospif(x, &s, &c);
  return make_float2(c, s);
}
__device__ __forceinline__ double2 expi_pi(double x) {
  double s, c;
  sincospi(x, &s, &c);
  return make_double2(c, s);
}
// Widening / narrowing between the arena's fp32 and a transform's element type.
template <typename C>
__device__ __forceinline__ C widen(float2 v) { return Cx<C>::mk(v.x, v.y); }
__device__ __forceinline__ float2 narrow(float2 v) { return v; }
__device__ __forceinline__ float2 narrow(double2 v) { return make_float2(static_cast<float>(v.x), static_cast<float>(v.y)); }

// ---- register DFTs of size R (DIT split, constant twiddles) --------------------------

template <int R, int DIR, typename C = float2>
struct Dft;

template <int DIR, typename C>
struct Dft<2, DIR, C> {
  static __device__ __forceinline__ void run(C* v) {
    const C a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <int DIR, typename C>
struct Dft<4, DIR, C> {
  static __device__ __forceinline__ void run(C* v) {
    const C t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    const C t2 = cadd(v[1], v[3]), t3 = cmul_i<DIR>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  }
};

template <int DIR, typename C>
struct Dft<8, DIR, C> {
  static __device__ __forceinline__ void run(C* v) {
    using T = RealOf<C>;
    C e[4] = {v[0], v[2], v[4], v[6]};
    C o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4, DIR, C>::run(e);
    Dft<4, DIR, C>::run(o);
    constexpr T h = static_cast<T>(0.70710678118654752440);
    // o[k] *= exp(dir*2*pi*i*k/8)
    o[1] = cmul(o[1], Cx<C>::mk(h, DIR * h));
    o[2] = cmul_i<DIR>(o[2]);
    o[3] = cmul(o[3], Cx<C>::mk(-h, DIR * h));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = cadd(e[k], o[k]);
      v[k + 4] = csub(e[k], o[k]);
    }
  }
};

template <int DIR, typename C>
struct Dft<16, DIR, C> {
  static __device__ __forceinline__ void run(C* v) {
    using T = RealOf<C>;
    C e[8], o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      e[k] = v[2 * k];
      o[k] = v[2 * k + 1];
    }
    Dft<8, DIR, C>::run(e);
    Dft<8, DIR, C>::run(o);
    // o[k] *= exp(dir*2*pi*i*k/16)
    constexpr T c1 = static_cast<T>(0.92387953251128675613), s1 = static_cast<T>(0.38268343236508977173),
                h = static_cast<T>(0.70710678118654752440);
    constexpr T cs[8] = {T(1), c1, h, s1, T(0), -s1, -h, -c1};
    constexpr T sn[8] = {T(0), s1, h, c1, T(1), c1, h, s1};
#pragma unroll
    for (int k = 1; k < 8; ++k) o[k] = cmul(o[k], Cx<C>::mk(cs[k], DIR * sn[k]));
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = cadd(e[k], o[k]);
      v[k + 8] = csub(e[k], o[k]);
    }
  }
};

template <int DIR, typename C>
struct Dft<3, DIR, C> {
  static __device__ __forceinline__ void run(C* v) {
    using T = RealOf<C>;
    constexpr T c = T(-0.5);
    constexpr T s = static_cast<T>(0.86602540378443864676) * DIR;  // sin(dir*2*pi/3)
    const C a = v[0], b = v[1], d = v[2];
    const C sum = cadd(b, d), dif = csub(b, d);
    v[0] = cadd(a, sum);
    const C m = caxpy(sum, c, a);
    const C r = cscale(Cx<C>::mk(-dif.y, dif.x), s);  // i*s*(b-d)
    v[1] = cadd(m, r);
    v[2] = csub(m, r);
  }
};

// Twiddles w[r] = exp(dir*2*pi*i * r * x / 2), r < R, for x = 2*j/(Ns*R) (so w[1] = exp(i*pi*dir*x)).
template <int R, int DIR, typename C>
__device__ __forceinline__ void pass_twiddles(RealOf<C> x, C* w) {
  using T = RealOf<C>;
  const T s = DIR * x;
  w[1] = expi_pi(s);
  if constexpr (R >= 3) w[2] = expi_pi(T(2) * s);
  if constexpr (R >= 4) w[3] = cmul(w[1], w[2]);
  if constexpr (R >= 8) {
    w[4] = expi_pi(T(4) * s);
    w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]);
    w[7] = cmul(w[3], w[4]);
  }
}

// Forward twiddle table: tw[k] = exp(-2*pi*i*k / kTwN), fp32 rounded from fp64, built once
// per device (twiddle_table() in tables.cu). Every pow2 transform up to kTwN points reads its
// pass twiddles from it (L1-resident, 64 KiB) instead of evaluating sin/cos per butterfly.
constexpr int kTwN = 8192;

// Per-pass twiddle tables, stored in the same allocation just BEFORE the kTwN table (at
// negative offsets from the pointer the kernels receive): for every pass size M = NS*R = 2^m
// (m = 1..13) and radix R = 2^k (k = 1..4, R <= M) a block [k][NS] of the power-of-two
// twiddles exp(-2 pi i j 2^i / M), j < NS, i < k (w, w^2, w^4, w^8; the others are <= 3
// products, TwBase::apply). A pass's threads (consecutive butterflies j) read consecutive
// entries — coalesced — where the strided kTwN table made every warp load touch 16-32 sectors
// (70% of a row kernel's L1 wavefronts), and a radix-8 butterfly loads 3 values, not 7.
__host__ __device__ constexpr int tw_pass_off(int m, int k) {
  int off = 0;
  for (int mm = 1; mm <= 13; ++mm) {
    for (int kk = 1; kk <= 4 && kk <= mm; ++kk) {
      if (mm == m && kk == k) return off;
      off += kk << (mm - kk);
    }
  }
  return off;
}
constexpr int kTwPassTotal = tw_pass_off(14, 1);
__host__ __device__ constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x / 2); }


// Bank-conflict-free smem layout for pow2 transforms: one float2 of padding per 16 elements.
// With the radix-16 first pass below, every Stockham pass then reads 16-aligned runs and
// writes either runs of >= 16 (NS >= 16) or the stride-17 pattern of the first pass — both
// hit 16 distinct 8-byte bank pairs per half-warp.
__host__ __device__ constexpr int sidx(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int padded(int n) { return n + (n >> 4); }

// One Stockham pass of radix R over COUNT independent transforms of size N held in smem
// at buf[f*FSTRIDE + i]; NS = product of earlier radices; NTHR threads participate.
// Twiddles exp(dir*2*pi*i * jm*r / (NS*R)) come from `tw` when given (N | kTwN), else sincospif.
// Table twiddles for one butterfly: loads w^1, w^2, w^4, w^8 (as many as R needs) from the
// forward table at stride `step` and conjugates them for the inverse transform.
template <int R, int DIR, typename C = float2>
struct TwBase {
  C w[4];
  __device__ __forceinline__ void load(const C* __restrict__ tw, int step) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if ((1 << i) < R) {
        C v = tw[step << i];
        if (DIR > 0) v.y = -v.y;
        w[i] = v;
      }
    }
  }
  // v[r] *= w^r for r = 1..R-1 (w^3 = w w^2, w^5..w^7 via w^4, w^9..w^15 via w^8: <= 3 products)
  __device__ __forceinline__ void apply(C* v) const {
    C p[16];
    p[1] = w[0];
    if constexpr (R > 2) p[2] = w[1];
    if constexpr (R > 3) p[3] = cmul(w[0], w[1]);
    if constexpr (R > 4) {
      p[4] = w[2];
      p[5] = cmul(p[1], p[4]);
      p[6] = cmul(p[2], p[4]);
      p[7] = cmul(p[3], p[4]);
    }
    if constexpr (R > 8) {
      p[8] = w[3];
#pragma unroll
      for (int r = 9; r < 16; ++r) p[r] = cmul(p[r - 8], p[8]);
    }
#pragma unroll
    for (int r = 1; r < R; ++r) v[r] = cmul(v[r], p[r]);
  }
};

// The twiddles of butterfly j of a pass (NS, R) from its per-pass table (w, w^2, w^4, w^8 of
// exp(-2 pi i j / (NS R)); TwBase::apply forms the rest).
template <int R, int NS, int DIR, typename C>
struct TwPass : TwBase<R, DIR, C> {
  __device__ __forceinline__ void load(const C* __restrict__ tw, int j) {
    const C* tp = tw - kTwPassTotal + tw_pass_off(ilog2c(NS * R), ilog2c(R));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if ((1 << i) < R) {
        C v = tp[i * NS + j];
        if (DIR > 0) v.y = -v.y;
        this->w[i] = v;
      }
    }
  }
};

// One Stockham pass of radix R over COUNT independent transforms of size N held in smem
// at buf[f*fstride + i] (padded layout when PAD); NS = product of earlier radices; NTHR
// threads participate. Twiddles exp(dir*2*pi*i * jm*r / (NS*R)) come from the table `tw`
// (TWN entries) when given, else sincospif; table loads are issued before the barrier-
// separated smem reads so their latency overlaps them.
template <int N, int R, int NS, int COUNT, int NTHR, int DIR, int TWN = kTwN, bool PAD = true, typename C>
__device__ __forceinline__ void stockham_pass(C* buf, int fstride, const C* __restrict__ tw) {
  using T = RealOf<C>;
  constexpr int M = N / R;                 // butterflies per transform
  constexpr int TOTAL = COUNT * M;
  constexpr int PER = (TOTAL + NTHR - 1) / NTHR;
  const int tid = threadIdx.x;
  C v[PER][R];
  // When the threads cover whole transforms (NTHR a multiple of M), a thread's butterfly index
  // j is the same for every q (one butterfly per transform): its twiddles are loaded once, not
  // PER times (the repeated table loads were most of the L1 traffic of the row kernels).
  constexpr bool kSharedJ = NTHR % M == 0;
  constexpr int NTW = kSharedJ ? 1 : PER;
  // kTwN-table transforms read the per-pass tables; others (fft_384) the strided table.
  using TW = std::conditional_t<TWN == kTwN, TwPass<R, NS, DIR, C>, TwBase<R, DIR, C>>;
  TW twb[NTW];
  if constexpr (NS > 1) {
    if (tw != nullptr) {
#pragma unroll
      for (int q = 0; q < NTW; ++q) {
        const int b = tid + q * NTHR;
        if (kSharedJ || TOTAL % NTHR == 0 || b < TOTAL) {
          const int j = b % M;
          if constexpr (TWN == kTwN) twb[q].load(tw, j % NS);
          else twb[q].load(tw, (j % NS) * (TWN / (NS * R)));
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int b = tid + q * NTHR;
    if (TOTAL % NTHR == 0 || b < TOTAL) {
      const int f = b / M, j = b - f * M;
      const C* base = buf + f * fstride;
      if constexpr (PAD && M % 16 == 0) {
        // j + r*M with M a multiple of 16: sidx(j + r*M) = sidx(j) + r*padded(M), so every
        // load is one base register plus an immediate offset (no per-element index math).
        const C* lb = base + sidx(j);
#pragma unroll
        for (int r = 0; r < R; ++r) v[q][r] = lb[r * padded(M)];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[q][r] = base[PAD ? sidx(j + r * M) : j + r * M];
      }
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
        if (tw != nullptr) {
          twb[kSharedJ ? 0 : q].apply(v[q]);
        } else {
          C w[R];
          pass_twiddles<R, DIR, C>(T(2) * static_cast<T>(jm) / static_cast<T>(NS * R), w);
#pragma unroll
          for (int r = 1; r < R; ++r) v[q][r] = cmul(v[q][r], w[r]);
        }
      }
      Dft<R, DIR, C>::run(v[q]);
      C* base = buf + f * fstride;
      const int o0 = (j / NS) * NS * R + jm;
      if constexpr (PAD && NS % 16 == 0) {
        C* sb = base + sidx(o0);  // o0 + r*NS, NS a multiple of 16: immediate offsets
#pragma unroll
        for (int r = 0; r < R; ++r) sb[r * padded(NS)] = v[q][r];
      } else if constexpr (PAD && NS == 1 && R == 16) {
        C* sb = base + 17 * j;    // o0 = 16 j: sidx(16 j + r) = 17 j + r
#pragma unroll
        for (int r = 0; r < R; ++r) sb[r] = v[q][r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) base[PAD ? sidx(o0 + r * NS) : o0 + r * NS] = v[q][r];
      }
    }
  }
  __syncthreads();
}

// Power-of-two FFT on the padded layout: a radix-16 first pass, then radix-8 passes,
// finishing with radix 4/2 (or 4+4 when 16 remain). Element i of transform f lives at
// buf[f*fstride + sidx(i)].
template <int LOG2N, int LOGNS, int COUNT, int NTHR, int DIR, typename C>
struct Pow2Fft {
  static __device__ __forceinline__ void run(C* buf, int fstride, const C* tw) {
    constexpr int REM = LOG2N - LOGNS;
    if constexpr (REM > 0) {
      constexpr int RL = (LOGNS == 0 && REM >= 4) ? 4 : ((REM == 4 || REM == 2) ? 2 : (REM == 1 ? 1 : 3));
      stockham_pass<(1 << LOG2N), (1 << RL), (1 << LOGNS), COUNT, NTHR, DIR>(buf, fstride, tw);
      Pow2Fft<LOG2N, LOGNS + RL, COUNT, NTHR, DIR, C>::run(buf, fstride, tw);
    }
  }
};

template <int LOG2N, int COUNT, int NTHR, int DIR, typename C>
__device__ __forceinline__ void fft_pow2(C* buf, int fstride, const C* tw) {
  static_assert((1 << LOG2N) <= kTwN, "pow2 smem FFT larger than the twiddle table");
  Pow2Fft<LOG2N, 0, COUNT, NTHR, DIR, C>::run(buf, fstride, tw);
}

// ---- register-ended transforms ------------------------------------------------------------
// The same pass plan with its first and/or last pass done straight from / into registers, so
// the staging smem store before the first pass and the smem read after the last one (and
// their barriers) disappear: a thread that loaded the 16 inputs of a radix-16 first-pass
// butterfly from global memory transforms them at once, and a thread that holds the R
// outputs of a last-pass butterfly writes them to global memory (twiddled) directly.
__host__ __device__ constexpr int pow2_rl(int log2n, int logns) {
  return (logns == 0 && log2n - logns >= 4) ? 4
         : ((log2n - logns == 4 || log2n - logns == 2) ? 2 : (log2n - logns == 1 ? 1 : 3));
}
__host__ __device__ constexpr int pow2_last_logns(int log2n) {
  int ns = 0;
  while (ns + pow2_rl(log2n, ns) < log2n) ns += pow2_rl(log2n, ns);
  return ns;
}
template <int LOG2N>
struct Pow2Plan {
  static constexpr int kLastLogNs = pow2_last_logns(LOG2N);
  static constexpr int kLastNs = 1 << kLastLogNs;         // butterflies per transform in the last pass
  static constexpr int kLastR = 1 << (LOG2N - kLastLogNs);
  static constexpr int kFirstM = (1 << LOG2N) / 16;        // butterflies per transform in the first pass
  static_assert(LOG2N >= 6 && pow2_rl(LOG2N, 0) == 4 && kLastLogNs >= 4, "register-ended plan needs 2+ passes");
};

template <int LOG2N, int LOGNS, int LOGEND, int COUNT, int NTHR, int DIR, typename C>
struct Pow2FftRange {
  static __device__ __forceinline__ void run(C* buf, int fstride, const C* tw) {
    if constexpr (LOGNS < LOGEND) {
      constexpr int RL = pow2_rl(LOG2N, LOGNS);
      stockham_pass<(1 << LOG2N), (1 << RL), (1 << LOGNS), COUNT, NTHR, DIR>(buf, fstride, tw);
      Pow2FftRange<LOG2N, LOGNS + RL, LOGEND, COUNT, NTHR, DIR, C>::run(buf, fstride, tw);
    }
  }
};

// First pass (radix 16, no twiddles) of butterfly j of the transform at `base`:
// v[r] = element j + r*N/16 on entry. Writes the pass outputs; the caller barriers.
template <int DIR, typename C>
__device__ __forceinline__ void fft_first_from_regs(C (&v)[16], C* base, int j) {
  Dft<16, DIR, C>::run(v);
  C* sb = base + 17 * j;  // outputs 16 j + r: sidx(16 j + r) = 17 j + r
#pragma unroll
  for (int r = 0; r < 16; ++r) sb[r] = v[r];
}

// Passes between the first and the last (they start and end with a barrier).
template <int LOG2N, int COUNT, int NTHR, int DIR, typename C>
__device__ __forceinline__ void fft_middle(C* buf, int fstride, const C* tw) {
  Pow2FftRange<LOG2N, 4, Pow2Plan<LOG2N>::kLastLogNs, COUNT, NTHR, DIR, C>::run(buf, fstride, tw);
}

// Every pass after the first (the first ran from registers; starts and ends with a barrier).
template <int LOG2N, int COUNT, int NTHR, int DIR, typename C>
__device__ __forceinline__ void fft_after_first(C* buf, int fstride, const C* tw) {
  Pow2FftRange<LOG2N, 4, LOG2N, COUNT, NTHR, DIR, C>::run(buf, fstride, tw);
}

// Every pass but the last (smem in, smem out; for a transform whose input was staged in smem).
template <int LOG2N, int COUNT, int NTHR, int DIR, typename C>
__device__ __forceinline__ void fft_all_but_last(C* buf, int fstride, const C* tw) {
  Pow2FftRange<LOG2N, 0, Pow2Plan<LOG2N>::kLastLogNs, COUNT, NTHR, DIR, C>::run(buf, fstride, tw);
}

// Last pass of butterfly j (< kLastNs) of the transform at `base`: on return v[r] = output
// element j + r*kLastNs (reads smem after the previous pass's barrier; writes nothing).
template <int LOG2N, int DIR, typename C>
__device__ __forceinline__ void fft_last_to_regs(const C* base, int j, const C* __restrict__ tw,
                                                 C (&v)[Pow2Plan<LOG2N>::kLastR]) {
  constexpr int NS = Pow2Plan<LOG2N>::kLastNs, R = Pow2Plan<LOG2N>::kLastR;
  TwPass<R, NS, DIR, C> twb;
  twb.load(tw, j);
  const C* lb = base + sidx(j);  // inputs j + r*NS, NS a multiple of 16: immediate offsets
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = lb[r * padded(NS)];
  twb.apply(v);
  Dft<R, DIR, C>::run(v);
}

// 384 = 16 * 8 * 3 (reverb STFT frames); tw384[k] = exp(-2*pi*i*k/384), usually in smem.
// Element i of transform f lives at buf[f*fstride + sidx(i)] (padded layout). Three passes with
// NS = 1, 16, 128 — every store run 16-aligned (the 3*8*4*4 plan's NS = 3 and 24 passes were
// bank-conflicted, as were its NS = 24 twiddle reads).
template <int COUNT, int NTHR, int DIR, typename C>
__device__ __forceinline__ void fft_384(C* buf, int fstride, const C* tw384) {
  stockham_pass<384, 16, 1, COUNT, NTHR, DIR, 384>(buf, fstride, tw384);
  stockham_pass<384, 8, 16, COUNT, NTHR, DIR, 384>(buf, fstride, tw384);
  stockham_pass<384, 3, 128, COUNT, NTHR, DIR, 384>(buf, fstride, tw384);
}

}  // namespace mgb
