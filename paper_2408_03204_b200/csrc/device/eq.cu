// K5/K6: equalizer — zero-phase FIR design + overlap-save FFT convolution.
//
// Reference: eq_slot `processors.cpp:65-68` -> zero_phase_fir(p, 2047) `dsp.cpp:106-136`
// (mirror the 1024 log-magnitudes, inverse DFT, circular centre, symmetric Hann) ->
// fft_convolve(ZeroPhase) `dsp.cpp:64-86` (linear convolution, (taps-1)/2 samples dropped
// from the head, zero padded edges). Same real kernel for both channels and every batch.
//
// Device plan per step:
//  1. eq_design: taps in fp64 by the equivalent cosine sum (odd N = 2047 has no pow2 FFT;
//     the sum is the exact IDFT of the real even spectrum), grid (4, slots).
//  2. eq_response: 8192-point FFT of the circularly centred taps -> real response R[k],
//     prescaled by 1/8192.
//  3. eq_conv: overlap-save, one CTA per 6146-sample output block and (slot, batch):
//     gather-sum the block's 8192-sample window (both channels packed as re/im, since the
//     kernel is real and shared), FFT, multiply by R, inverse FFT, store the 6146 samples
//     that did not wrap. Arena in -> arena out in one kernel.
#include "fft_smem.cuh"
#include "launch.hpp"

namespace mgb {

namespace {

constexpr int kN = 2047;  // kEqFirLength
constexpr int kLogFft = 13;
static_assert((1 << kLogFft) == kEqFft, "EQ FFT size");
constexpr int kEqBuf = padded(kEqFft);
constexpr int kEqOut = 6144;  // outputs per block (of the 8192 - 2046 = 6146 non-wrapped)
constexpr int kEqSmem = kEqBuf * 8;

// Taps by the exact cosine sum raw[j] = (m0 + 2 sum_{k=1}^{1023} m_k cos(2 pi k j / 2047)) / 2047
// in fp64. One warp per kDesignTpw taps j (independent recurrences interleaved for ILP);
// each lane runs 32-term Chebyshev recurrences started from the fp64 cos table (error
// ~1e-12); lanes are reduced with xor-shuffles in a fixed order.
// grid (1024 / (8 kDesignTpw), slots) x 256 threads (8 kDesignTpw taps per CTA).
constexpr int kDesignSplit = 32;
constexpr int kDesignTpw = 4;  // taps per warp
// exp of the 1024 log-magnitudes of every slot, once (fp64). grid (slots) x 1024.
__global__ void __launch_bounds__(1024) eq_mags(const double* params, double* mags) {
  const long i = static_cast<long>(blockIdx.x) * (kEqHalf + 1) + threadIdx.x;
  mags[i] = exp(params[i]);
}

__global__ void __launch_bounds__(256) eq_design(const double* __restrict__ mag_g, float* taps, const double* __restrict__ cos_tab) {
  __shared__ double mags[kEqHalf + 1];
  const int slot = blockIdx.y;
  for (int k = threadIdx.x; k <= kEqHalf; k += blockDim.x) mags[k] = __ldg(mag_g + static_cast<long>(slot) * (kEqHalf + 1) + k);
  __syncthreads();
  // Lane l sums k = 1 + l + 32 i (i < 32, k <= 1023): consecutive lanes read consecutive
  // magnitudes (no bank conflicts); the stride-32 recurrence is
  // cos((k + 32) t) = 2 cos(32 t) cos(k t) - cos((k - 32) t).
  const int lane = threadIdx.x & 31;
  const int j0 = (blockIdx.x * (256 / kDesignSplit) + threadIdx.x / kDesignSplit) * kDesignTpw;  // first tap
  double c_prev[kDesignTpw], c_cur[kDesignTpw], two_c[kDesignTpw], acc[kDesignTpw];
#pragma unroll
  for (int q = 0; q < kDesignTpw; ++q) {
    const long j = j0 + q;
    c_prev[q] = __ldg(cos_tab + (static_cast<long>(31 - lane) * j) % kN);  // cos((1 + l - 32) t)
    c_cur[q] = __ldg(cos_tab + (static_cast<long>(1 + lane) * j) % kN);
    two_c[q] = 2.0 * __ldg(cos_tab + (32L * j) % kN);
    acc[q] = 0.0;
  }
#pragma unroll 2
  for (int k = 1 + lane; k <= kEqHalf; k += 32) {
    const double m = mags[k];
#pragma unroll
    for (int q = 0; q < kDesignTpw; ++q) {
      acc[q] = fma(m, c_cur[q], acc[q]);
      const double nxt = fma(two_c[q], c_cur[q], -c_prev[q]);
      c_prev[q] = c_cur[q];
      c_cur[q] = nxt;
    }
  }
#pragma unroll
  for (int q = 0; q < kDesignTpw; ++q) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], off);
  }
  if (lane >= kDesignTpw) return;
  // lane q writes tap j0 + q
  double a = acc[0];
#pragma unroll
  for (int q = 1; q < kDesignTpw; ++q) a = lane == q ? acc[q] : a;
  const int j = j0 + lane;
  const double raw = (mags[0] + 2.0 * a) / kN;
  double s, c;
  sincospi(2.0 * (kEqHalf + j) / (kN - 1), &s, &c);
  const double w = 0.5 - 0.5 * c;  // symmetric Hann; w(half - j) == w(half + j)
  float* t = taps + static_cast<long>(slot) * 2048;
  t[kEqHalf + j] = static_cast<float>(w * raw);
  t[kEqHalf - j] = static_cast<float>(w * raw);
}

__global__ void __launch_bounds__(512) eq_response(const float* taps, float* resp, const float2* tw) {
  extern __shared__ float2 buf[];
  const int slot = blockIdx.x;
  const float* t = taps + static_cast<long>(slot) * 2048;
  for (int i = threadIdx.x; i < kEqFft; i += blockDim.x) {
    float v = 0.f;
    if (i <= kEqHalf) v = t[kEqHalf + i];
    else if (i >= kEqFft - kEqHalf) v = t[kEqHalf - (kEqFft - i)];
    buf[sidx(i)] = make_float2(v, 0.f);
  }
  __syncthreads();
  fft_pow2<kLogFft, 1, 512, -1>(buf, kEqBuf, tw);
  float* r = resp + static_cast<long>(slot) * kEqFft;
  for (int i = threadIdx.x; i < kEqFft; i += blockDim.x) r[i] = buf[sidx(i)].x * (1.f / kEqFft);
}

// Window geometry per FFT size: 8192 (6144 outputs per block, the throughput choice) or
// 4096 (2048 outputs per block: 2.2x less FFT work per CTA and 3x the CTAs, for steps whose
// 8192 grid would not fill the GPU, e.g. a 1-slot bus EQ). The taps span +-1023 < 2048, so
// the 4096-point response is exactly every other bin of the 8192-point one.
template <int LOG> struct EqWin {
  static constexpr int kFft = 1 << LOG;
  static constexpr int kOut = LOG == 13 ? 6144 : 2048;
  static constexpr int kThreads = LOG == 13 ? 512 : 256;
  static constexpr int kMinBlocks = 2;
  static constexpr int kSmem = padded(kFft) * 8;
  static_assert(kOut <= kFft - 2 * kEqHalf, "EQ block larger than the non-wrapped window");
};

// grid (blocks per signal, slots*B). Block covers outputs [out0, out0 + kOut) from the
// kFft-sample window starting at out0 - 1024; the circular convolution is exact for window
// indices [1023, kFft - 1024]. Window loads feed the first FFT pass directly and the last
// inverse pass stores directly (register-ended transforms, fft_smem.cuh), both coalesced.
template <int MODE, int LOG>
__global__ void __launch_bounds__(EqWin<LOG>::kThreads, EqWin<LOG>::kMinBlocks) eq_conv(StepArgs a, const float* resp, float2* spec) {
  using W = EqWin<LOG>;
  constexpr int kEqFft = W::kFft, kEqOut = W::kOut, kNt = W::kThreads;
  constexpr int kRs = kEqFft == 8192 ? 1 : 8192 / kEqFft;   // response bin stride
  const float rscale = static_cast<float>(kRs);            // response is prescaled by 1/8192
  extern __shared__ float2 buf[];
  const int sb = blockIdx.y;
  const int slot = sb / a.batch, b = sb - slot * a.batch;
  const int e0 = __ldg(a.row_ptr + slot), e1 = __ldg(a.row_ptr + slot + 1);
  const long out0 = static_cast<long>(blockIdx.x) * kEqOut;
  const long s0 = out0 - (kEqHalf + 1);
  const long boff = static_cast<long>(b) * 2 * a.length;
  float2* sp = spec + (static_cast<long>(sb) * gridDim.x + blockIdx.x) * kEqFft;  // MODE 1/2 scratch
  const float* rs = resp + static_cast<long>(slot) * 8192;
  if constexpr (MODE == 2) {
    // spectrum computed earlier by MODE 1: load it with the response product fused; loads
    // are issued 8 at a time ahead of their smem stores.
    constexpr int PER = kEqFft / kNt;
    static_assert(PER % 8 == 0, "eq_conv: spectrum load chunking");
#pragma unroll
    for (int q0 = 0; q0 < PER; q0 += 8) {
      float2 v[8];
      float r[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int t = threadIdx.x + (q0 + q) * kNt;
        v[q] = __ldg(sp + t);
        r[q] = __ldg(rs + kRs * t);
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) buf[sidx(threadIdx.x + (q0 + q) * kNt)] = cscale(v[q], rscale * r[q]);
    }
    __syncthreads();
  } else {
  // Gather-sum of the window straight into the radix-16 first-pass butterfly this thread
  // owns (elements t + r*N/16: consecutive threads read consecutive samples), edges
  // outermost so all 16 sample pairs are in flight at once; per element the sum runs in
  // edge order (as the reference's gather).
  constexpr int M1 = kEqFft / 16;
  static_assert(M1 == kNt, "eq_conv: threads must be the first pass's butterflies");
  float2 v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = make_float2(0.f, 0.f);
  for (int e = e0; e < e1; ++e) {
    const float* p = a.src + static_cast<long>(__ldg(a.col + e)) * a.rowstride + boff;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const long pos = s0 + threadIdx.x + r * M1;
      if (pos >= 0 && pos < a.length) {
        v[r].x += __ldg(p + pos);
        v[r].y += __ldg(p + a.length + pos);
      }
    }
  }
  fft_first_from_regs<-1>(v, buf, threadIdx.x);
  __syncthreads();
  fft_middle<LOG, 1, kNt, -1>(buf, padded(kEqFft), a.tw);
  // Last forward pass into registers: MODE 1 stores the spectrum, MODE 0 multiplies by the
  // response and writes the product back (in place: after every thread has read its inputs).
  constexpr int NS = Pow2Plan<LOG>::kLastNs, R = Pow2Plan<LOG>::kLastR, PL = NS / kNt;
  float2 o[PL][R];
#pragma unroll
  for (int p = 0; p < PL; ++p) fft_last_to_regs<LOG, -1>(buf, threadIdx.x + p * kNt, a.tw, o[p]);
  if constexpr (MODE == 1) {
#pragma unroll
    for (int p = 0; p < PL; ++p) {
#pragma unroll
      for (int r = 0; r < R; ++r) sp[threadIdx.x + p * kNt + r * NS] = o[p][r];
    }
    return;
  }
  __syncthreads();
#pragma unroll
  for (int p = 0; p < PL; ++p) {
    const int j = threadIdx.x + p * kNt;
    float2* sb = buf + sidx(j);
#pragma unroll
    for (int r = 0; r < R; ++r) sb[r * padded(NS)] = cscale(o[p][r], rscale * __ldg(rs + kRs * (j + r * NS)));
  }
  __syncthreads();
  }
  // Inverse: every pass but the last in smem, the last into registers and straight to the
  // arena (window index w = j + r*NS holds output out0 + w - 1024 for w in [1024, 1024 + kEqOut)).
  fft_all_but_last<LOG, 1, kNt, +1>(buf, padded(kEqFft), a.tw);
  constexpr int NS = Pow2Plan<LOG>::kLastNs, R = Pow2Plan<LOG>::kLastR, PL = NS / kNt;
  float* yl = a.dst + static_cast<long>(slot) * a.rowstride + boff;
  float* yr = yl + a.length;
#pragma unroll
  for (int p = 0; p < PL; ++p) {
    const int j = threadIdx.x + p * kNt;
    float2 y[R];
    fft_last_to_regs<LOG, +1>(buf, j, a.tw, y);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int w = j + r * NS;
      const long pos = out0 + w - (kEqHalf + 1);
      if (w >= kEqHalf + 1 && w < kEqHalf + 1 + kEqOut && pos < a.length) {
        yl[pos] = y[r].x;
        yr[pos] = y[r].y;
      }
    }
  }
}

}  // namespace

void eq_setup() {
  static const bool done = [] {
    cudaFuncSetAttribute(eq_response, cudaFuncAttributeMaxDynamicSharedMemorySize, kEqSmem);
    for (auto fn : {eq_conv<0, 13>, eq_conv<1, 13>, eq_conv<2, 13>, eq_conv<0, 12>}) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kEqSmem);
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    return true;
  }();
  (void)done;
}

void launch_eq_prologue(const StepArgs& a, float* taps_ws, float* resp_ws, cudaStream_t s) {
  if (a.slots == 0) return;
  eq_setup();
  // taps_ws holds [slots][2048] floats followed by [slots][1024] doubles of magnitudes.
  auto* mags = reinterpret_cast<double*>(taps_ws + 2048L * a.slots);
  note_prologue_kernel(reinterpret_cast<const void*>(eq_mags));
  note_prologue_kernel(reinterpret_cast<const void*>(eq_design));
  note_prologue_kernel(reinterpret_cast<const void*>(eq_response));
  eq_mags<<<a.slots, kEqHalf + 1, 0, s>>>(a.params, mags);
  eq_design<<<dim3(1024 / (256 / kDesignSplit * kDesignTpw), a.slots), 256, 0, s>>>(mags, taps_ws, cos_table(a.tw));
  eq_response<<<a.slots, 512, kEqSmem, s>>>(taps_ws, resp_ws, a.tw);
}

std::size_t eq_spectrum_bytes(int slots, int batch, long length) {
  return sizeof(float2) * kEqFft * static_cast<std::size_t>(slots) * batch * ((length + kEqOut - 1) / kEqOut);
}

namespace {
template <int LOG>
dim3 eq_grid(const StepArgs& a) {
  constexpr int out = EqWin<LOG>::kOut;
  return dim3(static_cast<unsigned>((a.length + out - 1) / out), static_cast<unsigned>(a.slots * a.batch));
}

int sm_count() {
  static const int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}
}  // namespace

bool eq_uses_small_window(const StepArgs& a) {
  const dim3 g = eq_grid<13>(a);
  return static_cast<long>(g.x) * g.y < sm_count();
}

void launch_eq_main(const StepArgs& a, const float* resp_ws, cudaStream_t s) {
  if (a.slots == 0 || a.batch == 0 || a.length == 0) return;
  eq_setup();
  if (eq_uses_small_window(a)) {
    eq_conv<0, 12><<<eq_grid<12>(a), EqWin<12>::kThreads, EqWin<12>::kSmem, s>>>(a, resp_ws, nullptr);
    return;
  }
  eq_conv<0, 13><<<eq_grid<13>(a), 512, kEqSmem, s>>>(a, resp_ws, nullptr);
}

void launch_eq_forward(const StepArgs& a, float2* spectrum, cudaStream_t s) {
  if (a.slots == 0 || a.batch == 0 || a.length == 0) return;
  eq_setup();
  eq_conv<1, 13><<<eq_grid<13>(a), 512, kEqSmem, s>>>(a, nullptr, spectrum);
}

void launch_eq_inverse(const StepArgs& a, const float* resp_ws, const float2* spectrum, cudaStream_t s) {
  if (a.slots == 0 || a.batch == 0 || a.length == 0) return;
  eq_setup();
  eq_conv<2, 13><<<eq_grid<13>(a), 512, kEqSmem, s>>>(a, resp_ws, const_cast<float2*>(spectrum));
}

}  // namespace mgb
