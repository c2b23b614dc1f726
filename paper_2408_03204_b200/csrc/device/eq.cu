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

__global__ void __launch_bounds__(256) eq_design(const double* params, float* taps) {
  __shared__ double cos_tab[kN];
  __shared__ double mags[kEqHalf + 1];
  const int slot = blockIdx.y;
  const double* lm = params + static_cast<long>(slot) * (kEqHalf + 1);
  for (int k = threadIdx.x; k < kN; k += blockDim.x) {
    double s, c;
    sincospi(2.0 * k / kN, &s, &c);
    cos_tab[k] = c;
  }
  for (int k = threadIdx.x; k <= kEqHalf; k += blockDim.x) mags[k] = exp(lm[k]);
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;  // 0..1023: |time index| from centre
  if (j > kEqHalf) return;
  double acc = 0.0;
  int idx = 0;  // (k*j) mod N
  for (int k = 1; k <= kEqHalf; ++k) {
    idx += j;
    if (idx >= kN) idx -= kN;
    acc = fma(mags[k], cos_tab[idx], acc);
  }
  const double raw = (mags[0] + 2.0 * acc) / kN;
  double s, c;
  sincospi(2.0 * (kEqHalf + j) / (kN - 1), &s, &c);
  const double w = 0.5 - 0.5 * c;  // symmetric Hann; w(half - j) == w(half + j)
  float* t = taps + static_cast<long>(slot) * 2048;
  t[kEqHalf + j] = static_cast<float>(w * raw);
  t[kEqHalf - j] = static_cast<float>(w * raw);
}

__global__ void __launch_bounds__(512) eq_response(const float* taps, float* resp) {
  extern __shared__ float2 buf[];
  const int slot = blockIdx.x;
  const float* t = taps + static_cast<long>(slot) * 2048;
  for (int i = threadIdx.x; i < kEqFft; i += blockDim.x) {
    float v = 0.f;
    if (i <= kEqHalf) v = t[kEqHalf + i];
    else if (i >= kEqFft - kEqHalf) v = t[kEqHalf - (kEqFft - i)];
    buf[i] = make_float2(v, 0.f);
  }
  __syncthreads();
  fft_pow2<kLogFft, 1, 512, -1>(buf, kEqFft);
  float* r = resp + static_cast<long>(slot) * kEqFft;
  for (int i = threadIdx.x; i < kEqFft; i += blockDim.x) r[i] = buf[i].x * (1.f / kEqFft);
}

// grid (blocks per signal, slots*B)
__global__ void __launch_bounds__(512) eq_conv(StepArgs a, const float* resp) {
  extern __shared__ float2 buf[];
  const int sb = blockIdx.y;
  const int slot = sb / a.batch, b = sb - slot * a.batch;
  const int e0 = __ldg(a.row_ptr + slot), e1 = __ldg(a.row_ptr + slot + 1);
  const long out0 = static_cast<long>(blockIdx.x) * kEqValid;
  const long s0 = out0 - kEqHalf;
  for (int t = threadIdx.x; t < kEqFft; t += blockDim.x) {
    const long pos = s0 + t;
    buf[t] = (pos >= 0 && pos < a.length) ? gather2(a, e0, e1, b, pos) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  fft_pow2<kLogFft, 1, 512, -1>(buf, kEqFft);
  const float* r = resp + static_cast<long>(slot) * kEqFft;
  for (int t = threadIdx.x; t < kEqFft; t += blockDim.x) buf[t] = cscale(buf[t], __ldg(r + t));
  __syncthreads();
  fft_pow2<kLogFft, 1, 512, +1>(buf, kEqFft);
  float* yl = a.dst + static_cast<long>(slot) * a.rowstride + static_cast<long>(b) * 2 * a.length;
  float* yr = yl + a.length;
  for (int t = threadIdx.x; t < kEqValid; t += blockDim.x) {
    const long pos = out0 + t;
    if (pos < a.length) {
      const float2 v = buf[kEqHalf + t];
      yl[pos] = v.x;
      yr[pos] = v.y;
    }
  }
}

}  // namespace

void launch_eq(const StepArgs& a, float* taps_ws, float* resp_ws, cudaStream_t s) {
  if (a.slots == 0) return;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(eq_response, cudaFuncAttributeMaxDynamicSharedMemorySize, kEqFft * 8);
    cudaFuncSetAttribute(eq_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, kEqFft * 8);
    configured = true;
  }
  eq_design<<<dim3(4, a.slots), 256, 0, s>>>(a.params, taps_ws);
  eq_response<<<a.slots, 512, kEqFft * 8, s>>>(taps_ws, resp_ws);
  if (a.batch == 0 || a.length == 0) return;
  const long blocks = (a.length + kEqValid - 1) / kEqValid;
  eq_conv<<<dim3(static_cast<unsigned>(blocks), a.slots * a.batch), 512, kEqFft * 8, s>>>(a, resp_ws);
}

}  // namespace mgb
