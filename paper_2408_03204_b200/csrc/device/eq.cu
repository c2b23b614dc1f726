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
#include <cstdlib>
#include <map>
#include <utility>
#include <mutex>
#include <stdexcept>
#include <vector>

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

// ---- FIR design as a product with a fixed basis -------------------------------------------
// The zero-phase FIR (dsp.cpp:106-136) is LINEAR in the magnitudes m_q = exp(lm_q): its taps
// are h[c + t] = h[c - t] = sum_q m_q D[q][t] with D[q][t] = w(c + t) c_q cos(2 pi q t / 2047)
// / 2047 (c = 1023, c_0 = 1, c_q = 2, w the symmetric Hann) — eq_design's cosine sum as a
// matrix. D (1024 x 1024, fp32 rounded from fp64 with exact-integer angle reduction) is built
// once per device; a step with many slots computes every slot's 1024 distinct taps as one fp32
// product (eq_basis_product<true>), then the 8192-point FFT per slot (eq_response): 0.45 ->
// 0.19 ms per config-5 union. The 8192-bin response is linear in m too, R = A m, A[k][q] = the
// response to the unit spectrum e_q in closed form (a sum of Dirichlet kernels, below): steps
// with few slots (config 2's 16 tracks) take the product with A directly (4x the multiply-adds
// of the taps product, but no per-slot FFT on the critical path).
constexpr int kBasisTileK = 32;                                          // bins per CTA (one per lane)
constexpr int kTapsK = kEqHalf + 1;                                      // design basis: 1024 distinct taps t
constexpr int kRespK = ((kEqFft / 2 + 1 + kBasisTileK - 1) / kBasisTileK) * kBasisTileK;  // response basis: 4128 bins
constexpr int kBasisSlots = 16;                                          // slots per CTA
constexpr int kBasisWarps = 16;                                          // q split over warps
constexpr int kBasisQ = (kEqHalf + 1) / kBasisWarps;                     // 64 q per warp
constexpr int kBasisTileBytes = (kEqHalf + 1) * kBasisTileK * 4;         // 128 KiB column block
constexpr int kBasisMBytes = (kEqHalf + 1) * kBasisSlots * 4;            // magnitude tile, 64 KiB
constexpr int kBasisSmem = kBasisTileBytes + kBasisMBytes;
constexpr int kBasisMinSlots = 4;    // fewer slots: the fp64 cosine-sum design (eq_design) is as fast
constexpr int kTapsMinSlots = 128;  // from here the design basis (4x fewer multiply-adds, then one FFT per
                                    // slot); below, the response basis (the per-slot FFT's latency
                                    // sat on config 2's critical path: 0.1945 -> 0.1986 ms)

// m[group][q][16 slots] = exp(lm) in fp32 (0 past the last slot): the basis kernel's
// magnitude tiles, built once per step instead of once per basis CTA (129 CTAs each
// re-reading 128 KiB of fp64 parameters was half of that kernel's L2 traffic and its
// latency chain). grid (ceil(slots / 16), 8) x 128: thread q writes one 64-byte row.
__global__ void __launch_bounds__(128) eq_mag_tiles(const double* __restrict__ params, int slots, float4* mt) {
  const int q = blockIdx.y * 128 + threadIdx.x, s0 = blockIdx.x * kBasisSlots;
  float v[kBasisSlots];
#pragma unroll
  for (int s = 0; s < kBasisSlots; ++s) {
    v[s] = s0 + s < slots ? expf(static_cast<float>(__ldg(params + static_cast<long>(s0 + s) * (kEqHalf + 1) + q))) : 0.f;
  }
  float4* row = mt + (static_cast<long>(blockIdx.x) * (kEqHalf + 1) + q) * (kBasisSlots / 4);
#pragma unroll
  for (int g = 0; g < kBasisSlots / 4; ++g) row[g] = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
}

// d = a * b + c on a pair of fp32 lanes (one FFMA2 instruction on sm_100).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// grid (kBasisK / 32, ceil(slots / 16)) x 512. The basis is stored tiled, [kBasisK / 32][1024 q]
// [32 taps], so a CTA's column block is one contiguous 128 KiB run, copied into smem with the
// slot group's magnitude tile (eq_mag_tiles). Lane l of warp w then sums tap t0 + l over q in
// [64 w, 64 w + 64) for 16 slots (conflict-free basis reads, broadcast float4 magnitude reads,
// slot pairs in FFMA2); the 16 warp partials are added in warp order. Output: taps[slot][2048]
// (h[c + t] and its mirror h[c - t]), eq_design's layout.
// TAPS = false: the response basis [kRespK / 32][1024 q][32 bins], output resp[slot][8192]
// (bins k <= 4096 and their mirrors 8192 - k).
template <bool TAPS>
__global__ void __launch_bounds__(512, 1) eq_basis_product(const float4* __restrict__ mtiles, int slots,
                                                           const float* __restrict__ basis, float* out) {
  extern __shared__ __align__(128) unsigned char bsm[];
  float* tile = reinterpret_cast<float*>(bsm);                                    // [1024][32]
  float4* msm = reinterpret_cast<float4*>(bsm + kBasisTileBytes);                 // [1024][4] float4
  const int s0 = blockIdx.y * kBasisSlots;
  const int ns = min(kBasisSlots, slots - s0);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // Basis column block and magnitude tile into smem with cp.async (LDGSTS): every thread has
  // its 24 16-byte copies in flight at once. (A TMA bulk copy per quarter measured ~24 GB/s
  // per SM here, a quarter of the HBM share: 10.5 us for this kernel instead of ~5.)
  {
    const char* src = reinterpret_cast<const char*>(basis) + static_cast<long>(blockIdx.x) * kBasisTileBytes;
    const char* msrc = reinterpret_cast<const char*>(mtiles + static_cast<long>(blockIdx.y) * (kEqHalf + 1) * (kBasisSlots / 4));
#pragma unroll
    for (int i = 0; i < kBasisTileBytes / (16 * 512); ++i) {
      const int off = (i * 512 + threadIdx.x) * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(bsm + off)), "l"(src + off) : "memory");
    }
#pragma unroll
    for (int i = 0; i < kBasisMBytes / (16 * 512); ++i) {
      const int off = (i * 512 + threadIdx.x) * 16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(bsm + kBasisTileBytes + off)), "l"(msrc + off)
                   : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  float2 acc2[kBasisSlots / 2];                         // slot pairs: one FFMA2 per pair
#pragma unroll
  for (int s = 0; s < kBasisSlots / 2; ++s) acc2[s] = make_float2(0.f, 0.f);
#pragma unroll 8
  for (int u = 0; u < kBasisQ; ++u) {
    const int q = w * kBasisQ + u;
    const float a = tile[q * kBasisTileK + lane];
    const float2 aa = make_float2(a, a);
    const float4* mq = msm + q * (kBasisSlots / 4);
#pragma unroll
    for (int g = 0; g < kBasisSlots / 4; ++g) {
      const float4 m = mq[g];
      acc2[2 * g + 0] = ffma2(aa, make_float2(m.x, m.y), acc2[2 * g + 0]);
      acc2[2 * g + 1] = ffma2(aa, make_float2(m.z, m.w), acc2[2 * g + 1]);
    }
  }
  float acc[kBasisSlots];
#pragma unroll
  for (int s = 0; s < kBasisSlots / 2; ++s) {
    acc[2 * s] = acc2[s].x;
    acc[2 * s + 1] = acc2[s].y;
  }
  __syncthreads();                                      // tile no longer read: reuse as partials
  float* part = tile;                                   // [16 warps][16 slots][32 lanes]
#pragma unroll
  for (int s = 0; s < kBasisSlots; ++s) part[(w * kBasisSlots + s) * 32 + lane] = acc[s];
  __syncthreads();
  {
    const int i = threadIdx.x;                          // 512 = 16 slots x 32 bins
    const int s = i >> 5, l = i & 31;
    float v = part[s * 32 + l];
#pragma unroll
    for (int ww = 1; ww < kBasisWarps; ++ww) v += part[(ww * kBasisSlots + s) * 32 + l];
    const int kk = blockIdx.x * kBasisTileK + l;
    if constexpr (TAPS) {
      if (s < ns) {
        float* h = out + static_cast<long>(s0 + s) * 2048;
        h[kEqHalf + kk] = v;
        if (kk > 0) h[kEqHalf - kk] = v;
      }
    } else if (s < ns && kk <= kEqFft / 2) {
      float* r = out + static_cast<long>(s0 + s) * kEqFft;
      r[kk] = v;
      if (kk > 0 && kk < kEqFft / 2) r[kEqFft - kk] = v;
    }
  }
}

// Design-basis entries (fp64, rounded to fp32): tiled[(t / 32) * 1024 + q][t % 32] =
// w(c + t) c_q cos(2 pi ((q t) mod 2047) / 2047) / 2047, the exact-integer angle reduction of
// eq_design's cosine table, w(c + t) = 0.5 - 0.5 cos(2 pi (c + t) / 2046) as eq_design.
__global__ void eq_taps_basis_build(float* tiled) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long>(kTapsK) * (kEqHalf + 1)) return;
  const int tl = static_cast<int>(i % kBasisTileK);
  const int q = static_cast<int>((i / kBasisTileK) % (kEqHalf + 1));
  const int t = static_cast<int>(i / (static_cast<long>(kBasisTileK) * (kEqHalf + 1))) * kBasisTileK + tl;
  const long qt = (static_cast<long>(q) * t) % kN;
  double sw, cw;
  sincospi(2.0 * (kEqHalf + t) / (kN - 1), &sw, &cw);
  const double w = 0.5 - 0.5 * cw;
  const double cq = q == 0 ? 1.0 : 2.0;
  tiled[i] = static_cast<float>(w * cq * cospi(2.0 * static_cast<double>(qt) / kN) / kN);
}

// Basis entries in closed form (fp64). With c = 1023, theta_q = 2 pi q / 2047 and
// phi_k = 2 pi k / 8192, the design of the unit spectrum e_q (dsp.cpp:106-136) is
// h_q[j] = w_j c_q cos(j theta_q) / 2047 (c_0 = 1, else 2; symmetric Hann w_j =
// 0.5 + 0.5 cos(pi j / 1023)), and its 8192-point response is
// R_q[k] = c_q / (2 * 2047) [F(theta_q + phi_k) + F(theta_q - phi_k)] with the window
// transform F(x) = sum_j w_j e^{ijx} = D(x)/2 + D(x + pi/1023)/4 + D(x - pi/1023)/4 and the
// Dirichlet kernel D(x) = sin(2047 x / 2) / sin(x / 2). Every angle is 2 pi n / d with exact
// integers n, d, reduced before sinpi, so each entry is correct to a few fp64 ulps.
__device__ double eq_dirichlet(long long n, long long d) {  // D(2 pi n / d)
  n %= d;
  if (2 * n > d) n -= d;
  if (2 * n <= -d) n += d;
  if (n == 0) return 2047.0;
  long long m = (2047LL * n) % (2 * d);                      // sin(2047 pi n / d): reduce mod 2d
  if (m > d) m -= 2 * d;
  if (m <= -d) m += 2 * d;
  return sinpi(static_cast<double>(m) / static_cast<double>(d)) / sinpi(static_cast<double>(n) / static_cast<double>(d));
}
__device__ double eq_window_transform(long long n, long long d) {  // F(2 pi n / d), d a multiple of 2046
  const long long s = d / 2046;                                   // pi / 1023 = 2 pi s / d
  return 0.5 * eq_dirichlet(n, d) + 0.25 * eq_dirichlet(n + s, d) + 0.25 * eq_dirichlet(n - s, d);
}
// tiled[(k / 32) * 1024 + q][k % 32] = R_q[k] / 8192 (the response prescale), 0 for k > 4096.
__global__ void eq_resp_basis_build(float* tiled) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long>(kRespK) * (kEqHalf + 1)) return;
  const int kl = static_cast<int>(i % kBasisTileK);
  const int q = static_cast<int>((i / kBasisTileK) % (kEqHalf + 1));
  const int k = static_cast<int>(i / (static_cast<long>(kBasisTileK) * (kEqHalf + 1))) * kBasisTileK + kl;
  double v = 0.0;
  if (k <= kEqFft / 2) {
    constexpr long long d = 2047LL * 8192LL * 2046LL;             // common denominator
    const long long nq = static_cast<long long>(q) * 8192LL * 2046LL, nk = static_cast<long long>(k) * 2047LL * 2046LL;
    const double cq = q == 0 ? 1.0 : 2.0;
    v = cq / (2.0 * 2047.0 * 8192.0) * (eq_window_transform(nq + nk, d) + eq_window_transform(nq - nk, d));
  }
  tiled[i] = static_cast<float>(v);
}

// Window geometry per FFT size: 8192 (6144 outputs per block, the throughput choice) or
// 4096 (2048 outputs per block: 2.2x less FFT work per CTA and 3x the CTAs, for steps whose
// 8192 grid would not fill the GPU, e.g. a 1-slot bus EQ). The taps span +-1023 < 2048, so
// the 4096-point response is exactly every other bin of the 8192-point one.
template <int LOG, typename C = float2> struct EqWin {
  static constexpr int kFft = 1 << LOG;
  static constexpr int kOut = LOG == 13 ? 6144 : 2048;
  static constexpr int kThreads = LOG == 13 ? 512 : 256;
  static constexpr int kMinBlocks = sizeof(C) == 8 ? 2 : 1;
  static constexpr int kSmem = padded(kFft) * static_cast<int>(sizeof(C));
  static_assert(kOut <= kFft - 2 * kEqHalf, "EQ block larger than the non-wrapped window");
};

// grid (blocks per signal, slots*B). Block covers outputs [out0, out0 + kOut) from the
// kFft-sample window starting at out0 - 1024; the circular convolution is exact for window
// indices [1023, kFft - 1024]. Window loads feed the first FFT pass directly and the last
// inverse pass stores directly (register-ended transforms, fft_smem.cuh), both coalesced.
// C: transform element type (float2, or double2: fp64 arithmetic, fp32 arena in and out).
template <int LOG, typename C>
__global__ void __launch_bounds__(EqWin<LOG, C>::kThreads, EqWin<LOG, C>::kMinBlocks) eq_conv(StepArgs a, const float* resp) {
  using W = EqWin<LOG, C>;
  using T = RealOf<C>;
  constexpr int kEqFft = W::kFft, kEqOut = W::kOut, kNt = W::kThreads;
  constexpr int kRs = kEqFft == 8192 ? 1 : 8192 / kEqFft;   // response bin stride
  const T rscale = static_cast<T>(kRs);                    // response is prescaled by 1/8192
  extern __shared__ __align__(16) unsigned char eq_smem[];
  C* buf = reinterpret_cast<C*>(eq_smem);
  const C* tw = twiddles<C>(a);
  const int sb = blockIdx.y;
  const int slot = sb / a.batch, b = sb - slot * a.batch;
  const int e0 = slot_e0(a, slot), e1 = slot_e1(a, slot);
  const long out0 = static_cast<long>(blockIdx.x) * kEqOut;
  const long s0 = out0 - (kEqHalf + 1);
  const long boff = static_cast<long>(b) * 2 * a.length;
  const float* rs = resp + static_cast<long>(slot) * 8192;
  // fp32 8192-point windows: the slot's response (32 KiB, L2-resident) is requested into shared
  // memory with cp.async now and read after the forward transform, instead of 16 L2 round
  // trips per thread in the middle of the kernel
  constexpr bool kStageResp = LOG == 13 && sizeof(C) == 8;
  float* rsm = reinterpret_cast<float*>(eq_smem + W::kSmem);
  if constexpr (kStageResp) {
#pragma unroll
    for (int i = 0; i < 8192 / 4 / kNt; ++i) {
      const int off = (i * kNt + threadIdx.x) * 4;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(rsm + off)), "l"(rs + off) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  {
  // Gather-sum of the window straight into the radix-16 first-pass butterfly this thread
  // owns (elements t + r*N/16: consecutive threads read consecutive samples), edges
  // outermost so all 16 sample pairs are in flight at once; per element the sum runs in
  // edge order (as the reference's gather).
  constexpr int M1 = kEqFft / 16;
  static_assert(M1 == kNt, "eq_conv: threads must be the first pass's butterflies");
  C v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = Cx<C>::mk(T(0), T(0));
  // 32-bit sample positions (L < 2^31), one unsigned compare for both bounds, addresses from
  // opaque row pointers (the 64-bit re-derivation per element was a fifth of the instructions)
  const int pos0 = static_cast<int>(s0) + static_cast<int>(threadIdx.x);
  const unsigned len = static_cast<unsigned>(a.length);
  for (int e = e0; e < e1; ++e) {
    const float* pl = opaque_ptr(a.src + edge_row(a, e) * a.rowstride + boff);
    const float* pr = opaque_ptr(pl + a.length);
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const unsigned pos = static_cast<unsigned>(pos0 + r * M1);
      if (pos < len) {
        v[r].x += static_cast<T>(__ldg(pl + pos));
        v[r].y += static_cast<T>(__ldg(pr + pos));
      }
    }
  }
  fft_first_from_regs<-1>(v, buf, threadIdx.x);
  __syncthreads();
  // Forward plan 16 x 8 x 4 x 16 (8192) or 16 x 16 x 16 (4096): its last pass is radix 16, so
  // butterfly j ends holding X[j + r N/16], r < 16 — exactly the inputs of the inverse's
  // radix-16 first-pass butterfly j. The product with the response and the inverse's first
  // pass run in registers: no smem round trip, no barrier between the two transforms.
  if constexpr (LOG == 13) {
    stockham_pass<kEqFft, 8, 16, 1, kNt, -1>(buf, padded(kEqFft), tw);
    stockham_pass<kEqFft, 4, 128, 1, kNt, -1>(buf, padded(kEqFft), tw);
  } else {
    stockham_pass<kEqFft, 16, 16, 1, kNt, -1>(buf, padded(kEqFft), tw);
  }
  constexpr int NL = kEqFft / 16;  // last-pass butterflies = threads
  static_assert(NL == kNt, "eq_conv: one last-pass butterfly per thread");
  const int j = threadIdx.x;
  {
    TwPass<16, NL, -1, C> twb;
    twb.load(tw, j);
    const C* lb = buf + sidx(j);
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = lb[r * padded(NL)];
    twb.apply(v);
    Dft<16, -1, C>::run(v);
  }
  if constexpr (kStageResp) {
    asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's own copies (the bins it
                                                      // reads are other threads': barrier below)
  }
  __syncthreads();  // every thread has read its last-pass inputs (and the response is staged)
  if constexpr (kStageResp) {
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = cscale(v[r], rscale * rsm[j + r * NL]);
  } else {
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = cscale(v[r], rscale * static_cast<T>(__ldg(rs + kRs * (j + r * NL))));
  }
  fft_first_from_regs<+1>(v, buf, j);
  }
  __syncthreads();
  // Inverse: the middle passes in smem, the last into registers and straight to the arena
  // (window index w = j + r*NS holds output out0 + w - 1024 for w in [1024, 1024 + kEqOut)).
  fft_middle<LOG, 1, kNt, +1>(buf, padded(kEqFft), tw);
  constexpr int NS = Pow2Plan<LOG>::kLastNs, R = Pow2Plan<LOG>::kLastR, PL = NS / kNt;
  float* yl = opaque_ptr(a.dst + static_cast<long>(slot) * a.rowstride + boff + out0);
  float* yr = opaque_ptr(yl + a.length);
  const int pend = static_cast<int>(min(a.length - out0, static_cast<long>(kEqOut)));  // outputs of this block
#pragma unroll
  for (int p = 0; p < PL; ++p) {
    const int j = threadIdx.x + p * kNt;
    C y[R];
    fft_last_to_regs<LOG, +1>(buf, j, tw, y);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int w = j + r * NS - (kEqHalf + 1);  // output out0 + w, stored for 0 <= w < pend
      if (static_cast<unsigned>(w) < static_cast<unsigned>(pend)) {
        st_global(yl + static_cast<unsigned>(w), static_cast<float>(y[r].x));
        st_global(yr + static_cast<unsigned>(w), static_cast<float>(y[r].y));
      }
    }
  }
}

}  // namespace

void eq_setup() {
  static const bool done = [] {
    cudaFuncSetAttribute(eq_response, cudaFuncAttributeMaxDynamicSharedMemorySize, kEqSmem);
    cudaFuncSetAttribute(eq_basis_product<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBasisSmem);
    cudaFuncSetAttribute(eq_basis_product<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kBasisSmem);
    for (auto fn : {eq_conv<13, float2>, eq_conv<12, float2>}) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kEqSmem + 8192 * 4);
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    for (auto fn : {eq_conv<13, double2>, eq_conv<12, double2>}) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kEqSmem);
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    return true;
  }();
  (void)done;
}

// Per-device bases (the design basis D [1024 q][1024 t] and the response basis A^T
// [1024 q][4128 bins], both tiled by 32 columns), built synchronously on first use
// (ProcessorSet's constructor calls it, before any stream capture).
const float* eq_basis(int device, bool taps) {
  static std::mutex mu;
  static std::map<std::pair<int, bool>, float*> bases;
  std::scoped_lock lock(mu);
  auto it = bases.find({device, taps});
  if (it != bases.end()) return it->second;
  eq_setup();
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  float* basis = nullptr;
  const long n = static_cast<long>(taps ? kTapsK : kRespK) * (kEqHalf + 1);
  bool ok = cudaMalloc(&basis, sizeof(float) * n) == cudaSuccess;
  if (ok) {
    if (taps) eq_taps_basis_build<<<static_cast<unsigned>((n + 255) / 256), 256>>>(basis);
    else eq_resp_basis_build<<<static_cast<unsigned>((n + 255) / 256), 256>>>(basis);
    ok = cudaDeviceSynchronize() == cudaSuccess;
  }
  cudaSetDevice(prev);
  if (!ok) {
    cudaFree(basis);
    throw std::runtime_error("EQ basis build failed");
  }
  bases.emplace(std::make_pair(device, taps), basis);
  return basis;
}

void launch_eq_prologue(const StepArgs& a, float* taps_ws, float* resp_ws, cudaStream_t s) {
  if (a.slots == 0) return;
  eq_setup();
  if (a.slots >= kBasisMinSlots) {
    int dev = 0;
    cudaGetDevice(&dev);
    const int groups = (a.slots + kBasisSlots - 1) / kBasisSlots;
    note_prologue_kernel(reinterpret_cast<const void*>(eq_mag_tiles));
    if (a.slots >= kTapsMinSlots) {
      note_prologue_kernel(reinterpret_cast<const void*>(eq_basis_product<true>));
      note_prologue_kernel(reinterpret_cast<const void*>(eq_response));
      // the magnitude tiles (64 KiB per 16 slots) borrow the response region (32 KiB per slot),
      // which eq_response overwrites only after the product has read them
      auto* mt = reinterpret_cast<float4*>(resp_ws);
      eq_mag_tiles<<<dim3(groups, (kEqHalf + 1) / 128), 128, 0, s>>>(a.params, a.slots, mt);
      eq_basis_product<true><<<dim3(kTapsK / kBasisTileK, groups), 512, kBasisSmem, s>>>(mt, a.slots, eq_basis(dev, true),
                                                                                        taps_ws);
      eq_response<<<a.slots, 512, kEqSmem, s>>>(taps_ws, resp_ws, a.tw);
      return;
    }
    note_prologue_kernel(reinterpret_cast<const void*>(eq_basis_product<false>));
    auto* mt = reinterpret_cast<float4*>(taps_ws);  // the taps region is unused on this path
    eq_mag_tiles<<<dim3(groups, (kEqHalf + 1) / 128), 128, 0, s>>>(a.params, a.slots, mt);
    eq_basis_product<false><<<dim3(kRespK / kBasisTileK, groups), 512, kBasisSmem, s>>>(mt, a.slots, eq_basis(dev, false),
                                                                                       resp_ws);
    return;
  }
  // taps_ws holds [slots][2048] floats followed by [slots][1024] doubles of magnitudes.
  auto* mags = reinterpret_cast<double*>(taps_ws + 2048L * a.slots);
  note_prologue_kernel(reinterpret_cast<const void*>(eq_mags));
  note_prologue_kernel(reinterpret_cast<const void*>(eq_design));
  note_prologue_kernel(reinterpret_cast<const void*>(eq_response));
  eq_mags<<<a.slots, kEqHalf + 1, 0, s>>>(a.params, mags);
  eq_design<<<dim3(1024 / (256 / kDesignSplit * kDesignTpw), a.slots), 256, 0, s>>>(mags, taps_ws, cos_table(a.tw));
  eq_response<<<a.slots, 512, kEqSmem, s>>>(taps_ws, resp_ws, a.tw);
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
  if (fft_fp64()) {
    if (eq_uses_small_window(a)) {
      eq_conv<12, double2><<<eq_grid<12>(a), EqWin<12>::kThreads, EqWin<12, double2>::kSmem, s>>>(a, resp_ws);
      return;
    }
    eq_conv<13, double2><<<eq_grid<13>(a), 512, EqWin<13, double2>::kSmem, s>>>(a, resp_ws);
    return;
  }
  if (eq_uses_small_window(a)) {
    eq_conv<12, float2><<<eq_grid<12>(a), EqWin<12>::kThreads, EqWin<12>::kSmem, s>>>(a, resp_ws);
    return;
  }
  eq_conv<13, float2><<<eq_grid<13>(a), 512, kEqSmem + 8192 * 4, s>>>(a, resp_ws);
}

}  // namespace mgb
