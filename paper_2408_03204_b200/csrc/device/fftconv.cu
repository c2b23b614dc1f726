// K8/K9 (reverb) and K10/K11 (multitap delay): long causal convolutions.
//
// Reference: the reverb step builds a stereo impulse response from a masked noise STFT
// (`processors.cpp:162-187`, istft `dsp.cpp:165-190`) and the delay step builds a sparse
// multitap kernel (`processors.cpp:189-227`); both then run fft_convolve(Causal) per
// (batch, channel) with a zero-padded next_pow2(L + taps - 1) FFT (`dsp.cpp:64-86`), which
// re-transforms the kernel on every call.
//
// Device plan per step (N = 2^a >= L + taps - 1, N = N1 * N2):
//   ir build      -> packed kernel h = h_L + i h_R (one complex signal per node)
//   cols_fwd<K>   -> column FFTs of h (length N1, stride N2) x four-step twiddle
//   rows<SPEC>    -> row FFTs: P = FFT_N(h) in the transposed (k1 + N1*k2) order
//   cols_fwd<S>   -> same for the signal x = u_L + i u_R, gathered from the arena (Eq. 1b)
//   rows<CONV>    -> row FFTs of x, channel split by conjugate pairing of rows k1 / N1-k1,
//                    Z = X_L H_L + i X_R H_R, inverse row FFTs x inverse twiddle
//   cols_inv      -> inverse column FFTs, real part -> left, imag part -> right, store the
//                    first L samples into the arena.
// The spectrum stays in four-step (transposed) order: forward and inverse are mirror
// images, so no transpose pass is ever made. Each pass is one smem-resident batch of FFTs.
#include <cmath>
#include <stdexcept>

#include "fft_smem.cuh"
#include "launch.hpp"

namespace mgb {

namespace {

// Column tile: complex elements per CTA (64 KiB either way: 8192 fp32 or 4096 fp64 values)
// and its threads, one per radix-16 first-pass butterfly.
template <typename CT> struct ColCfg {
  static constexpr int kElems = sizeof(CT) == 8 ? 8192 : 4096;
  static constexpr int kThreads = kElems / 16;
  static constexpr int kSmem(int n1) { return (kElems / n1) * (padded(n1) + 1) * static_cast<int>(sizeof(CT)); }
};
// Resident rows_conv threads per SM the register budget is sized for (half for fp64: twice the
// registers per complex value). The kernel spectrum is
// loaded where it is used (prefetching it into registers spilled; cp.async into shared memory
// measured no faster).
constexpr int kRconvThreadsPerSm = 1024;
// Resident CTAs per SM rows_bwd is compiled for: 4 up to 512-point rows (at 2 the 512-point
// kernel took 178 registers, 2 CTAs of 128 threads per SM: 0.76 -> 0.53 ms per config-4 launch
// at 4 with 44 B of spills; 6 spilled 700 B and was slower); 1 from 1024 points, whose 256/512
// threads need more than 128/64 registers.
template <int LN2>
constexpr int rbwd_min_blocks() { return LN2 >= 10 ? 1 : 4; }

inline std::size_t align256(std::size_t x) { return (x + 255) & ~static_cast<std::size_t>(255); }

// Packed impulse responses [slots][taps] float2, plus room for the delay tap records.
inline std::size_t ir_bytes(int slots, long taps) {
  return align256(sizeof(float2) * static_cast<std::size_t>(slots) * taps + sizeof(float) * 40 * 40 * slots);
}

// Multitap delay tap records (delay_taps): 2 channels x 20 taps, each [position as float
// bits, 39 FIR coefficients].
constexpr int kTaps = 40;       // 2 channels x 20
constexpr int kTapStride = 22;  // parameter row: per tap [re, im, 20 log-mags]
constexpr int kFir = 39;
constexpr int kFirHalf = 19;
constexpr int kTapRec = 40;

// Column-pass input: the packed kernel from an IR buffer, the arena signal (gathered), or
// the multitap delay kernel synthesised from its tap records (no dense IR in memory).
enum class ColSrc { Kernel, Signal, DelayTaps };

// Segmented overlap-save (launch.hpp ConvGeom): item = (slot*batch + b)*nseg + j, segment j
// transforms x[base_j, base_j + N), base_j = max(0, j*seg - pre), and owns the outputs
// [j*seg, (j+1)*seg). item0: first item of this launch (grids are chunked at 65535 in y).
struct SegArgs {
  long seg;
  long pre;
  int nseg;
  int item0;
  int mask_out;  // gather only the segment's own output samples (dY of the kernel gradient)
  const int* slot_map = nullptr;  // signal column pass over a subset of slots: launch slot -> step slot
};
SegArgs seg_args(const ConvGeom& g, int item0 = 0, bool mask_out = false, const int* slot_map = nullptr) {
  return SegArgs{g.seg, g.pre, g.nseg, item0, mask_out ? 1 : 0, slot_map};
}
__host__ __device__ __forceinline__ long seg_base(long seg, long pre, long j) {
  const long b = j * seg - pre;
  return b > 0 ? b : 0;
}
constexpr int kMaxGridY = 65535;

// ---- pass 1: column FFTs (forward) ------------------------------------------------------
// grid (N2 / C, items); item = slot (kernel) or slot*B + b (signal).
// Thread t owns column c = t % C and first-pass butterfly jt = t / C: elements n1 = jt + q*N1/16
// (q < 16) of its column, i.e. n = n0 + q*N/16. Index math is 32-bit within an item (N <= 2^22)
// on per-item base pointers: the 64-bit per-element arithmetic was a third of the instructions
// of these issue-bound kernels.
template <int LN1, ColSrc SRC, typename CT>
__global__ void __launch_bounds__(ColCfg<CT>::kThreads, 2) cols_fwd(StepArgs a, const float2* ir, long taps, int log_n,
                                                        CT* out, int window, SegArgs sg) {
  using T = RealOf<CT>;
  constexpr int N1 = 1 << LN1;
  constexpr int C = ColCfg<CT>::kElems / N1;
  constexpr int FS = padded(N1) + 1;
  constexpr int NT = ColCfg<CT>::kThreads;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CT* tile = reinterpret_cast<CT*>(smem_raw);
  const int log_n2 = log_n - LN1;
  const int N2 = 1 << log_n2;
  const int N = 1 << log_n;
  int item = sg.item0 + blockIdx.y;
  const int col0 = blockIdx.x * C;
  const int c = threadIdx.x % C, jt = threadIdx.x / C;
  const int nstep = N >> 4;
  const int n0 = jt * N2 + col0 + c;
  int slot = item, b = 0, e0 = 0, e1 = 0;
  long base = 0, lo = 0, hi = taps;  // sample m = base + n is loaded when lo <= m < hi
  if constexpr (SRC == ColSrc::Signal) {
    const int isb = item / sg.nseg, j = item - isb * sg.nseg;
    slot = isb / a.batch;
    b = isb - slot * a.batch;
    if (sg.slot_map != nullptr) {  // a subset of the step's slots: store at the step's own item
      slot = __ldg(sg.slot_map + slot);
      item = (slot * a.batch + b) * sg.nseg + j;
    }
    e0 = slot_e0(a, slot);
    e1 = slot_e1(a, slot);
    base = seg_base(sg.seg, sg.pre, j);
    const long first = static_cast<long>(j) * sg.seg;
    lo = sg.mask_out ? first : base;
    hi = min(first + sg.seg, a.length);
  }
  // Valid n of this item: [nlo, nhi).
  const int nlo = static_cast<int>(min(max(lo - base, 0L), static_cast<long>(N)));
  const int nhi = static_cast<int>(min(max(hi - base, 0L), static_cast<long>(N)));
  const unsigned span = static_cast<unsigned>(max(nhi - nlo, 0));  // n valid: unsigned(n - nlo) < span
  constexpr int EPT = ColCfg<CT>::kElems / NT;
  static_assert(EPT == 16, "cols_fwd: one radix-16 first-pass butterfly per thread");
  CT vals[EPT];
  if constexpr (SRC == ColSrc::DelayTaps) {
    // The dense multitap kernel (processors.cpp:210-227) has <= 40 x 39 nonzeros: zero the
    // tile, scatter the tap FIRs into it, read the butterfly inputs back. Windows of one parity
    // never overlap (w > 2*19), so the even taps then the odd taps add without races; an
    // element reached by two taps gets 0 + f_a + f_b in either order — the same float as the
    // dense synthesis's tap-order sum.
    __shared__ float rec[kTaps * kTapRec];
    const float* in = reinterpret_cast<const float*>(ir) + static_cast<long>(item) * kTaps * kTapRec;
    for (int q = threadIdx.x; q < kTaps * kTapRec; q += NT) rec[q] = __ldg(in + q);
    T* zt = reinterpret_cast<T*>(tile);
    for (int q = threadIdx.x; q < 2 * C * FS; q += NT) zt[q] = T(0);
    __syncthreads();
    constexpr int kPhase = 20 * kFir;  // (channel, tap of one parity, FIR index)
    for (int ph = 0; ph < 2; ++ph) {
      for (int q = threadIdx.x; q < kPhase; q += NT) {
        const int ch = q / (10 * kFir), rem = q - ch * (10 * kFir);
        const int m = 2 * (rem / kFir) + ph, jj = rem % kFir;
        const float* r = rec + (ch * 20 + m) * kTapRec;
        const int d = __float_as_int(r[0]);
        const int i = d - kFirHalf + jj;
        if (d < 0 || i < nlo || i >= nhi) continue;
        const int cc = (i & (N2 - 1)) - col0;
        if (cc < 0 || cc >= C) continue;
        T* e = zt + 2 * (cc * FS + sidx(i >> log_n2)) + ch;
        *e = *e + static_cast<T>(r[1 + jj]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < EPT; ++q) vals[q] = tile[c * FS + sidx(jt + q * (N1 / 16))];
    __syncthreads();
  } else {
    // All of this thread's loads are in flight before any smem store.
    const float* one = nullptr;  // in-degree-1 fast path
    if constexpr (SRC == ColSrc::Signal) {
      if (e1 - e0 == 1) one = opaque_ptr(a.src + edge_row(a, e0) * a.rowstride + static_cast<long>(b) * 2 * a.length + base);
    }
    const float2* irp = ir + static_cast<long>(item) * taps;
    if (SRC != ColSrc::Signal || one) {
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int n = n0 + q * nstep;
        CT v = Cx<CT>::mk(0.f, 0.f);
        if (static_cast<unsigned>(n - nlo) < span) {
          const unsigned un = static_cast<unsigned>(n);
          if constexpr (SRC == ColSrc::Signal) v = Cx<CT>::mk(__ldg(one + un), __ldg(one + a.length + un));
          else v = widen<CT>(__ldg(irp + un));
        }
        vals[q] = v;
      }
    } else {
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int n = n0 + q * nstep;
        vals[q] = (static_cast<unsigned>(n - nlo) < span) ? widen<CT>(gather2(a, e0, e1, b, base + n)) : Cx<CT>::mk(0.f, 0.f);
      }
    }
  }
  // vals[q] = element jt + q*N1/16 of column c: exactly the inputs of radix-16 first-pass
  // butterfly jt, so the first pass runs from registers.
  fft_first_from_regs<-1>(vals, tile + c * FS, jt);
  __syncthreads();
  fft_middle<LN1, C, NT, -1>(tile, FS, twiddles<CT>(a));
  // Last pass into registers, four-step twiddle exp(-2 pi i n2 k1 / N), store. Outputs of
  // butterfly j are k1 = j + r*NS: geometric in r, exact anchors (sincospif; n2 k1 < N <=
  // 2^24 is exact in fp32) every 4 outputs, <= 3 chained products in between.
  using Plan = Pow2Plan<LN1>;
  constexpr int NS = Plan::kLastNs, R = Plan::kLastR, JSTEP = NT / C;
  const int n2 = col0 + c;
  CT* o = out + static_cast<long>(item) * N + n2;
  const T inv_n = T(2) / static_cast<T>(N);
  const CT step = expi_pi(-static_cast<T>(n2 * NS) * inv_n);
#pragma unroll
  for (int p = 0; p < NS / JSTEP; ++p) {
    const int j = jt + p * JSTEP;
    CT v[R];
    fft_last_to_regs<LN1, -1>(tile + c * FS, j, twiddles<CT>(a), v);
    CT w = Cx<CT>::mk(1.f, 0.f);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int k1 = j + r * NS;
      w = (r % 4 == 0) ? expi_pi(-static_cast<T>(n2 * k1) * inv_n) : cmul(w, step);
      o[static_cast<unsigned>(k1 * N2)] = cmul(v[r], w);
    }
  }
}

// ---- delay kernel: column stage as a sparse DFT -------------------------------------------
// The multitap delay kernel (processors.cpp:210-227) has <= 40 taps x 39 FIR coefficients in
// a 2 s span: a column n2 of the four-step layout (samples n1*N2 + n2, N2 >= 64 > 39) meets
// each tap's FIR window at most once, ~3 times in all. Its N1-point DFT is therefore the sum
// of those few terms, f * w_N1^(n1 k1), evaluated directly: no zero fill, no scatter, no smem
// FFT passes — the kernel is bound by writing the 2 MiB column-stage spectrum per slot.
// Per CTA (C columns, as cols_fwd): warp w builds the hit lists of columns w, w + 16, ... in
// tap order (ballot + popc: deterministic), then thread (column c, group g) sums the hits of
// its column for k1 = g + G r (G = 512 / C, r < 16) and applies the four-step twiddle
// exp(-2 pi i n2 k1 / N). Twiddles from the table (exact anchors every 4 outputs, <= 3
// chained products in between). Same values as the transform of the synthesised kernel up to
// fp32 rounding (a direct sum of <= 40 terms).
constexpr int kDelayColThreads = 512;
constexpr int kDelayColBlocks = 4;  // column blocks per CTA (the records are loaded once)
template <int LN1>
__global__ void __launch_bounds__(kDelayColThreads) delay_cols(const float* taps_rec, long taps, int log_n, float2* out,
                                                           const float2* tw) {
  constexpr int N1 = 1 << LN1;
  constexpr int C = 8192 / N1;                  // columns per CTA (cols_fwd's tiling)
  constexpr int G = kDelayColThreads / C;       // k1 groups
  constexpr int R = N1 / G;                     // outputs per thread (16)
  constexpr int NW = kDelayColThreads / 32;
  static_assert(R == 16, "delay_cols: 16 outputs per thread");
  __shared__ float rec[kTaps * kTapRec];
  __shared__ int hn1[C][kTaps];
  __shared__ float2 hv[C][kTaps];
  __shared__ int hcnt[C];
  const int slot = blockIdx.y;
  const int log_n2 = log_n - LN1;
  const int N2 = 1 << log_n2;
  const int N = 1 << log_n;
  const float* in = taps_rec + static_cast<long>(slot) * kTaps * kTapRec;
  for (int q = threadIdx.x; q < kTaps * kTapRec; q += kDelayColThreads) rec[q] = __ldg(in + q);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nhi = static_cast<int>(min(taps, static_cast<long>(N)));
  const int c = threadIdx.x % C, g = threadIdx.x / C;
  constexpr int TS = 8192 / N1;  // table stride: w_N1^x = tw[x * TS]
  const float inv_n = 2.f / static_cast<float>(N);
  // Column blocks blockIdx.x, + gridDim.x, ...: the tap records are loaded once per CTA.
  for (int col0 = blockIdx.x * C; col0 < N2; col0 += gridDim.x * C) {
    __syncthreads();  // records loaded / previous block's hit lists consumed
    for (int cc = warp; cc < C; cc += NW) {
      const int n2 = col0 + cc;
      int base = 0;
      for (int m0 = 0; m0 < kTaps; m0 += 32) {
        const int m = m0 + lane;
        bool hit = false;
        int n1 = 0;
        float f = 0.f;
        if (m < kTaps) {
          const float* r = rec + m * kTapRec;
          const int d = __float_as_int(r[0]);
          if (d >= 0) {
            const int i0 = d - kFirHalf;
            const int i = i0 + ((n2 - i0) & (N2 - 1));  // first sample of column n2 at or after i0
            if (i <= d + kFirHalf && i >= 0 && i < nhi) {
              hit = true;
              n1 = i >> log_n2;
              f = r[1 + (i - i0)];
            }
          }
        }
        const unsigned mask = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int pos = base + __popc(mask & ((1u << lane) - 1u));
          hn1[cc][pos] = n1;
          hv[cc][pos] = m < kTaps / 2 ? make_float2(f, 0.f) : make_float2(0.f, f);  // left taps 0-19, right 20-39
        }
        base += __popc(mask);
      }
      if (lane == 0) hcnt[cc] = base;
    }
    __syncthreads();
    const int n2 = col0 + c;
    float2 acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = make_float2(0.f, 0.f);
    const int nh = hcnt[c];
    for (int h = 0; h < nh; ++h) {
      const int n1 = hn1[c][h];
      const float2 v = hv[c][h];
      // u = v w_N1^(n1 k1) chained on the product itself (v is real or imaginary: the anchor
      // product is exact up to one rounding), exact table anchors every 4 outputs.
      const float2 ws = __ldg(tw + ((n1 * G) & (N1 - 1)) * TS);
      float2 u = v;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        u = (r % 4 == 0) ? cmul(v, __ldg(tw + ((n1 * (g + G * r)) & (N1 - 1)) * TS)) : cmul(u, ws);
        acc[r] = cadd(acc[r], u);
      }
    }
    float2* o = out + static_cast<long>(slot) * N + n2;
    const float2 st = expi_pi(-static_cast<float>(n2 * G) * inv_n);
    float2 w = make_float2(1.f, 0.f);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int k1 = g + G * r;
      w = (r % 4 == 0) ? expi_pi(-static_cast<float>(n2 * k1) * inv_n) : cmul(w, st);
      o[static_cast<long>(k1) * N2] = cmul(acc[r], w);
    }
  }
}

// ---- pass 3 (last): inverse column FFTs, store into the arena --------------------------
// BUF: the whole transform goes back into the item's own spectrum in natural order (in place:
// a CTA owns its columns, and all its loads are consumed before its stores) for conv_ola.
template <int LN1, bool BUF, typename CT>
__global__ void __launch_bounds__(ColCfg<CT>::kThreads, 2) cols_inv(StepArgs a, int log_n, CT* X, SegArgs sg) {
  constexpr int N1 = 1 << LN1;
  constexpr int C = ColCfg<CT>::kElems / N1;
  constexpr int FS = padded(N1) + 1;
  constexpr int NT = ColCfg<CT>::kThreads;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CT* tile = reinterpret_cast<CT*>(smem_raw);
  const int N2 = 1 << (log_n - LN1);
  const int N = 1 << log_n;
  const int item = sg.item0 + blockIdx.y;
  const int c = threadIdx.x % C, jt = threadIdx.x / C;
  const int n2 = blockIdx.x * C + c;
  {
    const CT* xc = X + static_cast<long>(item) * N + n2;  // column n2: element n1 at xc[n1 * N2]
    constexpr int EPT = ColCfg<CT>::kElems / NT;
    CT vals[EPT];
#pragma unroll
    for (int q = 0; q < EPT; ++q) vals[q] = __ldg(xc + static_cast<unsigned>((jt + q * (N1 / 16)) * N2));
    // First pass from registers (vals[q] = element jt + q*N1/16 of column c), last pass into
    // registers and straight to the arena (outputs n1 = j + r*NS of column c).
    fft_first_from_regs<+1>(vals, tile + c * FS, jt);
  }
  __syncthreads();
  fft_middle<LN1, C, NT, +1>(tile, FS, twiddles<CT>(a));
  // (segment bookkeeping after the transform: nothing 64-bit stays live across it)
  const int isb = item / sg.nseg, jseg = item - isb * sg.nseg;
  const int slot = isb / a.batch, b = isb - slot * a.batch;
  const long base = seg_base(sg.seg, sg.pre, jseg);
  const long first = static_cast<long>(jseg) * sg.seg, end = min(first + sg.seg, a.length);
  CT* xc = X + static_cast<long>(item) * N + n2;
  using Plan = Pow2Plan<LN1>;
  constexpr int NS = Plan::kLastNs, R = Plan::kLastR, JSTEP = NT / C;
  // Output n = n1*N2 + n2 is sample base + n, stored when first <= base + n < end.
  if constexpr (BUF) {
#pragma unroll 1
    for (int p = 0; p < NS / JSTEP; ++p) {
      const int j = jt + p * JSTEP;
      CT v[R];
      fft_last_to_regs<LN1, +1>(tile + c * FS, j, twiddles<CT>(a), v);
#pragma unroll
      for (int r = 0; r < R; ++r) xc[static_cast<unsigned>((j + r * NS) * N2)] = v[r];
    }
    return;
  }
  // Offsets k >= 0 as unsigned: one IMAD.WIDE.U32 per store address, one compare per bound.
  const int nlo = static_cast<int>(min(max(first - base, 0L), static_cast<long>(N))) - n2;
  const int nhi = static_cast<int>(min(max(end - base, 0L), static_cast<long>(N))) - n2;
  const unsigned span = static_cast<unsigned>(max(nhi - nlo, 0));
  // Opaque row pointers: otherwise the compiler re-derives each store's address from a.dst.
  float* yl = opaque_ptr(a.dst + static_cast<long>(slot) * a.rowstride + static_cast<long>(b) * 2 * a.length + base + n2);
  float* yr = opaque_ptr(yl + a.length);
#pragma unroll
  for (int p = 0; p < NS / JSTEP; ++p) {
    const int j = jt + p * JSTEP;
    CT v[R];
    fft_last_to_regs<LN1, +1>(tile + c * FS, j, twiddles<CT>(a), v);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int k = (j + r * NS) * N2;
      if (static_cast<unsigned>(k - nlo) < span) {
        st_global(yl + static_cast<unsigned>(k), static_cast<float>(v[r].x));
        st_global(yr + static_cast<unsigned>(k), static_cast<float>(v[r].y));
      }
    }
  }
}

// Overlap-add of the segments' input-gradient contributions (backward, nseg > 1): segment j
// contributes to samples [base_j, (j+1)*seg); each sample sums its segments in order j = m/seg,
// ..., (m+pre)/seg (fixed order, deterministic). grid (ceil(L/256), slots*batch chunk).
template <typename CT>
__global__ void __launch_bounds__(256) conv_ola(StepArgs a, SegArgs sg, long N, const CT* buf) {
  using T = RealOf<CT>;
  // 32-bit index math (L, seg, pre < 2^31; the 64-bit divisions dominated this kernel)
  const int m = static_cast<int>(blockIdx.x) * 256 + static_cast<int>(threadIdx.x);
  if (m >= a.length) return;
  const int isb = sg.item0 + blockIdx.y;
  const int slot = isb / a.batch, b = isb - slot * a.batch;
  const int seg = static_cast<int>(sg.seg), pre = static_cast<int>(sg.pre);
  const int jhi = min((m + pre) / seg, sg.nseg - 1);
  CT acc = Cx<CT>::mk(0.f, 0.f);
  const CT* bi = buf + static_cast<long>(isb) * sg.nseg * N;
  for (int j = m / seg; j <= jhi; ++j) {
    const int base = max(j * seg - pre, 0);
    acc = cadd(acc, __ldg(bi + static_cast<long>(j) * N + (m - base)));
  }
  float* y = a.dst + static_cast<long>(slot) * a.rowstride + static_cast<long>(b) * 2 * a.length;
  y[m] = static_cast<float>(acc.x);
  y[a.length + m] = static_cast<float>(acc.y);
}

// ---- pass 2: row FFTs ---------------------------------------------------------------------
template <typename CT>
__device__ __forceinline__ CT zmix(CT xk, CT xm, CT pk, CT pm, RealOf<CT> s) {
  // xm = conj(X[N-k]), pm = conj(P[N-k]):  Z = ((xk+xm)(pk+pm) - i (xk-xm)(pk-pm)) / 4
  const CT s1 = cmul(cadd(xk, xm), cadd(pk, pm));
  const CT s2 = cmul(csub(xk, xm), csub(pk, pm));
  return cscale(cadd(s1, Cx<CT>::mk(s2.y, -s2.x)), s);
}

// Threads = radix-16 butterflies of the first pass (COUNT rows of 2^LN2 points), so no
// thread idles in it; later radix-8/4 passes give each thread 2 or 4 butterflies.
template <int LN2, int COUNT>
constexpr int row_threads() {
  constexpr int t = COUNT * (1 << LN2) / 16;
  return t < 32 ? 32 : (t > 512 ? 512 : t);
}
constexpr int kSpecRows = 4;  // kernel-spectrum rows per CTA

// Register-ended row transforms apply when a CTA's threads are exactly the radix-16 first
// pass's butterflies over its COUNT rows (row_threads not clamped).
template <int LN2, int COUNT>
constexpr bool rows_reg() {
  return row_threads<LN2, COUNT>() == COUNT * (1 << LN2) / 16 && LN2 >= 6;
}

// COUNT rows src[w] -> radix-16 first pass from registers into rows + w*RS, barrier, the
// remaining forward passes (thread t owns butterfly t % (N2/16) of row t / (N2/16)).
template <int LN2, int COUNT, int NT, typename CT>
__device__ __forceinline__ void rows_forward_from_global(CT* rows, int RS, const CT* s0, const CT* s1,
                                                         const CT* s2, const CT* s3, const CT* tw) {
  constexpr int M1 = (1 << LN2) / 16;
  const int w = threadIdx.x / M1, j = threadIdx.x - (threadIdx.x / M1) * M1;
  const CT* p = w == 0 ? s0 : (w == 1 ? s1 : (w == 2 ? s2 : s3));  // selects, no local array
  CT v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = p[j + r * M1];
  fft_first_from_regs<-1>(v, rows + w * RS, j);
  __syncthreads();
  fft_after_first<LN2, COUNT, NT, -1>(rows, RS, tw);
}

// Two rows (rows, rows + RS) inverse-transformed in smem up to the last pass, which goes to
// registers: output i of row w is scaled by the inverse four-step twiddle exp(+2 pi i r_w i / N)
// (geometric in i = j + r*NS, exact anchors every 4) and stored to dst_w[i]; row b is skipped
// when it is row a (self-paired rows). Half the threads per row, consecutive j per warp.
// ROWS = 4: two such pairs (rows 2, 3 -> dc, dd at row indices ra, rb), a quarter of the threads each.
template <int LN2, int NT, typename CT, int ROWS = 2>
__device__ __forceinline__ void rows_inverse_to_global(CT* rows, int RS, int ra, int rb, bool self, CT* da,
                                                       CT* db, RealOf<CT> inv_n, const CT* tw, CT* dc = nullptr,
                                                       CT* dd = nullptr) {
  using T = RealOf<CT>;
  fft_all_but_last<LN2, ROWS, NT, +1>(rows, RS, tw);
  constexpr int NS = Pow2Plan<LN2>::kLastNs, R = Pow2Plan<LN2>::kLastR, HT = NT / ROWS;
  static_assert(NS % HT == 0, "rows_inverse_to_global: threads must tile the last pass");
  const int w = threadIdx.x / HT, jt = threadIdx.x - (threadIdx.x / HT) * HT;
  if ((w & 1) && self) return;
  const int rw = (w & 1) ? rb : ra;
  CT* dst = w == 0 ? da : (w == 1 ? db : (w == 2 ? dc : dd));
  const CT step = expi_pi(static_cast<T>(static_cast<long>(rw) * NS) * inv_n);
#pragma unroll
  for (int p = 0; p < NS / HT; ++p) {
    const int j = jt + p * HT;
    CT v[R];
    fft_last_to_regs<LN2, +1>(rows + w * RS, j, tw, v);
    CT wt = Cx<CT>::mk(1.f, 0.f);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = j + r * NS;
      wt = (r % 4 == 0) ? expi_pi(static_cast<T>(static_cast<long>(rw) * i) * inv_n) : cmul(wt, step);
      dst[i] = cmul(v[r], wt);
    }
  }
}

// The channel-split product in registers at the forward transforms' last pass. Thread j runs
// the last-pass butterflies j of rows xa / ka and jb of rows xb / kb, where jb's outputs are
// the conjugate partners of j's (k -> N2 - 1 - k, or N2 - k for row pair 0): the product needs
// no smem round trip of the four spectra. Z_a / Z_b are stored in place into rows ka / kb (the
// positions this thread just read), ready for the inverse. Requires NS last-pass butterflies =
// the threads of one row group.
// pa / pb non-null: the kernel spectrum rows come from global memory (rows_conv: P already
// row-transformed) and Z goes in place into the X rows instead.
template <int LN2, typename CT>
__device__ __forceinline__ void rows_last_zmix(CT* rows, int RS, int xra, int xrb, int kra, int krb, int ra, int j,
                                               RealOf<CT> s, const CT* tw, const CT* pa = nullptr,
                                               const CT* pb = nullptr) {
  constexpr int NS = Pow2Plan<LN2>::kLastNs, R = Pow2Plan<LN2>::kLastR;
  const int jb = ra == 0 ? (NS - j) & (NS - 1) : NS - 1 - j;
  CT xa[R], xb[R], ka[R], kb[R];
  fft_last_to_regs<LN2, -1>(rows + xra * RS, j, tw, xa);
  fft_last_to_regs<LN2, -1>(rows + xrb * RS, jb, tw, xb);
  if (pa != nullptr) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      ka[r] = __ldg(pa + j + r * NS);
      kb[r] = __ldg(pb + jb + r * NS);
    }
  } else {
    fft_last_to_regs<LN2, -1>(rows + kra * RS, j, tw, ka);
    fft_last_to_regs<LN2, -1>(rows + krb * RS, jb, tw, kb);
  }
  CT* za = rows + (pa != nullptr ? xra : kra) * RS + sidx(j);
  CT* zb = rows + (pa != nullptr ? xrb : krb) * RS + sidx(jb);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    // output k = j + r NS of row a pairs with output jb + rp NS of row b
    const int rp = (ra == 0 && j == 0) ? (R - r) & (R - 1) : R - 1 - r;
    CT xo = xb[0], po = kb[0];
#pragma unroll
    for (int q = 1; q < R; ++q) {  // select without dynamic register indexing
      if (q == rp) {
        xo = xb[q];
        po = kb[q];
      }
    }
    za[r * padded(NS)] = zmix(xa[r], cconj(xo), ka[r], cconj(po), s);
    zb[rp * padded(NS)] = zmix(xo, cconj(xa[r]), po, cconj(ka[r]), s);
  }
}

// Forward row FFTs of the packed kernel, kSpecRows consecutive rows per CTA.
// grid (N1 / kSpecRows, slots)
template <int LN2, typename CT>
__global__ void __launch_bounds__(row_threads<LN2, kSpecRows>()) rows_spec(int log_n, CT* P, const CT* tw) {
  using T = RealOf<CT>;
  constexpr int N2 = 1 << LN2;
  constexpr int NT = row_threads<LN2, kSpecRows>();
  constexpr int RS = padded(N2);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CT* row = reinterpret_cast<CT*>(smem_raw);
  const long N = 1L << log_n;
  CT* p = P + static_cast<long>(blockIdx.y) * N + static_cast<long>(blockIdx.x) * kSpecRows * N2;
  // All of this thread's loads are issued before any smem store (loads in flight, not a
  // load -> store dependency per element).
  if constexpr (rows_reg<LN2, kSpecRows>()) {
    constexpr int M1 = N2 / 16;
    const int w = threadIdx.x / M1, j = threadIdx.x - (threadIdx.x / M1) * M1;
    CT v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = p[w * N2 + j + r * M1];
    fft_first_from_regs<-1>(v, row + w * RS, j);
    __syncthreads();
    fft_middle<LN2, kSpecRows, NT, -1>(row, RS, tw);
    constexpr int NS = Pow2Plan<LN2>::kLastNs, R = Pow2Plan<LN2>::kLastR;
    static_assert((kSpecRows * NS) % NT == 0, "rows_spec: threads must tile the last pass");
#pragma unroll
    for (int q = 0; q < kSpecRows * NS / NT; ++q) {
      const int bq = threadIdx.x + q * NT, f = bq / NS, jb = bq - f * NS;
      CT y[R];
      fft_last_to_regs<LN2, -1>(row + f * RS, jb, tw, y);
#pragma unroll
      for (int r = 0; r < R; ++r) p[f * N2 + jb + r * NS] = y[r];
    }
    return;
  }
  constexpr int PER = kSpecRows * N2 / NT;
  static_assert(PER * NT == kSpecRows * N2, "rows_spec: threads must tile the rows");
  CT v[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) v[q] = p[threadIdx.x + q * NT];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int i = threadIdx.x + q * NT;
    row[(i / N2) * RS + sidx(i % N2)] = v[q];
  }
  __syncthreads();
  fft_pow2<LN2, kSpecRows, NT, -1>(row, RS, tw);
  for (int i = threadIdx.x; i < kSpecRows * N2; i += NT) p[i] = row[(i / N2) * RS + sidx(i % N2)];
}

// Signal rows k1 = r and N1 - r together: forward FFTs, channel-split product with the
// kernel spectrum, inverse FFTs, inverse four-step twiddle. grid (N1/2 + 1, slots*B)
// `batch`: items per slot (batch * segments); item0: first item of this launch.
template <int LN2, typename CT>
__global__ void __launch_bounds__(row_threads<LN2, 2>(), kRconvThreadsPerSm / (sizeof(CT) / 8) / row_threads<LN2, 2>()) rows_conv(int log_n, int batch, CT* X, const CT* P, const CT* tw, int item0) {
  using T = RealOf<CT>;
  constexpr int N2 = 1 << LN2;
  constexpr int NT = row_threads<LN2, 2>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CT* rows = reinterpret_cast<CT*>(smem_raw);  // [2][N2]
  const long N = 1L << log_n;
  const int N1 = static_cast<int>(N >> LN2);
  const int item = item0 + blockIdx.y;
  const int slot = item / batch;
  const int ra = blockIdx.x, rb = (N1 - ra) & (N1 - 1);
  const bool self = ra == rb;
  CT* xa = X + static_cast<long>(item) * N + static_cast<long>(ra) * N2;
  CT* xb = X + static_cast<long>(item) * N + static_cast<long>(rb) * N2;
  const CT* pa = P + static_cast<long>(slot) * N + static_cast<long>(ra) * N2;
  const CT* pb = P + static_cast<long>(slot) * N + static_cast<long>(rb) * N2;
  constexpr int RS = padded(N2);  // second row's offset
  constexpr int KPT = N2 / NT;
  static_assert(KPT * NT == N2, "rows_conv: threads must tile a row");
  // Register-ended transforms when the threads are exactly the first pass's butterflies
  // (every LN2 >= 8): thread t loads the 16 inputs j + r*N2/16 of row t / (N2/16) and runs
  // that radix-16 butterfly from registers; the inverse's last pass writes global memory.
  constexpr bool REG = rows_reg<LN2, 2>();
  if constexpr (REG) {
    // (the kernel-spectrum prefetch is issued after the first pass, registers permitting)
    constexpr int M1 = N2 / 16;
    const int w = threadIdx.x / M1, j = threadIdx.x - (threadIdx.x / M1) * M1;
    const CT* src = w == 0 ? xa : xb;
    CT v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = src[j + r * M1];
    fft_first_from_regs<-1>(v, rows + w * RS, j);
    __syncthreads();
    if constexpr (2 * NT == Pow2Plan<LN2>::kLastNs) {
      // middle passes in smem; the last pass and the product in registers (rows_conv_fk's
      // scheme, two butterfly pairs per thread), Z in place in the X rows, then the inverse
      fft_middle<LN2, 2, NT, -1>(rows, RS, tw);
      const T sc = T(0.25) / static_cast<T>(N);
      rows_last_zmix<LN2>(rows, RS, 0, 1, -1, -1, ra, threadIdx.x, sc, tw, pa, pb);
      rows_last_zmix<LN2>(rows, RS, 0, 1, -1, -1, ra, threadIdx.x + NT, sc, tw, pa, pb);
      __syncthreads();
      rows_inverse_to_global<LN2, NT>(rows, RS, ra, rb, self, xa, xb, T(2) / static_cast<T>(N), tw);
      return;
    }
    fft_after_first<LN2, 2, NT, -1>(rows, RS, tw);
  } else {
    constexpr int PER = N2 / NT;
    static_assert(PER * NT == N2, "rows_conv: threads must tile a row");
    CT va[PER], vb[PER];  // loads in flight before any smem store
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      va[q] = xa[threadIdx.x + q * NT];
      vb[q] = xb[threadIdx.x + q * NT];
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      rows[sidx(threadIdx.x + q * NT)] = va[q];
      rows[RS + sidx(threadIdx.x + q * NT)] = vb[q];
    }
    __syncthreads();
    fft_pow2<LN2, 2, NT, -1>(rows, RS, tw);
  }
  const T s = T(0.25) / static_cast<T>(N);
#pragma unroll
  for (int q = 0; q < KPT; ++q) {
    const int k = threadIdx.x + q * NT;
    if (k >= N2) continue;
    const int kb = ra == 0 ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k);
    if (self && kb < k) continue;
    const CT xk = rows[sidx(k)], xo = rows[RS + sidx(kb)];
    const CT pk = __ldg(pa + k), po = __ldg(pb + kb);
    const CT zk = zmix(xk, cconj(xo), pk, cconj(po), s);
    const CT zo = zmix(xo, cconj(xk), po, cconj(pk), s);
    rows[sidx(k)] = zk;
    rows[RS + sidx(kb)] = zo;
    if (self) rows[sidx(kb)] = zo;
  }
  __syncthreads();
  const T inv_n = T(2) / static_cast<T>(N);
  if constexpr (REG) {
    rows_inverse_to_global<LN2, NT>(rows, RS, ra, rb, self, xa, xb, inv_n, tw);
    return;
  }
  fft_pow2<LN2, 2, NT, +1>(rows, RS, tw);
  // Inverse four-step twiddle exp(+2 pi i k1 i / N): geometric in this thread's i (step NT),
  // exact anchors every 4 elements as in cols_fwd.
  const CT step_a = expi_pi(static_cast<T>(static_cast<long>(ra) * NT) * inv_n);
  const CT step_b = expi_pi(static_cast<T>(static_cast<long>(rb) * NT) * inv_n);
  CT wa = Cx<CT>::mk(1.f, 0.f), wb = wa;
#pragma unroll
  for (int q = 0; q < N2 / NT; ++q) {
    const int i = threadIdx.x + q * NT;
    if (q % 4 == 0) {
      wa = expi_pi(static_cast<T>(static_cast<long>(ra) * i) * inv_n);
      wb = expi_pi(static_cast<T>(static_cast<long>(rb) * i) * inv_n);
    } else {
      wa = cmul(wa, step_a);
      wb = cmul(wb, step_b);
    }
    xa[i] = cmul(rows[sidx(i)], wa);
    if (!self) xb[i] = cmul(rows[RS + sidx(i)], wb);
  }
}


// rows_conv with the kernel's row stage fused in (large steps, see conv_fuse_kernel_rows):
// K holds the kernel's COLUMN-stage output (cols_fwd<Kernel>, no rows_spec pass); each CTA
// transforms the kernel rows ra / rb alongside the signal rows (4 transforms), so the kernel
// spectrum never makes a round trip through memory. grid (N1/2 + 1, slots*B)
// slot_map (optional): the launch covers a subset of the step's slots (launch slot -> slot).
template <int LN2, typename CT>
__global__ void __launch_bounds__(row_threads<LN2, 4>()) rows_conv_fk(int log_n, int batch, CT* X, const CT* K,
                                                                  const CT* tw, int item0, const int* slot_map) {
  using T = RealOf<CT>;
  constexpr int N2 = 1 << LN2;
  constexpr int NT = row_threads<LN2, 4>();
  constexpr int RS = padded(N2);
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CT* rows = reinterpret_cast<CT*>(smem_raw);  // [4][RS]: x a, x b, k a, k b
  const long N = 1L << log_n;
  const int N1 = static_cast<int>(N >> LN2);
  int item = item0 + blockIdx.y;
  int slot = item / batch;
  if (slot_map != nullptr) {
    const int sub = item - slot * batch;
    slot = __ldg(slot_map + slot);
    item = slot * batch + sub;
  }
  const int ra = blockIdx.x, rb = (N1 - ra) & (N1 - 1);
  const bool self = ra == rb;
  CT* xa = X + static_cast<long>(item) * N + static_cast<long>(ra) * N2;
  CT* xb = X + static_cast<long>(item) * N + static_cast<long>(rb) * N2;
  const CT* xa_in = xa;
  const CT* xb_in = xb;
  const CT* ka = K + static_cast<long>(slot) * N + static_cast<long>(ra) * N2;
  const CT* kb_ = K + static_cast<long>(slot) * N + static_cast<long>(rb) * N2;
  constexpr bool REG = rows_reg<LN2, 4>();
  if constexpr (REG && NT == Pow2Plan<LN2>::kLastNs) {
    // first pass from global, middle passes in smem, the last pass + product in registers
    constexpr int M1 = N2 / 16;
    {
      const int w = threadIdx.x / M1, j = threadIdx.x - (threadIdx.x / M1) * M1;
      const CT* p = w == 0 ? xa_in : (w == 1 ? xb_in : (w == 2 ? ka : kb_));
      CT v[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) v[r] = p[j + r * M1];
      fft_first_from_regs<-1>(v, rows + w * RS, j);
    }
    __syncthreads();
    fft_middle<LN2, 4, NT, -1>(rows, RS, tw);
    rows_last_zmix<LN2>(rows, RS, 0, 1, 2, 3, ra, threadIdx.x, T(0.25) / static_cast<T>(N), tw);
    __syncthreads();
    rows_inverse_to_global<LN2, NT>(rows + 2 * RS, RS, ra, rb, self, xa, xb, T(2) / static_cast<T>(N), tw);
    return;
  } else if constexpr (REG) {
    rows_forward_from_global<LN2, 4, NT>(rows, RS, xa_in, xb_in, ka, kb_, tw);
  } else {
    constexpr int PER = (N2 + NT - 1) / NT;
    CT v[4][PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int i = threadIdx.x + q * NT;
      if (N2 % NT == 0 || i < N2) {
        v[0][q] = xa_in[i];
        v[1][q] = xb_in[i];
        v[2][q] = __ldg(ka + i);
        v[3][q] = __ldg(kb_ + i);
      }
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int i = threadIdx.x + q * NT;
      if (N2 % NT == 0 || i < N2) {
#pragma unroll
        for (int r = 0; r < 4; ++r) rows[r * RS + sidx(i)] = v[r][q];
      }
    }
    __syncthreads();
    fft_pow2<LN2, 4, NT, -1>(rows, RS, tw);
  }
  const T s = T(0.25) / static_cast<T>(N);
  constexpr int KPT = (N2 + NT - 1) / NT;
  CT zk[KPT], zo[KPT];
#pragma unroll
  for (int q = 0; q < KPT; ++q) {
    const int k = threadIdx.x + q * NT;
    if (k >= N2) continue;
    const int kb = ra == 0 ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k);
    const CT xk = rows[sidx(k)], xo = rows[RS + sidx(kb)];
    const CT pk = rows[2 * RS + sidx(k)], po = rows[3 * RS + sidx(kb)];
    zk[q] = zmix(xk, cconj(xo), pk, cconj(po), s);
    zo[q] = zmix(xo, cconj(xk), po, cconj(pk), s);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < KPT; ++q) {
    const int k = threadIdx.x + q * NT;
    if (k >= N2) continue;
    const int kb = ra == 0 ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k);
    if (self && kb < k) continue;
    rows[sidx(k)] = zk[q];
    if (self) rows[sidx(kb)] = zo[q];
    else rows[RS + sidx(kb)] = zo[q];
  }
  __syncthreads();
  const T inv_n = T(2) / static_cast<T>(N);
  if constexpr (REG) {
    rows_inverse_to_global<LN2, NT>(rows, RS, ra, rb, self, xa, xb, inv_n, tw);
    return;
  }
  fft_pow2<LN2, 2, NT, +1>(rows, RS, tw);
  for (int i = threadIdx.x; i < N2; i += NT) {
    xa[i] = cmul(rows[sidx(i)], expi_pi(static_cast<T>(static_cast<long>(ra) * i) * inv_n));
    if (!self) xb[i] = cmul(rows[RS + sidx(i)], expi_pi(static_cast<T>(static_cast<long>(rb) * i) * inv_n));
  }
}

// Two conv steps sharing a signal spectrum (launch_conv_shared): for pair p, step A's item
// (slot pa[p]) and step B's item (slot pb[p]) convolve the same X (in Xa). One CTA per row pair
// and item pair transforms the two X rows once and both kernels' rows (6 forward row FFTs
// instead of 8), forms both channel-split products, inverts the 4 rows and stores A's result in
// place into Xa (only this CTA reads these rows) and B's into Xb.
template <int LN2>
constexpr int pair_threads() {
  constexpr int t = 6 * (1 << LN2) / 16;
  return t <= 32 ? 32 : (t <= 64 ? 64 : (t <= 128 ? 128 : (t <= 256 ? 256 : (t <= 512 ? 512 : 1024))));
}
template <int LN2, typename CT>
__global__ void __launch_bounds__(pair_threads<LN2>()) rows_conv_pair(int log_n, int batch, CT* Xa, CT* Xb,
                                                                   const CT* Ka, const CT* Kb, const int* pa,
                                                                   const int* pb, const CT* tw, int item0) {
  using T = RealOf<CT>;
  constexpr int N2 = 1 << LN2;
  constexpr int NT = pair_threads<LN2>();
  constexpr int RS = padded(N2);
  constexpr int M1 = N2 / 16;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CT* rows = reinterpret_cast<CT*>(smem_raw);  // [6][RS]: x a, x b, kA a, kA b, kB a, kB b
  const long N = 1L << log_n;
  const int N1 = static_cast<int>(N >> LN2);
  const int pi = item0 + blockIdx.y;
  const int p = pi / batch, sub = pi - p * batch;
  const int sa = __ldg(pa + p), sb = __ldg(pb + p);
  const long ia = static_cast<long>(sa) * batch + sub, ib = static_cast<long>(sb) * batch + sub;
  const int ra = blockIdx.x, rb = (N1 - ra) & (N1 - 1);
  const bool self = ra == rb;
  CT* xa = Xa + ia * N + static_cast<long>(ra) * N2;
  CT* xb = Xa + ia * N + static_cast<long>(rb) * N2;
  {
    const int w = threadIdx.x / M1, j = threadIdx.x - (threadIdx.x / M1) * M1;
    if (w < 6) {
      const long r = (w & 1) ? rb : ra;
      const CT* src = w < 2 ? Xa + ia * N : (w < 4 ? Ka + static_cast<long>(sa) * N : Kb + static_cast<long>(sb) * N);
      src += r * N2;
      CT v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = src[j + q * M1];
      fft_first_from_regs<-1>(v, rows + w * RS, j);
    }
  }
  __syncthreads();
  fft_after_first<LN2, 6, NT, -1>(rows, RS, tw);
  const T s = T(0.25) / static_cast<T>(N);
  constexpr int KPT = (N2 + NT - 1) / NT;
  CT zak[KPT], zao[KPT], zbk[KPT], zbo[KPT];
#pragma unroll
  for (int q = 0; q < KPT; ++q) {
    const int k = threadIdx.x + q * NT;
    if (k >= N2) continue;
    const int kb = ra == 0 ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k);
    const CT xk = rows[sidx(k)], xo = rows[RS + sidx(kb)];
    const CT ak = rows[2 * RS + sidx(k)], ao = rows[3 * RS + sidx(kb)];
    const CT bk = rows[4 * RS + sidx(k)], bo = rows[5 * RS + sidx(kb)];
    zak[q] = zmix(xk, cconj(xo), ak, cconj(ao), s);
    zao[q] = zmix(xo, cconj(xk), ao, cconj(ak), s);
    zbk[q] = zmix(xk, cconj(xo), bk, cconj(bo), s);
    zbo[q] = zmix(xo, cconj(xk), bo, cconj(bk), s);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < KPT; ++q) {
    const int k = threadIdx.x + q * NT;
    if (k >= N2) continue;
    const int kb = ra == 0 ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k);
    if (self && kb < k) continue;
    // Z_A into rows 0, 1 (the X rows' slots), Z_B into rows 2, 3: the inverse runs on rows 0..3
    rows[sidx(k)] = zak[q];
    rows[2 * RS + sidx(k)] = zbk[q];
    if (self) {
      rows[sidx(kb)] = zao[q];
      rows[2 * RS + sidx(kb)] = zbo[q];
    } else {
      rows[RS + sidx(kb)] = zao[q];
      rows[3 * RS + sidx(kb)] = zbo[q];
    }
  }
  __syncthreads();
  CT* ya = Xb + ib * N + static_cast<long>(ra) * N2;
  CT* yb = Xb + ib * N + static_cast<long>(rb) * N2;
  rows_inverse_to_global<LN2, NT, CT, 4>(rows, RS, ra, rb, self, xa, xb, T(2) / static_cast<T>(N), tw, ya, yb);
}

// ---- dispatch -----------------------------------------------------------------------------
// Launches over `items` grid rows in chunks of at most kMaxGridY (grid.y limit).
template <typename F>
void for_item_chunks(int items, F&& f) {
  for (int i0 = 0; i0 < items; i0 += kMaxGridY) f(i0, items - i0 < kMaxGridY ? items - i0 : kMaxGridY);
}

template <typename CT> const CT* tw_table(const StepArgs& a);
template <> const float2* tw_table<float2>(const StepArgs& a) { return a.tw; }
template <> const double2* tw_table<double2>(const StepArgs& a) { return a.tw64; }

template <int LN1, typename CT>
void cols_fwd_t(ColSrc src, const StepArgs& a, const float2* ir, long taps, const ConvGeom& g, int items,
                CT* out, int window, bool mask_out, cudaStream_t s, const int* slot_map = nullptr) {
  constexpr int C = ColCfg<CT>::kElems / (1 << LN1);
  constexpr int smem = ColCfg<CT>::kSmem(1 << LN1);
  static const bool attrs_set = [] {
    for (const void* fn : {reinterpret_cast<const void*>(cols_fwd<LN1, ColSrc::Signal, CT>),
                           reinterpret_cast<const void*>(cols_fwd<LN1, ColSrc::Kernel, CT>),
                           reinterpret_cast<const void*>(cols_fwd<LN1, ColSrc::DelayTaps, CT>)}) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    return true;
  }();
  (void)attrs_set;
  if (src == ColSrc::DelayTaps) {
    if constexpr (sizeof(CT) == 8 && LN1 >= 8) note_prologue_kernel(reinterpret_cast<const void*>(delay_cols<LN1>));
    else note_prologue_kernel(reinterpret_cast<const void*>(cols_fwd<LN1, ColSrc::DelayTaps, CT>));
  }
  if (src == ColSrc::Kernel) note_prologue_kernel(reinterpret_cast<const void*>(cols_fwd<LN1, ColSrc::Kernel, CT>));
  constexpr int nt = ColCfg<CT>::kThreads;
  for_item_chunks(items, [&](int i0, int n) {
    const dim3 grid(static_cast<unsigned>((1L << g.log_n2) / C), static_cast<unsigned>(n));
    const SegArgs sg = seg_args(g, i0, mask_out, slot_map);
    if (src == ColSrc::Signal) {
      cols_fwd<LN1, ColSrc::Signal, CT><<<grid, nt, smem, s>>>(a, ir, taps, g.log_n, out, window, sg);
    } else if (src == ColSrc::DelayTaps) {
      if constexpr (sizeof(CT) == 8 && LN1 >= 8) {  // fp32, <= 32 columns per CTA: the sparse direct DFT
        const dim3 dgrid(static_cast<unsigned>(std::max<long>(1, ((1L << g.log_n2) / C) / kDelayColBlocks)), static_cast<unsigned>(n));
        delay_cols<LN1><<<dgrid, kDelayColThreads, 0, s>>>(reinterpret_cast<const float*>(ir) + static_cast<long>(i0) * kTaps * kTapRec,
                                                          taps, g.log_n, out + static_cast<long>(i0) * (1L << g.log_n), a.tw);
      } else {
        cols_fwd<LN1, ColSrc::DelayTaps, CT><<<grid, nt, smem, s>>>(a, ir, taps, g.log_n, out, window, sg);
      }
    } else {
      cols_fwd<LN1, ColSrc::Kernel, CT><<<grid, nt, smem, s>>>(a, ir, taps, g.log_n, out, window, sg);
    }
  });
}

template <int LN1, typename CT>
void cols_inv_t(const StepArgs& a, const ConvGeom& g, CT* X, bool to_buf, cudaStream_t s) {
  constexpr int C = ColCfg<CT>::kElems / (1 << LN1);
  constexpr int smem = ColCfg<CT>::kSmem(1 << LN1);
  static const bool done = [] {
    for (const void* fn : {reinterpret_cast<const void*>(cols_inv<LN1, false, CT>), reinterpret_cast<const void*>(cols_inv<LN1, true, CT>)}) {
      cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    return true;
  }();
  (void)done;
  constexpr int nt = ColCfg<CT>::kThreads;
  for_item_chunks(a.slots * a.batch * g.nseg, [&](int i0, int n) {
    const dim3 grid(static_cast<unsigned>((1L << g.log_n2) / C), static_cast<unsigned>(n));
    if (to_buf) cols_inv<LN1, true, CT><<<grid, nt, smem, s>>>(a, g.log_n, X, seg_args(g, i0));
    else cols_inv<LN1, false, CT><<<grid, nt, smem, s>>>(a, g.log_n, X, seg_args(g, i0));
  });
}

template <int LN2, typename CT>
void rows_spec_t(const ConvGeom& g, int slots, CT* P, const CT* tw, cudaStream_t s) {
  constexpr int smem = kSpecRows * padded(1 << LN2) * static_cast<int>(sizeof(CT));
  static const bool done = [] {
    cudaFuncSetAttribute(rows_spec<LN2, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)done;
  note_prologue_kernel(reinterpret_cast<const void*>(rows_spec<LN2, CT>));
  for (int s0 = 0; s0 < slots; s0 += kMaxGridY) {
    const int n = slots - s0 < kMaxGridY ? slots - s0 : kMaxGridY;
    const dim3 grid(static_cast<unsigned>((1L << g.log_n1) / kSpecRows), static_cast<unsigned>(n));
    rows_spec<LN2, CT><<<grid, row_threads<LN2, kSpecRows>(), smem, s>>>(g.log_n, P + static_cast<long>(s0) * g.n, tw);
  }
}

template <int LN2, typename CT>
void rows_conv_t(const ConvGeom& g, int items, int per_slot, CT* X, const CT* P, const CT* tw, cudaStream_t s) {
  constexpr int smem = 2 * padded(1 << LN2) * static_cast<int>(sizeof(CT));
  static const bool done = [] {
    cudaFuncSetAttribute(rows_conv<LN2, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)done;
  for_item_chunks(items, [&](int i0, int n) {
    const dim3 grid(static_cast<unsigned>((1L << g.log_n1) / 2 + 1), static_cast<unsigned>(n));
    rows_conv<LN2, CT><<<grid, row_threads<LN2, 2>(), smem, s>>>(g.log_n, per_slot, X, P, tw, i0);
  });
}

template <int LN2, typename CT>
void rows_conv_fk_t(const ConvGeom& g, int items, int per_slot, CT* X, const CT* K, const CT* tw, cudaStream_t s,
                    const int* slot_map = nullptr) {
  constexpr int smem = 4 * padded(1 << LN2) * static_cast<int>(sizeof(CT));
  static const bool done = [] {
    cudaFuncSetAttribute(rows_conv_fk<LN2, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)done;
  for_item_chunks(items, [&](int i0, int n) {
    const dim3 grid(static_cast<unsigned>((1L << g.log_n1) / 2 + 1), static_cast<unsigned>(n));
    rows_conv_fk<LN2, CT><<<grid, row_threads<LN2, 4>(), smem, s>>>(g.log_n, per_slot, X, K, tw, i0, slot_map);
  });
}

template <int LN2, typename CT>
void rows_conv_pair_t(const ConvGeom& g, int items, int per_slot, CT* Xa, CT* Xb, const CT* Ka, const CT* Kb,
                      const int* pa, const int* pb, const CT* tw, cudaStream_t s) {
  constexpr int smem = 6 * padded(1 << LN2) * static_cast<int>(sizeof(CT));
  static const bool done = [] {
    cudaFuncSetAttribute(rows_conv_pair<LN2, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)done;
  for_item_chunks(items, [&](int i0, int n) {
    const dim3 grid(static_cast<unsigned>((1L << g.log_n1) / 2 + 1), static_cast<unsigned>(n));
    rows_conv_pair<LN2, CT><<<grid, pair_threads<LN2>(), smem, s>>>(g.log_n, per_slot, Xa, Xb, Ka, Kb, pa, pb, tw, i0);
  });
}

// log2 of the column length N1 = 2^(a/2) and row length N2 = 2^(a - a/2), a in [13, 22].
#define MGB_DISPATCH_LN(var, FN, CT, ...)                  \
  switch (var) {                                           \
    case 6: FN<6, CT>(__VA_ARGS__); break;                 \
    case 7: FN<7, CT>(__VA_ARGS__); break;                 \
    case 8: FN<8, CT>(__VA_ARGS__); break;                 \
    case 9: FN<9, CT>(__VA_ARGS__); break;                 \
    case 10: FN<10, CT>(__VA_ARGS__); break;               \
    case 11: FN<11, CT>(__VA_ARGS__); break;               \
    default: throw std::invalid_argument("fft convolution size out of range"); \
  }

// Kernel spectrum P (four-step order) of the packed kernels in `ir` ([slots][taps]).
template <typename CT>
void kernel_spectrum(ColSrc src, const StepArgs& a, const ConvGeom& g, const float2* ir, long taps, int window,
                     CT* P, cudaStream_t s) {
  MGB_DISPATCH_LN(g.log_n1, cols_fwd_t, CT, src, a, ir, taps, g, a.slots, P, window, false, s);
  // Large steps leave the row stage to rows_conv_fk (conv_fuse_kernel_rows).
  if (!conv_fuse_kernel_rows(g, a.slots)) MGB_DISPATCH_LN(g.log_n2, rows_spec_t, CT, g, a.slots, P, tw_table<CT>(a), s);
}

// ---- reverb impulse response (masked noise STFT -> ISTFT) ----------------------------------
constexpr int kRevBins = 193;      // kReverbStftLength / 2 + 1
constexpr int kRevParamBins = 192;
constexpr int kRevFpc = 16;        // adjoint: hops per CTA
constexpr int kRevThreads = 512;   // adjoint: threads per CTA
constexpr int kRevFS = padded(384);  // frame stride in smem (padded layout)
// Forward: 10 hops (11 frames) per CTA of 256 threads — 36 KB of frames, four CTAs per SM, so
// config 2's 12 reverbs (46 x 12 = 552 CTAs) fit one wave of 592 slots (16 hops x 512 threads
// made 348 CTAs for 296 slots: 1.18 waves).
constexpr int kRevFwdFpc = 10;
constexpr int kRevFwdThreads = 256;

// grid (ceil(frames / kRevFwdFpc), slots). Each CTA inverse-transforms frames m0-1 .. m0+9
// (mid and side packed as one complex transform each) and overlap-adds hops m0 .. m0+9.
// The per-bin mask exp(H0 + m Hdecay) is geometric in the frame index m: one exact expf
// anchor per bin for the CTA's first frame and the ratio exp(Hdecay), both with fp64
// exponents (processors.cpp:171-175), then <= 10 products. The noise STFT is read as one
// 16-byte (mid, side) value per (frame, bin).
__global__ void __launch_bounds__(kRevFwdThreads, 4) reverb_ir(const double* params, ReverbConst rc, float2* ir,
                                                            long ir_stride) {
  constexpr int kRevThreads = kRevFwdThreads, kRevFpc = kRevFwdFpc;
  extern __shared__ float2 fr[];  // [(kRevFpc + 1)][kRevFS]
  __shared__ float base[2][kRevBins], ratio[2][kRevBins];
  __shared__ float2 tw384[384];
  __shared__ float2 inv_cover[192];  // .x first hop, .y later hops
  const int slot = blockIdx.y;
  const double* row = params + static_cast<long>(slot) * 4 * kRevParamBins;
  const int m_first = blockIdx.x * kRevFpc - 1;
  for (int k = threadIdx.x; k < 384; k += kRevThreads) {
    tw384[k] = __ldg(tw384_table(rc.consts) + k);
    if (k < 192) inv_cover[k] = __ldg(cover_table(rc.consts) + k);
  }
  for (int idx = threadIdx.x; idx < 2 * kRevBins; idx += kRevThreads) {
    const int which = idx / kRevBins, k = idx - which * kRevBins;
    const int bin = k < kRevParamBins ? k : kRevParamBins - 1;
    const double* color = row + which * 2 * kRevParamBins;
    const double decay = color[kRevParamBins + bin];
    base[which][k] = expf(static_cast<float>(color[bin] + m_first * decay));
    ratio[which][k] = expf(static_cast<float>(decay));
  }
  __syncthreads();
  // Fill: thread owns one (bin-pair k, kk) column across all frames, walking the gains.
  for (int k = threadIdx.x; k < 384; k += kRevThreads) {
    const bool upper = k > 192;
    const int kk = upper ? 384 - k : k;
    float gm = base[0][kk], gs = base[1][kk];
    const float rm = ratio[0][kk], rs = ratio[1][kk];
#pragma unroll 4
    for (int f = 0; f <= kRevFpc; ++f) {
      const int m = m_first + f;
      float2 z = make_float2(0.f, 0.f);
      if (m >= 0 && m < rc.frames) {
        const float4 q = __ldg(rc.stft_ms + static_cast<long>(m) * kRevBins + kk);
        float2 M = make_float2(q.x * gm, q.y * gm);
        float2 S = make_float2(q.z * gs, q.w * gs);
        if (upper) {
          M = cconj(M);
          S = cconj(S);
        }
        z = make_float2(M.x - S.y, M.y + S.x);  // M + i S: both inverse transforms are real
      }
      fr[f * kRevFS + sidx(k)] = z;
      gm *= rm;
      gs *= rs;
    }
  }
  __syncthreads();
  fft_384<kRevFpc + 1, kRevThreads, +1>(fr, kRevFS, tw384);
  const long i0 = static_cast<long>(blockIdx.x) * kRevFpc * 192;
  for (int t = threadIdx.x; t < kRevFpc * 192; t += kRevThreads) {
    const long i = i0 + t;
    if (i >= rc.length) break;
    const int o = t % 192;
    const int f1 = t / 192 + 1;  // local frame starting in this hop
    float2 v = fr[f1 * kRevFS + sidx(o)];
    float sc = inv_cover[o].x;
    if (i >= 192) {
      v = cadd(v, fr[(f1 - 1) * kRevFS + sidx(o + 192)]);
      sc = inv_cover[o].y;
    }
    const float mid = v.x * sc, side = v.y * sc;
    ir[static_cast<long>(slot) * ir_stride + i] = make_float2(0.5f * (mid + side), 0.5f * (mid - side));
  }
}

// ---- multitap delay kernel -------------------------------------------------------------------

// Per tap record: fp64 position (processors.cpp:189-208: disabled taps, angle -> grid
// delay, window clamp) and the 39-tap zero-phase FIR (dsp.cpp:106-136 as the exact cosine
// sum). Output taps[slot][tap][kTapRec]. grid (kTaps, slots) x 64: one CTA per tap, one
// thread per coefficient.
__global__ void __launch_bounds__(64) delay_taps(const double* params, DelayConst dc, float* taps) {
  __shared__ double mag[20];
  __shared__ double cos39[kFir];
  const int tapi = blockIdx.x, slot = blockIdx.y;
  const double* tap = params + static_cast<long>(slot) * kTaps * kTapStride + tapi * kTapStride;
  float* out = taps + (static_cast<long>(slot) * kTaps + tapi) * kTapRec;
  const int t = threadIdx.x;
  if (t < 20) mag[t] = exp(tap[2 + t]);
  if (t < kFir) {
    double sk, ck;
    sincospi(2.0 * t / kFir, &sk, &ck);
    cos39[t] = ck;
  }
  if (t == 63) {  // second warp (lanes >= 39 idle in the FIR): the position
    double mx = tap[2];
    for (int k = 1; k < 20; ++k) mx = fmax(mx, tap[2 + k]);
    int d = -1;
    if (!(mx <= -60.0)) {
      const int m = tapi % 20;
      const double frac = -atan2(tap[1], tap[0]) / (2.0 * 3.14159265358979323846);
      long long dd = llround(frac * static_cast<double>(dc.span));
      dd %= dc.span;
      if (dd < 0) dd += dc.span;
      const long long lo = static_cast<long long>(m) * dc.window;
      const long long hi = min(static_cast<long long>(m + 1) * dc.window, static_cast<long long>(dc.span)) - 1;
      d = static_cast<int>(dd < lo ? lo : (dd > hi ? hi : dd));
    }
    out[0] = __int_as_float(d);
  }
  __syncthreads();
  if (t >= kFir) return;
  const int n = t;
  const int j = n >= kFirHalf ? n - kFirHalf : kFirHalf - n;
  double acc = 0.0;
  int idx = 0;
  for (int k = 0; k < kFir; ++k) {
    acc = fma(mag[k <= kFirHalf ? k : kFir - k], cos39[idx], acc);
    idx += j;
    if (idx >= kFir) idx -= kFir;
  }
  double s, c;
  sincospi(2.0 * n / (kFir - 1), &s, &c);
  out[1 + n] = static_cast<float>((0.5 - 0.5 * c) * acc / kFir);
}

// Dense multitap kernel (processors.cpp:210-227): every sample i of [0, span) sums, in tap
// order, the FIR taps of the (at most a few) windows whose clamped position lies within
// +-19 of i. Writes every sample (no memset, no scatter, deterministic).
// grid (ceil(span / 256), 2 channels, slots) x 256.
__global__ void __launch_bounds__(256) delay_dense(const float* taps, DelayConst dc, float2* ir, long ir_stride) {
  __shared__ float rec[20][kTapRec];
  const int c = blockIdx.y, slot = blockIdx.z;
  const float* in = taps + (static_cast<long>(slot) * kTaps + c * 20) * kTapRec;
  for (int q = threadIdx.x; q < 20 * kTapRec; q += blockDim.x) rec[q / kTapRec][q % kTapRec] = __ldg(in + q);
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dc.span) return;
  // Windows that can reach this CTA's samples (same range for every thread of the CTA).
  const int w = dc.window;
  const int first = blockIdx.x * blockDim.x;
  int m0 = (first - kFirHalf) / w - 1, m1 = (first + static_cast<int>(blockDim.x) + kFirHalf) / w;
  m0 = m0 < 0 ? 0 : m0;
  m1 = m1 > 19 ? 19 : m1;
  float acc = 0.f;
  for (int m = m0; m <= m1; ++m) {
    const int d = __float_as_int(rec[m][0]);
    const int j = i - d + kFirHalf;
    if (d >= 0 && j >= 0 && j < kFir) acc += rec[m][1 + j];
  }
  reinterpret_cast<float*>(ir + static_cast<long>(slot) * ir_stride + i)[c] = acc;
}

// ---- backward (adjoint) kernels -------------------------------------------------------------

// Backward row pass of a long convolution, fused: per row pair (ra, rb) of slot s, the kernel
// rows (KFFT: column-stage input, transformed here; else the finished spectrum P), then for
// every batch item the row FFTs of DY and X and
//  * the input gradient DY_c conj(H_c) (a correlation with the kernel): rows_conv's product
//    with the paired kernel values P[k] <-> P[N-k] swapped, which conjugates both channels'
//    kernel spectra; inverted and stored back into DY;
//  * the kernel-gradient spectrum sum_b DY_c conj(X_c), packed C_L + i C_R (both real):
//    conj(X_c) is the spectrum of x_c reversed, whose packed form is Z[N-k], so the same
//    product with X's pair swapped; inverted into X's b = 0 item at the end.
// `batch`: items per slot (batch * segments: the kernel gradient sums over both).
// grid (N1/2 + 1, slots chunk from slot0)
template <int LN2, bool KFFT, typename CT>
__global__ void __launch_bounds__(row_threads<LN2, 4>(), rbwd_min_blocks<LN2>()) rows_bwd(int log_n, int batch, CT* DY, CT* X,
                                                                 const CT* P, const CT* tw, int slot0) {
  using T = RealOf<CT>;
  constexpr int N2 = 1 << LN2;
  constexpr int NT = row_threads<LN2, 4>();
  constexpr int RS = padded(N2);
  extern __shared__ __align__(16) unsigned char smem_raw[];  // [8][RS]: dy a, dy b, x a, x b, h a, h b, acc a, acc b
  CT* rows = reinterpret_cast<CT*>(smem_raw);
  const long N = 1L << log_n;
  const int N1 = static_cast<int>(N >> LN2);
  const int slot = slot0 + blockIdx.y;
  const int ra = blockIdx.x, rb = (N1 - ra) & (N1 - 1);
  const bool self = ra == rb;
  const CT* pa = P + static_cast<long>(slot) * N + static_cast<long>(ra) * N2;
  const CT* pb = P + static_cast<long>(slot) * N + static_cast<long>(rb) * N2;
  CT* H = rows + 4 * RS;
  CT* A = rows + 6 * RS;
  for (int i = threadIdx.x; i < N2; i += NT) {
    H[sidx(i)] = __ldg(pa + i);
    H[RS + sidx(i)] = __ldg(pb + i);
    A[sidx(i)] = A[RS + sidx(i)] = Cx<CT>::mk(0.f, 0.f);
  }
  if constexpr (KFFT) {
    __syncthreads();
    fft_pow2<LN2, 2, NT, -1>(H, RS, tw);
  }
  const T s = T(0.25) / static_cast<T>(N);
  const T inv_n = T(2) / static_cast<T>(N);
  for (int b = 0; b < batch; ++b) {
    const long item = static_cast<long>(slot) * batch + b;
    CT* da = DY + item * N + static_cast<long>(ra) * N2;
    CT* db = DY + item * N + static_cast<long>(rb) * N2;
    const CT* xa = X + item * N + static_cast<long>(ra) * N2;
    const CT* xb = X + item * N + static_cast<long>(rb) * N2;
    __syncthreads();  // previous item's rows fully consumed
    if constexpr (rows_reg<LN2, 4>()) {
      rows_forward_from_global<LN2, 4, NT>(rows, RS, da, db, xa, xb, tw);
    } else {
      for (int i = threadIdx.x; i < N2; i += NT) {
        rows[sidx(i)] = da[i];
        rows[RS + sidx(i)] = db[i];
        rows[2 * RS + sidx(i)] = xa[i];
        rows[3 * RS + sidx(i)] = xb[i];
      }
      __syncthreads();
      fft_pow2<LN2, 4, NT, -1>(rows, RS, tw);
    }
    // Each (k, N-k) pair is read and written by one thread only: products in place.
    for (int k = threadIdx.x; k < N2; k += NT) {
      const int kb = ra == 0 ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k);
      if (self && kb < k) continue;
      const int ob = self ? sidx(kb) : RS + sidx(kb);
      const CT dk = rows[sidx(k)], dn = rows[RS + sidx(kb)];
      const CT xk = rows[2 * RS + sidx(k)], xn = rows[3 * RS + sidx(kb)];
      const CT hk = H[sidx(k)], hn = H[RS + sidx(kb)];
      // kernel gradient: DY_c conj(X_c) -> X's pair swapped
      // (a self-paired bin, k == kb, has one value: written once, as rows_conv does)
      if (!(self && kb == k)) A[sidx(k)] = cadd(A[sidx(k)], zmix(dk, cconj(dn), xn, cconj(xk), s));
      A[ob] = cadd(A[ob], zmix(dn, cconj(dk), xk, cconj(xn), s));
      // input gradient: conj(H_c) -> swapped kernel pair
      rows[sidx(k)] = zmix(dk, cconj(dn), hn, cconj(hk), s);
      rows[ob] = zmix(dn, cconj(dk), hk, cconj(hn), s);
    }
    __syncthreads();
    if constexpr (rows_reg<LN2, 4>()) {
      rows_inverse_to_global<LN2, NT>(rows, RS, ra, rb, self, da, db, inv_n, tw);
    } else {
      fft_pow2<LN2, 2, NT, +1>(rows, RS, tw);
      for (int i = threadIdx.x; i < N2; i += NT) {
        da[i] = cmul(rows[sidx(i)], expi_pi(static_cast<T>(static_cast<long>(ra) * i) * inv_n));
        if (!self) db[i] = cmul(rows[RS + sidx(i)], expi_pi(static_cast<T>(static_cast<long>(rb) * i) * inv_n));
      }
    }
  }
  __syncthreads();
  CT* oa = X + static_cast<long>(slot) * batch * N + static_cast<long>(ra) * N2;
  CT* ob = X + static_cast<long>(slot) * batch * N + static_cast<long>(rb) * N2;
  if constexpr (rows_reg<LN2, 4>()) {
    rows_inverse_to_global<LN2, NT>(A, RS, ra, rb, self, oa, ob, inv_n, tw);
    return;
  }
  fft_pow2<LN2, 2, NT, +1>(A, RS, tw);
  for (int i = threadIdx.x; i < N2; i += NT) {
    oa[i] = cmul(A[sidx(i)], expi_pi(static_cast<T>(static_cast<long>(ra) * i) * inv_n));
    if (!self) ob[i] = cmul(A[RS + sidx(i)], expi_pi(static_cast<T>(static_cast<long>(rb) * i) * inv_n));
  }
}

// Inverse column FFTs of slot items (X at item slot*batch) into a packed kernel-gradient
// buffer out[slot][taps] (x = left, y = right), first `taps` samples. grid (N2 / C, slots)
template <int LN1, typename CT>
__global__ void __launch_bounds__(ColCfg<CT>::kThreads, 2) cols_inv_buf(int log_n, int batch, const CT* X, float2* out,
                                                            long taps, const CT* tw, int slot0) {
  using T = RealOf<CT>;
  constexpr int N1 = 1 << LN1;
  constexpr int C = ColCfg<CT>::kElems / N1;
  constexpr int FS = padded(N1) + 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CT* tile = reinterpret_cast<CT*>(smem_raw);
  const long N2 = 1L << (log_n - LN1);
  const long N = 1L << log_n;
  const int slot = slot0 + blockIdx.y;
  const long col0 = static_cast<long>(blockIdx.x) * C;
  const CT* x = X + static_cast<long>(slot) * batch * N;
  // Register-ended column transform (as cols_inv): thread (c, j) loads the 16 inputs of its
  // first-pass butterfly and stores its last-pass outputs.
  constexpr int M1 = N1 / 16, JSTEP = ColCfg<CT>::kThreads / C;
  const int c = threadIdx.x % C, jt = threadIdx.x / C;
  CT v[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = __ldg(x + static_cast<long>(jt + r * M1) * N2 + col0 + c);
  fft_first_from_regs<+1>(v, tile + c * FS, jt);
  __syncthreads();
  fft_middle<LN1, C, ColCfg<CT>::kThreads, +1>(tile, FS, tw);
  constexpr int NS = Pow2Plan<LN1>::kLastNs, R = Pow2Plan<LN1>::kLastR;
#pragma unroll
  for (int p = 0; p < NS / JSTEP; ++p) {
    const int j = jt + p * JSTEP;
    CT y[R];
    fft_last_to_regs<LN1, +1>(tile + c * FS, j, tw, y);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long n = static_cast<long>(j + r * NS) * N2 + col0 + c;
      if (n < taps) out[static_cast<long>(slot) * taps + n] = narrow(y[r]);
    }
  }
}

// Reverb impulse-response adjoint (istft `dsp.cpp:165-190`, reverb_kernel
// `processors.cpp:162-187`): per frame m the time gradient of the masked frame is
// d fr[i] = dM[m hop + i] / (384 cover) (mid; side likewise, dM = (dL + dR)/2,
// dS = (dL - dR)/2), its forward 384-point FFT DFR gives the mask gradient
// d a[m][k] = c_k Re(N[m][k] conj(DFR[k])) (c_k = 1 for k = 0, 192, else 2), and
// a = exp(H0[p] + m Hd[p]), p = min(k, 191). Mid and side packed as one complex FFT.
// grid (ceil(frames / kRevFpc), slots); out partial[slot][blk][2 which][2][193] fp64.
__global__ void __launch_bounds__(kRevThreads) reverb_ir_adjoint(const double* params, ReverbConst rc, const float2* dh,
                                                                double* partial) {
  extern __shared__ float2 fr[];  // [kRevFpc][kRevFS]
  __shared__ float2 tw384[384];
  __shared__ float2 inv_cover[192];
  const int slot = blockIdx.y;
  const int m0 = blockIdx.x * kRevFpc;
  for (int k = threadIdx.x; k < 384; k += kRevThreads) {
    tw384[k] = __ldg(tw384_table(rc.consts) + k);
    if (k < 192) inv_cover[k] = __ldg(cover_table(rc.consts) + k);
  }
  __syncthreads();
  const float2* h = dh + static_cast<long>(slot) * rc.length;
  for (int t = threadIdx.x; t < kRevFpc * 384; t += kRevThreads) {
    const int f = t / 384, i = t - f * 384;
    const int m = m0 + f;
    const long idx = static_cast<long>(m) * 192 + i;
    float2 z = make_float2(0.f, 0.f);
    if (m < rc.frames && idx < rc.length) {
      const float2 g = __ldg(h + idx);
      const float sc = idx < 192 ? inv_cover[idx].x : inv_cover[idx % 192].y;
      z = make_float2(0.5f * (g.x + g.y) * sc, 0.5f * (g.x - g.y) * sc);
    }
    fr[f * kRevFS + sidx(i)] = z;
  }
  __syncthreads();
  fft_384<kRevFpc, kRevThreads, -1>(fr, kRevFS, tw384);
  const double* row = params + static_cast<long>(slot) * 4 * kRevParamBins;
  double* out = partial + (static_cast<long>(slot) * gridDim.x + blockIdx.x) * (4 * kRevBins);
  for (int item = threadIdx.x; item < 2 * kRevBins; item += kRevThreads) {
    const int which = item / kRevBins, k = item - which * kRevBins;
    const int bin = k < kRevParamBins ? k : kRevParamBins - 1;
    const double* color = row + which * 2 * kRevParamBins;
    const double c0 = color[bin], dec = color[kRevParamBins + bin];
    const float2* noise = which == 0 ? rc.stft_mid : rc.stft_side;
    const float ck = (k == 0 || k == 192) ? 1.f : 2.f;
    double g0 = 0.0, g1 = 0.0;
    for (int f = 0; f < kRevFpc; ++f) {
      const int m = m0 + f;
      if (m >= rc.frames) break;
      const float2 zk = fr[f * kRevFS + sidx(k)], zn = fr[f * kRevFS + sidx((384 - k) % 384)];
      // DFR_M = (Zk + conj Zn)/2, DFR_S = (Zk - conj Zn)/(2i)
      float2 d;
      if (which == 0) d = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y - zn.y));
      else d = make_float2(0.5f * (zk.y + zn.y), -0.5f * (zk.x - zn.x));
      const float2 nz = __ldg(noise + static_cast<long>(m) * kRevBins + k);
      const float da = ck * (nz.x * d.x + nz.y * d.y);
      const float a = expf(static_cast<float>(c0 + m * dec));
      g0 += static_cast<double>(da * a);
      g1 += static_cast<double>(m) * static_cast<double>(da * a);
    }
    out[which * 2 * kRevBins + k] = g0;
    out[which * 2 * kRevBins + kRevBins + k] = g1;
  }
}

// grid (slots) x 128: grad row [which][color 192 | decay 192]; bin 192 folds into param 191.
__global__ void reverb_grad_reduce(const double* partial, int blocks, double* grad) {
  const int slot = blockIdx.x;
  for (int item = threadIdx.x; item < 4 * kRevParamBins; item += blockDim.x) {
    const int which = item / (2 * kRevParamBins), r = item - which * 2 * kRevParamBins;
    const int kind = r / kRevParamBins, p = r - kind * kRevParamBins;
    double t = 0.0;
    for (int bk = 0; bk < blocks; ++bk) {
      const double* q = partial + (static_cast<long>(slot) * blocks + bk) * (4 * kRevBins) + which * 2 * kRevBins + kind * kRevBins;
      t += q[p];
      if (p == kRevParamBins - 1) t += q[kRevBins - 1];
    }
    grad[static_cast<long>(slot) * 4 * kRevParamBins + item] = t;
  }
}

// Multitap delay adjoint (delay_kernel `processors.cpp:210-227`, zero_phase_fir N = 39):
// the kernel gradient at the tap's 39 positions d - 19 + j is the FIR gradient; through the
// design, d lm[q] = (m_q / 39) e^{lm[q]} sum_j dfir[j] hann[j] cos(2 pi q (j - 19) / 39).
// Positions are piecewise constant in (Re z, Im z) (lround of the angle): gradient 0, as is
// every gradient of a disabled tap. grid (kTaps, slots) x 64.
__global__ void __launch_bounds__(64) delay_taps_adjoint(const double* params, const float* taps, const float2* dh,
                                                         long span, double* grad) {
  __shared__ double wd[kFir];
  const int tapi = blockIdx.x, slot = blockIdx.y, t = threadIdx.x;
  const float* rec = taps + (static_cast<long>(slot) * kTaps + tapi) * kTapRec;
  const int d = __float_as_int(rec[0]);
  const double* row = params + static_cast<long>(slot) * kTaps * kTapStride + tapi * kTapStride;
  double* g = grad + static_cast<long>(slot) * kTaps * kTapStride + tapi * kTapStride;
  if (d < 0) {
    if (t < kTapStride) g[t] = 0.0;
    return;
  }
  const int c = tapi / 20;
  if (t < kFir) {
    const long idx = static_cast<long>(d) - kFirHalf + t;
    double v = 0.0;
    if (idx >= 0 && idx < span) {
      const float2 q = __ldg(dh + static_cast<long>(slot) * span + idx);
      v = c == 0 ? q.x : q.y;
    }
    double s, co;
    sincospi(2.0 * t / (kFir - 1), &s, &co);
    wd[t] = v * (0.5 - 0.5 * co);
  }
  __syncthreads();
  if (t < 20) {
    double acc = 0.0;
    for (int j = 0; j < kFir; ++j) {
      double s, co;
      sincospi(2.0 * t * (j - kFirHalf) / kFir, &s, &co);
      acc = fma(wd[j], co, acc);
    }
    g[2 + t] = (t == 0 ? 1.0 : 2.0) / kFir * exp(row[2 + t]) * acc;
  } else if (t < 22) {
    g[t - 20] = 0.0;
  }
}

// ---- noise STFT (ProcessorSet construction) ---------------------------------------------------
// grid (frames): one frame per CTA, fp64 direct DFT of the periodic-Hann windowed frame.
__global__ void __launch_bounds__(256) noise_stft(const double* noise, long length, float2* out) {
  __shared__ double xw[384];
  __shared__ double cs[384], sn[384];
  const int m = blockIdx.x;
  for (int i = threadIdx.x; i < 384; i += blockDim.x) {
    const long idx = static_cast<long>(m) * 192 + i;
    double s, c;
    sincospi(2.0 * i / 384.0, &s, &c);
    xw[i] = idx < length ? noise[idx] * (0.5 - 0.5 * c) : 0.0;
    cs[i] = c;
    sn[i] = s;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < kRevBins; k += blockDim.x) {
    double re = 0.0, im = 0.0;
    int idx = 0;
    for (int i = 0; i < 384; ++i) {
      re = fma(xw[i], cs[idx], re);
      im = fma(-xw[i], sn[idx], im);
      idx += k;
      if (idx >= 384) idx -= 384;
    }
    out[static_cast<long>(m) * kRevBins + k] = make_float2(static_cast<float>(re), static_cast<float>(im));
  }
}

// (mid, side) noise STFT interleaved for reverb_ir's one-load-per-(frame, bin) fill.
__global__ void pack_mid_side(const float2* mid, const float2* side, long n, float4* out) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x) {
    const float2 a = mid[i], b = side[i];
    out[i] = make_float4(a.x, a.y, b.x, b.y);
  }
}

__global__ void f64_to_f32(const double* in, float* out, long n) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x) {
    out[i] = static_cast<float>(in[i]);
  }
}

__global__ void f32_to_f64(const float* in, double* out, long n) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x) {
    out[i] = static_cast<double>(in[i]);
  }
}

unsigned grid_for(long n) {
  long b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 148L * 16) b = 148L * 16;
  return static_cast<unsigned>(b);
}

}  // namespace

// Bytes per spectrum element of the current transform precision (fft_fp64()).
std::size_t spec_elem_bytes() { return fft_fp64() ? sizeof(double2) : sizeof(float2); }

static int g_conv_fuse = -1;  // -1 auto, 0 never, 1 always (mg_set_conv_fuse; tests)
void set_conv_fuse(int mode) { g_conv_fuse = mode; }

bool conv_fuse_kernel_rows(const ConvGeom& g, int slots) {
  if (g_conv_fuse >= 0) return g_conv_fuse == 1;
  // Kernel spectra that cannot stay in L2 (> 64 MiB over the step) are not worth a separate
  // rows pass: the signal's row kernel transforms the kernel rows itself.
  return spec_elem_bytes() * static_cast<std::size_t>(slots) * static_cast<std::size_t>(g.n) > (64u << 20);
}

static int g_conv_log = 0;  // 0 automatic (mg_set_conv_log; tests)
void set_conv_log(int log_n) { g_conv_log = log_n; }

// Transform size: the single next_pow2(L + taps - 1) transform of the reference when it is the
// cheapest, else the segment size 2^a (>= taps) minimising nseg * N * (log2 N + 6): FFT flops
// plus the per-point memory passes. E.g. taps 88,200: L = 2^17 -> one 2^18 transform (as the
// reference); L = 441,000 (10 s) -> three 2^18 segments instead of one 2^20 transform.
ConvGeom conv_geom(long length, long taps) {
  if (taps < 1) taps = 1;
  const long len = length > 0 ? length : 1;
  int single = kConvMinLog;
  while (single < 62 && (1L << single) < len + taps - 1) ++single;
  const int top = g_conv_log > 0 ? kConvMaxLog : (single < kConvMaxLog ? single : kConvMaxLog);
  int best = -1;
  double best_cost = 0.0;
  for (int a = kConvMinLog; a <= top; ++a) {
    const long n = 1L << a;
    if (n < taps) continue;
    const long seg = n - taps + 1;
    const double cost = static_cast<double>((len + seg - 1) / seg) * static_cast<double>(n) * (a + 6);
    if (g_conv_log > 0 ? a == g_conv_log : (best < 0 || cost < best_cost)) {
      best = a;
      best_cost = cost;
    }
  }
  if (best < 0) {
    throw std::invalid_argument(g_conv_log > 0 ? "fft convolution: forced transform size out of range"
                                               : "fft convolution: kernel longer than 2^22 taps");
  }
  ConvGeom g;
  g.log_n = best;
  g.log_n1 = best / 2;
  g.log_n2 = best - best / 2;
  g.n = 1L << best;
  g.pre = taps - 1;
  g.seg = g.n - taps + 1;
  g.nseg = static_cast<int>((len + g.seg - 1) / g.seg);
  return g;
}

void conv_geometry(long length, long taps, long* out) {
  const ConvGeom g = conv_geom(length, taps);
  out[0] = g.log_n;
  out[1] = g.log_n1;
  out[2] = g.log_n2;
  out[3] = g.nseg;
  out[4] = g.seg;
}

std::size_t conv_prologue_bytes(const ConvGeom& g, int slots, long taps) {
  return ir_bytes(slots, taps) + align256(spec_elem_bytes() * static_cast<std::size_t>(slots) * g.n);
}

std::size_t conv_main_bytes(const ConvGeom& g, int slots, int batch) {
  return align256(spec_elem_bytes() * static_cast<std::size_t>(slots) * batch * g.nseg * g.n);
}


void launch_reverb_ir(const double* params, int slots, const ReverbConst& rc, float2* ir, long ir_stride,
                      cudaStream_t s) {
  if (slots == 0) return;
  const dim3 grid(static_cast<unsigned>((rc.frames + kRevFwdFpc - 1) / kRevFwdFpc), static_cast<unsigned>(slots));
  note_prologue_kernel(reinterpret_cast<const void*>(reverb_ir));
  constexpr int smem = (kRevFwdFpc + 1) * kRevFS * 8;
  static const bool done = [] {
    cudaFuncSetAttribute(reverb_ir, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)done;
  reverb_ir<<<grid, kRevFwdThreads, smem, s>>>(params, rc, ir, ir_stride);
}

void launch_delay_ir(const double* params, int slots, const DelayConst& dc, float2* ir, long ir_stride,
                     cudaStream_t s) {
  if (slots == 0) return;
  // Tap records live right after the kernels' IR rows ([slots][ir_stride] float2).
  auto* taps = reinterpret_cast<float*>(ir + static_cast<long>(slots) * ir_stride);
  note_prologue_kernel(reinterpret_cast<const void*>(delay_taps));
  note_prologue_kernel(reinterpret_cast<const void*>(delay_dense));
  delay_taps<<<dim3(kTaps, slots), 64, 0, s>>>(params, dc, taps);
  const dim3 grid(static_cast<unsigned>((dc.span + 255) / 256), 2, static_cast<unsigned>(slots));
  delay_dense<<<grid, 256, 0, s>>>(taps, dc, ir, ir_stride);
}

namespace {
template <typename CT>
void conv_prologue(bool reverb, const StepArgs& a, const ReverbConst& rc, const DelayConst& dc, void* ws, cudaStream_t s) {
  const long taps = reverb ? rc.length : dc.span;
  const ConvGeom g = conv_geom(a.length, taps);
  auto* ir = static_cast<float2*>(ws);
  auto* P = reinterpret_cast<CT*>(static_cast<char*>(ws) + ir_bytes(a.slots, taps));
  if (reverb) {
    launch_reverb_ir(a.params, a.slots, rc, ir, taps, s);
    kernel_spectrum<CT>(ColSrc::Kernel, a, g, ir, taps, 0, P, s);
  } else {
    // Tap records only; the column pass synthesises the dense kernel on the fly.
    auto* rec = reinterpret_cast<float*>(ir + static_cast<long>(a.slots) * taps);
    note_prologue_kernel(reinterpret_cast<const void*>(delay_taps));
    delay_taps<<<dim3(kTaps, a.slots), 64, 0, s>>>(a.params, dc, rec);
    kernel_spectrum<CT>(ColSrc::DelayTaps, a, g, reinterpret_cast<const float2*>(rec), taps, dc.window, P, s);
  }
}

template <typename CT>
void conv_main(const StepArgs& a, long taps, const void* prologue_ws, void* ws, cudaStream_t s, cudaEvent_t kernel_ready) {
  const ConvGeom g = conv_geom(a.length, taps);
  const auto* P = reinterpret_cast<const CT*>(static_cast<const char*>(prologue_ws) + ir_bytes(a.slots, taps));
  auto* X = static_cast<CT*>(ws);
  const int per_slot = a.batch * g.nseg;
  const int items = a.slots * per_slot;
  MGB_DISPATCH_LN(g.log_n1, cols_fwd_t, CT, ColSrc::Signal, a, nullptr, 0, g, items, X, 0, false, s);
  // The signal's column pass needs no kernel spectrum: join the prologue only here.
  if (kernel_ready) cudaStreamWaitEvent(s, kernel_ready, 0);
  if (conv_fuse_kernel_rows(g, a.slots)) {
    MGB_DISPATCH_LN(g.log_n2, rows_conv_fk_t, CT, g, items, per_slot, X, P, tw_table<CT>(a), s);
  } else {
    MGB_DISPATCH_LN(g.log_n2, rows_conv_t, CT, g, items, per_slot, X, P, tw_table<CT>(a), s);
  }
  MGB_DISPATCH_LN(g.log_n1, cols_inv_t, CT, a, g, X, false, s);
}

// Adjacent long-convolution steps A, B whose slots read the same source rows (a console
// track's gain feeds both its delay and its reverb send): B's slots listed in `share` reuse A's
// signal spectrum instead of transforming the same row again. A's column pass, B's column pass
// over its own slots only, B's rows (reading A's spectra where shared, writing its own buffer),
// then A's rows in place (after B has read them), then both inverse column passes.
template <typename CT>
void conv_shared(const StepArgs& a, const StepArgs& b, long taps, const void* pws_a, const void* pws_b, void* ws_a,
                 void* ws_b, const ConvShare& sh, cudaStream_t s, cudaEvent_t ready_a, cudaEvent_t ready_b) {
  const ConvGeom g = conv_geom(a.length, taps);
  const auto* Pa = reinterpret_cast<const CT*>(static_cast<const char*>(pws_a) + ir_bytes(a.slots, taps));
  const auto* Pb = reinterpret_cast<const CT*>(static_cast<const char*>(pws_b) + ir_bytes(b.slots, taps));
  auto* Xa = static_cast<CT*>(ws_a);
  auto* Xb = static_cast<CT*>(ws_b);
  const int per_slot = a.batch * g.nseg;
  MGB_DISPATCH_LN(g.log_n1, cols_fwd_t, CT, ColSrc::Signal, a, nullptr, 0, g, a.slots * per_slot, Xa, 0, false, s);
  if (sh.n_own_b > 0) {
    MGB_DISPATCH_LN(g.log_n1, cols_fwd_t, CT, ColSrc::Signal, b, nullptr, 0, g, sh.n_own_b * per_slot, Xb, 0, false, s,
                    sh.own_b);
  }
  if (ready_a) cudaStreamWaitEvent(s, ready_a, 0);
  if (ready_b) cudaStreamWaitEvent(s, ready_b, 0);
  MGB_DISPATCH_LN(g.log_n2, rows_conv_pair_t, CT, g, sh.n_pairs * per_slot, per_slot, Xa, Xb, Pa, Pb, sh.pair_a,
                  sh.pair_b, tw_table<CT>(a), s);
  if (sh.n_own_a > 0) {
    MGB_DISPATCH_LN(g.log_n2, rows_conv_fk_t, CT, g, sh.n_own_a * per_slot, per_slot, Xa, Pa, tw_table<CT>(a), s,
                    sh.own_a);
  }
  if (sh.n_own_b > 0) {
    MGB_DISPATCH_LN(g.log_n2, rows_conv_fk_t, CT, g, sh.n_own_b * per_slot, per_slot, Xb, Pb, tw_table<CT>(b), s,
                    sh.own_b);
  }
  MGB_DISPATCH_LN(g.log_n1, cols_inv_t, CT, a, g, Xa, false, s);
  MGB_DISPATCH_LN(g.log_n1, cols_inv_t, CT, b, g, Xb, false, s);
}

template <int LN2, typename CT>
void rows_bwd_t(const ConvGeom& g, int slots, int per_slot, CT* DY, CT* X, const CT* P, bool kfft, const CT* tw,
                cudaStream_t s) {
  constexpr int smem = 8 * padded(1 << LN2) * static_cast<int>(sizeof(CT));
  static const bool done = [] {
    cudaFuncSetAttribute(rows_bwd<LN2, true, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(rows_bwd<LN2, false, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)done;
  for_item_chunks(slots, [&](int s0, int n) {
    const dim3 grid(static_cast<unsigned>((1L << g.log_n1) / 2 + 1), static_cast<unsigned>(n));
    if (kfft) rows_bwd<LN2, true, CT><<<grid, row_threads<LN2, 4>(), smem, s>>>(g.log_n, per_slot, DY, X, P, tw, s0);
    else rows_bwd<LN2, false, CT><<<grid, row_threads<LN2, 4>(), smem, s>>>(g.log_n, per_slot, DY, X, P, tw, s0);
  });
}

template <int LN1, typename CT>
void cols_inv_buf_t(const ConvGeom& g, int slots, int per_slot, const CT* X, float2* out, long taps, const CT* tw,
                    cudaStream_t s) {
  constexpr int C = ColCfg<CT>::kElems / (1 << LN1);
  constexpr int smem = ColCfg<CT>::kSmem(1 << LN1);
  static const bool done = [] {
    cudaFuncSetAttribute(cols_inv_buf<LN1, CT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return true;
  }();
  (void)done;
  for_item_chunks(slots, [&](int s0, int n) {
    const dim3 grid(static_cast<unsigned>((1L << g.log_n2) / C), static_cast<unsigned>(n));
    cols_inv_buf<LN1, CT><<<grid, ColCfg<CT>::kThreads, smem, s>>>(g.log_n, per_slot, X, out, taps, tw, s0);
  });
}

template <typename CT>
void conv_backward(bool reverb, const StepArgs& fw, const StepArgs& bw, const ReverbConst& rc, const DelayConst& dc,
                   const void* prologue_ws, void* ws, double* grad, cudaStream_t s) {
  const long taps = reverb ? rc.length : dc.span;
  const ConvGeom g = conv_geom(fw.length, taps);
  const auto* P = reinterpret_cast<const CT*>(static_cast<const char*>(prologue_ws) + ir_bytes(fw.slots, taps));
  // A large step's forward left the kernel spectrum at its column stage (rows_bwd transforms it).
  const bool kfft = conv_fuse_kernel_rows(g, fw.slots);
  const int per_slot = fw.batch * g.nseg;
  const int items = fw.slots * per_slot;
  const std::size_t spec = align256(sizeof(CT) * static_cast<std::size_t>(items) * g.n);
  auto* DY = static_cast<CT*>(ws);
  auto* X = reinterpret_cast<CT*>(static_cast<char*>(ws) + spec);
  auto* dh = reinterpret_cast<float2*>(static_cast<char*>(ws) + 2 * spec);
  auto* part = reinterpret_cast<double*>(static_cast<char*>(ws) + 2 * spec +
                                         align256(sizeof(float2) * static_cast<std::size_t>(fw.slots) * taps));
  const CT* tw = tw_table<CT>(fw);
  // dY masked to each segment's own outputs (kernel gradient), x laid out as in the forward.
  MGB_DISPATCH_LN(g.log_n1, cols_fwd_t, CT, ColSrc::Signal, bw, nullptr, 0, g, items, DY, 0, true, s);
  MGB_DISPATCH_LN(g.log_n1, cols_fwd_t, CT, ColSrc::Signal, fw, nullptr, 0, g, items, X, 0, false, s);
  MGB_DISPATCH_LN(g.log_n2, rows_bwd_t, CT, g, fw.slots, per_slot, DY, X, P, kfft, tw, s);
  if (g.nseg == 1) {
    MGB_DISPATCH_LN(g.log_n1, cols_inv_t, CT, bw, g, DY, false, s);
  } else {
    // Each segment's correlation with the kernel covers [base_j, (j+1)*seg): overlap-add.
    MGB_DISPATCH_LN(g.log_n1, cols_inv_t, CT, bw, g, DY, true, s);
    for_item_chunks(fw.slots * fw.batch, [&](int i0, int n) {
      const dim3 grid(static_cast<unsigned>((fw.length + 255) / 256), static_cast<unsigned>(n));
      conv_ola<CT><<<grid, 256, 0, s>>>(bw, seg_args(g, i0), g.n, DY);
    });
  }
  MGB_DISPATCH_LN(g.log_n1, cols_inv_buf_t, CT, g, fw.slots, per_slot, X, dh, taps, tw, s);
  if (reverb) {
    const int blocks = (rc.frames + kRevFpc - 1) / kRevFpc;
    static const bool done = [] {
      cudaFuncSetAttribute(reverb_ir_adjoint, cudaFuncAttributeMaxDynamicSharedMemorySize, kRevFpc * kRevFS * 8);
      return true;
    }();
    (void)done;
    reverb_ir_adjoint<<<dim3(static_cast<unsigned>(blocks), static_cast<unsigned>(fw.slots)), kRevThreads,
                        kRevFpc * kRevFS * 8, s>>>(fw.params, rc, dh, part);
    reverb_grad_reduce<<<fw.slots, 128, 0, s>>>(part, blocks, grad);
  } else {
    const auto* ir = static_cast<const float2*>(prologue_ws);
    const auto* rec = reinterpret_cast<const float*>(ir + static_cast<long>(fw.slots) * taps);
    delay_taps_adjoint<<<dim3(kTaps, fw.slots), 64, 0, s>>>(fw.params, rec, dh, dc.span, grad);
  }
}
}  // namespace

void launch_conv_prologue(bool reverb, const StepArgs& a, const ReverbConst& rc, const DelayConst& dc, void* ws,
                          cudaStream_t s) {
  if (a.slots == 0) return;
  if (fft_fp64()) conv_prologue<double2>(reverb, a, rc, dc, ws, s);
  else conv_prologue<float2>(reverb, a, rc, dc, ws, s);
}

void launch_conv_shared(const StepArgs& a, const StepArgs& b, long taps, const void* pws_a, const void* pws_b,
                        void* ws_a, void* ws_b, const ConvShare& sh, cudaStream_t s, cudaEvent_t ready_a,
                        cudaEvent_t ready_b) {
  if (fft_fp64()) {
    conv_shared<double2>(a, b, taps, pws_a, pws_b, ws_a, ws_b, sh, s, ready_a, ready_b);
  } else {
    conv_shared<float2>(a, b, taps, pws_a, pws_b, ws_a, ws_b, sh, s, ready_a, ready_b);
  }
}

void launch_conv_main(const StepArgs& a, long taps, const void* prologue_ws, void* ws, cudaStream_t s,
                      cudaEvent_t kernel_ready) {
  if (a.slots == 0 || a.batch == 0 || a.length == 0) {
    if (kernel_ready) cudaStreamWaitEvent(s, kernel_ready, 0);
    return;
  }
  if (fft_fp64()) conv_main<double2>(a, taps, prologue_ws, ws, s, kernel_ready);
  else conv_main<float2>(a, taps, prologue_ws, ws, s, kernel_ready);
}

std::size_t conv_bwd_bytes(const ConvGeom& g, int slots, int batch, long taps, int rev_frames) {
  const std::size_t spec = align256(spec_elem_bytes() * static_cast<std::size_t>(slots) * batch * g.nseg * g.n);
  const std::size_t blocks = static_cast<std::size_t>((rev_frames + kRevFpc - 1) / kRevFpc);
  return 2 * spec + align256(sizeof(float2) * static_cast<std::size_t>(slots) * taps) +
         align256(sizeof(double) * static_cast<std::size_t>(slots) * blocks * 4 * kRevBins);
}

void launch_conv_backward(bool reverb, const StepArgs& fw, const StepArgs& bw, const ReverbConst& rc,
                          const DelayConst& dc, const void* prologue_ws, void* ws, double* grad, cudaStream_t s) {
  if (fw.slots == 0 || fw.batch == 0 || fw.length == 0) return;
  if (fft_fp64()) conv_backward<double2>(reverb, fw, bw, rc, dc, prologue_ws, ws, grad, s);
  else conv_backward<float2>(reverb, fw, bw, rc, dc, prologue_ws, ws, grad, s);
}

void launch_noise_stft(const double* noise, long length, int frames, float2* out, cudaStream_t s) {
  noise_stft<<<frames, 256, 0, s>>>(noise, length, out);
}

void launch_pack_mid_side(const float2* mid, const float2* side, long n, float4* out, cudaStream_t s) {
  if (n > 0) pack_mid_side<<<grid_for(n), 256, 0, s>>>(mid, side, n, out);
}

void launch_f64_to_f32(const double* in, float* out, long n, cudaStream_t s) {
  if (n > 0) f64_to_f32<<<grid_for(n), 256, 0, s>>>(in, out, n);
}

void launch_f32_to_f64(const float* in, double* out, long n, cudaStream_t s) {
  if (n > 0) f32_to_f64<<<grid_for(n), 256, 0, s>>>(in, out, n);
}

}  // namespace mgb
