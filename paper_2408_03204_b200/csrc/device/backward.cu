// Reverse-mode pass over a rendered arena: parameter gradients (BASELINE configs 4/5, the
// optimisation setting).
//
// The reference has no autodiff (`SPEC.md:14`): its only gradient is the central
// difference of `fit.cpp:70-82`, which is what the tests compare these kernels with. The
// pass runs the steps in reverse. For a node v with aggregated input X_v (Eq. 1b) and output
// Y_v, the adjoint arena holds dL/dX_v in v's row; dL/dY_v is the sum of dL/dX_w over v's
// consumer edges (a transposed CSR, gathered in a fixed order, so no atomics). Per type:
//   mix/out/in  dX = dY
//   gain        dX = e^p dY (the forward kernel on the adjoint arena);  dp_c = sum dY_c Y_c
//   imager      dX = M dY (M symmetric: forward kernel);  dp = sum (dY_l - dY_r)(Y_l - Y_r)/2
//   eq          dX = h (x) dY (zero-phase h is even: forward kernel);  dh = corr(dY, X) then
//               through zero_phase_fir (`dsp.cpp:106-136`): a cosine sum in fp64
//   comp/gate   reverse affine scan (dynamics.cu)
//   reverb/delay  dX = corr(dY, h) (conjugate kernel spectrum), dh = corr(dY, X), then
//               through the ISTFT (`dsp.cpp:165-190`) / the tap FIRs (fftconv.cu)
// This file: the pointwise parameter reductions and the EQ correlation + FIR adjoint.
#include <algorithm>

#include "fft_smem.cuh"
#include "launch.hpp"

namespace mgb {

namespace {

constexpr int kPgThreads = 256;
constexpr int kPgPer = 8;  // samples per thread

// Partial sums of the pointwise parameter gradients. grid (blocks, slots*B).
// out[(sb * gridDim.x + blk) * 2 + j] (fp64).
template <PointOp OP>
__global__ void __launch_bounds__(kPgThreads) pw_param_grad(StepArgs fw, StepArgs bw, double* out) {
  __shared__ double red[kPgThreads / 32][2];
  const int sb = blockIdx.y;
  const int slot = sb / fw.batch, b = sb - slot * fw.batch;
  const int e0 = __ldg(bw.row_ptr + slot), e1 = __ldg(bw.row_ptr + slot + 1);
  const float* y = fw.dst + static_cast<long>(slot) * fw.rowstride + static_cast<long>(b) * 2 * fw.length;
  double s0 = 0.0, s1 = 0.0;
  const long n0 = (static_cast<long>(blockIdx.x) * kPgThreads + threadIdx.x) * kPgPer;
  for (int k = 0; k < kPgPer; ++k) {
    const long n = n0 + k;
    if (n >= fw.length) break;
    const float2 dy = gather2(bw, e0, e1, b, n);
    const float yl = __ldg(y + n), yr = __ldg(y + fw.length + n);
    if constexpr (OP == PointOp::Gain) {
      s0 += static_cast<double>(dy.x * yl);
      s1 += static_cast<double>(dy.y * yr);
    } else {
      s0 += 0.5 * static_cast<double>((dy.x - dy.y) * (yl - yr));
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, off);
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[warp][0] = s0;
    red[warp][1] = s1;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0.0;
    for (int w = 0; w < kPgThreads / 32; ++w) t += red[w][threadIdx.x];
    out[(static_cast<long>(sb) * gridDim.x + blockIdx.x) * 2 + threadIdx.x] = t;
  }
}

// Gain / imager backward in one pass (L % 4 == 0): gather dY over the consumer CSR (float4),
// dX = e^p dY (gain) or M dY (imager, M symmetric) stored into bw.dst, and the per-block
// partial sums of the parameter gradient (dY . Y). grid (ceil(L/4 / kPbThreads), slots*B).
constexpr int kPbThreads = 128;
template <PointOp OP>
__global__ void __launch_bounds__(kPbThreads) pointwise_bwd(StepArgs fw, StepArgs bw, double* out) {
  __shared__ double red[kPbThreads / 32][2];
  const int sb = blockIdx.y;
  const int slot = sb / fw.batch, b = sb - slot * fw.batch;
  const long n4 = fw.length >> 2;
  const long i = blockIdx.x * static_cast<long>(kPbThreads) + threadIdx.x;
  double s0 = 0.0, s1 = 0.0;
  if (i < n4) {
    const int e0 = __ldg(bw.row_ptr + slot), e1 = __ldg(bw.row_ptr + slot + 1);
    const long boff = static_cast<long>(b) * 2 * fw.length;
    float4 l = make_float4(0.f, 0.f, 0.f, 0.f), r = l;
    for (int e = e0; e < e1; ++e) {
      const float4* p = reinterpret_cast<const float4*>(bw.src + static_cast<long>(__ldg(bw.col + e)) * bw.rowstride + boff);
      l = f4add(l, __ldg(p + i));
      r = f4add(r, __ldg(p + n4 + i));
    }
    const float4* y = reinterpret_cast<const float4*>(fw.dst + static_cast<long>(slot) * fw.rowstride + boff);
    const float4 yl = __ldg(y + i), yr = __ldg(y + n4 + i);
    float4 ol, orr;
    if constexpr (OP == PointOp::Gain) {
      const float g0 = static_cast<float>(exp(fw.params[2 * slot])), g1 = static_cast<float>(exp(fw.params[2 * slot + 1]));
      s0 = static_cast<double>(l.x * yl.x + l.y * yl.y + l.z * yl.z + l.w * yl.w);
      s1 = static_cast<double>(r.x * yr.x + r.y * yr.y + r.z * yr.z + r.w * yr.w);
      ol = make_float4(g0 * l.x, g0 * l.y, g0 * l.z, g0 * l.w);
      orr = make_float4(g1 * r.x, g1 * r.y, g1 * r.z, g1 * r.w);
    } else {
      const float g = static_cast<float>(exp(fw.params[slot]));
      s0 = 0.5 * static_cast<double>((l.x - r.x) * (yl.x - yr.x) + (l.y - r.y) * (yl.y - yr.y) +
                                     (l.z - r.z) * (yl.z - yr.z) + (l.w - r.w) * (yl.w - yr.w));
      auto mix = [g](float a, float c, float& u, float& w) {
        const float m = a + c, sd = g * (a - c);
        u = 0.5f * (m + sd);
        w = 0.5f * (m - sd);
      };
      mix(l.x, r.x, ol.x, orr.x);
      mix(l.y, r.y, ol.y, orr.y);
      mix(l.z, r.z, ol.z, orr.z);
      mix(l.w, r.w, ol.w, orr.w);
    }
    float4* d = reinterpret_cast<float4*>(bw.dst + static_cast<long>(slot) * bw.rowstride + boff);
    d[i] = ol;
    d[n4 + i] = orr;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, off);
    s1 += __shfl_xor_sync(0xffffffffu, s1, off);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    red[warp][0] = s0;
    red[warp][1] = s1;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double t = 0.0;
    for (int w = 0; w < kPbThreads / 32; ++w) t += red[w][threadIdx.x];
    out[(static_cast<long>(sb) * gridDim.x + blockIdx.x) * 2 + threadIdx.x] = t;
  }
}

// grid (slots) x 32: grad[slot][j] = sum over rows_per_slot partial rows; for narrow tables
// (width <= 2) one warp per column, lanes strided over the rows, xor-tree in fixed order.
__global__ void reduce_partials(const double* partial, int rows_per_slot, int stride, int width, double* grad,
                                int grad_width) {
  const int slot = blockIdx.x;
  const double* p = partial + static_cast<long>(slot) * rows_per_slot * stride;
  for (int j = 0; j < width; ++j) {
    double t = 0.0;
    for (int r = threadIdx.x; r < rows_per_slot; r += 32) t += p[static_cast<long>(r) * stride + j];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (threadIdx.x == 0) grad[static_cast<long>(slot) * grad_width + j] = t;
  }
}

// ---- EQ ---------------------------------------------------------------------------------------
constexpr int kCorrLog = 13;
constexpr int kCorrFft = 1 << kCorrLog;
constexpr int kCorrOut = 6144;  // outputs per block (as the forward's 8192 window)
constexpr int kCorrThreads = 512;
constexpr int kCorrFS = padded(kCorrFft);

// dh[j] over `per` consecutive output blocks: with W = x[out0 - 1024 + u] (u < 8192) and
// D = dy[out0 + v] (v < 6144, zero-padded), sum_v D[v] W[v + s] = IFFT(conj(D^) W^)[s]; tap
// j = 2047 - s. The product spectra of the CTA's blocks are summed (fixed order) before ONE
// inverse transform. Channels packed as re/im: the real part of the product sums both
// channels' correlations. grid (ceil(blocks / per), slots*B); out[(sb * gridDim.x + cta) * 2048 + j].
// Register-ended transforms (as eq_conv): thread j loads the 16 inputs j + r*512 of its
// radix-16 first-pass butterfly straight from memory, and the forward plan 16 x 8 x 4 x 16 ends
// with a radix-16 pass whose butterfly j holds bins j + r*512 — the same bins every block, so
// the product spectrum accumulates in registers, and they are exactly the inputs of the
// inverse's radix-16 first-pass butterfly j. One smem buffer (the old kernel staged both
// windows and the accumulator in smem: 3x the smem traffic).
__device__ __forceinline__ void corr_load(const StepArgs& a, int e0, int e1, int b, long start, int count,
                                          float2 (&v)[16]) {
  constexpr int M1 = kCorrFft / 16;
  if (e1 - e0 == 1) {  // one input row (the common case): its base address once, not per sample
    const float* p = a.src + edge_row(a, e0) * a.rowstride + static_cast<long>(b) * 2 * a.length;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int i = threadIdx.x + r * M1;
      const long n = start + i;
      v[r] = (i < count && n >= 0 && n < a.length) ? make_float2(0.f + __ldg(p + n), 0.f + __ldg(p + a.length + n))
                                                   : make_float2(0.f, 0.f);
    }
    return;
  }
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const int i = threadIdx.x + r * M1;
    const long n = start + i;
    v[r] = (i < count && n >= 0 && n < a.length) ? gather2(a, e0, e1, b, n) : make_float2(0.f, 0.f);
  }
}
// Forward transform of v (first-pass inputs) through `buf`; on return v = bins j + r*512.
__device__ __forceinline__ void corr_forward(float2 (&v)[16], float2* buf, const float2* tw) {
  constexpr int NL = kCorrFft / 16;
  const int j = threadIdx.x;
  fft_first_from_regs<-1>(v, buf, j);
  __syncthreads();
  stockham_pass<kCorrFft, 8, 16, 1, kCorrThreads, -1>(buf, kCorrFS, tw);
  stockham_pass<kCorrFft, 4, 128, 1, kCorrThreads, -1>(buf, kCorrFS, tw);
  TwPass<16, NL, -1, float2> twb;
  twb.load(tw, j);
  const float2* lb = buf + sidx(j);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = lb[r * padded(NL)];
  twb.apply(v);
  Dft<16, -1, float2>::run(v);
  __syncthreads();  // buf is free again
}

__global__ void __launch_bounds__(kCorrThreads, 1) eq_corr(StepArgs fw, StepArgs bw, int per, float* out) {
  static_assert(kCorrFft / 16 == kCorrThreads, "eq_corr: one first-pass butterfly per thread");
  extern __shared__ float2 buf[];  // [kCorrFS] transforms, then [16][512] this thread's accumulated bins
  float2* acc = buf + kCorrFS;
  const int sb = blockIdx.y;
  const int slot = sb / fw.batch, b = sb - slot * fw.batch;
  const long nblk = (fw.length + kCorrOut - 1) / kCorrOut;
  const int fe0 = __ldg(fw.row_ptr + slot), fe1 = __ldg(fw.row_ptr + slot + 1);
  const int be0 = __ldg(bw.row_ptr + slot), be1 = __ldg(bw.row_ptr + slot + 1);
#pragma unroll
  for (int r = 0; r < 16; ++r) acc[r * kCorrThreads + threadIdx.x] = make_float2(0.f, 0.f);
  for (long blk = static_cast<long>(blockIdx.x) * per; blk < nblk && blk < static_cast<long>(blockIdx.x + 1) * per; ++blk) {
    const long out0 = blk * kCorrOut;
    float2 w[16], d[16];
    corr_load(fw, fe0, fe1, b, out0 - (kEqHalf + 1), kCorrFft, w);
    corr_forward(w, buf, fw.tw);
    corr_load(bw, be0, be1, b, out0, kCorrOut, d);
    corr_forward(d, buf, fw.tw);
#pragma unroll
    for (int r = 0; r < 16; ++r) {  // this thread's own entries: no barrier
      float2& a = acc[r * kCorrThreads + threadIdx.x];
      a = cadd(a, cmul(cconj(d[r]), w[r]));
    }
  }
  {
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = acc[r * kCorrThreads + threadIdx.x];
    fft_first_from_regs<+1>(v, buf, threadIdx.x);
  }
  __syncthreads();
  fft_middle<kCorrLog, 1, kCorrThreads, +1>(buf, kCorrFS, fw.tw);
  // Last inverse pass into registers: outputs k = jj + r*NS; tap 2047 - k for k in [1, 2047].
  constexpr int NS = Pow2Plan<kCorrLog>::kLastNs, R = Pow2Plan<kCorrLog>::kLastR;
  float* o = out + (static_cast<long>(sb) * gridDim.x + blockIdx.x) * 2048;
#pragma unroll
  for (int p = 0; p < NS / kCorrThreads; ++p) {
    const int jj = threadIdx.x + p * kCorrThreads;
    float2 y[R];
    fft_last_to_regs<kCorrLog, +1>(buf, jj, fw.tw, y);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int k = jj + r * NS;
      if (k >= 1 && k <= 2 * kEqHalf + 1) o[2 * kEqHalf + 1 - k] = y[r].x * (1.f / kCorrFft);
    }
  }
}

// Per slot: dtaps = sum of the block partials (fixed order), then the zero_phase_fir adjoint
//   d lm[q] = (m_q / N) e^{lm[q]} sum_t dtaps[t] hann[t] cos(2 pi q (t - c) / N),
// m_0 = 1, m_q = 2 (N = 2047, c = 1023). grid (slots) x 1024, fp64.
__global__ void __launch_bounds__(1024) eq_grad(const float* partial, int rows_per_slot, const double* params,
                                                const double* __restrict__ cos_tab, double* grad) {
  constexpr int N = 2 * kEqHalf + 1, C = kEqHalf;
  __shared__ double sym[kEqHalf + 1];  // S_j = (dh w)[c + j] + (dh w)[c - j], S_0 = (dh w)[c]
  __shared__ double cs[N];             // cos(2 pi i / N): the loop below gathers it at q t mod N
  const int slot = blockIdx.x;
  for (int i = threadIdx.x; i < N; i += blockDim.x) cs[i] = __ldg(cos_tab + i);
  const float* p = partial + static_cast<long>(slot) * rows_per_slot * 2048;
  const int j = threadIdx.x;  // 0..1023
  double hi = 0.0, lo = 0.0;
  for (int r = 0; r < rows_per_slot; ++r) {
    hi += p[static_cast<long>(r) * 2048 + C + j];
    if (j > 0) lo += p[static_cast<long>(r) * 2048 + C - j];
  }
  double s, c;
  sincospi(2.0 * (C + j) / (N - 1), &s, &c);
  const double w = 0.5 - 0.5 * c;  // symmetric Hann, w(c + j) == w(c - j)
  sym[j] = w * (hi + lo);
  __syncthreads();
  const int q = threadIdx.x;
  double acc = 0.0;
  int idx = 0;
  for (int t = 0; t <= kEqHalf; ++t) {
    acc = fma(sym[t], cs[idx], acc);  // (from L1 each warp's 32 scattered entries were ~32 wavefronts)
    idx += q;
    if (idx >= N) idx -= N;
  }
  const double lm = params[static_cast<long>(slot) * (kEqHalf + 1) + q];
  grad[static_cast<long>(slot) * (kEqHalf + 1) + q] = (q == 0 ? 1.0 : 2.0) / N * exp(lm) * acc;
}

// ---- optimisation helpers (fit.cpp:25-96 with analytic gradients) -----------------------------
constexpr int kMseBlocks = 592;  // 4 x 148 SMs, fixed (deterministic reduction order)
constexpr int kMseThreads = 256;

// grad = scale (y - t); per-block partial sums of (y - t)^2 in fp64.
__global__ void __launch_bounds__(kMseThreads) mse_grad(const float* y, const float* t, long n, float scale, float* g,
                                                       double* partial) {
  __shared__ double red[kMseThreads / 32];
  double acc = 0.0;
  for (long i = static_cast<long>(blockIdx.x) * kMseThreads + threadIdx.x; i < n; i += static_cast<long>(kMseBlocks) * kMseThreads) {
    const float d = y[i] - t[i];
    g[i] = scale * d;
    acc += static_cast<double>(d) * d;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kMseThreads / 32; ++w) s += red[w];
    partial[blockIdx.x] = s;
  }
}

__global__ void mse_finish(const double* partial, double inv_count, double* loss) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < kMseBlocks; i += 32) s += partial[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  (void)red;
  if (threadIdx.x == 0) *loss = s * inv_count;
}

// p -= lr g, then the legal-range projection of fit.cpp:13-21 for dynamics rows.
__global__ void sgd_update(double* p, const double* g, long n, double lr, int dyn) {
  for (long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x) {
    double v = p[i] - lr * g[i];
    if (dyn) {
      const int c = static_cast<int>(i % 4);
      if (c == 0) v = fmin(fmax(v, 1e-4), 1.0 - 1e-4);
      else if (c == 2) v = fmax(v, 1e-3);
      else if (c == 3) v = fmax(v, 1.0);
    }
    p[i] = v;
  }
}

}  // namespace

std::size_t mse_scratch_bytes() { return sizeof(double) * kMseBlocks; }

void launch_mse_loss_grad(const float* y, const float* target, long n, float* grad, double* loss, void* scratch,
                          cudaStream_t s) {
  auto* part = static_cast<double*>(scratch);
  const float scale = n > 0 ? 2.f / static_cast<float>(n) : 0.f;
  mse_grad<<<kMseBlocks, kMseThreads, 0, s>>>(y, target, n, scale, grad, part);
  mse_finish<<<1, 32, 0, s>>>(part, n > 0 ? 1.0 / static_cast<double>(n) : 0.0, loss);
}

void launch_sgd_step(bool dynamics, double* table, const double* grad, long n, double lr, cudaStream_t s) {
  if (n <= 0) return;
  const long blocks = std::min<long>((n + 255) / 256, 1184);
  sgd_update<<<static_cast<unsigned>(blocks), 256, 0, s>>>(table, grad, n, lr, dynamics ? 1 : 0);
}

std::size_t pw_grad_bytes(int slots, int batch, long length) {
  const long blocks = std::max((length + kPgThreads * kPgPer - 1) / (kPgThreads * kPgPer),
                               (length / 4 + kPbThreads - 1) / kPbThreads);
  return sizeof(double) * 2 * static_cast<std::size_t>(slots) * batch * blocks;
}

bool launch_pointwise_backward(PointOp op, const StepArgs& fw, const StepArgs& bw, void* ws, double* grad,
                               cudaStream_t s) {
  if (fw.length % 4 != 0 || op == PointOp::Copy || fw.slots == 0) return false;
  const long blocks = (fw.length / 4 + kPbThreads - 1) / kPbThreads;
  const dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(fw.slots * fw.batch));
  auto* part = static_cast<double*>(ws);
  if (op == PointOp::Gain) pointwise_bwd<PointOp::Gain><<<grid, kPbThreads, 0, s>>>(fw, bw, part);
  else pointwise_bwd<PointOp::Imager><<<grid, kPbThreads, 0, s>>>(fw, bw, part);
  const int width = op == PointOp::Gain ? 2 : 1;
  reduce_partials<<<fw.slots, 32, 0, s>>>(part, static_cast<int>(blocks) * fw.batch, 2, width, grad, width);
  return true;
}

void launch_pointwise_param_grad(PointOp op, const StepArgs& fw, const StepArgs& bw, void* ws, double* grad,
                                 cudaStream_t s) {
  if (fw.slots == 0 || op == PointOp::Copy) return;
  const long blocks = (fw.length + kPgThreads * kPgPer - 1) / (kPgThreads * kPgPer);
  const dim3 grid(static_cast<unsigned>(blocks), static_cast<unsigned>(fw.slots * fw.batch));
  auto* part = static_cast<double*>(ws);
  if (op == PointOp::Gain) pw_param_grad<PointOp::Gain><<<grid, kPgThreads, 0, s>>>(fw, bw, part);
  else pw_param_grad<PointOp::Imager><<<grid, kPgThreads, 0, s>>>(fw, bw, part);
  const int width = op == PointOp::Gain ? 2 : 1;
  reduce_partials<<<fw.slots, 32, 0, s>>>(part, static_cast<int>(blocks) * fw.batch, 2, width, grad, width);
}

std::size_t eq_grad_bytes(int slots, int batch, long length) {
  const long blocks = (length + kCorrOut - 1) / kCorrOut;
  return sizeof(float) * 2048 * static_cast<std::size_t>(slots) * batch * blocks;
}

void launch_eq_param_grad(const StepArgs& fw, const StepArgs& bw, void* ws, double* grad, cudaStream_t s) {
  if (fw.slots == 0) return;
  static const bool done = [] {
    cudaFuncSetAttribute(eq_corr, cudaFuncAttributeMaxDynamicSharedMemorySize, (kCorrFS + kCorrFft) * 8);
    return true;
  }();
  (void)done;
  const long blocks = (fw.length + kCorrOut - 1) / kCorrOut;
  // Blocks per CTA: fewer inverse transforms, but >= 8 waves of CTAs (1 per SM) over the step.
  const long items = static_cast<long>(fw.slots) * fw.batch;
  long per = std::max<long>(1, blocks * items / (8L * 148));
  per = std::min(per, blocks);
  const long ctas = (blocks + per - 1) / per;
  auto* part = static_cast<float*>(ws);
  eq_corr<<<dim3(static_cast<unsigned>(ctas), static_cast<unsigned>(items)), kCorrThreads, (kCorrFS + kCorrFft) * 8, s>>>(
      fw, bw, static_cast<int>(per), part);
  eq_grad<<<fw.slots, 1024, 0, s>>>(part, static_cast<int>(ctas) * fw.batch, fw.params, cos_table(fw.tw), grad);
}

}  // namespace mgb
