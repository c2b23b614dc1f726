// Host-side launchers for the per-step kernels (one translation unit per kernel family).
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

#include "step_common.cuh"

namespace mgb {

// Gather-sum + copy / gain / imager + store (mix, out, gain, imager steps); `epi`: fused
// pointwise followers (step_common.cuh), vector path only (pointwise_epi_ok).
void launch_pointwise(PointOp op, const StepArgs& a, cudaStream_t s, const PwEpi& epi = {});
bool pointwise_epi_ok(const StepArgs& a);

// A run of consecutive small pointwise steps (each slots*batch <= kPwChainMaxRows, L % 4 == 0)
// in one launch, steps applied in order per sample group (latency-bound bus tails).
constexpr int kPwChainMax = 8;
constexpr int kPwChainMaxRows = 4;
struct PwChain {
  StepArgs step[kPwChainMax];
  PointOp op[kPwChainMax];
  int n;
};
bool pointwise_chain_ok(const StepArgs& a);
void launch_pointwise_chain(const PwChain& c, cudaStream_t s);

// EQ: FIR design (fp64 cosine sum, `dsp.cpp:106-136`) -> 8192-bin zero-phase response
// (prologue: parameters only) ; overlap-save convolution fused with gather and store (main).
constexpr int kEqFft = 8192;
constexpr int kEqHalf = 1023;
constexpr int kEqValid = kEqFft - 2 * kEqHalf;
void launch_eq_prologue(const StepArgs& a, float* taps_ws /*slots*2048*/, float* resp_ws /*slots*8192*/, cudaStream_t s);
void launch_eq_main(const StepArgs& a, const float* resp_ws, cudaStream_t s);
// Per-device EQ bases (taps: the FIR design basis 1024 x 1024; else the response basis
// 1024 x 4128; fp32), built synchronously on first use.
const float* eq_basis(int device, bool taps);

// Compressor / noisegate: chained (decoupled look-back) scan of the energy envelope.
constexpr int kDynThreads = 512;
constexpr int kDynPerThread = 8;
constexpr int kDynTile = kDynThreads * kDynPerThread;
// `sync` (dyn_sync_bytes: tile ticket + per-tile status words) must be zero on entry; with
// zero_sync the launcher clears it itself, otherwise the caller did (render_arena clears
// every step's sync words with one memset per render).
std::size_t dyn_sync_bytes(int slots, int batch, long length);
void launch_dynamics(bool gate, const StepArgs& a, int envelope_taps, double energy_floor, void* sync,
                     bool zero_sync, cudaStream_t s, const PwEpi& epi = {});
// Steps with a full wave of dense sequences run the streaming scan (one CTA per sequence, no
// look-back); set_dyn_stream(0) forces the chained scan, 1 the streaming one where legal
// (dense, L % 4 == 0), -1 automatic (tests).
bool dyn_stream_ok(const StepArgs& a, const PwEpi& epi);
void set_dyn_stream(int mode);
// A compressor / noisegate step A followed by one (B) reading exactly A's rows slot by slot,
// both streaming-eligible: one kernel scans both (A's rows are written, never read back);
// `epi` = B's epilogue followers. set_dyn_pair(0) runs them as two launches (tests).
bool dyn_pair_ok(const StepArgs& a1, const StepArgs& a2);
// The shape part of dyn_pair_ok (plans decide their launch structure with it).
bool dyn_pair_shape(int slots, int batch, long length);
void launch_dynamics_pair(bool gate1, bool gate2, const StepArgs& a1, const StepArgs& a2, int envelope_taps,
                          double energy_floor, cudaStream_t s, const PwEpi& epi);
void set_dyn_pair(int mode);

// Backward of a compressor / noisegate step: `bw` gathers dy over the consumers' input
// gradients (transposed CSR) and stores du into bw.dst; parameter gradients [slots][4] fp64
// into `grad`. ws: dyn_bwd_bytes.
std::size_t dyn_bwd_bytes(int slots, int batch, long length);
void launch_dynamics_backward(bool gate, const StepArgs& fw, const StepArgs& bw, int envelope_taps,
                              double energy_floor, void* ws, double* grad, cudaStream_t s);

// FFT convolution with a long causal kernel (reverb, delay): four-step FFT of size N.
// Segmented overlap-save: the signal is cut into `nseg` segments of `seg` output samples;
// segment j transforms x[base_j, base_j + N) with base_j = max(0, j*seg - pre), pre = taps - 1,
// and keeps its outputs [j*seg, (j+1)*seg). One segment (seg >= L) is the reference's single
// next_pow2(L + taps - 1) transform (`dsp.cpp:64-86`); longer signals use several segments of
// the size that minimises the work, so any length renders with N <= 2^kConvMaxLog.
struct ConvGeom {
  int log_n = 0, log_n1 = 0, log_n2 = 0;
  long n = 0;
  long seg = 0;  // output samples per segment (N - taps + 1)
  long pre = 0;  // taps - 1
  int nseg = 1;
};
constexpr int kConvMinLog = 13;
constexpr int kConvMaxLog = 22;
ConvGeom conv_geom(long length, long taps);
// Tests: force the transform size 2^log (0 = automatic); conv_geom throws when 2^log < taps.
void set_conv_log(int log_n);
// [log_n, log_n1, log_n2, nseg, seg] of conv_geom (C ABI mg_conv_geometry).
void conv_geometry(long length, long taps, long* out);
// Large steps (kernel spectra beyond L2) fuse the kernel's row stage into the signal's row
// pass instead of a separate prologue pass.
bool conv_fuse_kernel_rows(const ConvGeom& g, int slots);
void set_conv_fuse(int mode);  // -1 auto (default), 0 never, 1 always

struct ReverbConst {
  const float2* stft_mid;  // [frames][193]
  const float2* stft_side;
  const float4* stft_ms;   // [frames][193] (mid, side) interleaved
  int frames;
  long length;  // reverb_length
  const float2* consts;  // twiddle_table(): 384-point twiddles and OLA covers
};
struct DelayConst {
  long span;
  int window;
};

// Prologue (parameters only): impulse responses + their spectra into `ws`
// (conv_prologue_bytes). Main (audio): gather -> FFT -> product -> inverse -> arena, using
// the prologue's spectra and a transient buffer of conv_main_bytes.
std::size_t conv_prologue_bytes(const ConvGeom& g, int slots, long taps);
std::size_t conv_main_bytes(const ConvGeom& g, int slots, int batch);
void launch_conv_prologue(bool reverb, const StepArgs& a, const ReverbConst& rc, const DelayConst& dc, void* ws,
                          cudaStream_t s);
// kernel_ready (optional): event of the prologue, waited on after the signal's column pass.
void launch_conv_main(const StepArgs& a, long taps, const void* prologue_ws, void* ws, cudaStream_t s,
                      cudaEvent_t kernel_ready = nullptr);

// Two adjacent conv steps A, B with the same transform (conv_fuse_kernel_rows for both) whose
// slots pair up on a common single source row (a console track's delay and reverb sends):
// pairs (pair_a[p], pair_b[p]) share A's signal spectrum (each A slot in at most one pair);
// own_a / own_b list the remaining slots of each step. ws_a / ws_b: conv_main_bytes each, both
// live until the call's kernels finish.
struct ConvShare {
  const int* pair_a = nullptr;
  const int* pair_b = nullptr;
  const int* own_a = nullptr;
  const int* own_b = nullptr;
  int n_pairs = 0, n_own_a = 0, n_own_b = 0;
};
void launch_conv_shared(const StepArgs& a, const StepArgs& b, long taps, const void* pws_a, const void* pws_b,
                        void* ws_a, void* ws_b, const ConvShare& sh, cudaStream_t s, cudaEvent_t ready_a,
                        cudaEvent_t ready_b);

// Backward of a reverb / delay step: dX = correlation with the kernel (stored into bw.dst),
// kernel gradient = correlation of dY with X, then through the IR build / tap FIRs into
// `grad` ([slots][768] / [slots][880] fp64). prologue_ws: the forward's prologue region.
std::size_t conv_bwd_bytes(const ConvGeom& g, int slots, int batch, long taps, int rev_frames);
void launch_conv_backward(bool reverb, const StepArgs& fw, const StepArgs& bw, const ReverbConst& rc,
                          const DelayConst& dc, const void* prologue_ws, void* ws, double* grad, cudaStream_t s);

// Pointwise (gain / imager) parameter gradients and the EQ correlation + FIR adjoint.
std::size_t pw_grad_bytes(int slots, int batch, long length);
// dX and the parameter gradient in one pass (returns false when L % 4 != 0: use the two-pass
// launch_pointwise + launch_pointwise_param_grad).
bool launch_pointwise_backward(PointOp op, const StepArgs& fw, const StepArgs& bw, void* ws, double* grad,
                               cudaStream_t s);
void launch_pointwise_param_grad(PointOp op, const StepArgs& fw, const StepArgs& bw, void* ws, double* grad,
                                 cudaStream_t s);
std::size_t eq_grad_bytes(int slots, int batch, long length);
void launch_eq_param_grad(const StepArgs& fw, const StepArgs& bw, void* ws, double* grad, cudaStream_t s);

// Optimisation helpers: MSE loss (fp64, deterministic) and its output gradient 2 (y - t) / n;
// plain gradient step with fit.cpp's legal-range projection of dynamics rows.
std::size_t mse_scratch_bytes();
void launch_mse_loss_grad(const float* y, const float* target, long n, float* grad, double* loss, void* scratch,
                          cudaStream_t s);
void launch_sgd_step(bool dynamics, double* table, const double* grad, long n, double lr, cudaStream_t s);

// Kernel-only entry points (for ProcessorSet::reverb_kernel / delay_kernel).
void launch_reverb_ir(const double* params, int slots, const ReverbConst& rc, float2* ir, long ir_stride,
                      cudaStream_t s);
void launch_delay_ir(const double* params, int slots, const DelayConst& dc, float2* ir, long ir_stride,
                     cudaStream_t s);

// Noise STFT for the reverb (ProcessorSet construction, `processors.cpp:151-160`).
void launch_noise_stft(const double* noise, long length, int frames, float2* out, cudaStream_t s);
void launch_pack_mid_side(const float2* mid, const float2* side, long n, float4* out, cudaStream_t s);

// Per-device constant tables, built on first use with a synchronous upload (call it before
// any stream capture; ProcessorSet does): kTwN forward twiddles (float2), followed by
// kCosN doubles cos(2 pi m / 2047) for the EQ FIR design (cos_table()).
constexpr int kCosN = 2047;
constexpr int kTw384Off = 8192 + kCosN;      // float2 offset of the 384-point twiddles
constexpr int kCoverOff = kTw384Off + 384;   // float2 offset of the reverb inverse covers
constexpr int kConstFloat2s = kCoverOff + 192;
const float2* twiddle_table(int device);
// kTwN forward twiddles exp(-2 pi i k / kTwN) in fp64 (the fp64 transforms' table).
const double2* twiddle_table64(int device);
// Arithmetic precision of the FFT-based steps (EQ, reverb, delay): false fp32, true fp64 (the
// arena stays fp32 either way). Process-wide; see DESIGN.md (precision).
bool fft_fp64();
void set_fft_fp64(bool on);
__host__ __device__ inline const double* cos_table(const float2* tw) { return reinterpret_cast<const double*>(tw + 8192); }
__host__ __device__ inline const float2* tw384_table(const float2* tw) { return tw + kTw384Off; }
// .x = 1/(384 w(o)) for the first hop, .y = 1/(384 (w(o) + w(o+192))) afterwards
__host__ __device__ inline const float2* cover_table(const float2* tw) { return tw + kCoverOff; }

// Kernels that only run in parameter-only prologues (RenderGraph gives them low priority).
void note_prologue_kernel(const void* fn);
bool is_prologue_kernel(const void* fn);

// Parameter reorder on the device (`schedule.cpp:454-471`, RenderData::reorder_params):
// out[t][r][:] = in[t][src_rows[t][r]][:] for every type with rows (BatchRenderer uploads the
// ORIGINAL-order tables and the plan's param_source_rows, and gathers here).
struct ParamGather {
  const double* in[10];
  const int* src_rows[10];
  double* out[10];
  int rows[10];
  int width[10];
};
void launch_param_gather(const ParamGather& g, cudaStream_t s);

// Arena conversion helpers for the host-buffer API.
void launch_f64_to_f32(const double* in, float* out, long n, cudaStream_t s);
void launch_f32_to_f64(const float* in, double* out, long n, cudaStream_t s);

}  // namespace mgb
