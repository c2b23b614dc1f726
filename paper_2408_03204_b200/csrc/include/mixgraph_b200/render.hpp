// Batched processors and the renderer (host API over the B200 engine).
//
// Drop-in for `proj/include/mixgraph/processors.hpp:15-76`, `render.hpp:11-32` and
// `audio_buffer.hpp:7-32`: same types, signatures, argument meaning and exceptions. The
// difference is where the work runs: a ProcessorSet owns device-resident constants (the
// reverb noise STFT) on the CUDA device current at construction, and render()/process()
// execute every step as sm_100a kernels over one fp32 HBM arena; host buffers are
// double, as in the reference, and converted at the boundary. There is no CPU fallback:
// without a usable CUDA device these calls throw std::runtime_error.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <span>
#include <utility>
#include <vector>

#include "mixgraph_b200/audio_buffer.hpp"
#include "mixgraph_b200/schedule.hpp"

typedef struct CUstream_st* cudaStream_t;
typedef struct CUevent_st* cudaEvent_t;

namespace mixgraph {

struct ProcessorConfig {
  double sample_rate = 44100.0;
  std::uint32_t reverb_seed = 0;
  int envelope_taps = 32768;
  double energy_floor = 1e-7;
};

struct DeviceConstants;  // engine-internal

class ProcessorSet {
 public:
  explicit ProcessorSet(const ProcessorConfig& config = {});
  ~ProcessorSet();
  ProcessorSet(const ProcessorSet&) = delete;
  ProcessorSet& operator=(const ProcessorSet&) = delete;

  const ProcessorConfig& config() const { return config_; }
  long delay_span() const { return delay_span_; }
  int delay_window() const { return delay_window_; }
  long reverb_length() const { return reverb_length_; }
  const std::vector<double>& reverb_noise_mid() const { return noise_mid_; }
  const std::vector<double>& reverb_noise_side() const { return noise_side_; }

  // Host-buffer operator (reference signature): in/out [slots][batch][2][length] double.
  void process(NodeType type, const double* in, double* out, int slots, int batch, long length,
               const ParamMatrix* params, int param_offset) const;
  AudioBuffer process_node(NodeType type, const AudioBuffer& input, std::span<const double> params) const;

  // Device operator: in/out device fp32 [slots][batch][2][length]; params device fp64
  // [>= param_offset + slots][param_width(type)]. Asynchronous on `stream`; no validation.
  void process_device(NodeType type, const float* in, float* out, int slots, int batch, long length,
                      const double* params, int param_offset, cudaStream_t stream) const;

  std::pair<std::vector<double>, std::vector<double>> reverb_kernel(std::span<const double> params) const;
  std::vector<double> delay_kernel(std::span<const double> params, int channel) const;
  std::vector<long> delay_positions(std::span<const double> params, int channel) const;

  const DeviceConstants& device() const { return *dev_; }
  int device_id() const;  // the CUDA device the constants live on

 private:
  ProcessorConfig config_;
  long delay_span_ = 0;
  int delay_window_ = 0;
  long reverb_length_ = 0;
  std::vector<double> noise_mid_, noise_side_;
  std::unique_ptr<DeviceConstants> dev_;
};

double compressor_gain_log(double g_u, double threshold, double knee_half_width, double ratio);
double noisegate_gain_log(double g_u, double threshold, double knee_half_width, double ratio);
void check_param_row(NodeType type, std::span<const double> row);

namespace dsp {
std::vector<double> uniform_noise(long n, std::uint32_t seed);
}

struct RenderOptions {
  bool keep_intermediates = false;
};

struct RenderResult {
  std::vector<AudioBuffer> outputs;
  std::vector<AudioBuffer> intermediates;
};

RenderResult render(const RenderData& rd, const ProcessorSet& processors, const ParamStore& params,
                    const std::vector<AudioBuffer>& sources, const RenderOptions& options = {});
RenderResult render(const RenderData& rd, const ProcessorSet& processors, const std::vector<AudioBuffer>& sources,
                    const RenderOptions& options = {});

// ---- device-resident render (the B200 hot path) ---------------------------------------
//
// `step_events`, when given, holds 2 * num_steps events recorded around every step (per-step
// device timing for the benchmark's roofline breakdown).
// A DevicePlan is RenderData's step table uploaded once: per step a CSR (row_ptr over the
// step's slots, col = gathered arena rows). render_arena() runs every step on `stream`
// over an arena of rd.buffer_rows rows x [batch][2][length] fp32 whose rows
// [0, num_inputs) hold the sources; outputs land in rows [output_begin, buffer_rows).
// `param_tables[t]` is a device pointer to the REORDERED fp64 table of NodeType t
// (RenderData::reorder_params layout), or null when the plan has no step of that type.
class DevicePlan {
 public:
  explicit DevicePlan(const RenderData& rd);
  // Borrowed residency (BatchRenderer): the step table is built on the host only; the owner
  // uploads host_index() to device memory it manages and calls attach() with that address
  // and with side streams / >= num_steps + 1 events it owns. No allocation, no sync.
  struct Deferred {};
  DevicePlan(const RenderData& rd, Deferred);
  void attach(const int* device_index, const std::array<cudaStream_t, 4>& aux, const cudaEvent_t* events);
  const std::vector<int>& host_index() const { return host_; }
  ~DevicePlan();
  DevicePlan(const DevicePlan&) = delete;
  DevicePlan& operator=(const DevicePlan&) = delete;

  const RenderData& data() const { return rd_; }
  const int* row_ptr(int step) const;
  const int* col(int step) const;
  // Transposed step table (backward pass): for the nodes of step k, the rows of their
  // consumers, one entry per edge, in (step, slot, edge) order; step num_steps = the sources.
  // Edges whose source row the forward read as silence (one-by-one quirk) are left out.
  const int* t_row_ptr(int step) const;
  const int* t_col(int step) const;
  const std::vector<int>& zero_rows() const { return zero_rows_; }
  // First source row when step k's slot s reads exactly row dense_src(k) + s (one edge per
  // slot, consecutive rows): its kernels then need no CSR loads. -1 otherwise.
  int dense_src(int step) const { return dense_[static_cast<std::size_t>(step)]; }
  // Step k (k >= 1) is a pointwise follower of step k-1 (gain / imager / mix / out whose
  // every node reads exactly one distinct node of step k-1): follow_map(k) maps step k-1's
  // slots to step k's slots (device); nullptr otherwise.
  bool follows(int step) const { return follow_off_[static_cast<std::size_t>(step)] >= 0; }
  const int* follow_map(int step) const;
  // Step k (k >= 1) and step k-1 are long convolutions and some of step k's slots read the same
  // single source row as a slot of step k-1 (a console track's delay and reverb sends; each
  // slot of step k-1 pairs at most once). share(k): device lists of the pairs (slot of k-1,
  // slot of k) and of each step's unpaired slots; shares(k) is false when nothing pairs.
  struct Share {
    int pairs = 0, own_prev = 0, own = 0;
    long off = -1;  // host_index offset: [pair_prev][pair][own_prev][own]
  };
  bool shares(int step) const { return share_[static_cast<std::size_t>(step)].off >= 0; }
  const Share& share_info(int step) const { return share_[static_cast<std::size_t>(step)]; }
  const int* share_ints(int step) const;  // device pointer to the step's lists
  std::size_t workspace_bytes(int batch, long length, const ProcessorSet& procs) const;
  // Workspace for a forward render followed by backward_arena (forward layout + scratch).
  std::size_t backward_workspace_bytes(int batch, long length, const ProcessorSet& procs) const;
  int kernels_per_render(int batch, long length) const;
  // owner[k] = the step whose launch computes step k: k itself, the head of its pointwise
  // chain, or the producer whose epilogue computes it (render_arena without per-step events).
  void step_owners(int batch, long length, int* owner) const;

  // Workspace: one persistent region per step for its parameter-only prologue, the steps'
  // synchronisation words, then one transient region shared by every step's audio pass.
  struct Layout {
    std::vector<std::size_t> prologue_off;
    std::vector<std::size_t> sync_off;  // per step: scan tickets / pass counters (zeroed per render)
    std::size_t sync_begin = 0, sync_bytes = 0;
    std::size_t main_off = 0;
    std::size_t main2_off = 0;  // second transient region (a step run concurrently with its predecessor)
    std::vector<char> paired;   // paired[k]: step k runs on the lane beside step k + 1
    std::vector<char> shared;   // shared[k]: step k reuses step k-1's signal spectra (launch_conv_shared)
    std::size_t share_off = 0;  // step k's transient region when shared[k] (after step k-1's)
    std::size_t total = 0;
  };
  Layout layout(int batch, long length, const ProcessorSet& procs) const;
  const std::array<cudaStream_t, 4>& aux_streams() const { return aux_; }
  // Second high-priority stream for a pair of independent, small conv steps (owned plans only).
  cudaStream_t lane() const { return lane_; }
  const cudaEvent_t* lane_events() const { return lane_events_.data(); }
  const cudaEvent_t* events() const { return borrowed_events_ ? borrowed_events_ : events_.data(); }

 private:
  void build_index();
  const RenderData& rd_;
  bool owned_ = true;
  std::array<cudaStream_t, 4> aux_{};  // low-priority side streams for the prologues
  std::vector<cudaEvent_t> events_;  // [0] fork, [k+1] prologue of step k done
  cudaStream_t lane_ = nullptr;
  std::vector<cudaEvent_t> lane_events_;  // [2k] fork before step k, [2k+1] step k done
  const cudaEvent_t* borrowed_events_ = nullptr;
  const int* d_index_ = nullptr;
  std::vector<int> host_;
  std::vector<long> rp_off_, col_off_, trp_off_, tcol_off_, follow_off_;
  std::vector<Share> share_;
  std::vector<int> zero_rows_;
  std::vector<int> dense_;
};

// Reverse-mode pass over a rendered arena (parameter gradients; the reference has no
// autodiff, its fit.cpp:70-82 uses central differences). `arena` and `workspace` must be
// those of the render_arena call that produced the forward (its prologue results are reused;
// workspace_bytes >= backward_workspace_bytes). `adjoint` ([rows][batch][2][length] fp32):
// on entry rows [output_begin, rows) hold dL/d(outputs); on exit row r holds dL/d(input of
// node r) — rows [0, num_inputs) are dL/d(sources). grad_tables[t]: device fp64 tables shaped
// like param_tables[t] (render order), overwritten with dL/d(params). Delay tap positions
// (Re z, Im z) are piecewise constant in the forward: their gradient is 0.
void backward_arena(const DevicePlan& plan, const ProcessorSet& processors, const double* const* param_tables,
                    const float* arena, float* adjoint, double* const* grad_tables, int batch, long length,
                    void* workspace, std::size_t workspace_bytes, cudaStream_t stream);

// Per-step device time (prologue + audio pass of step k, ms) from `reps` back-to-back
// repetitions captured as one CUDA graph and timed between one event pair (after one full
// render on `stream`; no host launch cost between repetitions). Diagnostic.
void profile_steps(const DevicePlan& plan, const ProcessorSet& processors, const double* const* param_tables,
                   float* arena, int batch, long length, void* workspace, std::size_t workspace_bytes,
                   cudaStream_t stream, int reps, float* step_ms);

// A whole render (main stream + side-stream prologues) captured once and instantiated as
// a CUDA graph with node priorities: launch() replays it on any stream. Pointers, shapes and
// parameter tables are baked in (update the tables' contents in place between launches).
typedef struct CUgraph_st* cudaGraph_t;
typedef struct CUgraphExec_st* cudaGraphExec_t;
class RenderGraph {
 public:
  RenderGraph(const DevicePlan& plan, const ProcessorSet& processors, const double* const* param_tables, float* arena,
              int batch, long length, void* workspace, std::size_t workspace_bytes);
  ~RenderGraph();
  RenderGraph(const RenderGraph&) = delete;
  RenderGraph& operator=(const RenderGraph&) = delete;
  void launch(cudaStream_t stream) const;

 private:
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t exec_ = nullptr;
};

// Streaming host API: renders submitted back to back overlap their host<->device copies with
// the previous render's kernels. `depth` arenas rotate; an H2D copy stream, a compute
// stream (graph replays) and a D2H copy stream are chained with events, so PCIe traffic in
// both directions runs concurrently with the GPU work. Host audio is float (f32_io, copied
// straight into the arena) or double (converted on the device). Host buffers passed to
// submit() must stay valid (and should be pinned) until sync().
// Double host audio (the reference's AudioBuffer type) is converted to/from fp32 on host
// worker threads (`host_threads`; < 0: half the host's hardware threads per local rank, up
// to 8), which halves its PCIe bytes: sources in submit() in 1 MiB chunks whose
// H2D copies start as each chunk is converted, outputs on a completion thread once their D2H
// landed. A fraction of the sources (1 - kHostFraction) still crosses PCIe as double and is
// converted on the device, so host memory bandwidth and PCIe work side by side. With
// host_threads = 0 every source goes as double (device conversion only).
class RenderPipeline {
 public:
  RenderPipeline(const DevicePlan& plan, const ProcessorSet& processors, int batch, long length, bool f32_io,
                 int depth = 2, int host_threads = -1);
  ~RenderPipeline();
  RenderPipeline(const RenderPipeline&) = delete;
  RenderPipeline& operator=(const RenderPipeline&) = delete;
  // params in render order (RenderData::reorder_params); validated like render().
  void submit(const ParamStore& params, const void* const* sources, void* const* outputs);
  void sync();
  std::size_t bytes_per_signal() const { return (f32_ ? sizeof(float) : sizeof(double)) * static_cast<std::size_t>(stride_); }

 private:
  struct Slot;
  const DevicePlan& plan_;
  const ProcessorSet& procs_;
  int batch_;
  long length_;
  bool f32_;
  long stride_;
  std::vector<std::unique_ptr<Slot>> slots_;
  cudaStream_t h2d_ = nullptr, compute_ = nullptr, d2h_ = nullptr;
  std::size_t next_ = 0;
  struct HostConvert;  // worker pool + completion thread (double host audio)
  std::unique_ptr<HostConvert> conv_;
  static constexpr double kHostFraction = 1.0;
  double host_fraction_ = kHostFraction;
};

// Renders a stream of plans whose topology changes every batch (BASELINE config 3: 64
// random consoles per step, render order recomputed per batch). Nothing is allocated or
// synchronised per plan: the arena, workspace, step tables and parameter tables live in
// device pools sized once (Capacity), `depth` slots rotate, and each submit() packs the new
// step table and the ORIGINAL-order parameter tables (as a dataset holds them) into pinned
// staging, uploads them on a copy stream and reorders the parameters on the device
// (`schedule.cpp:454-471`) before the render. The host therefore prepares batch i+1 while
// the GPU renders batch i. `rd` must stay alive until its slot is reused (`depth` submits
// later) or sync().
class BatchRenderer {
 public:
  struct Capacity {
    std::size_t rows = 0, workspace_bytes = 0, index_ints = 0, param_doubles = 0;
    void grow(const Capacity& o);
  };
  static Capacity capacity_for(const RenderData& rd, const ProcessorSet& processors, int batch, long length);
  BatchRenderer(const ProcessorSet& processors, int batch, long length, const Capacity& cap, int depth = 2);
  ~BatchRenderer();
  BatchRenderer(const BatchRenderer&) = delete;
  BatchRenderer& operator=(const BatchRenderer&) = delete;
  // orig_tables[t]: host fp64 [orig_rows[t]][param_width(t)] in original row order (null for
  // types without parameters); validated like render() when `validate`. sources: fp32
  // [source_rows][batch][2][length]; input k of the plan takes row k % source_rows (device
  // memory: copied on the device; host memory: should be pinned). outputs: host fp32
  // [num_outputs][batch][2][length], or null to keep them on the device (outputs()).
  void submit(const RenderData& rd, const double* const* orig_tables, const int* orig_rows, bool validate,
              const float* sources, int source_rows, bool sources_on_device, float* outputs);
  void sync();
  // Device arena of the most recent submit ([buffer_rows][batch][2][length] fp32).
  float* last_arena() const;
  cudaStream_t compute_stream() const { return compute_; }

 private:
  struct Slot;
  const ProcessorSet& procs_;
  int batch_;
  long length_;
  long stride_;
  Capacity cap_;
  std::vector<std::unique_ptr<Slot>> slots_;
  std::array<cudaStream_t, 4> aux_{};
  std::vector<cudaEvent_t> step_events_;
  cudaStream_t h2d_ = nullptr, compute_ = nullptr, d2h_ = nullptr;
  std::size_t next_ = 0;
};

// Host-buffer render over caller pointers (no intermediate host copies): sources[k] and
// outputs[o] each point at [batch][2][length] doubles (pinned memory makes the copies
// asynchronous DMA); intermediates (original row order) may be null. `plan` may be null.
void render_host(const RenderData& rd, const ProcessorSet& processors, const ParamStore& params,
                 const double* const* sources, int batch, long length, double* const* outputs,
                 double* const* intermediates, const DevicePlan* plan);

void render_arena(const DevicePlan& plan, const ProcessorSet& processors, const double* const* param_tables,
                  float* arena, int batch, long length, void* workspace, std::size_t workspace_bytes,
                  cudaStream_t stream, cudaEvent_t* step_events = nullptr, bool hoist = true);

}  // namespace mixgraph
