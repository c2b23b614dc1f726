// Render engine: processor constants, device step table, step dispatch, host-buffer API.
//
// Reference call stack this replaces (`render.cpp:14-81`, `processors.cpp:151-282`):
// render() allocates a double arena, then per step zero-fills step_in/step_out, sums the
// gathered rows, runs ProcessorSet::process and memcpy's the result back. Here the arena
// is fp32 in HBM and each step is one fused launch sequence that gathers straight from the
// arena rows and stores straight into the step's contiguous output rows (the contiguity
// is what node reordering buys, `schedule.cpp:397-413`): no step_in/step_out buffers.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <deque>
#include <functional>
#include <thread>
#include <unordered_map>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>

#include "host/convert.hpp"
#include "launch.hpp"
#include "mixgraph_b200/render.hpp"

namespace mixgraph {

namespace {

[[noreturn]] void fail(const std::string& msg) { throw std::invalid_argument(msg); }

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + what + ": " + cudaGetErrorString(e));
}

std::string tname(NodeType t) { return std::string(type_name(t)); }

// Grow-only device allocation.
struct DeviceBuffer {
  void* ptr = nullptr;
  std::size_t cap = 0;
  void* ensure(std::size_t bytes) {
    if (bytes > cap) {
      if (ptr) cudaFree(ptr);
      ptr = nullptr;
      cap = 0;
      cuda_check(cudaMalloc(&ptr, bytes), "cudaMalloc");
      cap = bytes;
    }
    return ptr;
  }
  ~DeviceBuffer() {
    if (ptr) cudaFree(ptr);
  }
};

// Per-thread, per-device resources of the host-buffer API (render / process).
struct Engine {
  int device = -1;
  cudaStream_t stream = nullptr;
  DeviceBuffer arena, ws, params, staging, aux;
  ~Engine() {
    if (stream) cudaStreamDestroy(stream);
  }
};

Engine& engine_for(int device) {
  thread_local std::map<int, std::unique_ptr<Engine>> engines;
  auto& e = engines[device];
  if (!e) {
    e = std::make_unique<Engine>();
    e->device = device;
    cuda_check(cudaSetDevice(device), "cudaSetDevice");
    cuda_check(cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  return *e;
}

inline std::size_t align256(std::size_t x) { return (x + 255) & ~static_cast<std::size_t>(255); }

// EQ prologue region: taps [slots][2048] f32 + magnitudes [slots][1024] f64, then the
// response [slots][8192] f32 (run_prologue / run_main locate it the same way).
std::size_t eq_taps_bytes(int slots) { return align256((sizeof(float) * 2048 + sizeof(double) * 1024) * slots); }
std::size_t eq_ws_bytes(int slots) { return eq_taps_bytes(slots) + align256(sizeof(float) * mgb::kEqFft * slots); }

}  // namespace

struct DeviceConstants {
  int device = 0;
  float2* stft_mid = nullptr;
  float2* stft_side = nullptr;
  float4* stft_ms = nullptr;
  int frames = 0;
  ~DeviceConstants() {
    if (stft_mid) cudaFree(stft_mid);
    if (stft_side) cudaFree(stft_side);
    if (stft_ms) cudaFree(stft_ms);
  }
};

// ---- scalar reference semantics (processors.cpp:110-149) ------------------------------

double compressor_gain_log(double g_u, double threshold, double knee, double ratio) {
  if (g_u >= threshold + knee) return threshold + (g_u - threshold) / ratio;
  if (g_u < threshold - knee) return g_u;
  const double d = g_u - threshold + knee;
  return g_u + (1.0 / ratio - 1.0) * d * d / (4.0 * knee);
}

double noisegate_gain_log(double g_u, double threshold, double knee, double ratio) {
  if (g_u >= threshold + knee) return g_u;
  if (g_u < threshold - knee) return threshold + ratio * (g_u - threshold);
  const double d = g_u - threshold - knee;
  return g_u + (1.0 - ratio) * d * d / (4.0 * knee);
}

void check_param_row(NodeType type, std::span<const double> row) {
  const std::string name = tname(type);
  for (double v : row) {
    if (!std::isfinite(v)) fail(name + ": non-finite parameter value");
  }
  if (type == NodeType::Compressor || type == NodeType::Noisegate) {
    if (!(row[0] > 0.0 && row[0] < 1.0)) fail(name + ": alpha must be in (0, 1)");
    if (!(row[2] > 0.0)) fail(name + ": knee half-width must be positive");
    if (!(row[3] >= 1.0)) fail(name + ": ratio must be >= 1");
  } else if (type == NodeType::Delay) {
    for (int tap = 0; tap < 2 * kDelayTapsPerChannel; ++tap) {
      if (std::hypot(row[static_cast<std::size_t>(tap * kDelayTapStride)], row[static_cast<std::size_t>(tap * kDelayTapStride + 1)]) >
          1.0 + 1e-9) {
        fail("delay: angular frequency outside the unit disk");
      }
    }
  }
}

namespace dsp {
// dsp.cpp:222-230: mt19937(seed), 2 * (u32 * 2^-32) - 1.
std::vector<double> uniform_noise(long n, std::uint32_t seed) {
  std::mt19937 gen(seed);
  std::vector<double> out(static_cast<std::size_t>(n));
  for (auto& v : out) v = 2.0 * (static_cast<double>(gen()) * (1.0 / 4294967296.0)) - 1.0;
  return out;
}
}  // namespace dsp

// ---- ProcessorSet -----------------------------------------------------------------------

ProcessorSet::ProcessorSet(const ProcessorConfig& config) : config_(config) {
  if (!(config_.sample_rate > 0)) fail("sample rate must be positive");
  delay_span_ = std::lround(kDelaySeconds * config_.sample_rate);
  delay_window_ = static_cast<int>(std::lround(kDelayWindowSeconds * config_.sample_rate));
  reverb_length_ = std::lround(kReverbSeconds * config_.sample_rate);
  noise_mid_ = dsp::uniform_noise(reverb_length_, config_.reverb_seed);
  noise_side_ = dsp::uniform_noise(reverb_length_, config_.reverb_seed + 1);

  dev_ = std::make_unique<DeviceConstants>();
  cuda_check(cudaGetDevice(&dev_->device), "cudaGetDevice");
  mgb::twiddle_table(dev_->device);
  mgb::twiddle_table64(dev_->device);
  mgb::eq_basis(dev_->device, true);
  mgb::eq_basis(dev_->device, false);
  dev_->frames = static_cast<int>((reverb_length_ + kReverbStftHop - 1) / kReverbStftHop);
  const std::size_t stft_bytes = sizeof(float2) * static_cast<std::size_t>(dev_->frames) * (kReverbStftLength / 2 + 1);
  cuda_check(cudaMalloc(&dev_->stft_mid, stft_bytes > 0 ? stft_bytes : 8), "cudaMalloc");
  cuda_check(cudaMalloc(&dev_->stft_side, stft_bytes > 0 ? stft_bytes : 8), "cudaMalloc");
  cuda_check(cudaMalloc(&dev_->stft_ms, stft_bytes > 0 ? 2 * stft_bytes : 16), "cudaMalloc");
  if (dev_->frames > 0) {
    Engine& e = engine_for(dev_->device);
    auto* d_noise = static_cast<double*>(e.aux.ensure(sizeof(double) * 2 * static_cast<std::size_t>(reverb_length_)));
    cuda_check(cudaMemcpyAsync(d_noise, noise_mid_.data(), sizeof(double) * reverb_length_, cudaMemcpyHostToDevice, e.stream), "H2D");
    cuda_check(cudaMemcpyAsync(d_noise + reverb_length_, noise_side_.data(), sizeof(double) * reverb_length_, cudaMemcpyHostToDevice, e.stream), "H2D");
    mgb::launch_noise_stft(d_noise, reverb_length_, dev_->frames, dev_->stft_mid, e.stream);
    mgb::launch_noise_stft(d_noise + reverb_length_, reverb_length_, dev_->frames, dev_->stft_side, e.stream);
    mgb::launch_pack_mid_side(dev_->stft_mid, dev_->stft_side, static_cast<long>(dev_->frames) * (kReverbStftLength / 2 + 1),
                              dev_->stft_ms, e.stream);
    cuda_check(cudaStreamSynchronize(e.stream), "noise stft");
  }
}

ProcessorSet::~ProcessorSet() = default;

int ProcessorSet::device_id() const { return dev_->device; }

namespace {

mgb::ReverbConst reverb_const(const ProcessorSet& p) {
  return {p.device().stft_mid, p.device().stft_side, p.device().stft_ms, p.device().frames, p.reverb_length(),
          mgb::twiddle_table(p.device().device)};
}
mgb::DelayConst delay_const(const ProcessorSet& p) { return {p.delay_span(), p.delay_window()}; }

bool has_prologue(NodeType t) { return t == NodeType::Eq || t == NodeType::Reverb || t == NodeType::Delay; }

// Parameter-only work (FIR design, impulse responses, kernel spectra) lives in a per-step
// persistent region so it can run ahead on a side stream; audio work uses a shared region.
std::size_t prologue_bytes(NodeType t, int slots, long length, const ProcessorSet& p) {
  switch (t) {
    case NodeType::Eq: return eq_ws_bytes(slots);
    case NodeType::Reverb:
      return mgb::conv_prologue_bytes(mgb::conv_geom(length, p.reverb_length()), slots, p.reverb_length());
    case NodeType::Delay: return mgb::conv_prologue_bytes(mgb::conv_geom(length, p.delay_span()), slots, p.delay_span());
    default: return 0;
  }
}

// Per-render synchronisation words (scan tickets and tile status): zero at the
// start of every step run. render_arena clears all steps' words with one memset.
std::size_t sync_bytes(NodeType t, int slots, int batch, long length) {
  switch (t) {
    case NodeType::Compressor:
    case NodeType::Noisegate: return mgb::dyn_sync_bytes(slots, batch, length);
    default: return 0;
  }
}

std::size_t main_bytes(NodeType t, int slots, int batch, long length, const ProcessorSet& p) {
  switch (t) {
    case NodeType::Reverb: return mgb::conv_main_bytes(mgb::conv_geom(length, p.reverb_length()), slots, batch);
    case NodeType::Delay: return mgb::conv_main_bytes(mgb::conv_geom(length, p.delay_span()), slots, batch);
    default: return 0;
  }
}

int step_kernels(NodeType t) {
  switch (t) {
    case NodeType::Eq: return 4;
    case NodeType::Compressor:
    case NodeType::Noisegate: return 1;
    case NodeType::Reverb: return 6;  // impulse responses, kernel spectrum (2), audio pass (3)
    case NodeType::Delay: return 6;   // tap records, kernel spectrum (2), audio pass (3)
    default: return 1;
  }
}

void run_prologue(NodeType t, const mgb::StepArgs& a, const ProcessorSet& p, void* pws, cudaStream_t s) {
  switch (t) {
    case NodeType::Eq: {
      auto* taps = static_cast<float*>(pws);
      auto* resp = reinterpret_cast<float*>(static_cast<char*>(pws) + eq_taps_bytes(a.slots));
      mgb::launch_eq_prologue(a, taps, resp, s);
      break;
    }
    case NodeType::Reverb: mgb::launch_conv_prologue(true, a, reverb_const(p), delay_const(p), pws, s); break;
    case NodeType::Delay: mgb::launch_conv_prologue(false, a, reverb_const(p), delay_const(p), pws, s); break;
    default: break;
  }
}

// One step's audio pass. a.params points at the step's first parameter row.
// `join`: the step's prologue event when it has not been waited on yet (conv steps join
// after their signal column pass; every other type joins first).
void run_main(NodeType t, const mgb::StepArgs& a, const ProcessorSet& p, void* pws, void* mws, void* sws, bool zero_sync,
              cudaStream_t s, cudaEvent_t join = nullptr, const mgb::PwEpi& epi = {}) {
  if (join && t != NodeType::Reverb && t != NodeType::Delay) {
    cuda_check(cudaStreamWaitEvent(s, join, 0), "wait");
    join = nullptr;
  }
  switch (t) {
    case NodeType::In:
    case NodeType::Out:
    case NodeType::Mix: mgb::launch_pointwise(mgb::PointOp::Copy, a, s, epi); break;
    case NodeType::Gain: mgb::launch_pointwise(mgb::PointOp::Gain, a, s, epi); break;
    case NodeType::Imager: mgb::launch_pointwise(mgb::PointOp::Imager, a, s, epi); break;
    case NodeType::Eq:
      mgb::launch_eq_main(a, reinterpret_cast<float*>(static_cast<char*>(pws) + eq_taps_bytes(a.slots)), s);
      break;
    case NodeType::Compressor:
    case NodeType::Noisegate:
      mgb::launch_dynamics(t == NodeType::Noisegate, a, p.config().envelope_taps, p.config().energy_floor, sws, zero_sync,
                           s, epi);
      break;
    case NodeType::Reverb: mgb::launch_conv_main(a, p.reverb_length(), pws, mws, s, join); break;
    case NodeType::Delay: mgb::launch_conv_main(a, p.delay_span(), pws, mws, s, join); break;
  }
}

bool is_pointwise(NodeType t) {
  return t == NodeType::In || t == NodeType::Out || t == NodeType::Mix || t == NodeType::Gain || t == NodeType::Imager;
}

mgb::PointOp point_op(NodeType t) {
  return t == NodeType::Gain ? mgb::PointOp::Gain : t == NodeType::Imager ? mgb::PointOp::Imager : mgb::PointOp::Copy;
}

bool chainable(NodeType t, int slots, int batch, long length) {
  return is_pointwise(t) && length % 4 == 0 && slots >= 1 && slots * batch <= mgb::kPwChainMaxRows;
}

// Length of the fused pointwise run starting at step k (1 = launch the step on its own).
int chain_length(const RenderData& rd, std::size_t k, int batch, long length) {
  int n = 0;
  while (k + n < rd.steps.size() && n < mgb::kPwChainMax) {
    const StepIndex& st = rd.steps[k + n];
    if (!chainable(st.type, st.store_end - st.store_begin, batch, length)) break;
    ++n;
  }
  return n >= 2 ? n : 1;
}

// Number of pointwise follower steps fused into step k's epilogue (render_arena): the
// producer is a compressor / noisegate scan or a pointwise step too large for a chain
// (vector path), the followers the consecutive steps the plan marked as followers.
int epi_followers(const DevicePlan& plan, std::size_t k, int batch, long length) {
  const RenderData& rd = plan.data();
  if (k + 1 >= rd.steps.size()) return 0;
  const StepIndex& st = rd.steps[k];
  const bool dyn = st.type == NodeType::Compressor || st.type == NodeType::Noisegate;
  const bool pw = is_pointwise(st.type) && st.type != NodeType::In && length % 4 == 0 &&
                  chain_length(rd, k, batch, length) == 1;
  if (!dyn && !pw) return 0;
  int n = 0;
  while (n < mgb::kPwEpiMax && k + 1 + n < rd.steps.size() && plan.follows(static_cast<int>(k + 1 + n))) ++n;
  return n;
}

// Steps k, k+1 run as one fused streaming scan (launch_dynamics_pair): both compressor /
// noisegate, dense, step k+1 reading step k's rows slot by slot (a console track's compressor
// -> noisegate).
bool dyn_pair(const DevicePlan& plan, std::size_t k, int batch, long length) {
  const RenderData& rd = plan.data();
  if (k + 1 >= rd.steps.size()) return false;
  auto dyn = [](NodeType t) { return t == NodeType::Compressor || t == NodeType::Noisegate; };
  const StepIndex& a = rd.steps[k];
  const StepIndex& b = rd.steps[k + 1];
  const int slots = a.store_end - a.store_begin;
  return dyn(a.type) && dyn(b.type) && slots == b.store_end - b.store_begin && plan.dense_src(static_cast<int>(k)) >= 0 &&
         plan.dense_src(static_cast<int>(k + 1)) == a.store_begin && mgb::dyn_pair_shape(slots, batch, length);
}

std::size_t step_ws_bytes(NodeType t, int slots, int batch, long length, const ProcessorSet& p) {
  return align256(prologue_bytes(t, slots, length, p)) + align256(sync_bytes(t, slots, batch, length)) +
         main_bytes(t, slots, batch, length, p);
}

void run_step(NodeType t, const mgb::StepArgs& a, const ProcessorSet& p, void* ws, cudaStream_t s) {
  const std::size_t pb = align256(prologue_bytes(t, a.slots, a.length, p));
  const std::size_t sb = align256(sync_bytes(t, a.slots, a.batch, a.length));
  run_prologue(t, a, p, ws, s);
  run_main(t, a, p, ws, static_cast<char*>(ws) + pb + sb, static_cast<char*>(ws) + pb, true, s);
}

}  // namespace

// ---- DevicePlan -------------------------------------------------------------------------

void DevicePlan::build_index() {
  std::vector<int>& host = host_;
  std::vector<char> written(static_cast<std::size_t>(rd_.buffer_rows), 0);
  for (int r = 0; r < rd_.num_inputs && r < rd_.buffer_rows; ++r) written[static_cast<std::size_t>(r)] = 1;
  for (const StepIndex& st : rd_.steps) {
    const int slots = st.store_end - st.store_begin;
    rp_off_.push_back(static_cast<long>(host.size()));
    std::size_t e = 0;
    for (int s = 0; s <= slots; ++s) {
      while (e < st.aggregate.size() && st.aggregate[e] < s) ++e;
      host.push_back(static_cast<int>(e));
    }
    col_off_.push_back(static_cast<long>(host.size()));
    for (int g : st.gather) {
      host.push_back(g);
      // A row read before any step stored it holds zeros in the reference (render.cpp:33).
      if (!written[static_cast<std::size_t>(g)]) {
        written[static_cast<std::size_t>(g)] = 1;
        zero_rows_.push_back(g);
      }
    }
    for (int r = st.store_begin; r < st.store_end; ++r) written[static_cast<std::size_t>(r)] = 1;
  }
  // Transposed table: consumers of each row over the edges whose source the forward read
  // after it was written (a row read before its step ran contributed silence).
  std::vector<std::vector<int>> cons(static_cast<std::size_t>(rd_.buffer_rows));
  std::vector<char> done(static_cast<std::size_t>(rd_.buffer_rows), 0);
  for (int r = 0; r < rd_.num_inputs && r < rd_.buffer_rows; ++r) done[static_cast<std::size_t>(r)] = 1;
  for (const StepIndex& st : rd_.steps) {
    for (std::size_t e = 0; e < st.gather.size(); ++e) {
      const int g = st.gather[e];
      if (done[static_cast<std::size_t>(g)]) cons[static_cast<std::size_t>(g)].push_back(st.store_begin + st.aggregate[e]);
    }
    for (int r = st.store_begin; r < st.store_end; ++r) done[static_cast<std::size_t>(r)] = 1;
  }
  auto emit = [&](int r0, int r1) {
    trp_off_.push_back(static_cast<long>(host.size()));
    int n = 0;
    for (int r = r0; r <= r1; ++r) {
      host.push_back(n);
      if (r < r1) n += static_cast<int>(cons[static_cast<std::size_t>(r)].size());
    }
    tcol_off_.push_back(static_cast<long>(host.size()));
    for (int r = r0; r < r1; ++r) host.insert(host.end(), cons[static_cast<std::size_t>(r)].begin(), cons[static_cast<std::size_t>(r)].end());
  };
  for (const StepIndex& st : rd_.steps) emit(st.store_begin, st.store_end);
  emit(0, rd_.num_inputs);
  // Dense steps: one edge per slot, from consecutive rows in slot order.
  dense_.assign(rd_.steps.size(), -1);
  for (std::size_t k = 0; k < rd_.steps.size(); ++k) {
    const StepIndex& st = rd_.steps[k];
    const int slots = st.store_end - st.store_begin;
    bool ok = slots > 0 && st.gather.size() == static_cast<std::size_t>(slots);
    for (int e = 0; ok && e < slots; ++e) {
      ok = st.aggregate[static_cast<std::size_t>(e)] == e && st.gather[static_cast<std::size_t>(e)] == st.gather[0] + e;
    }
    if (ok) dense_[k] = st.gather[0];
  }
  // Pointwise followers (fused into the previous step's epilogue by render_arena).
  follow_off_.assign(rd_.steps.size(), -1);
  for (std::size_t k = 1; k < rd_.steps.size(); ++k) {
    const StepIndex& st = rd_.steps[k];
    const StepIndex& pv = rd_.steps[k - 1];
    const NodeType t = st.type;
    if (t != NodeType::Gain && t != NodeType::Imager && t != NodeType::Mix && t != NodeType::Out) continue;
    const int slots = st.store_end - st.store_begin;
    if (slots == 0 || slots != pv.store_end - pv.store_begin || st.gather.size() != static_cast<std::size_t>(slots)) continue;
    std::vector<int> map(static_cast<std::size_t>(slots), -1);
    bool ok = true;
    for (int e = 0; e < slots && ok; ++e) {
      const int src = st.gather[static_cast<std::size_t>(e)] - pv.store_begin;
      ok = st.aggregate[static_cast<std::size_t>(e)] == e && src >= 0 && src < slots && map[static_cast<std::size_t>(src)] < 0;
      if (ok) map[static_cast<std::size_t>(src)] = e;
    }
    if (!ok) continue;
    follow_off_[k] = static_cast<long>(host.size());
    host.insert(host.end(), map.begin(), map.end());
  }
  // Shared signal spectra of adjacent long-convolution steps: slots with exactly one input edge
  // reading the same row (and step k reading none of step k-1's outputs).
  share_.assign(rd_.steps.size(), Share{});
  auto conv = [](NodeType t) { return t == NodeType::Reverb || t == NodeType::Delay; };
  auto single_sources = [](const StepIndex& st) {
    const int slots = st.store_end - st.store_begin;
    std::vector<int> cnt(static_cast<std::size_t>(slots), 0), src(static_cast<std::size_t>(slots), -1);
    for (std::size_t e = 0; e < st.gather.size(); ++e) {
      ++cnt[static_cast<std::size_t>(st.aggregate[e])];
      src[static_cast<std::size_t>(st.aggregate[e])] = st.gather[e];
    }
    for (int q = 0; q < slots; ++q) {
      if (cnt[static_cast<std::size_t>(q)] != 1) src[static_cast<std::size_t>(q)] = -1;
    }
    return src;
  };
  for (std::size_t k = 1; k < rd_.steps.size(); ++k) {
    const StepIndex& a = rd_.steps[k - 1];
    const StepIndex& b = rd_.steps[k];
    if (!conv(a.type) || !conv(b.type)) continue;
    bool reads_a = false;
    for (int g : b.gather) reads_a = reads_a || (g >= a.store_begin && g < a.store_end);
    if (reads_a) continue;
    std::unordered_map<int, int> slot_of;  // source row -> unpaired slot of step k-1
    const std::vector<int> sa = single_sources(a);
    for (int q = 0; q < static_cast<int>(sa.size()); ++q) {
      if (sa[static_cast<std::size_t>(q)] >= 0) slot_of.emplace(sa[static_cast<std::size_t>(q)], q);
    }
    const std::vector<int> sb = single_sources(b);
    std::vector<int> pa, pb, own_b;
    std::vector<char> paired_a(sa.size(), 0);
    for (int q = 0; q < static_cast<int>(sb.size()); ++q) {
      const auto it = sb[static_cast<std::size_t>(q)] >= 0 ? slot_of.find(sb[static_cast<std::size_t>(q)]) : slot_of.end();
      if (it != slot_of.end()) {
        pa.push_back(it->second);
        pb.push_back(q);
        paired_a[static_cast<std::size_t>(it->second)] = 1;
        slot_of.erase(it);
      } else {
        own_b.push_back(q);
      }
    }
    if (pa.empty()) continue;
    std::vector<int> own_a;
    for (int q = 0; q < static_cast<int>(sa.size()); ++q) {
      if (!paired_a[static_cast<std::size_t>(q)]) own_a.push_back(q);
    }
    Share& sh = share_[k];
    sh.off = static_cast<long>(host.size());
    sh.pairs = static_cast<int>(pa.size());
    sh.own_prev = static_cast<int>(own_a.size());
    sh.own = static_cast<int>(own_b.size());
    for (const std::vector<int>* v : {&pa, &pb, &own_a, &own_b}) host.insert(host.end(), v->begin(), v->end());
  }
}

const int* DevicePlan::share_ints(int step) const {
  const long off = share_[static_cast<std::size_t>(step)].off;
  return off < 0 ? nullptr : d_index_ + off;
}

const int* DevicePlan::follow_map(int step) const {
  const long off = follow_off_[static_cast<std::size_t>(step)];
  return off < 0 ? nullptr : d_index_ + off;
}

DevicePlan::DevicePlan(const RenderData& rd) : rd_(rd) {
  build_index();
  if (!host_.empty()) {
    int* d = nullptr;
    cuda_check(cudaMalloc(&d, sizeof(int) * host_.size()), "cudaMalloc");
    cuda_check(cudaMemcpy(d, host_.data(), sizeof(int) * host_.size(), cudaMemcpyHostToDevice), "H2D plan");
    d_index_ = d;
  }
  // Prologues are off the critical path: lowest priority, so the CTA scheduler prefers the
  // main stream's kernels whenever both have work (honoured inside RenderGraph too).
  int least = 0, greatest = 0;
  cuda_check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
  for (auto& a : aux_) cuda_check(cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, least), "cudaStreamCreate");
  events_.resize(rd.steps.size() + 1);
  for (auto& ev : events_) cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaStreamCreateWithPriority(&lane_, cudaStreamNonBlocking, greatest), "cudaStreamCreate");
  lane_events_.resize(2 * rd.steps.size());
  for (auto& ev : lane_events_) cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
}

DevicePlan::DevicePlan(const RenderData& rd, Deferred) : rd_(rd), owned_(false) { build_index(); }

void DevicePlan::attach(const int* device_index, const std::array<cudaStream_t, 4>& aux, const cudaEvent_t* events) {
  d_index_ = device_index;
  aux_ = aux;
  borrowed_events_ = events;
}

DevicePlan::~DevicePlan() {
  if (!owned_) return;
  for (cudaEvent_t ev : events_) cudaEventDestroy(ev);
  for (cudaEvent_t ev : lane_events_) cudaEventDestroy(ev);
  if (lane_) cudaStreamDestroy(lane_);
  for (cudaStream_t a : aux_) if (a) cudaStreamDestroy(a);
  if (d_index_) cudaFree(const_cast<int*>(d_index_));
}

const int* DevicePlan::row_ptr(int step) const { return d_index_ + rp_off_[static_cast<std::size_t>(step)]; }
const int* DevicePlan::col(int step) const { return d_index_ + col_off_[static_cast<std::size_t>(step)]; }
const int* DevicePlan::t_row_ptr(int step) const { return d_index_ + trp_off_[static_cast<std::size_t>(step)]; }
const int* DevicePlan::t_col(int step) const { return d_index_ + tcol_off_[static_cast<std::size_t>(step)]; }

namespace {
// Steps k and k+1 may run side by side (two streams) when both are long convolutions whose
// grids are small (the kernel spectra fit L2: under one or two waves per pass, e.g. config 2's
// 12 reverbs and 7 delays) and step k+1 reads none of step k's output rows.
bool pairable(const RenderData& rd, std::size_t k, long length, const ProcessorSet& p) {
  if (k + 1 >= rd.steps.size()) return false;
  const StepIndex& a = rd.steps[k];
  const StepIndex& b = rd.steps[k + 1];
  auto conv = [](NodeType t) { return t == NodeType::Reverb || t == NodeType::Delay; };
  if (!conv(a.type) || !conv(b.type)) return false;
  for (const StepIndex* st : {&a, &b}) {
    const long taps = st->type == NodeType::Reverb ? p.reverb_length() : p.delay_span();
    if (mgb::conv_fuse_kernel_rows(mgb::conv_geom(length, taps), st->store_end - st->store_begin)) return false;
  }
  for (int g : b.gather) {
    if (g >= a.store_begin && g < a.store_end) return false;
  }
  return true;
}

// Step k reuses step k-1's signal spectra (launch_conv_shared) when the plan found shared
// sources and both steps use the same transform with the kernel rows fused into the row pass
// (large steps: the rows kernel reads the other step's spectra).
bool shareable(const DevicePlan& plan, std::size_t k, long length, const ProcessorSet& p) {
  if (k == 0 || !plan.shares(static_cast<int>(k))) return false;
  const RenderData& rd = plan.data();
  long taps[2];
  for (int i = 0; i < 2; ++i) {
    const StepIndex& st = rd.steps[k - 1 + static_cast<std::size_t>(i)];
    taps[i] = st.type == NodeType::Reverb ? p.reverb_length() : p.delay_span();
    if (!mgb::conv_fuse_kernel_rows(mgb::conv_geom(length, taps[i]), st.store_end - st.store_begin)) return false;
  }
  const mgb::ConvGeom ga = mgb::conv_geom(length, taps[0]), gb = mgb::conv_geom(length, taps[1]);
  return ga.log_n == gb.log_n && ga.log_n1 == gb.log_n1 && ga.seg == gb.seg && ga.nseg == gb.nseg && taps[0] == taps[1];
}
}  // namespace

DevicePlan::Layout DevicePlan::layout(int batch, long length, const ProcessorSet& procs) const {
  Layout l;
  std::size_t off = 0, main = 256, main2 = 0;
  l.paired.assign(rd_.steps.size(), 0);
  if (owned_) {
    for (std::size_t k = 0; k + 1 < rd_.steps.size(); ++k) {
      if (pairable(rd_, k, length, procs)) {
        l.paired[k] = 1;
        const StepIndex& b = rd_.steps[k + 1];
        main2 = std::max(main2, main_bytes(b.type, b.store_end - b.store_begin, batch, length, procs));
        ++k;
      }
    }
  }
  l.shared.assign(rd_.steps.size(), 0);
  for (std::size_t k = 1; k < rd_.steps.size(); ++k) {
    if (shareable(*this, k, length, procs) && !l.paired[k - 1]) {
      l.shared[k] = 1;
      const StepIndex& a = rd_.steps[k - 1];
      const StepIndex& b = rd_.steps[k];
      const std::size_t ma = align256(main_bytes(a.type, a.store_end - a.store_begin, batch, length, procs));
      l.share_off = std::max(l.share_off, ma);
      main = std::max(main, ma + main_bytes(b.type, b.store_end - b.store_begin, batch, length, procs));
    }
  }
  for (const StepIndex& st : rd_.steps) {
    const int slots = st.store_end - st.store_begin;
    l.prologue_off.push_back(off);
    off += align256(prologue_bytes(st.type, slots, length, procs));
    main = std::max(main, main_bytes(st.type, slots, batch, length, procs));
  }
  l.sync_begin = off;
  for (const StepIndex& st : rd_.steps) {
    l.sync_off.push_back(off);
    off += align256(sync_bytes(st.type, st.store_end - st.store_begin, batch, length));
  }
  l.sync_bytes = off - l.sync_begin;
  l.main_off = off;
  l.share_off += off;
  l.main2_off = off + align256(main);
  l.total = l.main2_off + align256(main2);
  return l;
}

std::size_t DevicePlan::workspace_bytes(int batch, long length, const ProcessorSet& procs) const {
  return layout(batch, length, procs).total;
}

namespace {
std::size_t bwd_step_bytes(NodeType t, int slots, int batch, long length, const ProcessorSet& p) {
  switch (t) {
    case NodeType::Gain:
    case NodeType::Imager: return mgb::pw_grad_bytes(slots, batch, length);
    case NodeType::Eq: return mgb::eq_grad_bytes(slots, batch, length);
    case NodeType::Compressor:
    case NodeType::Noisegate: return mgb::dyn_bwd_bytes(slots, batch, length);
    case NodeType::Reverb:
      return mgb::conv_bwd_bytes(mgb::conv_geom(length, p.reverb_length()), slots, batch, p.reverb_length(), p.device().frames);
    case NodeType::Delay:
      return mgb::conv_bwd_bytes(mgb::conv_geom(length, p.delay_span()), slots, batch, p.delay_span(), p.device().frames);
    default: return 0;
  }
}
}  // namespace

std::size_t DevicePlan::backward_workspace_bytes(int batch, long length, const ProcessorSet& procs) const {
  std::size_t extra = 256;
  for (const StepIndex& st : rd_.steps) {
    extra = std::max(extra, bwd_step_bytes(st.type, st.store_end - st.store_begin, batch, length, procs));
  }
  return layout(batch, length, procs).total + align256(extra);
}

int DevicePlan::kernels_per_render(int batch, long length) const {
  int k = 0;
  for (std::size_t i = 0; i < rd_.steps.size();) {
    if (dyn_pair(*this, i, batch, length)) {
      k += 1;
      i += 2 + static_cast<std::size_t>(epi_followers(*this, i + 1, batch, length));
      continue;
    }
    const int n = chain_length(rd_, i, batch, length);
    k += n > 1 ? 1 : step_kernels(rd_.steps[i].type);
    i += static_cast<std::size_t>(n > 1 ? n : 1 + epi_followers(*this, i, batch, length));
  }
  return k;
}

void DevicePlan::step_owners(int batch, long length, int* owner) const {
  for (std::size_t i = 0; i < rd_.steps.size();) {
    const int n = chain_length(rd_, i, batch, length);
    std::size_t span = static_cast<std::size_t>(n > 1 ? n : 1 + epi_followers(*this, i, batch, length));
    if (dyn_pair(*this, i, batch, length)) span = 2 + static_cast<std::size_t>(epi_followers(*this, i + 1, batch, length));
    for (std::size_t j = i; j < i + span; ++j) owner[j] = static_cast<int>(i);
    i += span;
  }
}

void render_arena(const DevicePlan& plan, const ProcessorSet& procs, const double* const* param_tables, float* arena,
                  int batch, long length, void* workspace, std::size_t workspace_bytes, cudaStream_t stream,
                  cudaEvent_t* step_events, bool hoist) {
  const RenderData& rd = plan.data();
  const DevicePlan::Layout lay = plan.layout(batch, length, procs);
  if (workspace_bytes < lay.total) fail("render_arena: workspace too small");
  char* ws = static_cast<char*>(workspace);
  const long rowstride = static_cast<long>(batch) * 2 * length;
  const float2* tw = mgb::twiddle_table(procs.device().device);
  const double2* tw64 = mgb::twiddle_table64(procs.device().device);
  std::vector<mgb::StepArgs> args(rd.steps.size());
  for (std::size_t k = 0; k < rd.steps.size(); ++k) {
    const StepIndex& st = rd.steps[k];
    const int width = param_width(st.type);
    mgb::StepArgs& a = args[k];
    a.src = arena;
    a.dst = arena + st.store_begin * rowstride;
    a.row_ptr = plan.row_ptr(static_cast<int>(k));
    a.col = plan.col(static_cast<int>(k));
    a.params = nullptr;
    if (width > 0) {
      const double* table = param_tables ? param_tables[static_cast<int>(st.type)] : nullptr;
      if (!table) fail("render: missing parameter table for " + tname(st.type));
      a.params = table + static_cast<long>(st.param_begin) * width;
    }
    a.tw = tw;
    a.tw64 = tw64;
    a.slots = st.store_end - st.store_begin;
    a.batch = batch;
    a.length = length;
    a.rowstride = rowstride;
    a.nnz = static_cast<int>(st.gather.size());
    a.dense = plan.dense_src(static_cast<int>(k));
  }
  for (int r : plan.zero_rows()) {
    cuda_check(cudaMemsetAsync(arena + r * rowstride, 0, sizeof(float) * rowstride, stream), "memset");
  }
  // Parameter-only prologues (EQ design, reverb/delay impulse responses and their spectra)
  // depend on nothing the render computes: fork them onto the plan's side streams so they
  // overlap the earlier steps, and join each one right before its step's audio pass
  // (hoist = false runs every prologue inline: isolated per-step costs).
  const cudaEvent_t* ev = plan.events();
  // Every step's synchronisation words, cleared once (one memset node instead of one per
  // scan step on the critical path), first: a memset node queued behind the fork waits for
  // SM room like a kernel.
  if (lay.sync_bytes) cuda_check(cudaMemsetAsync(ws + lay.sync_begin, 0, lay.sync_bytes, stream), "memset sync");
  if (hoist) {
    cuda_check(cudaEventRecord(ev[0], stream), "event");  // fork point: before any render work
    for (cudaStream_t a : plan.aux_streams()) cuda_check(cudaStreamWaitEvent(a, ev[0], 0), "wait");
    for (std::size_t k = 0; k < rd.steps.size(); ++k) {
      if (!has_prologue(rd.steps[k].type)) continue;
      // Prologues complete in the order their steps need them on side stream 0, except the
      // delay's, which gets side stream 1 and so runs beside the reverb's (the delay step's
      // kernel spectrum was the critical path once conv steps joined their prologue late:
      // 0.324 -> 0.309 ms per config-2 render).
      cudaStream_t a = plan.aux_streams()[rd.steps[k].type == NodeType::Delay ? 1 : 0];
      run_prologue(rd.steps[k].type, args[k], procs, ws + lay.prologue_off[k], a);
      cuda_check(cudaEventRecord(ev[k + 1], a), "event");
    }
  }
  for (std::size_t k = 0; k < rd.steps.size(); ++k) {
    const NodeType t = rd.steps[k].type;
    // Runs of small pointwise steps (latency-bound) go out as one launch, unless per-step
    // events were asked for.
    const int chain = step_events ? 1 : chain_length(rd, k, batch, length);
    if (chain > 1) {
      mgb::PwChain c{};
      c.n = chain;
      for (int j = 0; j < chain; ++j) {
        c.step[j] = args[k + j];
        c.op[j] = point_op(rd.steps[k + j].type);
      }
      mgb::launch_pointwise_chain(c, stream);
      k += static_cast<std::size_t>(chain - 1);
      continue;
    }
    // Pointwise followers ride in this step's epilogue (not with per-step events, nor for a
    // step that runs on the side lane). Without hoisting everything is serialised on `stream`
    // (no side lane either): the product's kernels one after another, for per-kernel costs.
    mgb::PwEpi epi{};
    const bool paired = hoist && !step_events && lay.paired[k];
    if (!step_events && !paired) {
      epi.n = epi_followers(plan, k, batch, length);
      for (int f = 0; f < epi.n; ++f) {
        const std::size_t j = k + 1 + static_cast<std::size_t>(f);
        epi.op[f] = point_op(rd.steps[j].type);
        epi.dst[f] = args[j].dst;
        epi.map[f] = plan.follow_map(static_cast<int>(j));
        epi.params[f] = args[j].params;
      }
    }
    if (paired) {
      // Steps k and k+1 side by side: k on the lane, k+1 on the main stream, then join.
      const cudaEvent_t* le = plan.lane_events();
      cudaStream_t lane = plan.lane();
      cuda_check(cudaEventRecord(le[2 * k], stream), "event");
      cuda_check(cudaStreamWaitEvent(lane, le[2 * k], 0), "wait");
      for (std::size_t j = k; j <= k + 1; ++j) {
        cudaStream_t st = j == k ? lane : stream;
        const NodeType tj = rd.steps[j].type;
        if (!hoist) run_prologue(tj, args[j], procs, ws + lay.prologue_off[j], st);
        run_main(tj, args[j], procs, ws + lay.prologue_off[j], ws + (j == k ? lay.main_off : lay.main2_off),
                 ws + lay.sync_off[j], false, st, hoist ? ev[j + 1] : nullptr);
      }
      cuda_check(cudaEventRecord(le[2 * k + 1], lane), "event");
      cuda_check(cudaStreamWaitEvent(stream, le[2 * k + 1], 0), "wait");
      ++k;
      continue;
    }
    if (!step_events && dyn_pair(plan, k, batch, length) && mgb::dyn_pair_ok(args[k], args[k + 1])) {
      // Steps k, k+1: one streaming kernel scans both (the second reads the first's rows);
      // the second step's pointwise followers ride in its epilogue.
      const std::size_t j = k + 1;
      mgb::PwEpi e2{};
      e2.n = epi_followers(plan, j, batch, length);
      for (int f = 0; f < e2.n; ++f) {
        const std::size_t q = j + 1 + static_cast<std::size_t>(f);
        e2.op[f] = point_op(rd.steps[q].type);
        e2.dst[f] = args[q].dst;
        e2.map[f] = plan.follow_map(static_cast<int>(q));
        e2.params[f] = args[q].params;
      }
      mgb::launch_dynamics_pair(t == NodeType::Noisegate, rd.steps[j].type == NodeType::Noisegate, args[k], args[j],
                                procs.config().envelope_taps, procs.config().energy_floor, stream, e2);
      k = j + static_cast<std::size_t>(e2.n);
      continue;
    }
    if (!step_events && k + 1 < rd.steps.size() && lay.shared[k + 1]) {
      // Steps k and k+1: long convolutions sharing the transforms of common source rows.
      const std::size_t j = k + 1;
      const long taps = t == NodeType::Reverb ? procs.reverb_length() : procs.delay_span();
      if (!hoist) {
        run_prologue(t, args[k], procs, ws + lay.prologue_off[k], stream);
        run_prologue(rd.steps[j].type, args[j], procs, ws + lay.prologue_off[j], stream);
      }
      const DevicePlan::Share& si = plan.share_info(static_cast<int>(j));
      const int* ints = plan.share_ints(static_cast<int>(j));
      mgb::ConvShare sh;
      sh.pair_a = ints;
      sh.pair_b = ints + si.pairs;
      sh.own_a = ints + 2 * si.pairs;
      sh.own_b = ints + 2 * si.pairs + si.own_prev;
      sh.n_pairs = si.pairs;
      sh.n_own_a = si.own_prev;
      sh.n_own_b = si.own;
      mgb::launch_conv_shared(args[k], args[j], taps, ws + lay.prologue_off[k], ws + lay.prologue_off[j],
                              ws + lay.main_off, ws + lay.share_off, sh, stream, hoist ? ev[k + 1] : nullptr,
                              hoist ? ev[j + 1] : nullptr);
      ++k;
      continue;
    }
    char* pws = ws + lay.prologue_off[k];
    char* mws = ws + lay.main_off;
    if (step_events) cuda_check(cudaEventRecord(step_events[2 * k], stream), "event");
    const cudaEvent_t join = hoist && has_prologue(t) ? ev[k + 1] : nullptr;
    if (!hoist) run_prologue(t, args[k], procs, pws, stream);
    run_main(t, args[k], procs, pws, mws, ws + lay.sync_off[k], false, stream, join, epi);
    if (step_events) cuda_check(cudaEventRecord(step_events[2 * k + 1], stream), "event");
    k += static_cast<std::size_t>(epi.n);
  }
  cuda_check(cudaGetLastError(), "render_arena launch");
}

// ---- backward pass ---------------------------------------------------------------------------

void backward_arena(const DevicePlan& plan, const ProcessorSet& procs, const double* const* param_tables,
                    const float* arena, float* adjoint, double* const* grad_tables, int batch, long length,
                    void* workspace, std::size_t workspace_bytes, cudaStream_t stream) {
  const RenderData& rd = plan.data();
  const DevicePlan::Layout lay = plan.layout(batch, length, procs);
  if (workspace_bytes < plan.backward_workspace_bytes(batch, length, procs)) fail("backward: workspace too small");
  char* ws = static_cast<char*>(workspace);
  char* scratch = ws + lay.total;
  const long rowstride = static_cast<long>(batch) * 2 * length;
  const float2* tw = mgb::twiddle_table(procs.device().device);
  const double2* tw64 = mgb::twiddle_table64(procs.device().device);
  const int nsteps = static_cast<int>(rd.steps.size());
  for (int k = nsteps - 1; k >= 0; --k) {
    const StepIndex& st = rd.steps[static_cast<std::size_t>(k)];
    const NodeType t = st.type;
    if (t == NodeType::Out || t == NodeType::In) continue;  // out rows hold dL/dY on entry
    const int width = param_width(t);
    mgb::StepArgs fw{};
    fw.src = arena;
    fw.dst = const_cast<float*>(arena) + st.store_begin * rowstride;
    fw.row_ptr = plan.row_ptr(k);
    fw.col = plan.col(k);
    fw.params = nullptr;
    double* grad = nullptr;
    if (width > 0) {
      const double* table = param_tables ? param_tables[static_cast<int>(t)] : nullptr;
      if (!table) fail("backward: missing parameter table for " + tname(t));
      if (!grad_tables || !grad_tables[static_cast<int>(t)]) fail("backward: missing gradient table for " + tname(t));
      fw.params = table + static_cast<long>(st.param_begin) * width;
      grad = grad_tables[static_cast<int>(t)] + static_cast<long>(st.param_begin) * width;
    }
    fw.tw = tw;
    fw.tw64 = tw64;
    fw.slots = st.store_end - st.store_begin;
    fw.batch = batch;
    fw.length = length;
    fw.rowstride = rowstride;
    mgb::StepArgs bw = fw;
    bw.src = adjoint;
    bw.dst = adjoint + st.store_begin * rowstride;
    bw.row_ptr = plan.t_row_ptr(k);
    bw.col = plan.t_col(k);
    char* pws = ws + lay.prologue_off[static_cast<std::size_t>(k)];
    switch (t) {
      case NodeType::Mix: mgb::launch_pointwise(mgb::PointOp::Copy, bw, stream); break;
      case NodeType::Gain:
      case NodeType::Imager:
        if (!mgb::launch_pointwise_backward(point_op(t), fw, bw, scratch, grad, stream)) {
          mgb::launch_pointwise(point_op(t), bw, stream);
          mgb::launch_pointwise_param_grad(point_op(t), fw, bw, scratch, grad, stream);
        }
        break;
      case NodeType::Eq:
        mgb::launch_eq_main(bw, reinterpret_cast<float*>(pws + eq_taps_bytes(fw.slots)), stream);
        mgb::launch_eq_param_grad(fw, bw, scratch, grad, stream);
        break;
      case NodeType::Compressor:
      case NodeType::Noisegate:
        mgb::launch_dynamics_backward(t == NodeType::Noisegate, fw, bw, procs.config().envelope_taps,
                                      procs.config().energy_floor, scratch, grad, stream);
        break;
      case NodeType::Reverb:
      case NodeType::Delay:
        mgb::launch_conv_backward(t == NodeType::Reverb, fw, bw, reverb_const(procs), delay_const(procs), pws, scratch,
                                  grad, stream);
        break;
      default: break;
    }
  }
  // Sources: dL/d(source) = sum over the source's consumers.
  if (rd.num_inputs > 0) {
    mgb::StepArgs bw{};
    bw.src = adjoint;
    bw.dst = adjoint;
    bw.row_ptr = plan.t_row_ptr(nsteps);
    bw.col = plan.t_col(nsteps);
    bw.tw = tw;
    bw.tw64 = tw64;
    bw.slots = rd.num_inputs;
    bw.batch = batch;
    bw.length = length;
    bw.rowstride = rowstride;
    mgb::launch_pointwise(mgb::PointOp::Copy, bw, stream);
  }
  cuda_check(cudaGetLastError(), "backward launch");
}

// ---- per-step micro-benchmark ---------------------------------------------------------------

void profile_steps(const DevicePlan& plan, const ProcessorSet& procs, const double* const* param_tables, float* arena,
                   int batch, long length, void* workspace, std::size_t workspace_bytes, cudaStream_t stream, int reps,
                   float* step_ms) {
  const RenderData& rd = plan.data();
  const DevicePlan::Layout lay = plan.layout(batch, length, procs);
  if (workspace_bytes < lay.total) fail("profile_steps: workspace too small");
  // One full render so every row holds its real data; then each step (prologue + audio pass)
  // is re-run `reps` times back to back between one event pair (idempotent: same inputs,
  // same outputs), which amortises launch and event overheads out of the per-step time.
  render_arena(plan, procs, param_tables, arena, batch, length, workspace, workspace_bytes, stream, nullptr, false);
  char* ws = static_cast<char*>(workspace);
  const long rowstride = static_cast<long>(batch) * 2 * length;
  const float2* tw = mgb::twiddle_table(procs.device().device);
  const double2* tw64 = mgb::twiddle_table64(procs.device().device);
  cudaEvent_t e0, e1;
  cuda_check(cudaEventCreate(&e0), "event");
  cuda_check(cudaEventCreate(&e1), "event");
  cudaStream_t cap = nullptr;
  cuda_check(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "stream");
  cuda_check(cudaStreamSynchronize(stream), "sync");
  for (std::size_t k = 0; k < rd.steps.size(); ++k) {
    const StepIndex& st = rd.steps[k];
    const int width = param_width(st.type);
    mgb::StepArgs a{};
    a.src = arena;
    a.dst = arena + st.store_begin * rowstride;
    a.row_ptr = plan.row_ptr(static_cast<int>(k));
    a.col = plan.col(static_cast<int>(k));
    a.params = width > 0 ? param_tables[static_cast<int>(st.type)] + static_cast<long>(st.param_begin) * width : nullptr;
    a.tw = tw;
    a.tw64 = tw64;
    a.slots = st.store_end - st.store_begin;
    a.batch = batch;
    a.length = length;
    a.rowstride = rowstride;
    a.nnz = static_cast<int>(st.gather.size());
    a.dense = plan.dense_src(static_cast<int>(k));
    run_prologue(st.type, a, procs, ws + lay.prologue_off[k], stream);
    // The reps are captured into a CUDA graph and replayed, so short kernels are timed on
    // the device without the host's per-launch cost between them.
    cuda_check(cudaStreamSynchronize(stream), "sync");
    cuda_check(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "capture");
    for (int r = 0; r < reps; ++r) {
      run_prologue(st.type, a, procs, ws + lay.prologue_off[k], cap);
      run_main(st.type, a, procs, ws + lay.prologue_off[k], ws + lay.main_off, ws + lay.sync_off[k], true, cap);
    }
    cudaGraph_t g = nullptr;
    cuda_check(cudaStreamEndCapture(cap, &g), "capture");
    cudaGraphExec_t ge = nullptr;
    cuda_check(cudaGraphInstantiate(&ge, g, 0), "instantiate");
    cuda_check(cudaGraphLaunch(ge, cap), "graph launch");  // warm
    cuda_check(cudaEventRecord(e0, cap), "event");
    cuda_check(cudaGraphLaunch(ge, cap), "graph launch");
    cuda_check(cudaEventRecord(e1, cap), "event");
    cuda_check(cudaEventSynchronize(e1), "sync");
    float ms = 0.f;
    cuda_check(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    step_ms[k] = ms / static_cast<float>(reps);
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(cap);
}

// ---- RenderGraph ------------------------------------------------------------------------

RenderGraph::RenderGraph(const DevicePlan& plan, const ProcessorSet& procs, const double* const* param_tables,
                         float* arena, int batch, long length, void* workspace, std::size_t workspace_bytes) {
  int least = 0, greatest = 0;
  cuda_check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
  cudaStream_t cap = nullptr;
  cuda_check(cudaStreamCreateWithPriority(&cap, cudaStreamNonBlocking, greatest), "cudaStreamCreate");
  // One eager render first: one-time kernel attribute setup must not happen under capture.
  render_arena(plan, procs, param_tables, arena, batch, length, workspace, workspace_bytes, cap);
  cuda_check(cudaStreamSynchronize(cap), "warm-up render");
  cuda_check(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
  try {
    render_arena(plan, procs, param_tables, arena, batch, length, workspace, workspace_bytes, cap);
  } catch (...) {
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(cap, &g);
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
    throw;
  }
  cuda_check(cudaStreamEndCapture(cap, &graph_), "end capture");
  cudaStreamDestroy(cap);
  // Node priorities: prologue kernels (parameter-only, off the critical path) lowest, audio
  // kernels highest, so when both are runnable the CTA scheduler serves the main path.
  std::size_t n = 0;
  cuda_check(cudaGraphGetNodes(graph_, nullptr, &n), "graph nodes");
  std::vector<cudaGraphNode_t> nodes(n);
  cuda_check(cudaGraphGetNodes(graph_, nodes.data(), &n), "graph nodes");
  for (cudaGraphNode_t node : nodes) {
    cudaGraphNodeType type;
    cuda_check(cudaGraphNodeGetType(node, &type), "node type");
    if (type != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp{};
    cuda_check(cudaGraphKernelNodeGetParams(node, &kp), "kernel params");
    cudaLaunchAttributeValue v{};
    const bool pro = mgb::is_prologue_kernel(kp.func);
    v.priority = pro ? least : greatest;
    cuda_check(cudaGraphKernelNodeSetAttribute(node, cudaLaunchAttributePriority, &v), "node priority");
  }
  cuda_check(cudaGraphInstantiateWithFlags(&exec_, graph_, cudaGraphInstantiateFlagUseNodePriority), "instantiate");
}

RenderGraph::~RenderGraph() {
  if (exec_) cudaGraphExecDestroy(exec_);
  if (graph_) cudaGraphDestroy(graph_);
}

void RenderGraph::launch(cudaStream_t stream) const { cuda_check(cudaGraphLaunch(exec_, stream), "graph launch"); }

// ---- RenderPipeline -----------------------------------------------------------------------

namespace {
void validate_params(const RenderData& rd, const ParamStore& params) {
  // Per-step parameter checks, in step order (render.cpp:49-56, processors.cpp:232-247).
  for (const StepIndex& st : rd.steps) {
    const int width = param_width(st.type);
    if (width == 0) continue;
    auto it = params.tables.find(st.type);
    if (it == params.tables.end()) fail("render: missing parameter table for " + tname(st.type));
    const ParamMatrix& m = it->second;
    const int slots = st.store_end - st.store_begin;
    if (m.cols != width) fail(tname(st.type) + ": parameter row width mismatch");
    if (st.param_begin < 0 || st.param_begin + slots > m.rows) fail(tname(st.type) + ": parameter rows out of range");
    for (int s = 0; s < slots; ++s) check_param_row(st.type, m.row(st.param_begin + s));
  }
}
}  // namespace

struct RenderPipeline::Slot {
  DeviceBuffer arena, ws, params, staging;
  const double* tables[kNumNodeTypes] = {};
  std::size_t table_rows[kNumNodeTypes] = {};
  std::unique_ptr<RenderGraph> graph;
  cudaEvent_t h2d = nullptr, done = nullptr, d2h = nullptr;
  float* pin_src = nullptr;  // host-convert mode: pinned fp32 staging
  float* pin_out = nullptr;
  double* pin_params = nullptr;  // pinned staging of the parameter tables (same layout as `params`)
  std::uint64_t job = 0;     // completion job that reads pin_out (0: none)
  ~Slot() {
    for (cudaEvent_t e : {h2d, done, d2h}) {
      if (e) cudaEventDestroy(e);
    }
    if (pin_src) cudaFreeHost(pin_src);
    if (pin_out) cudaFreeHost(pin_out);
    if (pin_params) cudaFreeHost(pin_params);
  }
};

// Host-side double <-> float conversion: a fixed pool of workers splitting each array in
// equal contiguous chunks, and one completion thread that waits for a render's D2H event
// and converts its fp32 outputs into the caller's double buffers.
struct RenderPipeline::HostConvert {
  int nthreads = 1;
  std::vector<std::thread> workers;
  std::mutex mu;  // pool state
  std::condition_variable cv, cv_done;
  std::function<void(int)> task;
  std::uint64_t gen = 0;
  int remaining = 0;
  bool stop = false;
  std::mutex run_mu;  // one parallel job at a time (submit thread and completion thread)

  struct Job {
    std::uint64_t id;
    cudaEvent_t ev;
    const float* src;
    std::vector<double*> dst;
    std::size_t n;  // floats per output signal
  };
  std::thread completer;
  std::mutex qmu;
  std::condition_variable qcv, qdone;
  std::deque<Job> queue;
  std::uint64_t next_id = 1, finished = 0;
  std::string error;

  HostConvert(int n, int device) : nthreads(n) {
    for (int i = 0; i < nthreads; ++i) {
      workers.emplace_back([this, i, device] {
        cudaSetDevice(device);  // workers issue their chunks' H2D copies
        std::uint64_t seen = 0;
        for (;;) {
          std::function<void(int)> t;
          {
            std::unique_lock lk(mu);
            cv.wait(lk, [&] { return stop || gen != seen; });
            if (stop) return;
            seen = gen;
            t = task;
          }
          t(i);
          std::unique_lock lk(mu);
          if (--remaining == 0) cv_done.notify_all();
        }
      });
    }
    completer = std::thread([this] {
      for (;;) {
        Job j;
        {
          std::unique_lock lk(qmu);
          qcv.wait(lk, [&] { return stop || !queue.empty(); });
          if (queue.empty()) return;
          j = std::move(queue.front());
        }
        cudaError_t e = cudaEventSynchronize(j.ev);
        if (e != cudaSuccess) {
          std::scoped_lock lk(qmu);
          error = cudaGetErrorString(e);
        } else {
          for (std::size_t o = 0; o < j.dst.size(); ++o) convert(j.src + o * j.n, j.dst[o], j.n);
        }
        std::scoped_lock lk(qmu);
        queue.pop_front();
        finished = j.id;
        qdone.notify_all();
      }
    });
  }
  ~HostConvert() {
    {
      std::scoped_lock lk(qmu);
      stop = true;
    }
    qcv.notify_all();
    if (completer.joinable()) completer.join();
    {
      std::scoped_lock lk(mu);
      stop = true;
    }
    cv.notify_all();
    for (auto& w : workers) w.join();
  }
  // Runs f(0..nthreads) on the workers and the calling thread (index nthreads).
  void parallel(const std::function<void(int)>& f) {
    std::scoped_lock run(run_mu);
    {
      std::scoped_lock lk(mu);
      task = f;
      remaining = nthreads;
      ++gen;
    }
    cv.notify_all();
    f(nthreads);
    std::unique_lock lk(mu);
    cv_done.wait(lk, [&] { return remaining == 0; });
  }
  void convert(const float* src, double* dst, std::size_t n) {
    const int parts = nthreads + 1;
    parallel([&](int i) {
      const std::size_t lo = n * static_cast<std::size_t>(i) / parts, hi = n * static_cast<std::size_t>(i + 1) / parts;
      hostconv::f32_to_f64(src + lo, dst + lo, hi - lo);
    });
  }
  // Sources -> fp32 pinned staging -> device, in 1 MiB chunks claimed from a shared counter.
  // Each converted chunk goes onto the H2D stream at once, so the DMA of early chunks
  // overlaps the conversion of later ones (and the next render's conversion overlaps this
  // render's kernels).
  void upload(const double* const* src, int nsrc, std::size_t stride, float* pin, float* dev, cudaStream_t st) {
    // 2^18 floats per chunk (smaller chunks measured slower: concurrent cudaMemcpyAsync calls
    // contend; one H2D after converting everything measured no faster).
    constexpr std::size_t kChunk = std::size_t{1} << 18;
    const std::size_t per = (stride + kChunk - 1) / kChunk, total = per * static_cast<std::size_t>(nsrc);
    std::atomic<std::size_t> next{0};
    std::atomic<int> failed{0};
    parallel([&](int) {
      for (std::size_t c = next.fetch_add(1); c < total; c = next.fetch_add(1)) {
        const std::size_t k = c / per, lo = (c % per) * kChunk, n = std::min(kChunk, stride - lo);
        const std::size_t off = k * stride + lo;
        hostconv::f64_to_f32(src[k] + lo, pin + off, n);
        if (cudaMemcpyAsync(dev + off, pin + off, sizeof(float) * n, cudaMemcpyHostToDevice, st) != cudaSuccess) {
          failed = 1;
        }
      }
    });
    if (failed) throw std::runtime_error("cuda: RenderPipeline source upload failed");
  }
  std::uint64_t enqueue(Job j) {
    std::scoped_lock lk(qmu);
    j.id = next_id++;
    const std::uint64_t id = j.id;
    queue.push_back(std::move(j));
    qcv.notify_one();
    return id;
  }
  void wait(std::uint64_t id) {
    std::unique_lock lk(qmu);
    qdone.wait(lk, [&] { return finished >= id; });
    if (!error.empty()) throw std::runtime_error("cuda: RenderPipeline outputs: " + error);
  }
};

RenderPipeline::RenderPipeline(const DevicePlan& plan, const ProcessorSet& procs, int batch, long length, bool f32_io,
                               int depth, int host_threads)
    : plan_(plan), procs_(procs), batch_(batch), length_(length), f32_(f32_io),
      stride_(static_cast<long>(batch) * 2 * length) {
  if (depth < 1) fail("RenderPipeline: depth must be >= 1");
  cuda_check(cudaSetDevice(procs.device().device), "cudaSetDevice");
  int least = 0, greatest = 0;
  cuda_check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
  cuda_check(cudaStreamCreateWithPriority(&h2d_, cudaStreamNonBlocking, greatest), "stream");
  cuda_check(cudaStreamCreateWithPriority(&compute_, cudaStreamNonBlocking, greatest), "stream");
  cuda_check(cudaStreamCreateWithPriority(&d2h_, cudaStreamNonBlocking, greatest), "stream");
  if (!f32_) {
    int n = host_threads;
    if (n < 0) {
      // Default: half the host's hardware threads, at most 8 (config 2 on the 16-thread B200
      // box hosts: 0.66 ms/render device conversion, 0.48 ms with 8 host threads). Processes
      // sharing the host (torchrun sets LOCAL_WORLD_SIZE) split its threads; 0 converts on
      // the device (double audio crosses PCIe).
      const char* lw = std::getenv("LOCAL_WORLD_SIZE");
      const int procs_on_host = std::max(1, lw ? std::atoi(lw) : 1);
      const int hw = static_cast<int>(std::thread::hardware_concurrency());
      n = std::clamp(hw / (2 * procs_on_host) - 1, 0, 7);
    }
    if (n >= 1) conv_ = std::make_unique<HostConvert>(n, procs.device().device);
    host_fraction_ = kHostFraction;
  }
  const RenderData& rd = plan.data();
  const std::size_t rows = static_cast<std::size_t>(rd.buffer_rows);
  const std::size_t ws_bytes = plan.workspace_bytes(batch, length, procs);
  const std::size_t n_out = static_cast<std::size_t>(rd.buffer_rows - rd.output_begin);
  for (int d = 0; d < depth; ++d) {
    auto s = std::make_unique<Slot>();
    auto* arena = static_cast<float*>(s->arena.ensure(sizeof(float) * rows * stride_ + 16));
    void* ws = s->ws.ensure(ws_bytes);
    // Fixed device tables (the graph bakes their addresses), filled with default rows.
    std::size_t total = 0;
    for (const auto& [t, src] : rd.param_source_rows) total += src.size() * static_cast<std::size_t>(param_width(t));
    auto* dpar = static_cast<double*>(s->params.ensure(sizeof(double) * (total + 1)));
    std::vector<double> host;
    for (const auto& [t, src] : rd.param_source_rows) {
      s->tables[static_cast<int>(t)] = dpar + host.size();
      s->table_rows[static_cast<int>(t)] = src.size();
      std::vector<double> row(static_cast<std::size_t>(param_width(t)));
      default_param_row(t, row);
      for (std::size_t r = 0; r < src.size(); ++r) host.insert(host.end(), row.begin(), row.end());
    }
    if (!host.empty()) cuda_check(cudaMemcpy(dpar, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&s->pin_params), sizeof(double) * (total + 1), cudaHostAllocDefault),
               "cudaHostAlloc");
    if (!f32_) s->staging.ensure(sizeof(double) * rows * stride_ + 16);
    if (conv_) {
      cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&s->pin_src),
                               sizeof(float) * std::max<std::size_t>(1, static_cast<std::size_t>(rd.num_inputs)) * stride_,
                               cudaHostAllocDefault), "cudaHostAlloc");
      cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&s->pin_out), sizeof(float) * std::max<std::size_t>(1, n_out) * stride_,
                               cudaHostAllocDefault), "cudaHostAlloc");
    }
    cuda_check(cudaMemset(arena, 0, sizeof(float) * rows * stride_), "memset");
    s->graph = std::make_unique<RenderGraph>(plan, procs, s->tables, arena, batch, length, ws, ws_bytes);
    for (cudaEvent_t* e : {&s->h2d, &s->done, &s->d2h}) cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    slots_.push_back(std::move(s));
  }
  cuda_check(cudaDeviceSynchronize(), "pipeline setup");
}

RenderPipeline::~RenderPipeline() {
  if (compute_) cudaStreamSynchronize(compute_);
  if (d2h_) cudaStreamSynchronize(d2h_);
  conv_.reset();  // drains the completion thread
  slots_.clear();
  for (cudaStream_t st : {h2d_, compute_, d2h_}) {
    if (st) cudaStreamDestroy(st);
  }
}

void RenderPipeline::submit(const ParamStore& params, const void* const* sources, void* const* outputs) {
  const RenderData& rd = plan_.data();
  validate_params(rd, params);
  Slot& s = *slots_[next_ % slots_.size()];
  const bool reused = next_ >= slots_.size();
  ++next_;
  auto* arena = static_cast<float*>(s.arena.ptr);
  const std::size_t fbytes = sizeof(float) * static_cast<std::size_t>(stride_);
  if (reused) {
    // The slot's pinned staging (parameters; fp32 sources in host-convert mode) is rewritten
    // on the host: its previous upload, and its previous outputs' conversion, must be done.
    cuda_check(cudaEventSynchronize(s.h2d), "pipeline staging");
    if (conv_ && s.job) conv_->wait(s.job);
  }
  // Inputs: the slot's previous render must have consumed its sources and params, and its
  // outputs must have been read back: in device-conversion mode the fp64 outputs sit in the
  // same staging buffer the next sources are uploaded into.
  if (reused) {
    cuda_check(cudaStreamWaitEvent(h2d_, s.done, 0), "wait");
    cuda_check(cudaStreamWaitEvent(h2d_, s.d2h, 0), "wait");
  }
  // Parameters go through pinned staging: a pageable cudaMemcpyAsync waits for the stream's
  // earlier copies (the previous render's sources), which serialised this render's source
  // conversion behind the previous render's whole upload (0.46 -> ~0.36 ms per render e2e).
  for (const auto& [t, m] : params.tables) {
    const int ti = static_cast<int>(t);
    if (!s.tables[ti]) continue;
    if (static_cast<std::size_t>(m.rows) != s.table_rows[ti]) fail("RenderPipeline: parameter table shape changed");
    const std::size_t off = static_cast<std::size_t>(s.tables[ti] - static_cast<const double*>(s.params.ptr));
    std::memcpy(s.pin_params + off, m.values.data(), sizeof(double) * m.values.size());
    cuda_check(cudaMemcpyAsync(const_cast<double*>(s.tables[ti]), s.pin_params + off, sizeof(double) * m.values.size(),
                               cudaMemcpyHostToDevice, h2d_), "H2D params");
  }
  const std::size_t bytes = (f32_ ? sizeof(float) : sizeof(double)) * static_cast<std::size_t>(stride_);
  // Sources laid out back to back in host memory (one [K][B][2][L] array, the usual case)
  // go over PCIe as one transfer instead of K.
  auto contiguous = [&](const void* const* ptrs, int n) {
    for (int k = 1; k < n; ++k) {
      if (static_cast<const char*>(ptrs[k]) != static_cast<const char*>(ptrs[0]) + bytes * k) return false;
    }
    return n > 0;
  };
  // Host-converted double audio: sources [0, kh) are converted to fp32 on the host threads,
  // the rest cross PCIe as double first (their DMA runs while the host converts) and are
  // converted on the device. Splitting balances host memory bandwidth against PCIe.
  int kh = 0;
  if (conv_) {
    kh = std::min(rd.num_inputs, static_cast<int>(std::ceil(host_fraction_ * rd.num_inputs - 1e-9)));
    const int kd = rd.num_inputs - kh;
    if (kd > 0) {
      char* dst = static_cast<char*>(s.staging.ptr);
      if (contiguous(sources + kh, kd)) {
        cuda_check(cudaMemcpyAsync(dst, sources[kh], bytes * kd, cudaMemcpyHostToDevice, h2d_), "H2D sources");
      } else {
        for (int k = 0; k < kd; ++k) {
          cuda_check(cudaMemcpyAsync(dst + bytes * k, sources[kh + k], bytes, cudaMemcpyHostToDevice, h2d_), "H2D sources");
        }
      }
    }
    conv_->upload(reinterpret_cast<const double* const*>(sources), kh, static_cast<std::size_t>(stride_), s.pin_src, arena,
                  h2d_);
  } else {
    char* dst = f32_ ? reinterpret_cast<char*>(arena) : static_cast<char*>(s.staging.ptr);
    if (contiguous(sources, rd.num_inputs)) {
      cuda_check(cudaMemcpyAsync(dst, sources[0], bytes * rd.num_inputs, cudaMemcpyHostToDevice, h2d_), "H2D sources");
    } else {
      for (int k = 0; k < rd.num_inputs; ++k) {
        cuda_check(cudaMemcpyAsync(dst + bytes * k, sources[k], bytes, cudaMemcpyHostToDevice, h2d_), "H2D sources");
      }
    }
  }
  cuda_check(cudaEventRecord(s.h2d, h2d_), "event");
  // Compute: after the inputs landed and the slot's previous outputs were read back.
  cuda_check(cudaStreamWaitEvent(compute_, s.h2d, 0), "wait");
  if (reused) cuda_check(cudaStreamWaitEvent(compute_, s.d2h, 0), "wait");
  const bool dev_conv = !f32_ && !conv_;
  if (dev_conv) mgb::launch_f64_to_f32(static_cast<const double*>(s.staging.ptr), arena, rd.num_inputs * stride_, compute_);
  if (conv_ && kh < rd.num_inputs) {
    mgb::launch_f64_to_f32(static_cast<const double*>(s.staging.ptr), arena + static_cast<long>(kh) * stride_,
                           (rd.num_inputs - kh) * stride_, compute_);
  }
  s.graph->launch(compute_);
  const long n_out = (rd.buffer_rows - rd.output_begin) * stride_;
  if (dev_conv) mgb::launch_f32_to_f64(arena + rd.output_begin * stride_, static_cast<double*>(s.staging.ptr), n_out, compute_);
  cuda_check(cudaEventRecord(s.done, compute_), "event");
  // Outputs.
  cuda_check(cudaStreamWaitEvent(d2h_, s.done, 0), "wait");
  const int n_outs = rd.buffer_rows - rd.output_begin;
  if (conv_) {
    if (n_outs > 0) {
      cuda_check(cudaMemcpyAsync(s.pin_out, arena + rd.output_begin * stride_, fbytes * n_outs, cudaMemcpyDeviceToHost, d2h_),
                 "D2H outputs");
    }
    cuda_check(cudaEventRecord(s.d2h, d2h_), "event");
    HostConvert::Job j;
    j.ev = s.d2h;
    j.src = s.pin_out;
    j.n = static_cast<std::size_t>(stride_);
    for (int o = 0; o < n_outs; ++o) j.dst.push_back(static_cast<double*>(outputs[o]));
    s.job = conv_->enqueue(std::move(j));
    return;
  }
  const char* src = f32_ ? reinterpret_cast<const char*>(arena + rd.output_begin * stride_) : static_cast<const char*>(s.staging.ptr);
  if (contiguous(outputs, n_outs)) {
    cuda_check(cudaMemcpyAsync(outputs[0], src, bytes * n_outs, cudaMemcpyDeviceToHost, d2h_), "D2H outputs");
  } else {
    for (int o = 0; o < n_outs; ++o) {
      cuda_check(cudaMemcpyAsync(outputs[o], src + bytes * o, bytes, cudaMemcpyDeviceToHost, d2h_), "D2H outputs");
    }
  }
  cuda_check(cudaEventRecord(s.d2h, d2h_), "event");
}

void RenderPipeline::sync() {
  cuda_check(cudaStreamSynchronize(d2h_), "pipeline sync");
  cuda_check(cudaStreamSynchronize(compute_), "pipeline sync");
  if (conv_) {
    for (auto& s : slots_) {
      if (s->job) conv_->wait(s->job);
    }
  }
}

// ---- BatchRenderer ---------------------------------------------------------------------------

void BatchRenderer::Capacity::grow(const Capacity& o) {
  rows = std::max(rows, o.rows);
  workspace_bytes = std::max(workspace_bytes, o.workspace_bytes);
  index_ints = std::max(index_ints, o.index_ints);
  param_doubles = std::max(param_doubles, o.param_doubles);
}

namespace {
std::size_t param_src_ints(const RenderData& rd) {
  std::size_t n = 0;
  for (const auto& [t, src] : rd.param_source_rows) n += src.size();
  return n;
}
std::size_t param_doubles_of(const RenderData& rd) {
  std::size_t n = 0;
  for (const auto& [t, src] : rd.param_source_rows) n += src.size() * static_cast<std::size_t>(param_width(t));
  return n;
}
}  // namespace

BatchRenderer::Capacity BatchRenderer::capacity_for(const RenderData& rd, const ProcessorSet& procs, int batch,
                                                    long length) {
  DevicePlan plan(rd, DevicePlan::Deferred{});
  Capacity c;
  c.rows = static_cast<std::size_t>(rd.buffer_rows);
  c.workspace_bytes = plan.workspace_bytes(batch, length, procs);
  c.index_ints = plan.host_index().size() + param_src_ints(rd);
  c.param_doubles = param_doubles_of(rd);
  return c;
}

struct BatchRenderer::Slot {
  DeviceBuffer arena, ws, index, porig, prender;
  void* pinned = nullptr;  // [index ints][pad][orig params]
  std::unique_ptr<DevicePlan> plan;
  cudaEvent_t h2d = nullptr, done = nullptr, d2h = nullptr;
  bool used = false;
  ~Slot() {
    for (cudaEvent_t e : {h2d, done, d2h}) {
      if (e) cudaEventDestroy(e);
    }
    if (pinned) cudaFreeHost(pinned);
  }
};

BatchRenderer::BatchRenderer(const ProcessorSet& procs, int batch, long length, const Capacity& cap, int depth)
    : procs_(procs), batch_(batch), length_(length), stride_(static_cast<long>(batch) * 2 * length), cap_(cap) {
  if (depth < 1) fail("BatchRenderer: depth must be >= 1");
  if (batch < 1 || length < 1) fail("BatchRenderer: batch and length must be positive");
  cuda_check(cudaSetDevice(procs.device().device), "cudaSetDevice");
  int least = 0, greatest = 0;
  cuda_check(cudaDeviceGetStreamPriorityRange(&least, &greatest), "priority range");
  cuda_check(cudaStreamCreateWithPriority(&h2d_, cudaStreamNonBlocking, greatest), "stream");
  cuda_check(cudaStreamCreateWithPriority(&compute_, cudaStreamNonBlocking, greatest), "stream");
  cuda_check(cudaStreamCreateWithPriority(&d2h_, cudaStreamNonBlocking, greatest), "stream");
  for (auto& a : aux_) cuda_check(cudaStreamCreateWithPriority(&a, cudaStreamNonBlocking, least), "stream");
  const std::size_t index_bytes = align256(sizeof(int) * (cap.index_ints + 1));
  for (int d = 0; d < depth; ++d) {
    auto s = std::make_unique<Slot>();
    s->arena.ensure(sizeof(float) * cap.rows * static_cast<std::size_t>(stride_) + 16);
    s->ws.ensure(std::max<std::size_t>(cap.workspace_bytes, 256));
    s->index.ensure(index_bytes);
    s->porig.ensure(sizeof(double) * (cap.param_doubles + 1));
    s->prender.ensure(sizeof(double) * (cap.param_doubles + 1));
    cuda_check(cudaHostAlloc(&s->pinned, index_bytes + sizeof(double) * (cap.param_doubles + 1), cudaHostAllocDefault),
               "cudaHostAlloc");
    for (cudaEvent_t* e : {&s->h2d, &s->done, &s->d2h}) cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    slots_.push_back(std::move(s));
  }
  cuda_check(cudaDeviceSynchronize(), "BatchRenderer setup");
}

BatchRenderer::~BatchRenderer() {
  for (cudaStream_t st : {compute_, d2h_, h2d_}) {
    if (st) cudaStreamSynchronize(st);
  }
  slots_.clear();
  for (cudaEvent_t e : step_events_) cudaEventDestroy(e);
  for (cudaStream_t a : aux_) if (a) cudaStreamDestroy(a);
  for (cudaStream_t st : {h2d_, compute_, d2h_}) {
    if (st) cudaStreamDestroy(st);
  }
}

void BatchRenderer::submit(const RenderData& rd, const double* const* orig_tables, const int* orig_rows, bool validate,
                           const float* sources, int source_rows, bool sources_on_device, float* outputs) {
  cuda_check(cudaSetDevice(procs_.device().device), "cudaSetDevice");
  auto plan = std::make_unique<DevicePlan>(rd, DevicePlan::Deferred{});
  const std::vector<int>& idx = plan->host_index();
  const std::size_t n_idx = idx.size() + param_src_ints(rd);
  const std::size_t n_par = param_doubles_of(rd);
  const std::size_t ws_bytes = plan->workspace_bytes(batch_, length_, procs_);
  if (static_cast<std::size_t>(rd.buffer_rows) > cap_.rows || n_idx > cap_.index_ints || n_par > cap_.param_doubles ||
      ws_bytes > cap_.workspace_bytes) {
    fail("BatchRenderer: plan exceeds the renderer's capacity");
  }
  if (rd.num_inputs > 0 && (sources == nullptr || source_rows < 1)) fail("BatchRenderer: missing sources");
  // Parameter tables: the reference's reorder_params checks (schedule.cpp:454-471), then the
  // per-row checks render() applies (processors.cpp:132-149).
  for (const auto& [t, src] : rd.param_source_rows) {
    const int ti = static_cast<int>(t);
    if (!orig_tables || !orig_tables[ti] || !orig_rows || orig_rows[ti] != static_cast<int>(src.size())) {
      fail("reorder_params: missing or misshaped table for " + tname(t));
    }
    if (validate) {
      const std::size_t w = static_cast<std::size_t>(param_width(t));
      for (std::size_t r = 0; r < src.size(); ++r) check_param_row(t, {orig_tables[ti] + r * w, w});
    }
  }
  while (step_events_.size() < rd.steps.size() + 1) {
    cudaEvent_t e = nullptr;
    cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    step_events_.push_back(e);
  }

  Slot& s = *slots_[next_ % slots_.size()];
  ++next_;
  // The pinned staging is rewritten on the host: its previous upload must have finished.
  if (s.used) cuda_check(cudaEventSynchronize(s.h2d), "BatchRenderer staging");
  int* pin_idx = static_cast<int*>(s.pinned);
  std::memcpy(pin_idx, idx.data(), sizeof(int) * idx.size());
  const std::size_t index_bytes = align256(sizeof(int) * (cap_.index_ints + 1));
  auto* pin_par = reinterpret_cast<double*>(static_cast<char*>(s.pinned) + index_bytes);
  int* dev_idx = static_cast<int*>(s.index.ptr);
  auto* dev_orig = static_cast<double*>(s.porig.ptr);
  auto* dev_render = static_cast<double*>(s.prender.ptr);
  mgb::ParamGather g{};
  const double* tables[kNumNodeTypes] = {};
  std::size_t io = idx.size(), po = 0;
  for (const auto& [t, src] : rd.param_source_rows) {
    const int ti = static_cast<int>(t);
    const std::size_t w = static_cast<std::size_t>(param_width(t));
    std::memcpy(pin_idx + io, src.data(), sizeof(int) * src.size());
    std::memcpy(pin_par + po, orig_tables[ti], sizeof(double) * src.size() * w);
    g.in[ti] = dev_orig + po;
    g.src_rows[ti] = dev_idx + io;
    g.out[ti] = dev_render + po;
    g.rows[ti] = static_cast<int>(src.size());
    g.width[ti] = static_cast<int>(w);
    tables[ti] = dev_render + po;
    io += src.size();
    po += src.size() * w;
  }
  float* arena = static_cast<float*>(s.arena.ptr);
  // Uploads: the slot's previous render must be done with its device tables and arena.
  if (s.used) cuda_check(cudaStreamWaitEvent(h2d_, s.done, 0), "wait");
  if (n_idx) cuda_check(cudaMemcpyAsync(dev_idx, pin_idx, sizeof(int) * n_idx, cudaMemcpyHostToDevice, h2d_), "H2D plan");
  if (n_par) cuda_check(cudaMemcpyAsync(dev_orig, pin_par, sizeof(double) * n_par, cudaMemcpyHostToDevice, h2d_), "H2D params");
  const std::size_t row_bytes = sizeof(float) * static_cast<std::size_t>(stride_);
  if (!sources_on_device && rd.num_inputs > 0) {
    // Host sources: consecutive inputs that map to consecutive source rows go as one copy.
    for (int k = 0; k < rd.num_inputs;) {
      const int r0 = k % source_rows;
      const int n = std::min(rd.num_inputs - k, source_rows - r0);
      cuda_check(cudaMemcpyAsync(arena + static_cast<long>(k) * stride_, sources + static_cast<long>(r0) * stride_,
                                 row_bytes * n, cudaMemcpyHostToDevice, h2d_), "H2D sources");
      k += n;
    }
  }
  cuda_check(cudaEventRecord(s.h2d, h2d_), "event");
  // Compute: after the uploads, and after the slot's previous outputs were read back.
  cuda_check(cudaStreamWaitEvent(compute_, s.h2d, 0), "wait");
  if (s.used) cuda_check(cudaStreamWaitEvent(compute_, s.d2h, 0), "wait");
  if (sources_on_device && rd.num_inputs > 0) {
    for (int k = 0; k < rd.num_inputs;) {
      const int r0 = k % source_rows;
      const int n = std::min(rd.num_inputs - k, source_rows - r0);
      cuda_check(cudaMemcpyAsync(arena + static_cast<long>(k) * stride_, sources + static_cast<long>(r0) * stride_,
                                 row_bytes * n, cudaMemcpyDeviceToDevice, compute_), "D2D sources");
      k += n;
    }
  }
  mgb::launch_param_gather(g, compute_);
  plan->attach(dev_idx, aux_, step_events_.data());
  s.plan = std::move(plan);  // the previous plan of this slot is no longer referenced by queued work
  render_arena(*s.plan, procs_, tables, arena, batch_, length_, s.ws.ptr, cap_.workspace_bytes, compute_);
  cuda_check(cudaEventRecord(s.done, compute_), "event");
  if (outputs) {
    cuda_check(cudaStreamWaitEvent(d2h_, s.done, 0), "wait");
    const int n_outs = rd.buffer_rows - rd.output_begin;
    cuda_check(cudaMemcpyAsync(outputs, arena + static_cast<long>(rd.output_begin) * stride_, row_bytes * n_outs,
                               cudaMemcpyDeviceToHost, d2h_), "D2H outputs");
  }
  cuda_check(cudaEventRecord(s.d2h, d2h_), "event");
  s.used = true;
}

void BatchRenderer::sync() {
  for (cudaStream_t st : {h2d_, compute_, d2h_}) cuda_check(cudaStreamSynchronize(st), "BatchRenderer sync");
}

float* BatchRenderer::last_arena() const {
  if (next_ == 0) return nullptr;
  return static_cast<float*>(slots_[(next_ - 1) % slots_.size()]->arena.ptr);
}

// ---- host-buffer API ----------------------------------------------------------------------

void ProcessorSet::process_device(NodeType type, const float* in, float* out, int slots, int batch, long length,
                                  const double* params, int param_offset, cudaStream_t stream) const {
  // Identity CSR: slot s reads input row s.
  Engine& e = engine_for(dev_->device);
  std::vector<int> idx(static_cast<std::size_t>(2 * slots + 1));
  for (int s = 0; s <= slots; ++s) idx[static_cast<std::size_t>(s)] = s;
  for (int s = 0; s < slots; ++s) idx[static_cast<std::size_t>(slots + 1 + s)] = s;
  const std::size_t ws_bytes = std::max<std::size_t>(256, step_ws_bytes(type, slots, batch, length, *this));
  char* aux = static_cast<char*>(e.aux.ensure(align256(sizeof(int) * idx.size()) + ws_bytes));
  cuda_check(cudaMemcpyAsync(aux, idx.data(), sizeof(int) * idx.size(), cudaMemcpyHostToDevice, stream), "H2D csr");
  mgb::StepArgs a{};
  a.src = in;
  a.dst = out;
  a.row_ptr = reinterpret_cast<const int*>(aux);
  a.col = reinterpret_cast<const int*>(aux) + slots + 1;
  a.params = params ? params + static_cast<long>(param_offset) * param_width(type) : nullptr;
  a.slots = slots;
  a.batch = batch;
  a.length = length;
  a.tw = mgb::twiddle_table(dev_->device);
  a.tw64 = mgb::twiddle_table64(dev_->device);
  a.rowstride = static_cast<long>(batch) * 2 * length;
  a.nnz = slots;
  a.dense = 0;  // the identity CSR is dense: slot s reads row 0 + s
  run_step(type, a, *this, aux + align256(sizeof(int) * idx.size()), stream);
  cuda_check(cudaGetLastError(), "process launch");
  // The CSR lives in a reused staging buffer: finish before it can be overwritten.
  cuda_check(cudaStreamSynchronize(stream), "process");
}

void ProcessorSet::process(NodeType type, const double* in, double* out, int slots, int batch, long length,
                           const ParamMatrix* params, int param_offset) const {
  const int width = param_width(type);
  const std::string name = tname(type);
  if (width > 0) {
    if (params == nullptr) fail(name + ": missing parameters");
    if (params->cols != width) fail(name + ": parameter row width mismatch");
    if (param_offset < 0 || param_offset + slots > params->rows) fail(name + ": parameter rows out of range");
    for (int s = 0; s < slots; ++s) check_param_row(type, params->row(param_offset + s));
  }
  if (slots <= 0 || batch <= 0 || length <= 0) return;
  Engine& e = engine_for(dev_->device);
  const std::size_t n = static_cast<std::size_t>(slots) * batch * 2 * static_cast<std::size_t>(length);
  auto* stage = static_cast<double*>(e.staging.ensure(sizeof(double) * n));
  auto* io = static_cast<float*>(e.arena.ensure(sizeof(float) * 2 * n));
  double* d_par = nullptr;
  if (width > 0) {
    d_par = static_cast<double*>(e.params.ensure(sizeof(double) * static_cast<std::size_t>(slots) * width));
    cuda_check(cudaMemcpyAsync(d_par, params->row(param_offset).data(), sizeof(double) * static_cast<std::size_t>(slots) * width,
                               cudaMemcpyHostToDevice, e.stream), "H2D params");
  }
  cuda_check(cudaMemcpyAsync(stage, in, sizeof(double) * n, cudaMemcpyHostToDevice, e.stream), "H2D in");
  mgb::launch_f64_to_f32(stage, io, static_cast<long>(n), e.stream);
  process_device(type, io, io + n, slots, batch, length, d_par, 0, e.stream);
  mgb::launch_f32_to_f64(io + n, stage, static_cast<long>(n), e.stream);
  cuda_check(cudaMemcpyAsync(out, stage, sizeof(double) * n, cudaMemcpyDeviceToHost, e.stream), "D2H out");
  cuda_check(cudaStreamSynchronize(e.stream), "process");
}

AudioBuffer ProcessorSet::process_node(NodeType type, const AudioBuffer& input, std::span<const double> params) const {
  if (input.channels != 2) fail("process_node: processors are stereo (2 channels)");
  const int width = param_width(type);
  if (static_cast<int>(params.size()) != width) {
    fail(tname(type) + ": expected " + std::to_string(width) + " parameters");
  }
  AudioBuffer out(input.batch, 2, input.length, input.sample_rate);
  ParamMatrix table(width > 0 ? 1 : 0, width);
  if (width > 0) std::copy(params.begin(), params.end(), table.row(0).begin());
  process(type, input.samples.data(), out.samples.data(), 1, input.batch, input.length, width > 0 ? &table : nullptr, 0);
  return out;
}

std::pair<std::vector<double>, std::vector<double>> ProcessorSet::reverb_kernel(std::span<const double> params) const {
  Engine& e = engine_for(dev_->device);
  const long len = reverb_length_;
  auto* d_row = static_cast<double*>(e.params.ensure(sizeof(double) * param_width(NodeType::Reverb)));
  auto* d_ir = static_cast<float2*>(e.arena.ensure(sizeof(float2) * static_cast<std::size_t>(len) + 16));
  cuda_check(cudaMemcpyAsync(d_row, params.data(), sizeof(double) * param_width(NodeType::Reverb), cudaMemcpyHostToDevice, e.stream), "H2D");
  mgb::launch_reverb_ir(d_row, 1, reverb_const(*this), d_ir, len, e.stream);
  std::vector<float> h(static_cast<std::size_t>(2 * len));
  cuda_check(cudaMemcpyAsync(h.data(), d_ir, sizeof(float2) * static_cast<std::size_t>(len), cudaMemcpyDeviceToHost, e.stream), "D2H");
  cuda_check(cudaStreamSynchronize(e.stream), "reverb_kernel");
  std::vector<double> l(static_cast<std::size_t>(len)), r(static_cast<std::size_t>(len));
  for (long i = 0; i < len; ++i) {
    l[static_cast<std::size_t>(i)] = h[static_cast<std::size_t>(2 * i)];
    r[static_cast<std::size_t>(i)] = h[static_cast<std::size_t>(2 * i + 1)];
  }
  return {std::move(l), std::move(r)};
}

std::vector<double> ProcessorSet::delay_kernel(std::span<const double> params, int channel) const {
  Engine& e = engine_for(dev_->device);
  const long span = delay_span_;
  auto* d_row = static_cast<double*>(e.params.ensure(sizeof(double) * param_width(NodeType::Delay)));
  auto* d_ir = static_cast<float2*>(e.arena.ensure(sizeof(float2) * static_cast<std::size_t>(span) + 40 * 40 * 4 + 16));
  cuda_check(cudaMemcpyAsync(d_row, params.data(), sizeof(double) * param_width(NodeType::Delay), cudaMemcpyHostToDevice, e.stream), "H2D");
  mgb::launch_delay_ir(d_row, 1, delay_const(*this), d_ir, span, e.stream);
  std::vector<float> h(static_cast<std::size_t>(2 * span));
  cuda_check(cudaMemcpyAsync(h.data(), d_ir, sizeof(float2) * static_cast<std::size_t>(span), cudaMemcpyDeviceToHost, e.stream), "D2H");
  cuda_check(cudaStreamSynchronize(e.stream), "delay_kernel");
  std::vector<double> k(static_cast<std::size_t>(span));
  for (long i = 0; i < span; ++i) k[static_cast<std::size_t>(i)] = h[static_cast<std::size_t>(2 * i + channel)];
  return k;
}

std::vector<long> ProcessorSet::delay_positions(std::span<const double> params, int channel) const {
  // processors.cpp:189-208 (fp64, same libm on the host); the device kernel mirrors it.
  std::vector<long> pos(kDelayTapsPerChannel, -1);
  for (int m = 0; m < kDelayTapsPerChannel; ++m) {
    const std::size_t base = static_cast<std::size_t>(channel * kDelayTapsPerChannel + m) * kDelayTapStride;
    double mx = params[base + 2];
    for (int k = 1; k < kDelayFirBins; ++k) mx = std::max(mx, params[base + 2 + static_cast<std::size_t>(k)]);
    if (mx <= kDelayDisabledLogMag) continue;
    const double frac = -std::atan2(params[base + 1], params[base]) / (2.0 * std::numbers::pi);
    long d = std::lround(frac * static_cast<double>(delay_span_));
    d %= delay_span_;
    if (d < 0) d += delay_span_;
    const long lo = static_cast<long>(m) * delay_window_;
    const long hi = std::min(static_cast<long>(m + 1) * delay_window_, delay_span_) - 1;
    pos[static_cast<std::size_t>(m)] = std::clamp(d, lo, hi);
  }
  return pos;
}

void render_host(const RenderData& rd, const ProcessorSet& procs, const ParamStore& params,
                 const double* const* sources, int batch, long length, double* const* outputs,
                 double* const* intermediates, const DevicePlan* cached_plan) {
  // Per-step parameter checks, in step order (render.cpp:49-56, processors.cpp:232-247).
  for (const StepIndex& st : rd.steps) {
    const int width = param_width(st.type);
    if (width == 0) continue;
    auto it = params.tables.find(st.type);
    if (it == params.tables.end()) fail("render: missing parameter table for " + tname(st.type));
    const ParamMatrix& m = it->second;
    const int slots = st.store_end - st.store_begin;
    if (m.cols != width) fail(tname(st.type) + ": parameter row width mismatch");
    if (st.param_begin < 0 || st.param_begin + slots > m.rows) fail(tname(st.type) + ": parameter rows out of range");
    for (int s = 0; s < slots; ++s) check_param_row(st.type, m.row(st.param_begin + s));
  }

  Engine& e = engine_for(procs.device().device);
  const long stride = static_cast<long>(batch) * 2 * length;
  const std::size_t rows = static_cast<std::size_t>(rd.buffer_rows);
  std::unique_ptr<DevicePlan> own;
  if (!cached_plan) own = std::make_unique<DevicePlan>(rd);
  const DevicePlan& plan = cached_plan ? *cached_plan : *own;
  const std::size_t ws_bytes = plan.workspace_bytes(batch, length, procs);
  auto* arena = static_cast<float*>(e.arena.ensure(sizeof(float) * rows * stride + 16));
  void* ws = e.ws.ensure(ws_bytes);

  // Parameters: every table, one upload.
  std::size_t total = 0;
  for (const auto& [t, m] : params.tables) total += m.values.size();
  auto* d_par = static_cast<double*>(e.params.ensure(sizeof(double) * (total + 1)));
  const double* tables[kNumNodeTypes] = {};
  std::vector<double> host;
  host.reserve(total);
  for (const auto& [t, m] : params.tables) {
    tables[static_cast<int>(t)] = d_par + host.size();
    host.insert(host.end(), m.values.begin(), m.values.end());
  }
  if (!host.empty()) {
    cuda_check(cudaMemcpyAsync(d_par, host.data(), sizeof(double) * host.size(), cudaMemcpyHostToDevice, e.stream), "H2D params");
  }
  // Sources (double, caller memory) -> staging -> fp32 arena rows [0, K).
  const std::size_t n_src = static_cast<std::size_t>(rd.num_inputs) * stride;
  auto* stage = static_cast<double*>(e.staging.ensure(sizeof(double) * std::max<std::size_t>(n_src, rows * stride) + 16));
  for (int k = 0; k < rd.num_inputs; ++k) {
    cuda_check(cudaMemcpyAsync(stage + static_cast<std::size_t>(k) * stride, sources[k], sizeof(double) * stride,
                               cudaMemcpyHostToDevice, e.stream), "H2D sources");
  }
  mgb::launch_f64_to_f32(stage, arena, static_cast<long>(n_src), e.stream);
  render_arena(plan, procs, tables, arena, batch, length, ws, ws_bytes, e.stream);

  // Rows back to double on the device, then straight into the caller's buffers.
  const long first = intermediates ? 0 : rd.output_begin;
  mgb::launch_f32_to_f64(arena + first * stride, stage, (rd.buffer_rows - first) * stride, e.stream);
  auto row_of = [&](long r) { return stage + static_cast<std::size_t>(r - first) * stride; };
  for (int r = rd.output_begin; r < rd.buffer_rows; ++r) {
    cuda_check(cudaMemcpyAsync(outputs[r - rd.output_begin], row_of(r), sizeof(double) * stride, cudaMemcpyDeviceToHost,
                               e.stream), "D2H outputs");
  }
  for (int r = 0; intermediates && r < rd.buffer_rows; ++r) {
    cuda_check(cudaMemcpyAsync(intermediates[r], row_of(rd.sigma[static_cast<std::size_t>(r)]), sizeof(double) * stride,
                               cudaMemcpyDeviceToHost, e.stream), "D2H intermediates");
  }
  cuda_check(cudaStreamSynchronize(e.stream), "render");
}

RenderResult render(const RenderData& rd, const ProcessorSet& procs, const ParamStore& params,
                    const std::vector<AudioBuffer>& sources, const RenderOptions& options) {
  // render.cpp:17-30
  if (static_cast<int>(sources.size()) != rd.num_inputs) {
    fail("render: expected " + std::to_string(rd.num_inputs) + " sources, got " + std::to_string(sources.size()));
  }
  if (sources.empty()) fail("render: graph has no input nodes to take signal shape from");
  const int batch = sources[0].batch;
  const long length = sources[0].length;
  const double fs = sources[0].sample_rate;
  for (const AudioBuffer& s : sources) {
    if (s.channels != 2) fail("render: sources must be stereo");
    if (s.batch != batch || s.length != length || s.sample_rate != fs) {
      fail("render: sources must share batch, length and sample rate");
    }
  }
  RenderResult result;
  std::vector<const double*> src;
  for (const AudioBuffer& s : sources) src.push_back(s.samples.data());
  std::vector<double*> outs, inter;
  for (int r = rd.output_begin; r < rd.buffer_rows; ++r) {
    result.outputs.emplace_back(batch, 2, length, fs);
  }
  for (auto& o : result.outputs) outs.push_back(o.samples.data());
  if (options.keep_intermediates) {
    for (int r = 0; r < rd.buffer_rows; ++r) result.intermediates.emplace_back(batch, 2, length, fs);
    for (auto& o : result.intermediates) inter.push_back(o.samples.data());
  }
  render_host(rd, procs, params, src.data(), batch, length, outs.data(), options.keep_intermediates ? inter.data() : nullptr,
              nullptr);
  return result;
}

RenderResult render(const RenderData& rd, const ProcessorSet& procs, const std::vector<AudioBuffer>& sources,
                    const RenderOptions& options) {
  return render(rd, procs, rd.flat.params, sources, options);
}

}  // namespace mixgraph
