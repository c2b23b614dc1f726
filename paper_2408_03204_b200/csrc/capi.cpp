// C ABI (include/mixgraph_b200.h): thin extern "C" layer over the C++ API.
// Exceptions become status codes; std::invalid_argument keeps its message (MG_EINVAL).
#include "../../include/mixgraph_b200.h"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>

#include "mixgraph_b200/graph_io.hpp"
#include "mixgraph_b200/render.hpp"

namespace mgb {  // device/launch.hpp (nvcc-only header): optimisation helpers
std::size_t mse_scratch_bytes();
void launch_mse_loss_grad(const float* y, const float* target, long n, float* grad, double* loss, void* scratch,
                          cudaStream_t s);
void launch_sgd_step(bool dynamics, double* table, const double* grad, long n, double lr, cudaStream_t s);
void set_conv_fuse(int mode);
void set_dyn_stream(int mode);
void set_dyn_pair(int mode);
void set_conv_log(int log_n);
void set_fft_fp64(bool on);
void conv_geometry(long length, long taps, long* out);
bool fft_fp64();
}  // namespace mgb

using namespace mixgraph;

struct mg_plan {
  RenderData rd;
  std::map<int, std::unique_ptr<DevicePlan>> dev;  // per device, uploaded lazily on first use
  std::vector<cudaEvent_t> events;  // per-step timing events (profiled renders)
  std::mutex mu;
  std::mutex render_mu;  // serialises enqueue: the plan's fork/join events are shared
  ~mg_plan() {
    for (cudaEvent_t e : events) cudaEventDestroy(e);
  }
};

struct mg_graph {
  std::unique_ptr<RenderGraph> g;
};

struct mg_pipeline {
  std::unique_ptr<RenderPipeline> p;
  const mg_plan* plan;
};

struct mg_batch {
  std::unique_ptr<BatchRenderer> b;
};

struct mg_doc {
  std::pair<Graph, ParamStore> d;
};

struct mg_audio {
  AudioBuffer b;
};

struct mg_processors {
  std::unique_ptr<ProcessorSet> ps;
};

namespace {

thread_local std::string g_err;

template <typename F>
int32_t guarded(F&& f) {
  try {
    f();
    return MG_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return MG_EINVAL;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return MG_EINVAL;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MG_ERUNTIME;
  } catch (...) {
    g_err = "unknown error";
    return MG_ERUNTIME;
  }
}

NodeType to_type(int32_t t) {
  if (t < 0 || t >= kNumNodeTypes) throw std::invalid_argument("unknown node type " + std::to_string(t));
  return static_cast<NodeType>(t);
}

Graph make_graph(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne) {
  std::vector<NodeType> tv(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) tv[static_cast<std::size_t>(i)] = to_type(types[i]);
  std::vector<Edge> ev(static_cast<std::size_t>(ne));
  for (int i = 0; i < ne; ++i) ev[static_cast<std::size_t>(i)] = Edge{edges[4 * i], edges[4 * i + 1], edges[4 * i + 2], edges[4 * i + 3]};
  Graph g;
  g.append_unchecked(tv, ev);
  return g;
}

ParamStore make_store(const double* const* tables, const int32_t* rows) {
  ParamStore s;
  for (int t = 0; t < kNumNodeTypes; ++t) {
    const int w = param_width(static_cast<NodeType>(t));
    if (w == 0 || !tables || !tables[t]) continue;
    ParamMatrix m(rows[t], w);
    std::memcpy(m.values.data(), tables[t], sizeof(double) * m.values.size());
    s.tables.emplace(static_cast<NodeType>(t), std::move(m));
  }
  return s;
}

void export_graph(const Graph& g, int32_t* types, int32_t cap_nodes, int32_t* edges, int32_t cap_edges, int32_t* nn,
                  int32_t* ne) {
  *nn = g.num_nodes();
  *ne = static_cast<int32_t>(g.edges().size());
  if (types && g.num_nodes() <= cap_nodes) {
    for (int i = 0; i < g.num_nodes(); ++i) types[i] = static_cast<int32_t>(g.node_type(i));
  }
  if (edges && static_cast<int>(g.edges().size()) <= cap_edges) {
    for (std::size_t i = 0; i < g.edges().size(); ++i) {
      const Edge& e = g.edges()[i];
      edges[4 * i] = e.src;
      edges[4 * i + 1] = e.dst;
      edges[4 * i + 2] = e.outlet;
      edges[4 * i + 3] = e.inlet;
    }
  }
}

// Graph built through the checked builder (add_node / connect), as the reference's callers do.
Graph checked_graph(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne) {
  Graph g;
  for (int i = 0; i < n; ++i) g.add_node(to_type(types[i]));
  for (int i = 0; i < ne; ++i) g.connect(edges[4 * i], edges[4 * i + 1], edges[4 * i + 2], edges[4 * i + 3]);
  return g;
}

void copy_text(const std::string& s, char* buf, int64_t cap, int64_t* len) {
  *len = static_cast<int64_t>(s.size());
  if (buf && static_cast<int64_t>(s.size()) < cap) std::memcpy(buf, s.c_str(), s.size() + 1);
}

}  // namespace

extern "C" {

const char* mg_last_error(void) { return g_err.c_str(); }
int32_t mg_abi_version(void) { return 2; }
int32_t mg_param_width(int32_t t) { return (t < 0 || t >= kNumNodeTypes) ? -1 : param_width(static_cast<NodeType>(t)); }

int32_t mg_graph_validate(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne) {
  return guarded([&] { make_graph(types, n, edges, ne).validate(); });
}

int32_t mg_plan_create(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, int32_t strategy,
                       int32_t beam_width, int32_t optimal_cap, mg_plan** out) {
  return guarded([&] {
    if (strategy < 0 || strategy > 3) throw std::invalid_argument("unknown strategy");
    // to_flat without the default parameter tables: C-ABI renders always pass their own
    // tables, and building/reordering defaults (tens of MB for a 64-graph union) would
    // dominate the plan build.
    const Graph g = make_graph(types, n, edges, ne);
    g.validate();
    FlatGraph fg;
    fg.node_types = g.node_types();
    fg.edges = g.edges();
    fg.num_inputs = static_cast<int>(std::count(fg.node_types.begin(), fg.node_types.end(), NodeType::In));
    fg.num_outputs = static_cast<int>(std::count(fg.node_types.begin(), fg.node_types.end(), NodeType::Out));
    ScheduleOptions o;
    o.strategy = static_cast<Strategy>(strategy);
    o.beam_width = beam_width;
    o.optimal_node_cap = optimal_cap;
    auto p = std::make_unique<mg_plan>();
    p->rd = compute_render_data(fg, o);
    *out = p.release();
  });
}

void mg_plan_destroy(mg_plan* p) { delete p; }

int32_t mg_plan_info(const mg_plan* p, int32_t* info) {
  info[0] = static_cast<int32_t>(p->rd.steps.size());
  info[1] = p->rd.buffer_rows;
  info[2] = p->rd.num_inputs;
  info[3] = p->rd.output_begin;
  info[4] = static_cast<int32_t>(p->rd.flat.edges.size());
  info[5] = static_cast<int32_t>(p->rd.schedule.type_string.size());
  return MG_OK;
}

int32_t mg_plan_type_codes(const mg_plan* p, char* buf, int32_t cap) {
  const std::string s = p->rd.schedule.type_codes();
  if (static_cast<int>(s.size()) + 1 > cap) {
    g_err = "mg_plan_type_codes: buffer too small";
    return MG_EINVAL;
  }
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return MG_OK;
}

int32_t mg_plan_subsets(const mg_plan* p, int32_t* sizes, int32_t* rows) {
  int off = 0;
  for (std::size_t k = 0; k < p->rd.schedule.subsets.size(); ++k) {
    sizes[k] = static_cast<int32_t>(p->rd.schedule.subsets[k].size());
    for (int r : p->rd.schedule.subsets[k]) rows[off++] = r;
  }
  return MG_OK;
}

int32_t mg_plan_sigma(const mg_plan* p, int32_t* sigma) {
  for (std::size_t i = 0; i < p->rd.sigma.size(); ++i) sigma[i] = p->rd.sigma[i];
  return MG_OK;
}

int32_t mg_plan_flat(const mg_plan* p, int32_t* types, int32_t* edges) {
  const FlatGraph& f = p->rd.flat;
  for (std::size_t i = 0; i < f.node_types.size(); ++i) types[i] = static_cast<int32_t>(f.node_types[i]);
  for (std::size_t i = 0; i < f.edges.size(); ++i) {
    edges[4 * i] = f.edges[i].src;
    edges[4 * i + 1] = f.edges[i].dst;
    edges[4 * i + 2] = f.edges[i].outlet;
    edges[4 * i + 3] = f.edges[i].inlet;
  }
  return MG_OK;
}

int32_t mg_plan_step(const mg_plan* p, int32_t k, int32_t* head, int32_t* gather, int32_t* aggregate) {
  return guarded([&] {
    const StepIndex& s = p->rd.steps.at(static_cast<std::size_t>(k));
    head[0] = static_cast<int32_t>(s.type);
    head[1] = s.param_begin;
    head[2] = s.param_end;
    head[3] = s.store_begin;
    head[4] = s.store_end;
    head[5] = static_cast<int32_t>(s.gather.size());
    if (gather) std::copy(s.gather.begin(), s.gather.end(), gather);
    if (aggregate) std::copy(s.aggregate.begin(), s.aggregate.end(), aggregate);
  });
}

int32_t mg_plan_param_source_rows(const mg_plan* p, int32_t t, int32_t* out) {
  auto it = p->rd.param_source_rows.find(static_cast<NodeType>(t));
  if (it == p->rd.param_source_rows.end()) return 0;
  if (out) std::copy(it->second.begin(), it->second.end(), out);
  return static_cast<int32_t>(it->second.size());
}

int32_t mg_plan_reorder_params(const mg_plan* p, const double* const* original, const int32_t* rows,
                               double* const* reordered) {
  return guarded([&] {
    ParamStore r = p->rd.reorder_params(make_store(original, rows));
    for (auto& [t, m] : r.tables) {
      if (reordered[static_cast<int>(t)]) std::memcpy(reordered[static_cast<int>(t)], m.values.data(), sizeof(double) * m.values.size());
    }
  });
}

int32_t mg_validate_schedule(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, const int32_t* ts,
                             int32_t num_subsets, const int32_t* sizes, const int32_t* rows) {
  return guarded([&] {
    FlatGraph fg;
    Graph g = make_graph(types, n, edges, ne);
    fg.node_types = g.node_types();
    fg.edges = g.edges();
    Schedule s;
    int off = 0;
    for (int k = 0; k < num_subsets; ++k) {
      s.type_string.push_back(to_type(ts[k]));
      s.subsets.emplace_back(rows + off, rows + off + sizes[k]);
      off += sizes[k];
    }
    validate_schedule(fg, s);
  });
}

int32_t mg_processors_create(double fs, uint32_t seed, int32_t env_taps, double floor_, int32_t device, mg_processors** out) {
  return guarded([&] {
    if (device >= 0 && cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("cudaSetDevice failed");
    ProcessorConfig c;
    c.sample_rate = fs;
    c.reverb_seed = seed;
    c.envelope_taps = env_taps;
    c.energy_floor = floor_;
    auto p = std::make_unique<mg_processors>();
    p->ps = std::make_unique<ProcessorSet>(c);
    *out = p.release();
  });
}

void mg_processors_destroy(mg_processors* p) { delete p; }

int32_t mg_processors_info(const mg_processors* p, int64_t* info) {
  info[0] = p->ps->delay_span();
  info[1] = p->ps->delay_window();
  info[2] = p->ps->reverb_length();
  return MG_OK;
}

DevicePlan& device_plan(const mg_plan* cp, const mg_processors* procs);

int32_t mg_render(const mg_plan* p, const mg_processors* procs, const double* const* tables, const int32_t* rows,
                  const double* sources, int32_t num_sources, int32_t batch, int64_t length, double fs, double* outputs,
                  double* intermediates) {
  return guarded([&] {
    (void)fs;
    const RenderData& rd = p->rd;
    if (num_sources != rd.num_inputs) {
      throw std::invalid_argument("render: expected " + std::to_string(rd.num_inputs) + " sources, got " +
                                  std::to_string(num_sources));
    }
    if (num_sources == 0) throw std::invalid_argument("render: graph has no input nodes to take signal shape from");
    const std::size_t stride = static_cast<std::size_t>(batch) * 2 * static_cast<std::size_t>(length);
    std::vector<const double*> src;
    for (int k = 0; k < num_sources; ++k) src.push_back(sources + stride * k);
    std::vector<double*> outs, inter;
    for (int r = rd.output_begin; r < rd.buffer_rows; ++r) outs.push_back(outputs + stride * (r - rd.output_begin));
    for (int r = 0; intermediates && r < rd.buffer_rows; ++r) inter.push_back(intermediates + stride * r);
    DevicePlan& dp = device_plan(p, procs);
    std::scoped_lock lock(const_cast<mg_plan*>(p)->render_mu);
    render_host(rd, *procs->ps, make_store(tables, rows), src.data(), batch, static_cast<long>(length), outs.data(),
                intermediates ? inter.data() : nullptr, &dp);
  });
}

// The plan's device-side step table, streams and events live on one device: one DevicePlan per
// device the plan is rendered on (the ProcessorSet's; nullptr: the current device), created
// and used with that device current.
DevicePlan& device_plan(const mg_plan* cp, const mg_processors* procs) {
  auto* p = const_cast<mg_plan*>(cp);
  int device = 0;
  if (procs) {
    device = procs->ps->device_id();
  } else if (cudaGetDevice(&device) != cudaSuccess) {
    throw std::runtime_error("cudaGetDevice failed");
  }
  if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("cudaSetDevice failed");
  std::scoped_lock lock(p->mu);
  auto& d = p->dev[device];
  if (!d) d = std::make_unique<DevicePlan>(p->rd);
  return *d;
}

int32_t mg_plan_workspace_bytes(const mg_plan* p, const mg_processors* procs, int32_t batch, int64_t length, uint64_t* bytes) {
  return guarded([&] { *bytes = device_plan(p, procs).workspace_bytes(batch, static_cast<long>(length), *procs->ps); });
}

int32_t mg_plan_kernel_count(const mg_plan* p, int32_t batch, int64_t length, int32_t* count) {
  return guarded([&] { *count = device_plan(p, nullptr).kernels_per_render(batch, static_cast<long>(length)); });
}

int32_t mg_plan_fusion_candidates(const mg_plan* p, int32_t* share_pairs, int32_t* reads_prev_rows) {
  return guarded([&] {
    const DevicePlan plan(p->rd, DevicePlan::Deferred{});  // host-side analysis only, no device
    for (std::size_t k = 0; k < p->rd.steps.size(); ++k) {
      const int ks = static_cast<int>(k);
      share_pairs[k] = plan.shares(ks) ? plan.share_info(ks).pairs : 0;
      reads_prev_rows[k] = k > 0 && plan.dense_src(ks) >= 0 && plan.dense_src(ks) == p->rd.steps[k - 1].store_begin &&
                                   p->rd.steps[k].store_end - p->rd.steps[k].store_begin ==
                                       p->rd.steps[k - 1].store_end - p->rd.steps[k - 1].store_begin
                               ? 1
                               : 0;
    }
  });
}

int32_t mg_plan_shared_pairs(const mg_plan* p, const mg_processors* procs, int32_t batch, int64_t length,
                             int32_t* pairs) {
  return guarded([&] {
    const DevicePlan& dp = device_plan(p, procs);
    const DevicePlan::Layout lay = dp.layout(batch, static_cast<long>(length), *procs->ps);
    for (std::size_t k = 0; k < p->rd.steps.size(); ++k) {
      pairs[k] = lay.shared[k] ? dp.share_info(static_cast<int>(k)).pairs : 0;
    }
  });
}

int32_t mg_plan_step_owners(const mg_plan* p, int32_t batch, int64_t length, int32_t* owner) {
  return guarded([&] { device_plan(p, nullptr).step_owners(batch, static_cast<long>(length), owner); });
}

int32_t mg_render_arena(const mg_plan* p, const mg_processors* procs, const double* const* d_tables, float* d_arena,
                        int32_t batch, int64_t length, void* d_ws, uint64_t ws_bytes, void* stream) {
  return guarded([&] {
    DevicePlan& dp = device_plan(p, procs);
    std::scoped_lock lock(const_cast<mg_plan*>(p)->render_mu);
    render_arena(dp, *procs->ps, d_tables, d_arena, batch, static_cast<long>(length), d_ws, ws_bytes,
                 static_cast<cudaStream_t>(stream));
  });
}

int32_t mg_render_arena_profiled(const mg_plan* cp, const mg_processors* procs, const double* const* d_tables,
                                 float* d_arena, int32_t batch, int64_t length, void* d_ws, uint64_t ws_bytes,
                                 void* stream, float* step_ms, int32_t hoist) {
  return guarded([&] {
    auto* p = const_cast<mg_plan*>(cp);
    DevicePlan& dp = device_plan(p, procs);
    {
      std::scoped_lock lock(p->mu);
      while (p->events.size() < 2 * p->rd.steps.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) throw std::runtime_error("cudaEventCreate failed");
        p->events.push_back(e);
      }
    }
    auto s = static_cast<cudaStream_t>(stream);
    std::scoped_lock rlock(p->render_mu);
    render_arena(dp, *procs->ps, d_tables, d_arena, batch, static_cast<long>(length), d_ws, ws_bytes, s,
                 step_ms ? p->events.data() : nullptr, hoist != 0);
    if (step_ms) {
      if (cudaStreamSynchronize(s) != cudaSuccess) throw std::runtime_error("render failed");
      for (std::size_t k = 0; k < p->rd.steps.size(); ++k) {
        cudaEventElapsedTime(&step_ms[k], p->events[2 * k], p->events[2 * k + 1]);
      }
    }
  });
}

int32_t mg_profile_steps(const mg_plan* p, const mg_processors* procs, const double* const* d_tables, float* d_arena,
                         int32_t batch, int64_t length, void* d_ws, uint64_t ws_bytes, void* stream, int32_t reps,
                         float* step_ms) {
  return guarded([&] {
    DevicePlan& dp = device_plan(p, procs);
    std::scoped_lock lock(const_cast<mg_plan*>(p)->render_mu);
    profile_steps(dp, *procs->ps, d_tables, d_arena, batch, static_cast<long>(length), d_ws, ws_bytes,
                  static_cast<cudaStream_t>(stream), reps, step_ms);
  });
}

int32_t mg_render_graph_create(const mg_plan* p, const mg_processors* procs, const double* const* d_tables,
                               float* d_arena, int32_t batch, int64_t length, void* d_ws, uint64_t ws_bytes,
                               mg_graph** out) {
  return guarded([&] {
    DevicePlan& dp = device_plan(p, procs);
    std::scoped_lock lock(const_cast<mg_plan*>(p)->render_mu);
    auto g = std::make_unique<mg_graph>();
    g->g = std::make_unique<RenderGraph>(dp, *procs->ps, d_tables, d_arena, batch, static_cast<long>(length), d_ws,
                                         ws_bytes);
    *out = g.release();
  });
}

int32_t mg_render_graph_launch(const mg_graph* g, void* stream) {
  return guarded([&] { g->g->launch(static_cast<cudaStream_t>(stream)); });
}

void mg_render_graph_destroy(mg_graph* g) { delete g; }

int32_t mg_pipeline_create(const mg_plan* p, const mg_processors* procs, int32_t batch, int64_t length, int32_t f32_io,
                           int32_t depth, int32_t host_threads, mg_pipeline** out) {
  return guarded([&] {
    DevicePlan& dp = device_plan(p, procs);
    std::scoped_lock lock(const_cast<mg_plan*>(p)->render_mu);
    auto q = std::make_unique<mg_pipeline>();
    q->plan = p;
    q->p = std::make_unique<RenderPipeline>(dp, *procs->ps, batch, static_cast<long>(length), f32_io != 0, depth,
                                            host_threads);
    *out = q.release();
  });
}

int32_t mg_pipeline_submit(mg_pipeline* q, const double* const* tables, const int32_t* rows, const void* sources,
                           void* outputs) {
  return guarded([&] {
    const RenderData& rd = q->plan->rd;
    // sources / outputs are contiguous [K][B][2][L] / [O][B][2][L] host arrays
    std::vector<const void*> src;
    std::vector<void*> dst;
    const std::size_t bytes = q->p->bytes_per_signal();
    for (int k = 0; k < rd.num_inputs; ++k) src.push_back(static_cast<const char*>(sources) + bytes * k);
    for (int o = 0; o < rd.buffer_rows - rd.output_begin; ++o) dst.push_back(static_cast<char*>(outputs) + bytes * o);
    q->p->submit(make_store(tables, rows), src.data(), dst.data());
  });
}

int32_t mg_pipeline_sync(mg_pipeline* q) {
  return guarded([&] { q->p->sync(); });
}

void mg_pipeline_destroy(mg_pipeline* q) { delete q; }

int32_t mg_backward_workspace_bytes(const mg_plan* p, const mg_processors* procs, int32_t batch, int64_t length,
                                    uint64_t* bytes) {
  return guarded([&] { *bytes = device_plan(p, procs).backward_workspace_bytes(batch, static_cast<long>(length), *procs->ps); });
}

int32_t mg_render_backward_arena(const mg_plan* p, const mg_processors* procs, const double* const* d_tables,
                                 const float* d_arena, float* d_adjoint, double* const* d_grad_tables, int32_t batch,
                                 int64_t length, void* d_workspace, uint64_t workspace_bytes, void* stream) {
  return guarded([&] {
    DevicePlan& dp = device_plan(p, procs);
    std::scoped_lock lock(const_cast<mg_plan*>(p)->render_mu);
    backward_arena(dp, *procs->ps, d_tables, d_arena, d_adjoint, d_grad_tables, batch, static_cast<long>(length),
                   d_workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
  });
}

void mg_set_conv_fuse(int32_t mode) { mgb::set_conv_fuse(mode); }
void mg_set_dyn_stream(int32_t mode) { mgb::set_dyn_stream(mode); }
void mg_set_dyn_pair(int32_t mode) { mgb::set_dyn_pair(mode); }

void mg_set_conv_log(int32_t log_n) { mgb::set_conv_log(log_n); }

int32_t mg_conv_geometry(int64_t length, int64_t taps, int64_t* out) {
  return guarded([&] {
    long g[5];
    mgb::conv_geometry(static_cast<long>(length), static_cast<long>(taps), g);
    for (int i = 0; i < 5; ++i) out[i] = g[i];
  });
}

void mg_set_fft_precision(int32_t bits) { mgb::set_fft_fp64(bits == 64); }
int32_t mg_fft_precision(void) { return mgb::fft_fp64() ? 64 : 32; }

uint64_t mg_mse_scratch_bytes(void) { return mgb::mse_scratch_bytes(); }

int32_t mg_mse_loss_grad(const float* d_y, const float* d_target, int64_t n, float* d_grad, double* d_loss,
                         void* d_scratch, void* stream) {
  return guarded([&] {
    mgb::launch_mse_loss_grad(d_y, d_target, static_cast<long>(n), d_grad, d_loss, d_scratch,
                              static_cast<cudaStream_t>(stream));
  });
}

int32_t mg_sgd_step(int32_t node_type, double* d_table, const double* d_grad, int32_t rows, double learning_rate,
                    void* stream) {
  return guarded([&] {
    const NodeType t = to_type(node_type);
    const bool dyn = t == NodeType::Compressor || t == NodeType::Noisegate;
    mgb::launch_sgd_step(dyn, d_table, d_grad, static_cast<long>(rows) * param_width(t), learning_rate,
                         static_cast<cudaStream_t>(stream));
  });
}

int32_t mg_batch_capacity(const mg_plan* p, const mg_processors* procs, int32_t batch, int64_t length, uint64_t* cap) {
  return guarded([&] {
    const BatchRenderer::Capacity c = BatchRenderer::capacity_for(p->rd, *procs->ps, batch, static_cast<long>(length));
    cap[0] = c.rows;
    cap[1] = c.workspace_bytes;
    cap[2] = c.index_ints;
    cap[3] = c.param_doubles;
  });
}

int32_t mg_batch_create(const mg_processors* procs, int32_t batch, int64_t length, const uint64_t* cap, int32_t depth,
                        mg_batch** out) {
  return guarded([&] {
    BatchRenderer::Capacity c;
    c.rows = cap[0];
    c.workspace_bytes = cap[1];
    c.index_ints = cap[2];
    c.param_doubles = cap[3];
    auto b = std::make_unique<mg_batch>();
    b->b = std::make_unique<BatchRenderer>(*procs->ps, batch, static_cast<long>(length), c, depth);
    *out = b.release();
  });
}

int32_t mg_batch_submit(mg_batch* b, const mg_plan* p, const double* const* tables, const int32_t* rows, int32_t validate,
                        const float* sources, int32_t source_rows, int32_t sources_on_device, float* outputs) {
  return guarded([&] {
    b->b->submit(p->rd, tables, rows, validate != 0, sources, source_rows, sources_on_device != 0, outputs);
  });
}

int32_t mg_batch_sync(mg_batch* b) {
  return guarded([&] { b->b->sync(); });
}

int32_t mg_batch_last_arena(const mg_batch* b, void** arena) {
  return guarded([&] { *arena = b->b->last_arena(); });
}

void mg_batch_destroy(mg_batch* b) { delete b; }

int32_t mg_process(const mg_processors* procs, int32_t t, const double* in, double* out, int32_t slots, int32_t batch,
                   int64_t length, const double* params, int32_t param_rows, int32_t param_offset) {
  return guarded([&] {
    const NodeType type = to_type(t);
    ParamMatrix m;
    const ParamMatrix* pm = nullptr;
    if (params) {
      m = ParamMatrix(param_rows, param_width(type));
      std::memcpy(m.values.data(), params, sizeof(double) * m.values.size());
      pm = &m;
    }
    procs->ps->process(type, in, out, slots, batch, static_cast<long>(length), pm, param_offset);
  });
}

int32_t mg_reverb_kernel(const mg_processors* procs, const double* row, double* left, double* right) {
  return guarded([&] {
    auto [l, r] = procs->ps->reverb_kernel({row, static_cast<std::size_t>(param_width(NodeType::Reverb))});
    std::memcpy(left, l.data(), sizeof(double) * l.size());
    std::memcpy(right, r.data(), sizeof(double) * r.size());
  });
}

int32_t mg_delay_kernel(const mg_processors* procs, const double* row, int32_t channel, double* kernel, int64_t* positions) {
  return guarded([&] {
    std::span<const double> r{row, static_cast<std::size_t>(param_width(NodeType::Delay))};
    if (positions) {
      auto pos = procs->ps->delay_positions(r, channel);
      for (std::size_t i = 0; i < pos.size(); ++i) positions[i] = pos[i];
    }
    if (kernel) {
      auto k = procs->ps->delay_kernel(r, channel);
      std::memcpy(kernel, k.data(), sizeof(double) * k.size());
    }
  });
}

double mg_compressor_gain_log(double g, double t, double w, double r) { return compressor_gain_log(g, t, w, r); }
double mg_noisegate_gain_log(double g, double t, double w, double r) { return noisegate_gain_log(g, t, w, r); }

int32_t mg_check_param_row(int32_t t, const double* row) {
  return guarded([&] {
    const NodeType type = to_type(t);
    check_param_row(type, {row, static_cast<std::size_t>(param_width(type))});
  });
}

int32_t mg_default_param_row(int32_t t, double* row) {
  return guarded([&] {
    const NodeType type = to_type(t);
    default_param_row(type, {row, static_cast<std::size_t>(param_width(type))});
  });
}

int32_t mg_uniform_noise(int64_t n, uint32_t seed, double* out) {
  return guarded([&] {
    auto v = dsp::uniform_noise(static_cast<long>(n), seed);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}

// ---- file-level I/O (graph_io.cpp:19-143, wav.cpp:39-133) --------------------------------

int32_t mg_graph_to_json(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, const double* const* tables,
                         const int32_t* rows, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] { copy_text(graph_to_json(checked_graph(types, n, edges, ne), make_store(tables, rows)), buf, cap, len); });
}

int32_t mg_save_graph(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, const double* const* tables,
                      const int32_t* rows, const char* path) {
  return guarded([&] { save_graph(checked_graph(types, n, edges, ne), make_store(tables, rows), path); });
}

int32_t mg_graph_from_json(const char* text, int64_t len, mg_doc** out) {
  return guarded([&] {
    *out = nullptr;
    auto d = std::make_unique<mg_doc>();
    d->d = graph_from_json(std::string(text, static_cast<std::size_t>(len)));
    *out = d.release();
  });
}

int32_t mg_load_graph(const char* path, mg_doc** out) {
  return guarded([&] {
    *out = nullptr;
    auto d = std::make_unique<mg_doc>();
    d->d = load_graph(path);
    *out = d.release();
  });
}

int32_t mg_doc_info(const mg_doc* doc, int32_t* num_nodes, int32_t* num_edges, int32_t* rows) {
  return guarded([&] {
    *num_nodes = doc->d.first.num_nodes();
    *num_edges = static_cast<int32_t>(doc->d.first.edges().size());
    for (int t = 0; t < kNumNodeTypes; ++t) {
      const NodeType nt = static_cast<NodeType>(t);
      rows[t] = doc->d.second.has(nt) ? doc->d.second.table(nt).rows : -1;
    }
  });
}

int32_t mg_doc_graph(const mg_doc* doc, int32_t* types, int32_t* edges) {
  return guarded([&] {
    int32_t nn = 0, ne = 0;
    const Graph& g = doc->d.first;
    export_graph(g, types, g.num_nodes(), edges, static_cast<int32_t>(g.edges().size()), &nn, &ne);
  });
}

int32_t mg_doc_params(const mg_doc* doc, int32_t node_type, double* out) {
  return guarded([&] {
    const ParamMatrix& m = doc->d.second.table(to_type(node_type));
    std::memcpy(out, m.values.data(), sizeof(double) * m.values.size());
  });
}

void mg_doc_destroy(mg_doc* doc) { delete doc; }

int32_t mg_export_dot(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, char* buf, int64_t cap,
                      int64_t* len) {
  return guarded([&] { copy_text(export_dot(checked_graph(types, n, edges, ne)), buf, cap, len); });
}

int32_t mg_write_wav(const double* samples, int32_t batch, int32_t channels, int64_t length, double sample_rate,
                     const char* path) {
  return guarded([&] {
    AudioBuffer b(batch, channels, static_cast<long>(length), sample_rate);
    std::memcpy(b.samples.data(), samples, sizeof(double) * b.samples.size());
    write_wav(b, path);
  });
}

int32_t mg_read_wav(const char* path, mg_audio** out) {
  return guarded([&] {
    *out = nullptr;
    auto a = std::make_unique<mg_audio>();
    a->b = read_wav(path);
    *out = a.release();
  });
}

int32_t mg_audio_info(const mg_audio* a, int64_t* length, double* sample_rate) {
  return guarded([&] {
    *length = a->b.length;
    *sample_rate = a->b.sample_rate;
  });
}

int32_t mg_audio_samples(const mg_audio* a, double* out) {
  return guarded([&] { std::memcpy(out, a->b.samples.data(), sizeof(double) * a->b.samples.size()); });
}

void mg_audio_destroy(mg_audio* a) { delete a; }

}  // extern "C"
