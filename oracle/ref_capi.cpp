// ORACLE — test infrastructure only. Never linked into or called by the product.
//
// A C-ABI over the UNMODIFIED reference (`/root/reference/proj/src/*.cpp`, compiled by
// oracle/Makefile into oracle/_ref/libmixgraph_ref.so together with the FFTW-API stand-in
// in oracle/shim/). tests/ (parity checker), __graft_entry__.smoke() and bench.py's CPU
// baseline load it with ctypes. Each entry point forwards to the reference function named
// in its comment; nothing here re-implements reference arithmetic.
//
// Parameter tables cross the boundary the way the product's C-ABI takes them
// (include/mixgraph_b200.h): `tables[t]` points at a row-major [rows[t]][param_width(t)]
// double matrix for NodeType t (enum order, `proj/include/mixgraph/types.hpp:12-23`), or
// is NULL when the graph has no node of that type.
#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "mixgraph/console.hpp"
#include "mixgraph/dsp.hpp"
#include "mixgraph/fit.hpp"
#include "mixgraph/graph.hpp"
#include "mixgraph/graph_io.hpp"
#include "mixgraph/wav.hpp"
#include "mixgraph/processors.hpp"
#include "mixgraph/reference.hpp"
#include "mixgraph/render.hpp"
#include "mixgraph/schedule.hpp"
#include "support/test_util.hpp"

using namespace mixgraph;

namespace {

thread_local std::string g_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_error = e.what();
    return 2;
  }
}

FlatGraph make_flat(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne) {
  Graph g;
  for (int i = 0; i < n; ++i) g.add_node(static_cast<NodeType>(types[i]));
  for (int i = 0; i < ne; ++i) g.connect(edges[4 * i], edges[4 * i + 1], edges[4 * i + 2], edges[4 * i + 3]);
  return to_flat(g);  // graph.cpp:188-199 (validates)
}

ParamStore make_store(const double* const* tables, const int32_t* rows) {
  ParamStore store;
  for (int t = 0; t < kNumNodeTypes; ++t) {
    const int w = param_width(static_cast<NodeType>(t));
    if (w == 0 || tables == nullptr || tables[t] == nullptr) continue;
    ParamMatrix m(rows[t], w);
    std::memcpy(m.values.data(), tables[t], sizeof(double) * static_cast<std::size_t>(rows[t]) * w);
    store.tables.emplace(static_cast<NodeType>(t), std::move(m));
  }
  return store;
}

int export_graph(const Graph& g, int32_t* types, int32_t cap_nodes, int32_t* edges, int32_t cap_edges,
                 int32_t* n_nodes, int32_t* n_edges) {
  *n_nodes = g.num_nodes();
  *n_edges = static_cast<int32_t>(g.edges().size());
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
  return 0;
}

const ProcessorSet& processors_for(double fs, uint32_t seed, int32_t env_taps, double floor_) {
  static std::mutex mu;
  static std::map<std::tuple<double, uint32_t, int32_t, double>, std::unique_ptr<ProcessorSet>> cache;
  std::scoped_lock lock(mu);
  auto key = std::make_tuple(fs, seed, env_taps, floor_);
  auto it = cache.find(key);
  if (it == cache.end()) {
    ProcessorConfig c;
    c.sample_rate = fs;
    c.reverb_seed = seed;
    c.envelope_taps = env_taps;
    c.energy_floor = floor_;
    it = cache.emplace(key, std::make_unique<ProcessorSet>(c)).first;  // processors.cpp:151-160
  }
  return *it->second;
}

std::vector<AudioBuffer> make_sources(const double* src, int32_t k, int32_t batch, int64_t length, double fs) {
  std::vector<AudioBuffer> out;
  const std::size_t stride = static_cast<std::size_t>(batch) * 2 * static_cast<std::size_t>(length);
  for (int i = 0; i < k; ++i) {
    AudioBuffer b(batch, 2, static_cast<long>(length), fs);
    std::memcpy(b.samples.data(), src + stride * i, sizeof(double) * stride);
    out.push_back(std::move(b));
  }
  return out;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_error.c_str(); }

// console.cpp:10-44
int ref_console(int32_t tracks, double prune, uint32_t seed, int32_t* types, int32_t cap_nodes,
                int32_t* edges, int32_t cap_edges, int32_t* n_nodes, int32_t* n_edges) {
  return guarded([&] {
    ConsoleOptions o;
    o.send_prune_probability = prune;
    o.seed = seed;
    export_graph(generate_console(tracks, o), types, cap_nodes, edges, cap_edges, n_nodes, n_edges);
  });
}

// tests/support/test_util.cpp:17-61 with a fresh mt19937(seed)
int ref_random_dag(uint32_t seed, int32_t min_nodes, int32_t max_nodes, int32_t heavy, int32_t* types,
                   int32_t cap_nodes, int32_t* edges, int32_t cap_edges, int32_t* n_nodes, int32_t* n_edges) {
  return guarded([&] {
    std::mt19937 rng(seed);
    export_graph(testutil::random_dag(rng, min_nodes, max_nodes, heavy != 0), types, cap_nodes, edges,
                 cap_edges, n_nodes, n_edges);
  });
}

// tests/support/test_util.cpp:190-211
int ref_four_track_snippet(int32_t* types, int32_t cap_nodes, int32_t* edges, int32_t cap_edges,
                           int32_t* n_nodes, int32_t* n_edges) {
  return guarded([&] {
    export_graph(testutil::four_track_mix_snippet(), types, cap_nodes, edges, cap_edges, n_nodes, n_edges);
  });
}

// tests/support/test_util.cpp:63-113 with a fresh mt19937(seed); tables in original node order.
int ref_random_legal_params(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, uint32_t seed,
                            double* const* tables) {
  return guarded([&] {
    FlatGraph fg = make_flat(types, n, edges, ne);
    std::mt19937 rng(seed);
    ParamStore s = testutil::random_legal_params(fg, rng);
    for (auto& [t, m] : s.tables) {
      if (tables[static_cast<int>(t)]) std::memcpy(tables[static_cast<int>(t)], m.values.data(), sizeof(double) * m.values.size());
    }
  });
}

// graph.cpp:130-155
int ref_default_param_row(int32_t type, double* row) {
  return guarded([&] {
    std::vector<double> r(static_cast<std::size_t>(param_width(static_cast<NodeType>(type))));
    default_param_row(static_cast<NodeType>(type), r);
    std::memcpy(row, r.data(), sizeof(double) * r.size());
  });
}

// schedule.cpp:473-525
int ref_plan_create(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, int32_t strategy,
                    int32_t beam_width, int32_t optimal_cap, void** out) {
  return guarded([&] {
    FlatGraph fg = make_flat(types, n, edges, ne);
    ScheduleOptions o;
    o.strategy = static_cast<Strategy>(strategy);
    o.beam_width = beam_width;
    o.optimal_node_cap = optimal_cap;
    *out = new RenderData(compute_render_data(fg, o));
  });
}

void ref_plan_destroy(void* p) { delete static_cast<RenderData*>(p); }

// info[0..5] = num_steps, buffer_rows, num_inputs, output_begin, num_edges, type_string length
int ref_plan_info(const void* p, int32_t* info) {
  const auto* rd = static_cast<const RenderData*>(p);
  info[0] = static_cast<int32_t>(rd->steps.size());
  info[1] = rd->buffer_rows;
  info[2] = rd->num_inputs;
  info[3] = rd->output_begin;
  info[4] = static_cast<int32_t>(rd->flat.edges.size());
  info[5] = static_cast<int32_t>(rd->schedule.type_string.size());
  return 0;
}

// schedule.cpp:301-306 (Schedule::type_codes)
int ref_plan_type_codes(const void* p, char* buf, int32_t cap) {
  std::string s = static_cast<const RenderData*>(p)->schedule.type_codes();
  if (static_cast<int>(s.size()) + 1 > cap) return 1;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}

// Schedule subsets (original rows): sizes[k] per subset, rows concatenated.
int ref_plan_subsets(const void* p, int32_t* sizes, int32_t* rows) {
  const auto* rd = static_cast<const RenderData*>(p);
  int off = 0;
  for (std::size_t k = 0; k < rd->schedule.subsets.size(); ++k) {
    sizes[k] = static_cast<int32_t>(rd->schedule.subsets[k].size());
    for (int r : rd->schedule.subsets[k]) rows[off++] = r;
  }
  return 0;
}

int ref_plan_sigma(const void* p, int32_t* sigma) {
  const auto* rd = static_cast<const RenderData*>(p);
  for (std::size_t i = 0; i < rd->sigma.size(); ++i) sigma[i] = rd->sigma[i];
  return 0;
}

// reordered graph (schedule.cpp:421-452): node types and edges [src,dst,outlet,inlet]
int ref_plan_flat(const void* p, int32_t* types, int32_t* edges) {
  const auto* rd = static_cast<const RenderData*>(p);
  for (std::size_t i = 0; i < rd->flat.node_types.size(); ++i) types[i] = static_cast<int32_t>(rd->flat.node_types[i]);
  for (std::size_t i = 0; i < rd->flat.edges.size(); ++i) {
    edges[4 * i] = rd->flat.edges[i].src;
    edges[4 * i + 1] = rd->flat.edges[i].dst;
    edges[4 * i + 2] = rd->flat.edges[i].outlet;
    edges[4 * i + 3] = rd->flat.edges[i].inlet;
  }
  return 0;
}

// StepIndex (schedule.hpp:60-68): head[0..5] = type, param_begin, param_end, store_begin,
// store_end, |gather|; gather/aggregate may be NULL.
int ref_plan_step(const void* p, int32_t k, int32_t* head, int32_t* gather, int32_t* aggregate) {
  const auto* rd = static_cast<const RenderData*>(p);
  const StepIndex& s = rd->steps.at(static_cast<std::size_t>(k));
  head[0] = static_cast<int32_t>(s.type);
  head[1] = s.param_begin;
  head[2] = s.param_end;
  head[3] = s.store_begin;
  head[4] = s.store_end;
  head[5] = static_cast<int32_t>(s.gather.size());
  for (std::size_t i = 0; gather && i < s.gather.size(); ++i) gather[i] = s.gather[i];
  for (std::size_t i = 0; aggregate && i < s.aggregate.size(); ++i) aggregate[i] = s.aggregate[i];
  return 0;
}

// RenderData::param_source_rows (schedule.cpp:515-523); returns the row count.
int ref_plan_param_source_rows(const void* p, int32_t type, int32_t* out) {
  const auto* rd = static_cast<const RenderData*>(p);
  auto it = rd->param_source_rows.find(static_cast<NodeType>(type));
  if (it == rd->param_source_rows.end()) return 0;
  for (std::size_t i = 0; out && i < it->second.size(); ++i) out[i] = it->second[i];
  return static_cast<int>(it->second.size());
}

// render.cpp:14-81 with params = rd.reorder_params(original) (schedule.cpp:454-471).
// sources [K][B][2][L]; outputs [num_outputs][B][2][L]; intermediates [rows][B][2][L] or NULL.
int ref_render(const void* p, double fs, uint32_t seed, int32_t env_taps, double floor_,
               const double* const* tables, const int32_t* rows, const double* sources, int32_t batch,
               int64_t length, double* outputs, double* intermediates) {
  return guarded([&] {
    const auto* rd = static_cast<const RenderData*>(p);
    const ProcessorSet& procs = processors_for(fs, seed, env_taps, floor_);
    ParamStore original = make_store(tables, rows);
    ParamStore params = rd->reorder_params(original);
    auto src = make_sources(sources, rd->num_inputs, batch, length, fs);
    RenderOptions o;
    o.keep_intermediates = intermediates != nullptr;
    RenderResult r = render(*rd, procs, params, src, o);
    const std::size_t stride = static_cast<std::size_t>(batch) * 2 * static_cast<std::size_t>(length);
    for (std::size_t i = 0; i < r.outputs.size(); ++i) std::memcpy(outputs + stride * i, r.outputs[i].samples.data(), sizeof(double) * stride);
    for (std::size_t i = 0; intermediates && i < r.intermediates.size(); ++i) {
      std::memcpy(intermediates + stride * i, r.intermediates[i].samples.data(), sizeof(double) * stride);
    }
  });
}

// render.cpp:14-81 restated with each step's slots spread over `threads` host threads, for
// full-size parity of the large BASELINE configs on the GPU box's cores (test infrastructure).
// Per slot it runs exactly the reference's arithmetic: the gather sum ((0 + x0) + x1) + ... in
// gather order (render.cpp:44-48), then ProcessorSet::process on that one slot
// (processors.cpp:229-282 loops over slots independently; the set is immutable and shared,
// processors.hpp:24-25). Rows live from their store to their last reader (outputs and the
// `keep` nodes to the end), so the fp64 arena of a 966-node 10 s graph never exists at once;
// a row read before any step stored it reads zeros, as the reference's zero-filled buffer.
// outputs [num_outputs][B][2][L]; kept [n_keep][B][2][L] = rows sigma[keep[j]] (original ids).
// round_f32 (diagnostic): every stored row (and the sources) rounded to float, i.e. the
// reference's fp64 arithmetic with an fp32 arena — the error floor of any fp32-storage renderer.
// perturb > 0 (conditioning probe): every processed row gets uniform noise of amplitude
// perturb * (row peak), mt19937(row) — the global per-step error an FFT-based fp32 renderer
// makes; the output's response to it measures the graph's amplification of such errors.
int ref_render_parallel(const void* p, double fs, uint32_t seed, int32_t env_taps, double floor_,
                        const double* const* tables, const int32_t* rows, const double* sources, int32_t batch,
                        int64_t length, int32_t threads, const int32_t* keep, int32_t n_keep, double* outputs,
                        double* kept, int32_t round_f32, double perturb) {
  return guarded([&] {
    const auto* rd = static_cast<const RenderData*>(p);
    const ProcessorSet& procs = processors_for(fs, seed, env_taps, floor_);
    const ParamStore params = rd->reorder_params(make_store(tables, rows));
    const std::size_t stride = static_cast<std::size_t>(batch) * 2 * static_cast<std::size_t>(length);
    const int nrows = rd->buffer_rows;
    // last step reading each row; -1: never read
    std::vector<int> last(static_cast<std::size_t>(nrows), -1);
    for (std::size_t k = 0; k < rd->steps.size(); ++k) {
      for (int g : rd->steps[k].gather) last[static_cast<std::size_t>(g)] = static_cast<int>(k);
    }
    std::vector<char> pinned(static_cast<std::size_t>(nrows), 0);
    for (int r = rd->output_begin; r < nrows; ++r) pinned[static_cast<std::size_t>(r)] = 1;
    for (int j = 0; j < n_keep; ++j) pinned[static_cast<std::size_t>(rd->sigma.at(static_cast<std::size_t>(keep[j])))] = 1;
    std::vector<std::unique_ptr<double[]>> buf(static_cast<std::size_t>(nrows));
    for (int k = 0; k < rd->num_inputs; ++k) {
      buf[static_cast<std::size_t>(k)] = std::make_unique<double[]>(stride);
      std::memcpy(buf[static_cast<std::size_t>(k)].get(), sources + stride * k, sizeof(double) * stride);
      if (round_f32) {
        double* r = buf[static_cast<std::size_t>(k)].get();
        for (std::size_t j = 0; j < stride; ++j) r[j] = static_cast<double>(static_cast<float>(r[j]));
      }
    }
    const int nthreads = std::max(1, threads);
    for (std::size_t k = 0; k < rd->steps.size(); ++k) {
      const StepIndex& step = rd->steps[k];
      const int slots = step.store_end - step.store_begin;
      const ParamMatrix* table = nullptr;
      if (param_width(step.type) > 0) {
        auto it = params.tables.find(step.type);
        if (it == params.tables.end()) throw std::invalid_argument("render: missing parameter table");
        table = &it->second;
      }
      // edge range [first[s], first[s+1]) of each slot (aggregate is non-decreasing)
      std::vector<std::size_t> first(static_cast<std::size_t>(slots) + 1, step.gather.size());
      for (std::size_t i = step.gather.size(); i-- > 0;) first[static_cast<std::size_t>(step.aggregate[i])] = i;
      for (int s = slots - 1; s >= 0; --s) first[static_cast<std::size_t>(s)] = std::min(first[static_cast<std::size_t>(s)], first[static_cast<std::size_t>(s) + 1]);
      std::vector<std::unique_ptr<double[]>> out(static_cast<std::size_t>(slots));
      std::atomic<int> next{0};
      std::mutex err_mu;
      std::string err;
      auto work = [&] {
        std::vector<double> in(stride);
        for (int s = next.fetch_add(1); s < slots; s = next.fetch_add(1)) {
          try {
            std::fill(in.begin(), in.end(), 0.0);
            for (std::size_t i = first[static_cast<std::size_t>(s)]; i < first[static_cast<std::size_t>(s) + 1]; ++i) {
              const double* src = buf[static_cast<std::size_t>(step.gather[i])].get();
              if (!src) continue;  // never stored: the reference's zero-filled row
              for (std::size_t j = 0; j < stride; ++j) in[j] += src[j];
            }
            auto y = std::make_unique<double[]>(stride);
            std::fill(y.get(), y.get() + stride, 0.0);
            procs.process(step.type, in.data(), y.get(), 1, batch, static_cast<long>(length), table, step.param_begin + s);
            if (perturb > 0.0) {
              double peak = 0.0;
              for (std::size_t j = 0; j < stride; ++j) peak = std::max(peak, std::abs(y[j]));
              std::mt19937 noise(static_cast<std::uint32_t>(step.store_begin + s));
              for (std::size_t j = 0; j < stride; ++j) y[j] += perturb * peak * (2.0 * (noise() * (1.0 / 4294967296.0)) - 1.0);
            }
            if (round_f32) {
              for (std::size_t j = 0; j < stride; ++j) y[j] = static_cast<double>(static_cast<float>(y[j]));
            }
            out[static_cast<std::size_t>(s)] = std::move(y);
          } catch (const std::exception& e) {
            std::scoped_lock lk(err_mu);
            if (err.empty()) err = e.what();
          }
        }
      };
      std::vector<std::thread> pool;
      for (int t = 1; t < std::min(nthreads, slots); ++t) pool.emplace_back(work);
      work();
      for (auto& th : pool) th.join();
      if (!err.empty()) throw std::invalid_argument(err);
      for (int s = 0; s < slots; ++s) buf[static_cast<std::size_t>(step.store_begin + s)] = std::move(out[static_cast<std::size_t>(s)]);
      for (int g : step.gather) {
        if (last[static_cast<std::size_t>(g)] == static_cast<int>(k) && !pinned[static_cast<std::size_t>(g)]) buf[static_cast<std::size_t>(g)].reset();
      }
      for (int r = step.store_begin; r < step.store_end; ++r) {
        if (last[static_cast<std::size_t>(r)] < 0 && !pinned[static_cast<std::size_t>(r)]) buf[static_cast<std::size_t>(r)].reset();
      }
    }
    auto row_or_zero = [&](int r, double* dst) {
      const double* src = buf[static_cast<std::size_t>(r)].get();
      if (src) std::memcpy(dst, src, sizeof(double) * stride);
      else std::fill(dst, dst + stride, 0.0);
    };
    for (int r = rd->output_begin; r < nrows; ++r) row_or_zero(r, outputs + stride * (r - rd->output_begin));
    for (int j = 0; j < n_keep; ++j) row_or_zero(rd->sigma.at(static_cast<std::size_t>(keep[j])), kept + stride * j);
  });
}

// fit.cpp:25-96 (central-difference gradient descent). trainable: n_trainable NodeType ids;
// tables: init params (original order), overwritten with the fitted params; loss_history
// holds steps + 1 values.
int ref_fit(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, double fs, const double* const* tables,
            const int32_t* rows, double* const* out_tables, const double* sources, const double* target, int32_t batch,
            int64_t length, const int32_t* trainable, int32_t n_trainable, int32_t steps, double learning_rate,
            double fd_step, double* loss_history) {
  return guarded([&] {
    FlatGraph fg = make_flat(types, n, edges, ne);
    const ProcessorSet& procs = processors_for(fs, 0, 32768, 1e-7);
    ParamStore init = make_store(tables, rows);
    auto src = make_sources(sources, fg.num_inputs, batch, length, fs);
    auto tgt = make_sources(target, fg.num_outputs, batch, length, fs);
    FitOptions o;
    o.trainable.clear();
    for (int i = 0; i < n_trainable; ++i) o.trainable.push_back(static_cast<NodeType>(trainable[i]));
    o.steps = steps;
    o.learning_rate = learning_rate;
    o.fd_step = fd_step;
    FitResult r = fit(fg, init, procs, src, tgt, o);
    for (std::size_t i = 0; i < r.loss_history.size(); ++i) loss_history[i] = r.loss_history[i];
    for (auto& [t, m] : r.params.tables) {
      if (out_tables[static_cast<int>(t)]) std::memcpy(out_tables[static_cast<int>(t)], m.values.data(), sizeof(double) * m.values.size());
    }
  });
}

// reference.cpp:155-328 (per-node oracle: direct convolutions, recursive envelope)
int ref_render_reference(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, double fs,
                         uint32_t seed, int32_t env_taps, double floor_, const double* const* tables,
                         const int32_t* rows, const double* sources, int32_t batch, int64_t length,
                         double* outputs) {
  return guarded([&] {
    FlatGraph fg = make_flat(types, n, edges, ne);
    const ProcessorSet& procs = processors_for(fs, seed, env_taps, floor_);
    ParamStore params = make_store(tables, rows);
    auto src = make_sources(sources, fg.num_inputs, batch, length, fs);
    auto outs = render_reference(fg, procs, params, src);
    const std::size_t stride = static_cast<std::size_t>(batch) * 2 * static_cast<std::size_t>(length);
    for (std::size_t i = 0; i < outs.size(); ++i) std::memcpy(outputs + stride * i, outs[i].samples.data(), sizeof(double) * stride);
  });
}

// processors.cpp:229-282 (ProcessorSet::process); params [rows][width] or NULL.
int ref_process(int32_t type, const double* in, double* out, int32_t slots, int32_t batch, int64_t length,
                const double* params, int32_t rows, int32_t param_offset, double fs, uint32_t seed,
                int32_t env_taps, double floor_) {
  return guarded([&] {
    const ProcessorSet& procs = processors_for(fs, seed, env_taps, floor_);
    const NodeType t = static_cast<NodeType>(type);
    ParamMatrix m;
    const ParamMatrix* pm = nullptr;
    if (params) {
      m = ParamMatrix(rows, param_width(t));
      std::memcpy(m.values.data(), params, sizeof(double) * m.values.size());
      pm = &m;
    }
    procs.process(t, in, out, slots, batch, static_cast<long>(length), pm, param_offset);
  });
}

// processors.cpp:162-187; left/right hold reverb_length() samples.
int ref_reverb_kernel(double fs, uint32_t seed, const double* row, double* left, double* right, int64_t* len) {
  return guarded([&] {
    const ProcessorSet& procs = processors_for(fs, seed, 32768, 1e-7);
    *len = procs.reverb_length();
    if (!left) return;
    auto [l, r] = procs.reverb_kernel({row, static_cast<std::size_t>(param_width(NodeType::Reverb))});
    std::memcpy(left, l.data(), sizeof(double) * l.size());
    std::memcpy(right, r.data(), sizeof(double) * r.size());
  });
}

// processors.cpp:189-227; kernel holds delay_span() samples, positions 20 entries.
int ref_delay_kernel(double fs, const double* row, int32_t channel, double* kernel, int64_t* positions,
                     int64_t* span) {
  return guarded([&] {
    const ProcessorSet& procs = processors_for(fs, 0, 32768, 1e-7);
    *span = procs.delay_span();
    std::span<const double> r{row, static_cast<std::size_t>(param_width(NodeType::Delay))};
    if (positions) {
      auto p = procs.delay_positions(r, channel);
      for (std::size_t i = 0; i < p.size(); ++i) positions[i] = p[i];
    }
    if (kernel) {
      auto k = procs.delay_kernel(r, channel);
      std::memcpy(kernel, k.data(), sizeof(double) * k.size());
    }
  });
}

// dsp.cpp:106-136
int ref_zero_phase_fir(const double* log_mags, int32_t fir_length, double* taps) {
  return guarded([&] {
    auto f = dsp::zero_phase_fir({log_mags, static_cast<std::size_t>((fir_length + 1) / 2)}, fir_length);
    std::memcpy(taps, f.taps.data(), sizeof(double) * f.taps.size());
  });
}

// dsp.cpp:222-230
int ref_uniform_noise(int64_t n, uint32_t seed, double* out) {
  return guarded([&] {
    auto v = dsp::uniform_noise(static_cast<long>(n), seed);
    std::memcpy(out, v.data(), sizeof(double) * v.size());
  });
}

// dsp.cpp:138-163: noise STFT [frames][bins] complex (interleaved re, im)
int ref_stft(const double* x, int64_t n, int32_t fft_length, int32_t hop, double* out, int32_t* frames) {
  return guarded([&] {
    auto s = dsp::stft({x, static_cast<std::size_t>(n)}, fft_length, hop);
    *frames = s.num_frames;
    if (out) std::memcpy(out, s.bins.data(), sizeof(double) * 2 * s.bins.size());
  });
}

// processors.cpp:110-130
double ref_compressor_gain_log(double g, double t, double w, double r) { return compressor_gain_log(g, t, w, r); }
double ref_noisegate_gain_log(double g, double t, double w, double r) { return noisegate_gain_log(g, t, w, r); }

// ---- file-level I/O (graph_io.cpp:19-143, wav.cpp:39-133) --------------------------------

namespace {
Graph graph_from_arrays(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne) {
  Graph g;
  for (int i = 0; i < n; ++i) g.add_node(static_cast<NodeType>(types[i]));
  for (int i = 0; i < ne; ++i) g.connect(edges[4 * i], edges[4 * i + 1], edges[4 * i + 2], edges[4 * i + 3]);
  return g;
}
int copy_text(const std::string& s, char* buf, int64_t cap, int64_t* len) {
  *len = static_cast<int64_t>(s.size());
  if (buf && static_cast<int64_t>(s.size()) < cap) std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}
}  // namespace

// graph_to_json (graph_io.cpp:19-49); `with_params` = 0 passes an empty ParamStore.
int ref_graph_to_json(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, const double* const* tables,
                      const int32_t* rows, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] { copy_text(graph_to_json(graph_from_arrays(types, n, edges, ne), make_store(tables, rows)), buf, cap, len); });
}

// graph_from_json (graph_io.cpp:51-117) -> heap (Graph, ParamStore)
int ref_graph_from_json(const char* text, void** doc) {
  return guarded([&] { *doc = new std::pair<Graph, ParamStore>(graph_from_json(text)); });
}
int ref_load_graph(const char* path, void** doc) {
  return guarded([&] { *doc = new std::pair<Graph, ParamStore>(load_graph(path)); });
}
int ref_save_graph(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, const double* const* tables,
                   const int32_t* rows, const char* path) {
  return guarded([&] { save_graph(graph_from_arrays(types, n, edges, ne), make_store(tables, rows), path); });
}
int ref_doc_info(const void* doc, int32_t* n_nodes, int32_t* n_edges, int32_t* rows) {
  return guarded([&] {
    const auto& d = *static_cast<const std::pair<Graph, ParamStore>*>(doc);
    *n_nodes = d.first.num_nodes();
    *n_edges = static_cast<int32_t>(d.first.edges().size());
    for (int t = 0; t < kNumNodeTypes; ++t) {
      rows[t] = d.second.has(static_cast<NodeType>(t)) ? d.second.table(static_cast<NodeType>(t)).rows : -1;
    }
  });
}
int ref_doc_graph(const void* doc, int32_t* types, int32_t* edges) {
  return guarded([&] {
    const auto& d = *static_cast<const std::pair<Graph, ParamStore>*>(doc);
    int32_t nn = 0, ne = 0;
    export_graph(d.first, types, d.first.num_nodes(), edges, static_cast<int32_t>(d.first.edges().size()), &nn, &ne);
  });
}
int ref_doc_params(const void* doc, int32_t type, double* out) {
  return guarded([&] {
    const auto& d = *static_cast<const std::pair<Graph, ParamStore>*>(doc);
    const ParamMatrix& m = d.second.table(static_cast<NodeType>(type));
    std::memcpy(out, m.values.data(), sizeof(double) * m.values.size());
  });
}
void ref_doc_destroy(void* doc) { delete static_cast<std::pair<Graph, ParamStore>*>(doc); }

// export_dot (graph_io.cpp:129-143)
int ref_export_dot(const int32_t* types, int32_t n, const int32_t* edges, int32_t ne, char* buf, int64_t cap,
                   int64_t* len) {
  return guarded([&] { copy_text(export_dot(graph_from_arrays(types, n, edges, ne)), buf, cap, len); });
}

// write_wav / read_wav (wav.cpp:39-133); samples [batch][channels][length]
int ref_write_wav(const double* samples, int32_t batch, int32_t channels, int64_t length, double fs, const char* path) {
  return guarded([&] {
    AudioBuffer b(batch, channels, static_cast<long>(length), fs);
    std::memcpy(b.samples.data(), samples, sizeof(double) * b.samples.size());
    write_wav(b, path);
  });
}
int ref_read_wav(const char* path, double* out, int64_t cap, int64_t* length, double* fs) {
  return guarded([&] {
    const AudioBuffer b = read_wav(path);
    *length = b.length;
    *fs = b.sample_rate;
    if (out && static_cast<int64_t>(b.samples.size()) <= cap) std::memcpy(out, b.samples.data(), sizeof(double) * b.samples.size());
  });
}

}  // extern "C"
