// C entry points of the synthetic workload generators (test / benchmark support, not the
// product): generate_console (`proj/src/console.cpp:10-44`) and random_legal_params
// (`proj/tests/support/test_util.cpp:63-113`), restated bit-identically in workload.cpp.
// Links against the product library for Graph / ParamStore (libmgb200.so).
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "mixgraph_b200/graph.hpp"

namespace mixgraph::workload {
Graph generate_console(int tracks, double prune, std::uint32_t seed);
ParamStore random_legal_params(const std::vector<NodeType>& types, std::uint32_t seed);
}  // namespace mixgraph::workload

using namespace mixgraph;

namespace {
thread_local std::string g_err;

template <typename F>
int32_t guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* wl_last_error(void) { return g_err.c_str(); }

int32_t wl_generate_console(int32_t tracks, double prune, uint32_t seed, int32_t* types, int32_t cap_nodes,
                            int32_t* edges, int32_t cap_edges, int32_t* nn, int32_t* ne) {
  return guarded([&] {
    const Graph g = workload::generate_console(tracks, prune, seed);
    *nn = g.num_nodes();
    *ne = static_cast<int32_t>(g.edges().size());
    if (*nn > cap_nodes || *ne > cap_edges) throw std::invalid_argument("wl_generate_console: buffers too small");
    for (int i = 0; i < g.num_nodes(); ++i) types[i] = static_cast<int32_t>(g.node_type(i));
    for (std::size_t i = 0; i < g.edges().size(); ++i) {
      const Edge& e = g.edges()[i];
      edges[4 * i] = e.src;
      edges[4 * i + 1] = e.dst;
      edges[4 * i + 2] = e.outlet;
      edges[4 * i + 3] = e.inlet;
    }
  });
}

int32_t wl_random_legal_params(const int32_t* types, int32_t n, uint32_t seed, double* const* tables) {
  return guarded([&] {
    std::vector<NodeType> tv(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) {
      if (types[i] < 0 || types[i] >= kNumNodeTypes) throw std::invalid_argument("unknown node type");
      tv[static_cast<std::size_t>(i)] = static_cast<NodeType>(types[i]);
    }
    ParamStore s = workload::random_legal_params(tv, seed);
    for (auto& [t, m] : s.tables) {
      if (tables[static_cast<int>(t)]) std::memcpy(tables[static_cast<int>(t)], m.values.data(), sizeof(double) * m.values.size());
    }
  });
}

}  // extern "C"
