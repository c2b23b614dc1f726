// Synthetic workload generators used by the benchmark and tests.
//
// These reproduce the reference's generators bit-for-bit so that the GPU path and the
// reference CPU renderer see identical inputs: generate_console (`proj/src/console.cpp:10-44`)
// and random_legal_params (`proj/tests/support/test_util.cpp:63-113`). Both consume a
// std::mt19937 stream in a fixed order; tests/test_workload.py compares them with the
// compiled reference.
#include <cmath>
#include <numbers>
#include <random>
#include <stdexcept>

#include "mixgraph_b200/graph.hpp"

namespace mixgraph::workload {

namespace {
double uniform(std::mt19937& rng, double lo, double hi) { return lo + (hi - lo) * (static_cast<double>(rng()) * (1.0 / 4294967296.0)); }
}  // namespace

Graph generate_console(int tracks, double prune, std::uint32_t seed) {
  if (tracks < 1) throw std::invalid_argument("generate_console: need at least one track");
  std::mt19937 rng(seed);
  auto keep = [&] { return prune <= 0.0 || static_cast<double>(rng()) * (1.0 / 4294967296.0) >= prune; };
  Graph g;
  std::vector<int> gains;
  std::vector<std::pair<int, int>> sends;
  for (int k = 0; k < tracks; ++k) {
    const int in = g.add_node(NodeType::In);
    auto [first, gain] = g.add_serial_chain({NodeType::Eq, NodeType::Compressor, NodeType::Noisegate, NodeType::Imager, NodeType::Gain});
    g.connect(in, first);
    gains.push_back(gain);
    if (keep()) sends.emplace_back(gain, g.add_node(NodeType::Delay));
    if (keep()) sends.emplace_back(gain, g.add_node(NodeType::Reverb));
  }
  const int bus = g.add_node(NodeType::Mix);
  for (int gain : gains) g.connect(gain, bus);
  for (auto [gain, send] : sends) {
    g.connect(gain, send);
    g.connect(send, bus);
  }
  auto [b0, b1] = g.add_serial_chain({NodeType::Eq, NodeType::Compressor, NodeType::Imager, NodeType::Gain});
  g.connect(bus, b0);
  const int out = g.add_node(NodeType::Out);
  g.connect(b1, out);
  return g;
}

ParamStore random_legal_params(const std::vector<NodeType>& types, std::uint32_t seed) {
  std::mt19937 rng(seed);
  ParamStore store = default_params(types);
  for (auto& [t, table] : store.tables) {  // enum order, as std::map iterates
    for (int r = 0; r < table.rows; ++r) {
      auto row = table.row(r);
      switch (t) {
        case NodeType::Gain:
          row[0] = uniform(rng, -1.0, 1.0);
          row[1] = uniform(rng, -1.0, 1.0);
          break;
        case NodeType::Imager: row[0] = uniform(rng, -1.0, 1.0); break;
        case NodeType::Eq:
          for (auto& v : row) v = uniform(rng, -0.5, 0.5);
          break;
        case NodeType::Reverb:
          for (int k = 0; k < kReverbNumBins; ++k) {
            row[static_cast<std::size_t>(k)] = uniform(rng, -2.0, 0.0);
            row[static_cast<std::size_t>(kReverbNumBins + k)] = uniform(rng, -1.5, -0.02);
            row[static_cast<std::size_t>(2 * kReverbNumBins + k)] = uniform(rng, -2.0, 0.0);
            row[static_cast<std::size_t>(3 * kReverbNumBins + k)] = uniform(rng, -1.5, -0.02);
          }
          break;
        case NodeType::Compressor:
        case NodeType::Noisegate:
          row[0] = uniform(rng, 0.9, 0.9995);
          row[1] = uniform(rng, -3.0, 0.5);
          row[2] = uniform(rng, 0.1, 1.0);
          row[3] = uniform(rng, 1.0, 8.0);
          break;
        case NodeType::Delay:
          for (int tap = 0; tap < 2 * kDelayTapsPerChannel; ++tap) {
            auto sub = row.subspan(static_cast<std::size_t>(tap) * kDelayTapStride, kDelayTapStride);
            const double radius = uniform(rng, 0.7, 1.0);
            const double angle = uniform(rng, -std::numbers::pi, std::numbers::pi);
            sub[0] = radius * std::cos(angle);
            sub[1] = radius * std::sin(angle);
            const bool active = rng() % 5 != 0;
            for (int k = 0; k < kDelayFirBins; ++k) sub[static_cast<std::size_t>(2 + k)] = active ? uniform(rng, -1.0, 0.5) : -80.0;
          }
          break;
        default: break;
      }
    }
  }
  return store;
}

}  // namespace mixgraph::workload
