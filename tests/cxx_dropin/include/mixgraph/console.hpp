// Drop-in shim for the reference's console generator (`proj/include/mixgraph/console.hpp`):
// test support, served by the bit-identical restatement in workloads/libmgbwork.so.
#pragma once

#include <cstdint>

#include "mixgraph_b200/graph.hpp"

namespace mixgraph {

namespace workload {
Graph generate_console(int tracks, double prune, std::uint32_t seed);
}  // namespace workload

struct ConsoleOptions {
  double send_prune_probability = 0.0;
  std::uint32_t seed = 0;
};

inline Graph generate_console(int tracks, const ConsoleOptions& options) {
  return workload::generate_console(tracks, options.send_prune_probability, options.seed);
}
inline Graph generate_console(int tracks) { return generate_console(tracks, ConsoleOptions{}); }

}  // namespace mixgraph
