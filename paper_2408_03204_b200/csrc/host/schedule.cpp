// Render-order computation (host, integer work).
//
// Output contract: identical to `proj/src/schedule.cpp` for every strategy —
//  * interior nodes = everything but in/out; dependencies = UNIQUE interior predecessors
//    (schedule.cpp:33-67);
//  * greedy: largest computable per-type subset, ties to the lowest enum value (:163-184);
//  * one-by-one: min-heap on row id with in-degree = #unique preds decremented once per
//    interior EDGE (:186-203 — parallel edges decrement more than once; kept as-is);
//  * beam/optimal: candidates expanded in LETTER order, dedup by covered set keeping the
//    lexicographically smaller (by letter) type string, beam ordered by (covered desc,
//    length asc, letters asc) (:205-296), then replayed (:141-161);
//  * sigma = stable sort of rows by step (:397-413); StepIndex slot-major, edge order
//    within a slot (:473-511); param_source_rows (:515-523).
// Data structures are new: CSR adjacency, incremental ready lists for greedy/replay, and
// beam candidates that carry their ready frontier instead of rescanning all nodes.
#include <algorithm>
#include <bit>
#include <cstdint>
#include <deque>
#include <queue>
#include <sstream>
#include <stdexcept>
#include <unordered_map>

#include "mixgraph_b200/schedule.hpp"

namespace mixgraph {

namespace {

[[noreturn]] void fail(const std::string& msg) { throw std::invalid_argument(msg); }

constexpr int kTypes = kNumNodeTypes;

// Interior sub-DAG in CSR form.
struct Dag {
  int n = 0;                     // all nodes
  int m = 0;                     // interior nodes
  std::vector<int> row;          // interior index -> row (ascending)
  std::vector<int> idx;          // row -> interior index or -1
  std::vector<uint8_t> type;     // interior index -> NodeType
  std::vector<int> in_rows, out_rows;
  std::vector<int> pred_off, pred;    // unique preds, sorted
  std::vector<int> usucc_off, usucc;  // unique successors
  std::vector<int> esucc_off, esucc;  // successors per interior edge (multiplicity, edge order)
};

Dag analyze(const FlatGraph& fg) {
  Dag d;
  d.n = fg.num_nodes();
  d.idx.assign(static_cast<std::size_t>(d.n), -1);
  for (int r = 0; r < d.n; ++r) {
    const NodeType t = fg.node_types[static_cast<std::size_t>(r)];
    if (t == NodeType::In) {
      d.in_rows.push_back(r);
    } else if (t == NodeType::Out) {
      d.out_rows.push_back(r);
    } else {
      d.idx[static_cast<std::size_t>(r)] = static_cast<int>(d.row.size());
      d.row.push_back(r);
      d.type.push_back(static_cast<uint8_t>(t));
    }
  }
  d.m = static_cast<int>(d.row.size());
  std::vector<std::pair<int, int>> ie;  // (dst, src) interior edges, edge order
  d.esucc_off.assign(static_cast<std::size_t>(d.m) + 1, 0);
  for (const Edge& e : fg.edges) {
    const int s = d.idx[static_cast<std::size_t>(e.src)], t = d.idx[static_cast<std::size_t>(e.dst)];
    if (s >= 0 && t >= 0) {
      ie.emplace_back(t, s);
      ++d.esucc_off[static_cast<std::size_t>(s) + 1];
    }
  }
  for (int j = 0; j < d.m; ++j) d.esucc_off[static_cast<std::size_t>(j) + 1] += d.esucc_off[static_cast<std::size_t>(j)];
  d.esucc.resize(ie.size());
  {
    std::vector<int> fill(d.esucc_off.begin(), d.esucc_off.end() - 1);
    for (auto [t, s] : ie) d.esucc[static_cast<std::size_t>(fill[static_cast<std::size_t>(s)]++)] = t;
  }
  // Unique predecessor lists (sorted) and the matching unique successor lists.
  std::vector<std::pair<int, int>> pairs = ie;
  std::sort(pairs.begin(), pairs.end());
  pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
  d.pred_off.assign(static_cast<std::size_t>(d.m) + 1, 0);
  d.usucc_off.assign(static_cast<std::size_t>(d.m) + 1, 0);
  for (auto [t, s] : pairs) {
    ++d.pred_off[static_cast<std::size_t>(t) + 1];
    ++d.usucc_off[static_cast<std::size_t>(s) + 1];
  }
  for (int j = 0; j < d.m; ++j) {
    d.pred_off[static_cast<std::size_t>(j) + 1] += d.pred_off[static_cast<std::size_t>(j)];
    d.usucc_off[static_cast<std::size_t>(j) + 1] += d.usucc_off[static_cast<std::size_t>(j)];
  }
  d.pred.resize(pairs.size());
  d.usucc.resize(pairs.size());
  std::vector<int> pf(d.pred_off.begin(), d.pred_off.end() - 1), sf(d.usucc_off.begin(), d.usucc_off.end() - 1);
  for (auto [t, s] : pairs) {
    d.pred[static_cast<std::size_t>(pf[static_cast<std::size_t>(t)]++)] = s;
    d.usucc[static_cast<std::size_t>(sf[static_cast<std::size_t>(s)]++)] = t;
  }
  return d;
}

int npred(const Dag& d, int j) { return d.pred_off[static_cast<std::size_t>(j) + 1] - d.pred_off[static_cast<std::size_t>(j)]; }

using Step = std::pair<NodeType, std::vector<int>>;  // type, rows (ascending)

// Letter order of the types (c d e g i m n o r s), used by beam / optimal expansion.
const std::array<int, kTypes>& letter_order() {
  static const std::array<int, kTypes> order = [] {
    std::array<int, kTypes> o{};
    for (int i = 0; i < kTypes; ++i) o[static_cast<std::size_t>(i)] = i;
    std::sort(o.begin(), o.end(), [](int a, int b) {
      return type_code(static_cast<NodeType>(a)) < type_code(static_cast<NodeType>(b));
    });
    return o;
  }();
  return order;
}

bool letters_less(const std::vector<NodeType>& x, const std::vector<NodeType>& y) {
  return std::lexicographical_compare(x.begin(), x.end(), y.begin(), y.end(), [](NodeType p, NodeType q) {
    return type_code(p) < type_code(q);
  });
}

// Incremental frontier: per-type ready lists over interior indices.
struct Frontier {
  std::vector<int> missing;                   // unique preds not yet done
  std::array<std::vector<int>, kTypes> ready;  // interior indices (unsorted)
  int remaining = 0;

  explicit Frontier(const Dag& d) : missing(static_cast<std::size_t>(d.m)), remaining(d.m) {
    for (int j = 0; j < d.m; ++j) {
      missing[static_cast<std::size_t>(j)] = npred(d, j);
      if (missing[static_cast<std::size_t>(j)] == 0) ready[d.type[static_cast<std::size_t>(j)]].push_back(j);
    }
  }

  // Takes every ready node of type t; returns their rows ascending.
  std::vector<int> take(const Dag& d, int t) {
    std::vector<int> nodes = std::move(ready[static_cast<std::size_t>(t)]);
    ready[static_cast<std::size_t>(t)].clear();
    std::sort(nodes.begin(), nodes.end());
    for (int j : nodes) {
      for (int k = d.usucc_off[static_cast<std::size_t>(j)]; k < d.usucc_off[static_cast<std::size_t>(j) + 1]; ++k) {
        const int s = d.usucc[static_cast<std::size_t>(k)];
        if (--missing[static_cast<std::size_t>(s)] == 0) ready[d.type[static_cast<std::size_t>(s)]].push_back(s);
      }
    }
    remaining -= static_cast<int>(nodes.size());
    for (int& j : nodes) j = d.row[static_cast<std::size_t>(j)];
    return nodes;
  }
};

std::vector<Step> greedy_steps(const Dag& d) {
  Frontier f(d);
  std::vector<Step> steps;
  while (f.remaining > 0) {
    int best = -1;
    for (int t = 0; t < kTypes; ++t) {  // enum order, strict '>' keeps the lowest on ties
      if (!f.ready[static_cast<std::size_t>(t)].empty() &&
          (best < 0 || f.ready[static_cast<std::size_t>(t)].size() > f.ready[static_cast<std::size_t>(best)].size())) {
        best = t;
      }
    }
    steps.emplace_back(static_cast<NodeType>(best), f.take(d, best));
  }
  return steps;
}

std::vector<Step> one_by_one_steps(const Dag& d) {
  std::vector<int> indeg(static_cast<std::size_t>(d.m));
  std::priority_queue<int, std::vector<int>, std::greater<int>> heap;
  for (int j = 0; j < d.m; ++j) {
    indeg[static_cast<std::size_t>(j)] = npred(d, j);
    if (indeg[static_cast<std::size_t>(j)] == 0) heap.push(d.row[static_cast<std::size_t>(j)]);
  }
  std::vector<Step> steps;
  while (!heap.empty()) {
    const int r = heap.top();
    heap.pop();
    const int j = d.idx[static_cast<std::size_t>(r)];
    steps.emplace_back(static_cast<NodeType>(d.type[static_cast<std::size_t>(j)]), std::vector<int>{r});
    for (int k = d.esucc_off[static_cast<std::size_t>(j)]; k < d.esucc_off[static_cast<std::size_t>(j) + 1]; ++k) {
      const int w = d.esucc[static_cast<std::size_t>(k)];
      if (--indeg[static_cast<std::size_t>(w)] == 0) heap.push(d.row[static_cast<std::size_t>(w)]);
    }
  }
  return steps;
}

std::vector<Step> replay(const Dag& d, const std::vector<NodeType>& types) {
  Frontier f(d);
  std::vector<Step> steps;
  for (NodeType t : types) {
    if (t == NodeType::In || t == NodeType::Out) fail("type string steps must be interior types");
    if (f.ready[static_cast<std::size_t>(t)].empty()) {
      fail(std::string("type string step '") + type_code(t) + "' has no computable node");
    }
    steps.emplace_back(t, f.take(d, static_cast<int>(t)));
  }
  if (f.remaining != 0) fail("type string leaves interior nodes unprocessed");
  return steps;
}

// ---- search strategies over covered sets --------------------------------------------

using Bits = std::vector<std::uint64_t>;

struct BitsHash {
  std::size_t operator()(const Bits& b) const {
    std::uint64_t h = 0x9E3779B97F4A7C15ull;
    for (std::uint64_t w : b) h = (h ^ w) * 0x100000001B3ull + (h >> 29);
    return static_cast<std::size_t>(h);
  }
};

inline bool has(const Bits& b, int i) { return (b[static_cast<std::size_t>(i) >> 6] >> (i & 63)) & 1u; }
inline void put(Bits& b, int i) { b[static_cast<std::size_t>(i) >> 6] |= std::uint64_t{1} << (i & 63); }

// Beam candidate: covered set plus its ready frontier per type.
struct Cand {
  Bits done;
  std::array<std::vector<int>, kTypes> ready;
  std::vector<NodeType> types;
  int count = 0;
};

// Successor frontier after covering `take` (all of one type's ready list).
void advance(const Dag& d, const Cand& parent, int t, Cand& child) {
  child.done = parent.done;
  const auto& take = parent.ready[static_cast<std::size_t>(t)];
  for (int j : take) put(child.done, j);
  for (int u = 0; u < kTypes; ++u) {
    if (u != t) child.ready[static_cast<std::size_t>(u)] = parent.ready[static_cast<std::size_t>(u)];
  }
  child.ready[static_cast<std::size_t>(t)].clear();
  for (int j : take) {
    for (int k = d.usucc_off[static_cast<std::size_t>(j)]; k < d.usucc_off[static_cast<std::size_t>(j) + 1]; ++k) {
      const int s = d.usucc[static_cast<std::size_t>(k)];
      if (has(child.done, s)) continue;
      bool ok = true;
      for (int q = d.pred_off[static_cast<std::size_t>(s)]; q < d.pred_off[static_cast<std::size_t>(s) + 1]; ++q) {
        if (!has(child.done, d.pred[static_cast<std::size_t>(q)])) {
          ok = false;
          break;
        }
      }
      if (ok) child.ready[d.type[static_cast<std::size_t>(s)]].push_back(s);
    }
  }
  // A node completed by several members of `take` was pushed once per member.
  for (auto& r : child.ready) {
    std::sort(r.begin(), r.end());
    r.erase(std::unique(r.begin(), r.end()), r.end());
  }
  child.types = parent.types;
  child.types.push_back(static_cast<NodeType>(t));
  child.count = parent.count + static_cast<int>(take.size());
}

std::vector<NodeType> beam_steps(const Dag& d, int width) {
  if (width < 1) fail("beam width must be >= 1");
  if (d.m == 0) return {};
  Cand root;
  root.done.assign(static_cast<std::size_t>((d.m + 63) / 64), 0);
  for (int j = 0; j < d.m; ++j) {
    if (npred(d, j) == 0) root.ready[d.type[static_cast<std::size_t>(j)]].push_back(j);
  }
  for (auto& r : root.ready) std::sort(r.begin(), r.end());
  std::vector<Cand> beam;
  beam.push_back(std::move(root));
  for (int iter = 0; iter < d.m; ++iter) {
    std::vector<Cand> uniq;
    std::unordered_map<Bits, std::size_t, BitsHash> seen;
    for (const Cand& c : beam) {
      for (int t : letter_order()) {
        if (c.ready[static_cast<std::size_t>(t)].empty()) continue;
        Cand nc;
        advance(d, c, t, nc);
        auto [it, fresh] = seen.try_emplace(nc.done, uniq.size());
        if (fresh) {
          uniq.push_back(std::move(nc));
        } else if (letters_less(nc.types, uniq[it->second].types)) {
          uniq[it->second] = std::move(nc);
        }
      }
    }
    std::sort(uniq.begin(), uniq.end(), [](const Cand& x, const Cand& y) {
      if (x.count != y.count) return x.count > y.count;
      if (x.types.size() != y.types.size()) return x.types.size() < y.types.size();
      return letters_less(x.types, y.types);
    });
    if (static_cast<int>(uniq.size()) > width) uniq.resize(static_cast<std::size_t>(width));
    beam = std::move(uniq);
    if (beam.front().count == d.m) return beam.front().types;
  }
  fail("beam search failed to cover the graph");
}

std::vector<NodeType> optimal_steps(const Dag& d, int node_cap) {
  if (d.n > node_cap) {
    std::ostringstream os;
    os << "optimal scheduling is capped at " << node_cap << " nodes (graph has " << d.n
       << "); use the beam strategy or raise the cap";
    fail(os.str());
  }
  if (d.m == 0) return {};
  const std::size_t words = static_cast<std::size_t>((d.m + 63) / 64);
  std::vector<Bits> states{Bits(words, 0)};
  std::vector<std::pair<int, NodeType>> parent{{-1, NodeType::In}};
  std::unordered_map<Bits, int, BitsHash> index{{states[0], 0}};
  std::deque<int> queue{0};
  std::array<std::vector<int>, kTypes> comp;
  while (!queue.empty()) {
    const int s = queue.front();
    queue.pop_front();
    const Bits done = states[static_cast<std::size_t>(s)];
    for (auto& c : comp) c.clear();
    for (int j = 0; j < d.m; ++j) {
      if (has(done, j)) continue;
      bool ok = true;
      for (int q = d.pred_off[static_cast<std::size_t>(j)]; q < d.pred_off[static_cast<std::size_t>(j) + 1]; ++q) {
        if (!has(done, d.pred[static_cast<std::size_t>(q)])) {
          ok = false;
          break;
        }
      }
      if (ok) comp[d.type[static_cast<std::size_t>(j)]].push_back(j);
    }
    for (int t : letter_order()) {
      if (comp[static_cast<std::size_t>(t)].empty()) continue;
      Bits next = done;
      for (int j : comp[static_cast<std::size_t>(t)]) put(next, j);
      if (index.count(next)) continue;
      const int id = static_cast<int>(states.size());
      index.emplace(next, id);
      states.push_back(next);
      parent.emplace_back(s, static_cast<NodeType>(t));
      int covered = 0;
      for (std::uint64_t w : next) covered += std::popcount(w);
      if (covered == d.m) {
        std::vector<NodeType> out;
        for (int cur = id; parent[static_cast<std::size_t>(cur)].first >= 0; cur = parent[static_cast<std::size_t>(cur)].first) {
          out.push_back(parent[static_cast<std::size_t>(cur)].second);
        }
        std::reverse(out.begin(), out.end());
        return out;
      }
      queue.push_back(id);
    }
  }
  fail("optimal search failed to cover the graph");
}

Schedule assemble(const Dag& d, std::vector<Step>&& steps) {
  Schedule s;
  s.type_string.push_back(NodeType::In);
  s.subsets.push_back(d.in_rows);
  for (auto& [t, rows] : steps) {
    s.type_string.push_back(t);
    s.subsets.push_back(std::move(rows));
  }
  if (!d.out_rows.empty()) {
    s.type_string.push_back(NodeType::Out);
    s.subsets.push_back(d.out_rows);
  }
  return s;
}

// Occurrence index of every row within its type, in the given node order.
std::vector<int> occurrences(const std::vector<NodeType>& types) {
  std::vector<int> occ(types.size());
  int counter[kTypes] = {};
  for (std::size_t r = 0; r < types.size(); ++r) occ[r] = counter[static_cast<int>(types[r])]++;
  return occ;
}

}  // namespace

std::string_view strategy_name(Strategy s) {
  switch (s) {
    case Strategy::OneByOne: return "one-by-one";
    case Strategy::Greedy: return "greedy";
    case Strategy::Beam: return "beam";
    case Strategy::Optimal: return "optimal";
  }
  return "?";
}

std::optional<Strategy> strategy_from_name(std::string_view name) {
  if (name == "one-by-one" || name == "one_by_one") return Strategy::OneByOne;
  if (name == "greedy") return Strategy::Greedy;
  if (name == "beam") return Strategy::Beam;
  if (name == "optimal") return Strategy::Optimal;
  return std::nullopt;
}

std::string Schedule::type_codes() const {
  std::string s;
  for (NodeType t : type_string) s.push_back(type_code(t));
  return s;
}

Schedule make_schedule(const FlatGraph& fg, const ScheduleOptions& options) {
  const Dag d = analyze(fg);
  switch (options.strategy) {
    case Strategy::OneByOne: return assemble(d, one_by_one_steps(d));
    case Strategy::Greedy: return assemble(d, greedy_steps(d));
    case Strategy::Beam: return assemble(d, replay(d, beam_steps(d, options.beam_width)));
    case Strategy::Optimal: return assemble(d, replay(d, optimal_steps(d, options.optimal_node_cap)));
  }
  fail("unknown strategy");
}

Schedule make_schedule(const FlatGraph& fg, Strategy strategy) {
  ScheduleOptions o;
  o.strategy = strategy;
  return make_schedule(fg, o);
}

Schedule schedule_from_type_string(const FlatGraph& fg, const std::vector<NodeType>& steps) {
  const Dag d = analyze(fg);
  return assemble(d, replay(d, steps));
}

void validate_schedule(const FlatGraph& fg, const Schedule& s) {
  const int n = fg.num_nodes();
  if (s.subsets.size() != s.type_string.size() || s.subsets.empty()) fail("schedule: type string and subsets disagree");
  if (s.type_string[0] != NodeType::In) fail("schedule: type string must start with in");
  std::vector<int> step_of(static_cast<std::size_t>(n), -1);
  for (std::size_t k = 0; k < s.subsets.size(); ++k) {
    if (k > 0 && s.subsets[k].empty()) fail("schedule: empty subset at step " + std::to_string(k));
    for (int r : s.subsets[k]) {
      if (r < 0 || r >= n) fail("schedule: partition violated: unknown node " + std::to_string(r));
      if (step_of[static_cast<std::size_t>(r)] >= 0) fail("schedule: partition violated: node " + std::to_string(r) + " appears twice");
      step_of[static_cast<std::size_t>(r)] = static_cast<int>(k);
      if (fg.node_types[static_cast<std::size_t>(r)] != s.type_string[k]) {
        std::ostringstream os;
        os << "schedule: homogeneity violated: node " << r << " of type " << type_name(fg.node_types[static_cast<std::size_t>(r)])
           << " in a " << type_name(s.type_string[k]) << " step " << k;
        fail(os.str());
      }
    }
  }
  const int last = static_cast<int>(s.subsets.size()) - 1;
  for (int r = 0; r < n; ++r) {
    const int k = step_of[static_cast<std::size_t>(r)];
    if (k < 0) fail("schedule: partition violated: node " + std::to_string(r) + " missing");
    const NodeType t = fg.node_types[static_cast<std::size_t>(r)];
    if (t == NodeType::In && k != 0) fail("schedule: in node " + std::to_string(r) + " must be in V_0");
    if (t == NodeType::Out && k != last) fail("schedule: out node " + std::to_string(r) + " must be in the final subset");
  }
  for (const Edge& e : fg.edges) {
    const int a = step_of[static_cast<std::size_t>(e.src)], b = step_of[static_cast<std::size_t>(e.dst)];
    if (a >= b) {
      std::ostringstream os;
      os << "schedule: causality violated: edge " << e.src << "->" << e.dst << " goes from step " << a << " to step " << b;
      fail(os.str());
    }
  }
}

std::vector<int> optimize_node_order(const FlatGraph& fg, const Schedule& s) {
  // Counting-sort form of the reference's stable sort by step.
  const int n = fg.num_nodes();
  std::vector<int> step_of(static_cast<std::size_t>(n), -1);
  for (std::size_t k = 0; k < s.subsets.size(); ++k) {
    for (int r : s.subsets[k]) step_of[static_cast<std::size_t>(r)] = static_cast<int>(k);
  }
  std::vector<int> start(s.subsets.size() + 1, 0);
  for (int r = 0; r < n; ++r) {
    if (step_of[static_cast<std::size_t>(r)] < 0) fail("optimize_node_order: schedule does not cover node " + std::to_string(r));
    ++start[static_cast<std::size_t>(step_of[static_cast<std::size_t>(r)]) + 1];
  }
  for (std::size_t k = 0; k + 1 < start.size(); ++k) start[k + 1] += start[k];
  std::vector<int> sigma(static_cast<std::size_t>(n));
  for (int r = 0; r < n; ++r) sigma[static_cast<std::size_t>(r)] = start[static_cast<std::size_t>(step_of[static_cast<std::size_t>(r)])]++;
  return sigma;
}

std::vector<int> inverse_permutation(const std::vector<int>& sigma) {
  std::vector<int> inv(sigma.size());
  for (std::size_t i = 0; i < sigma.size(); ++i) inv[static_cast<std::size_t>(sigma[i])] = static_cast<int>(i);
  return inv;
}

FlatGraph reorder_flat(const FlatGraph& fg, const std::vector<int>& sigma) {
  const int n = fg.num_nodes();
  FlatGraph out;
  out.node_types.resize(static_cast<std::size_t>(n));
  for (int r = 0; r < n; ++r) out.node_types[static_cast<std::size_t>(sigma[static_cast<std::size_t>(r)])] = fg.node_types[static_cast<std::size_t>(r)];
  out.edges.reserve(fg.edges.size());
  for (const Edge& e : fg.edges) {
    out.edges.push_back(Edge{sigma[static_cast<std::size_t>(e.src)], sigma[static_cast<std::size_t>(e.dst)], e.outlet, e.inlet});
  }
  out.num_inputs = fg.num_inputs;
  out.num_outputs = fg.num_outputs;
  // Parameter rows follow their nodes (row l of P[t] = l-th occurrence of t).
  const std::vector<int> inv = inverse_permutation(sigma);
  const std::vector<int> occ = occurrences(fg.node_types);
  for (const auto& [t, table] : fg.params.tables) {
    ParamMatrix m(table.rows, table.cols);
    int next = 0;
    for (int j = 0; j < n; ++j) {
      const int old = inv[static_cast<std::size_t>(j)];
      if (fg.node_types[static_cast<std::size_t>(old)] != t) continue;
      auto src = table.row(occ[static_cast<std::size_t>(old)]);
      std::copy(src.begin(), src.end(), m.row(next++).begin());
    }
    out.params.tables.emplace(t, std::move(m));
  }
  return out;
}

ParamStore RenderData::reorder_params(const ParamStore& original) const {
  ParamStore out;
  for (const auto& [t, src_rows] : param_source_rows) {
    auto it = original.tables.find(t);
    if (it == original.tables.end() || it->second.rows != static_cast<int>(src_rows.size()) ||
        it->second.cols != param_width(t)) {
      fail(std::string("reorder_params: missing or misshaped table for ") + std::string(type_name(t)));
    }
    ParamMatrix m(it->second.rows, it->second.cols);
    for (std::size_t j = 0; j < src_rows.size(); ++j) {
      auto src = it->second.row(src_rows[j]);
      std::copy(src.begin(), src.end(), m.row(static_cast<int>(j)).begin());
    }
    out.tables.emplace(t, std::move(m));
  }
  return out;
}

RenderData compute_render_data(const FlatGraph& fg, const ScheduleOptions& options) {
  RenderData rd;
  rd.schedule = make_schedule(fg, options);
  rd.sigma = optimize_node_order(fg, rd.schedule);
  rd.flat = reorder_flat(fg, rd.sigma);
  const int n = fg.num_nodes();
  rd.num_inputs = fg.num_inputs;
  rd.buffer_rows = n;
  rd.output_begin = n - fg.num_outputs;

  const std::vector<int> occ = occurrences(rd.flat.node_types);
  // Incoming edges per destination row, edge order (CSR).
  std::vector<int> off(static_cast<std::size_t>(n) + 1, 0);
  for (const Edge& e : rd.flat.edges) ++off[static_cast<std::size_t>(e.dst) + 1];
  for (int v = 0; v < n; ++v) off[static_cast<std::size_t>(v) + 1] += off[static_cast<std::size_t>(v)];
  std::vector<int> src(rd.flat.edges.size()), fill(off.begin(), off.end() - 1);
  for (const Edge& e : rd.flat.edges) src[static_cast<std::size_t>(fill[static_cast<std::size_t>(e.dst)]++)] = e.src;

  int row0 = static_cast<int>(rd.schedule.subsets[0].size());
  rd.steps.reserve(rd.schedule.subsets.size());
  for (std::size_t k = 1; k < rd.schedule.subsets.size(); ++k) {
    StepIndex si;
    si.type = rd.schedule.type_string[k];
    const int size = static_cast<int>(rd.schedule.subsets[k].size());
    si.store_begin = row0;
    si.store_end = row0 + size;
    if (param_width(si.type) > 0) {
      si.param_begin = occ[static_cast<std::size_t>(row0)];
      si.param_end = si.param_begin + size;
    }
    const int e0 = off[static_cast<std::size_t>(row0)], e1 = off[static_cast<std::size_t>(row0 + size)];
    si.gather.assign(src.begin() + e0, src.begin() + e1);
    si.aggregate.reserve(static_cast<std::size_t>(e1 - e0));
    for (int slot = 0; slot < size; ++slot) {
      si.aggregate.insert(si.aggregate.end(), static_cast<std::size_t>(off[static_cast<std::size_t>(row0 + slot) + 1] - off[static_cast<std::size_t>(row0 + slot)]), slot);
    }
    rd.steps.push_back(std::move(si));
    row0 += size;
  }

  const std::vector<int> inv = inverse_permutation(rd.sigma);
  const std::vector<int> old_occ = occurrences(fg.node_types);
  for (int j = 0; j < n; ++j) {
    const NodeType t = rd.flat.node_types[static_cast<std::size_t>(j)];
    if (param_width(t) == 0) continue;
    rd.param_source_rows[t].push_back(old_occ[static_cast<std::size_t>(inv[static_cast<std::size_t>(j)])]);
  }
  return rd;
}

}  // namespace mixgraph
