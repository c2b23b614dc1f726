// Graph documents, DOT export and float WAV files (host-only, no device work).
//
// Behaviour follows `proj/src/graph_io.cpp:19-143` and `proj/src/wav.cpp:39-133`; the
// reference's JSON dependency (nlohmann/json, not vendored in the snapshot) is replaced by
// the small DOM below. What is reproduced of it is what a document shows: objects with
// sorted keys (std::map), `dump(2)` layout, integers as integers and doubles in the
// shortest round-trip form laid out like its `to_chars` (fixed notation for decimal
// exponents in (-4, 15], `d.ddde+XX` otherwise, `.0` on integral values, non-finite as
// null), last value wins for a repeated key.
#include "mixgraph_b200/graph_io.hpp"

#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string_view>
#include <vector>

namespace mixgraph {

namespace {

[[noreturn]] void fail(const std::string& msg) { throw std::invalid_argument(msg); }
[[noreturn]] void fail_doc(const std::string& msg) { fail("graph document: " + msg); }

// ---- JSON DOM ----------------------------------------------------------------------------

struct Json {
  enum class Kind { Null, Bool, Int, Float, String, Array, Object } kind = Kind::Null;
  bool b = false;
  std::int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Json> items;        // Array elements, or Object values (parallel to keys)
  std::vector<std::string> keys;  // Object keys, sorted, unique

  bool is_object() const { return kind == Kind::Object; }
  bool is_array() const { return kind == Kind::Array; }
  bool is_number() const { return kind == Kind::Int || kind == Kind::Float; }
  const Json* find(std::string_view key) const {
    if (!is_object()) return nullptr;
    for (std::size_t k = 0; k < keys.size(); ++k) {
      if (keys[k] == key) return &items[k];
    }
    return nullptr;
  }
  // Element count as the reference's library reports it: arrays/objects their size, null 0,
  // any other value 1.
  std::size_t size() const {
    if (kind == Kind::Array || kind == Kind::Object) return items.size();
    return kind == Kind::Null ? 0 : 1;
  }
  double as_double(const std::string& what) const {
    if (kind == Kind::Int) return static_cast<double>(i);
    if (kind == Kind::Float) return d;
    fail_doc(what + " must be a number");
  }
  int as_int(const std::string& what) const {
    if (kind == Kind::Int) return static_cast<int>(i);
    if (kind == Kind::Float) return static_cast<int>(d);
    fail_doc(what + " must be a number");
  }
};

class Parser {
 public:
  explicit Parser(std::string_view t) : t_(t) {}

  Json document() {
    Json v = value(0);
    ws();
    if (p_ != t_.size()) error("unexpected trailing characters");
    return v;
  }

 private:
  std::string_view t_;
  std::size_t p_ = 0;

  [[noreturn]] void error(const std::string& what) const {
    std::size_t line = 1, col = 1;
    for (std::size_t k = 0; k < p_ && k < t_.size(); ++k) {
      if (t_[k] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
    }
    fail_doc("parse error at line " + std::to_string(line) + ", column " + std::to_string(col) + ": " + what);
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < t_.size() && t_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) error(std::string("expected '") + c + "'");
  }
  bool literal(std::string_view w) {
    if (t_.substr(p_, w.size()) == w) {
      p_ += w.size();
      return true;
    }
    return false;
  }

  Json value(int depth) {
    if (depth > 512) error("nesting too deep");
    ws();
    if (p_ >= t_.size()) error("unexpected end of input");
    Json v;
    const char c = t_[p_];
    if (c == '{') {
      ++p_;
      v.kind = Json::Kind::Object;
      if (eat('}')) return v;
      do {
        ws();
        std::string k = string();
        expect(':');
        Json item = value(depth + 1);
        // Sorted keys, a repeated key replaces the earlier value.
        auto it = std::lower_bound(v.keys.begin(), v.keys.end(), k);
        const std::size_t at = static_cast<std::size_t>(it - v.keys.begin());
        if (it != v.keys.end() && *it == k) {
          v.items[at] = std::move(item);
        } else {
          v.keys.insert(it, std::move(k));
          v.items.insert(v.items.begin() + static_cast<std::ptrdiff_t>(at), std::move(item));
        }
      } while (eat(','));
      expect('}');
    } else if (c == '[') {
      ++p_;
      v.kind = Json::Kind::Array;
      if (eat(']')) return v;
      do {
        v.items.push_back(value(depth + 1));
      } while (eat(','));
      expect(']');
    } else if (c == '"') {
      v.kind = Json::Kind::String;
      v.s = string();
    } else if (literal("true")) {
      v.kind = Json::Kind::Bool;
      v.b = true;
    } else if (literal("false")) {
      v.kind = Json::Kind::Bool;
    } else if (literal("null")) {
      v.kind = Json::Kind::Null;
    } else if (c == '-' || (c >= '0' && c <= '9')) {
      number(v);
    } else {
      error(std::string("invalid literal '") + c + "'");
    }
    return v;
  }

  std::string string() {
    if (p_ >= t_.size() || t_[p_] != '"') error("expected string");
    ++p_;
    std::string out;
    for (;;) {
      if (p_ >= t_.size()) error("unterminated string");
      const char c = t_[p_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) error("control character in string");
      if (c != '\\') {
        out.push_back(c);
        continue;
      }
      if (p_ >= t_.size()) error("unterminated string");
      const char e = t_[p_++];
      switch (e) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          std::uint32_t cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (!literal("\\u")) error("unpaired surrogate");
            const std::uint32_t lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) error("unpaired surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          }
          utf8(out, cp);
          break;
        }
        default: error("invalid escape");
      }
    }
  }
  std::uint32_t hex4() {
    if (p_ + 4 > t_.size()) error("truncated \\u escape");
    std::uint32_t v = 0;
    auto [ptr, ec] = std::from_chars(t_.data() + p_, t_.data() + p_ + 4, v, 16);
    if (ec != std::errc() || ptr != t_.data() + p_ + 4) error("invalid \\u escape");
    p_ += 4;
    return v;
  }
  static void utf8(std::string& out, std::uint32_t cp) {
    if (cp < 0x80) {
      out.push_back(static_cast<char>(cp));
    } else if (cp < 0x800) {
      out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
      out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else {
      out.push_back(static_cast<char>(0xF0 | (cp >> 18)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    }
  }
  // JSON number grammar: -?(0|[1-9][0-9]*)(.[0-9]+)?([eE][+-]?[0-9]+)? ; integers without
  // fraction/exponent stay integers (floats when out of int64 range).
  void number(Json& v) {
    const std::size_t b = p_;
    auto digits = [&] {
      const std::size_t s = p_;
      while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
      return p_ - s;
    };
    if (t_[p_] == '-') ++p_;
    if (p_ < t_.size() && t_[p_] == '0') {
      ++p_;
    } else if (digits() == 0) {
      error("invalid number");
    }
    bool integral = true;
    if (p_ < t_.size() && t_[p_] == '.') {
      ++p_;
      integral = false;
      if (digits() == 0) error("invalid number");
    }
    if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
      ++p_;
      integral = false;
      if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
      if (digits() == 0) error("invalid number");
    }
    const char* first = t_.data() + b;
    const char* last = t_.data() + p_;
    if (integral) {
      std::int64_t iv = 0;
      auto [ptr, ec] = std::from_chars(first, last, iv);
      if (ec == std::errc() && ptr == last) {
        v.kind = Json::Kind::Int;
        v.i = iv;
        return;
      }
    }
    double dv = 0.0;
    auto [ptr, ec] = std::from_chars(first, last, dv);
    if (ptr != last || (ec != std::errc() && ec != std::errc::result_out_of_range)) error("invalid number");
    if (ec == std::errc::result_out_of_range) error("number out of range");
    v.kind = Json::Kind::Float;
    v.d = dv;
  }
};

// ---- writer --------------------------------------------------------------------------------

// Shortest round-trip digits, laid out like the reference library's dtoa (`dump`).
void put_double(std::string& out, double x) {
  if (!std::isfinite(x)) {
    out += "null";
    return;
  }
  if (x == 0.0) {
    out += std::signbit(x) ? "-0.0" : "0.0";
    return;
  }
  char buf[64];
  const auto r = std::to_chars(buf, buf + sizeof(buf), x, std::chars_format::scientific);
  std::string_view sv(buf, static_cast<std::size_t>(r.ptr - buf));
  if (sv.front() == '-') {
    out.push_back('-');
    sv.remove_prefix(1);
  }
  const std::size_t epos = sv.find('e');
  std::string digits;
  for (char c : sv.substr(0, epos)) {
    if (c != '.') digits.push_back(c);
  }
  int e10 = 0;
  std::string_view es = sv.substr(epos + 1);
  if (es.front() == '+') es.remove_prefix(1);
  std::from_chars(es.data(), es.data() + es.size(), e10);
  const int k = static_cast<int>(digits.size());
  const int n = e10 + 1;  // value = 0.d1..dk x 10^n
  constexpr int kMinExp = -4, kMaxExp = 15;
  if (k <= n && n <= kMaxExp) {
    out += digits;
    out.append(static_cast<std::size_t>(n - k), '0');
    out += ".0";
  } else if (0 < n && n <= kMaxExp) {
    out.append(digits, 0, static_cast<std::size_t>(n));
    out.push_back('.');
    out.append(digits, static_cast<std::size_t>(n));
  } else if (kMinExp < n && n <= 0) {
    out += "0.";
    out.append(static_cast<std::size_t>(-n), '0');
    out += digits;
  } else {
    out.push_back(digits[0]);
    if (k > 1) {
      out.push_back('.');
      out.append(digits, 1);
    }
    int ee = n - 1;
    out.push_back('e');
    out.push_back(ee < 0 ? '-' : '+');
    ee = std::abs(ee);
    if (ee < 10) out.push_back('0');
    out += std::to_string(ee);
  }
}

void indent(std::string& out, int level) { out.append(static_cast<std::size_t>(2 * level), ' '); }

}  // namespace

std::string graph_to_json(const Graph& g, const ParamStore& params) {
  // Keys in sorted order at every level: edges, nodes, params, version.
  std::string out = "{\n";
  indent(out, 1);
  out += "\"edges\": ";
  if (g.edges().empty()) {
    out += "[]";
  } else {
    out += "[\n";
    for (std::size_t i = 0; i < g.edges().size(); ++i) {
      const Edge& e = g.edges()[i];
      indent(out, 2);
      out += "{\n";
      indent(out, 3);
      out += "\"dst\": " + std::to_string(e.dst);
      if (e.inlet != 0) {
        out += ",\n";
        indent(out, 3);
        out += "\"inlet\": " + std::to_string(e.inlet);
      }
      if (e.outlet != 0) {
        out += ",\n";
        indent(out, 3);
        out += "\"outlet\": " + std::to_string(e.outlet);
      }
      out += ",\n";
      indent(out, 3);
      out += "\"src\": " + std::to_string(e.src) + "\n";
      indent(out, 2);
      out += i + 1 < g.edges().size() ? "},\n" : "}\n";
    }
    indent(out, 1);
    out += "]";
  }
  out += ",\n";
  indent(out, 1);
  out += "\"nodes\": ";
  if (g.num_nodes() == 0) {
    out += "[]";
  } else {
    out += "[\n";
    for (int v = 0; v < g.num_nodes(); ++v) {
      indent(out, 2);
      out += "{\n";
      indent(out, 3);
      out += "\"id\": " + std::to_string(v) + ",\n";
      indent(out, 3);
      out += "\"type\": \"" + std::string(type_name(g.node_type(v))) + "\"\n";
      indent(out, 2);
      out += v + 1 < g.num_nodes() ? "},\n" : "}\n";
    }
    indent(out, 1);
    out += "]";
  }
  if (!params.tables.empty()) {
    // Object keys sorted by type name.
    std::vector<std::pair<std::string, const ParamMatrix*>> named;
    for (const auto& [t, m] : params.tables) named.emplace_back(std::string(type_name(t)), &m);
    std::sort(named.begin(), named.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    out += ",\n";
    indent(out, 1);
    out += "\"params\": {\n";
    for (std::size_t ti = 0; ti < named.size(); ++ti) {
      const ParamMatrix& m = *named[ti].second;
      indent(out, 2);
      out += "\"" + named[ti].first + "\": ";
      if (m.rows == 0) {
        out += "[]";
      } else {
        out += "[\n";
        for (int r = 0; r < m.rows; ++r) {
          indent(out, 3);
          if (m.cols == 0) {
            out += "[]";
          } else {
            out += "[\n";
            for (int c = 0; c < m.cols; ++c) {
              indent(out, 4);
              put_double(out, m.at(r, c));
              out += c + 1 < m.cols ? ",\n" : "\n";
            }
            indent(out, 3);
            out += "]";
          }
          out += r + 1 < m.rows ? ",\n" : "\n";
        }
        indent(out, 2);
        out += "]";
      }
      out += ti + 1 < named.size() ? ",\n" : "\n";
    }
    indent(out, 1);
    out += "}";
  }
  out += ",\n";
  indent(out, 1);
  out += "\"version\": 1\n}\n";
  return out;
}

std::pair<Graph, ParamStore> graph_from_json(const std::string& text) {
  const Json doc = Parser(text).document();
  const Json* nodes = doc.find("nodes");
  if (!doc.is_object() || !nodes) fail_doc("missing 'nodes'");
  if (!nodes->is_array()) fail_doc("'nodes' must be an array");

  Graph g;
  for (std::size_t i = 0; i < nodes->items.size(); ++i) {
    const Json& jn = nodes->items[i];
    const Json* jt = jn.find("type");
    if (!jt) fail_doc("node " + std::to_string(i) + " missing 'type'");
    if (jt->kind != Json::Kind::String) fail_doc("node " + std::to_string(i) + " 'type' must be a string");
    const auto t = type_from_name(jt->s);
    if (!t) fail_doc("unknown node type '" + jt->s + "'");
    const Json* jid = jn.find("id");
    const int id = jid ? jid->as_int("node " + std::to_string(i) + " 'id'") : static_cast<int>(i);
    if (id != static_cast<int>(i)) {
      fail_doc("node ids must be dense 0..N-1 in order (node " + std::to_string(i) + " has id " + std::to_string(id) + ")");
    }
    g.add_node(*t);
  }
  if (const Json* edges = doc.find("edges")) {
    if (!edges->is_array()) fail_doc("'edges' must be an array");
    for (std::size_t i = 0; i < edges->items.size(); ++i) {
      const Json& je = edges->items[i];
      const Json* s = je.find("src");
      const Json* d = je.find("dst");
      if (!s || !d) fail_doc("edge " + std::to_string(i) + " missing 'src' or 'dst'");
      const std::string what = "edge " + std::to_string(i);
      const Json* o = je.find("outlet");
      const Json* in = je.find("inlet");
      g.connect(s->as_int(what + " 'src'"), d->as_int(what + " 'dst'"), o ? o->as_int(what + " 'outlet'") : 0,
                in ? in->as_int(what + " 'inlet'") : 0);
    }
  }
  g.validate();

  ParamStore params = default_params(g.node_types());
  if (const Json* jp = doc.find("params")) {
    if (!jp->is_object()) fail_doc("'params' must be an object");
    for (std::size_t k = 0; k < jp->keys.size(); ++k) {
      const std::string& name = jp->keys[k];
      const Json& rows = jp->items[k];
      const auto t = type_from_name(name);
      if (!t) fail_doc("unknown parameter type '" + name + "'");
      if (param_width(*t) == 0) fail_doc("type '" + name + "' takes no parameters");
      if (!params.has(*t)) fail_doc("no '" + name + "' nodes in the graph");
      ParamMatrix& table = params.table(*t);
      if (static_cast<int>(rows.size()) != table.rows) {
        fail_doc("'" + name + "' has " + std::to_string(rows.size()) + " rows, expected " + std::to_string(table.rows));
      }
      if (!rows.is_array()) fail_doc("'" + name + "' must be an array of rows");
      for (int r = 0; r < table.rows; ++r) {
        const Json& row = rows.items[static_cast<std::size_t>(r)];
        if (static_cast<int>(row.size()) != table.cols) {
          fail_doc("'" + name + "' row " + std::to_string(r) + " has width " + std::to_string(row.size()) + ", expected " +
                   std::to_string(table.cols));
        }
        if (!row.is_array()) fail_doc("'" + name + "' row " + std::to_string(r) + " must be an array");
        for (int c = 0; c < table.cols; ++c) {
          table.at(r, c) = row.items[static_cast<std::size_t>(c)].as_double("'" + name + "' row " + std::to_string(r) + " values");
        }
      }
    }
  }
  return {std::move(g), std::move(params)};
}

void save_graph(const Graph& g, const ParamStore& params, const std::string& path) {
  std::ofstream out(path, std::ios::binary);
  if (!out) fail("save_graph: cannot open '" + path + "' for writing");
  out << graph_to_json(g, params);
  if (!out) fail("save_graph: write to '" + path + "' failed");
}

std::pair<Graph, ParamStore> load_graph(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) fail("load_graph: cannot open '" + path + "'");
  std::ostringstream buf;
  buf << in.rdbuf();
  return graph_from_json(buf.str());
}

std::string export_dot(const Graph& g) {
  std::string out = "digraph {\n  rankdir=LR;\n";
  for (int v = 0; v < g.num_nodes(); ++v) {
    out += "  n" + std::to_string(v) + " [label=\"" + type_code(g.node_type(v)) + "\"];\n";
  }
  for (const Edge& e : g.edges()) out += "  n" + std::to_string(e.src) + " -> n" + std::to_string(e.dst) + ";\n";
  out += "}\n";
  return out;
}

// ---- WAV -----------------------------------------------------------------------------------

namespace {

[[noreturn]] void wav_fail(const std::string& msg) { throw std::runtime_error(msg); }

void put_le(std::string& out, std::uint32_t v, int bytes) {
  for (int i = 0; i < bytes; ++i) out.push_back(static_cast<char>((v >> (8 * i)) & 0xffu));
}
std::uint32_t get_le(const std::string& s, std::size_t pos, int bytes) {
  std::uint32_t v = 0;
  for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | static_cast<unsigned char>(s[pos + static_cast<std::size_t>(i)]);
  return v;
}
constexpr std::uint16_t kWaveFormatIeeeFloat = 3;

}  // namespace

void write_wav(const AudioBuffer& buffer, const std::string& path) {
  if (buffer.batch != 1) wav_fail("write_wav: only single-source buffers (batch 1) can be written");
  if (buffer.channels != 2) wav_fail("write_wav: only stereo buffers can be written");
  const auto frames = static_cast<std::uint32_t>(buffer.length);
  const auto rate = static_cast<std::uint32_t>(buffer.sample_rate);
  const std::uint32_t data_bytes = frames * 2u * 4u;
  std::string out;
  out.reserve(static_cast<std::size_t>(data_bytes) + 64);
  // RIFF header, fmt (IEEE float, 2 ch, 32 bit), fact (frame count), data.
  out += "RIFF";
  put_le(out, 4 + (8 + 16) + (8 + 4) + 8 + data_bytes, 4);
  out += "WAVEfmt ";
  put_le(out, 16, 4);
  put_le(out, kWaveFormatIeeeFloat, 2);
  put_le(out, 2, 2);
  put_le(out, rate, 4);
  put_le(out, rate * 8u, 4);
  put_le(out, 8, 2);
  put_le(out, 32, 2);
  out += "fact";
  put_le(out, 4, 4);
  put_le(out, frames, 4);
  out += "data";
  put_le(out, data_bytes, 4);
  const std::size_t head = out.size();
  out.resize(head + data_bytes);
  const double* l = buffer.channel(0, 0);
  const double* r = buffer.channel(0, 1);
  char* dst = out.data() + head;
  for (std::uint32_t i = 0; i < frames; ++i) {
    const float lr[2] = {static_cast<float>(l[i]), static_cast<float>(r[i])};
    std::uint32_t bits[2];
    std::memcpy(bits, lr, 8);
    for (int c = 0; c < 2; ++c) {
      for (int b = 0; b < 4; ++b) *dst++ = static_cast<char>((bits[c] >> (8 * b)) & 0xffu);
    }
  }
  std::ofstream file(path, std::ios::binary);
  if (!file) wav_fail("write_wav: cannot open '" + path + "' for writing");
  file.write(out.data(), static_cast<std::streamsize>(out.size()));
  if (!file) wav_fail("write_wav: write to '" + path + "' failed");
}

AudioBuffer read_wav(const std::string& path) {
  std::ifstream file(path, std::ios::binary);
  if (!file) wav_fail("read_wav: cannot open '" + path + "'");
  const std::string data((std::istreambuf_iterator<char>(file)), std::istreambuf_iterator<char>());
  if (data.size() < 12 || data.compare(0, 4, "RIFF") != 0 || data.compare(8, 4, "WAVE") != 0) {
    wav_fail("read_wav: '" + path + "' is not a RIFF/WAVE file");
  }
  bool have_fmt = false;
  std::uint32_t format = 0, channels = 0, bits = 0, rate = 0;
  std::size_t data_pos = 0, data_len = 0;
  for (std::size_t pos = 12; pos + 8 <= data.size();) {
    const std::string id = data.substr(pos, 4);
    const std::uint32_t size = get_le(data, pos + 4, 4);
    const std::size_t body = pos + 8;
    if (body + size > data.size()) wav_fail("read_wav: truncated chunk '" + id + "'");
    if (id == "fmt ") {
      if (size < 16) wav_fail("read_wav: fmt chunk too small");
      format = get_le(data, body, 2);
      channels = get_le(data, body + 2, 2);
      rate = get_le(data, body + 4, 4);
      bits = get_le(data, body + 14, 2);
      have_fmt = true;
    } else if (id == "data") {
      data_pos = body;
      data_len = size;
    }
    pos = body + size + (size & 1u);  // chunks are word-aligned
  }
  if (!have_fmt || data_pos == 0) wav_fail("read_wav: missing fmt or data chunk");
  if (format != kWaveFormatIeeeFloat || bits != 32) wav_fail("read_wav: unsupported encoding (need 32-bit float PCM)");
  if (channels != 2) wav_fail("read_wav: unsupported channel count " + std::to_string(channels) + " (need 2)");
  const std::size_t frames = data_len / 8;
  AudioBuffer buffer(1, 2, static_cast<long>(frames), static_cast<double>(rate));
  double* l = buffer.channel(0, 0);
  double* r = buffer.channel(0, 1);
  for (std::size_t i = 0; i < frames; ++i) {
    float lr[2];
    const std::uint32_t raw[2] = {get_le(data, data_pos + 8 * i, 4), get_le(data, data_pos + 8 * i + 4, 4)};
    std::memcpy(lr, raw, 8);
    l[i] = lr[0];
    r[i] = lr[1];
  }
  return buffer;
}

}  // namespace mixgraph
