// Graph documents (JSON), DOT export and stereo float WAV I/O: the file-level drop-in.
//
// Drop-in for `proj/include/mixgraph/graph_io.hpp:9-29` / `proj/src/graph_io.cpp:19-143`
// and `proj/include/mixgraph/wav.hpp:9-14` / `proj/src/wav.cpp:39-133`: same functions,
// document layout, error behaviour (std::invalid_argument "graph document: ..." for
// documents, std::runtime_error "read_wav: ..." / "write_wav: ..." for audio files).
//
// Document layout (graph_io.hpp:11-18):
//   {"edges": [{"dst": 1, "src": 0}, ...], "nodes": [{"id": 0, "type": "in"}, ...],
//    "params": {"gain": [[0.0, 0.0], ...], ...}, "version": 1}
// written with sorted keys and two-space indentation; `outlet`/`inlet` only when non-zero;
// numbers in shortest round-trip form, so every parameter value reloads bit-exactly.
// The reference's JSON library (nlohmann/json, un-vendored) is replaced by a small parser
// and writer here (graph_io.cpp); its observable format is reproduced.
#pragma once

#include <string>
#include <utility>

#include "mixgraph_b200/audio_buffer.hpp"
#include "mixgraph_b200/graph.hpp"

namespace mixgraph {

std::string graph_to_json(const Graph& g, const ParamStore& params);
std::pair<Graph, ParamStore> graph_from_json(const std::string& text);

void save_graph(const Graph& g, const ParamStore& params, const std::string& path);
std::pair<Graph, ParamStore> load_graph(const std::string& path);

// Deterministic DOT document, one node per graph node labelled with its letter code.
std::string export_dot(const Graph& g);

// 32-bit float PCM RIFF/WAVE, little-endian, stereo; batch axis must be 1.
void write_wav(const AudioBuffer& buffer, const std::string& path);
AudioBuffer read_wav(const std::string& path);

}  // namespace mixgraph
