// pybind11 module `mixgraph._core`: the Python binding the reference declares
// (`proj/CMakeLists.txt:47-74`, pybind11_add_module(_core bindings/module.cpp), whose source is
// absent from the reference), over the product's C++ API (mixgraph_b200/*.hpp, libmgb200.so).
// Names and argument meaning follow the C++ API; arrays cross as numpy: sources and outputs
// [K][B][2][L] float64 (the reference's AudioBuffer layout), parameter tables as
// {NodeType: [rows][width] float64}.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "mixgraph_b200/graph.hpp"
#include "mixgraph_b200/render.hpp"
#include "mixgraph_b200/schedule.hpp"
#include "mixgraph_b200/types.hpp"

namespace py = pybind11;
using namespace mixgraph;

namespace {

using Array = py::array_t<double, py::array::c_style | py::array::forcecast>;

NodeType to_type(const py::handle& h) {
  if (py::isinstance<py::str>(h)) {
    const std::string s = h.cast<std::string>();
    if (auto t = s.size() == 1 ? type_from_code(s[0]) : type_from_name(s)) return *t;
    throw std::invalid_argument("unknown node type '" + s + "'");
  }
  return h.cast<NodeType>();
}

ParamStore to_store(const py::dict& d) {
  ParamStore s;
  for (auto [k, v] : d) {
    const NodeType t = to_type(k);
    Array a = Array::ensure(v);
    if (!a || a.ndim() != 2 || a.shape(1) != param_width(t)) {
      throw std::invalid_argument(std::string(type_name(t)) + ": parameter table must be [rows][" +
                                  std::to_string(param_width(t)) + "]");
    }
    ParamMatrix m(static_cast<int>(a.shape(0)), static_cast<int>(a.shape(1)));
    std::memcpy(m.values.data(), a.data(), sizeof(double) * m.values.size());
    s.tables.emplace(t, std::move(m));
  }
  return s;
}

py::dict from_store(const ParamStore& s) {
  py::dict d;
  for (const auto& [t, m] : s.tables) {
    Array a({m.rows, m.cols});
    std::memcpy(a.mutable_data(), m.values.data(), sizeof(double) * m.values.size());
    d[py::cast(t)] = a;
  }
  return d;
}

std::vector<AudioBuffer> to_buffers(const Array& src, double fs) {
  if (src.ndim() != 4 || src.shape(2) != 2) throw std::invalid_argument("sources must be [K][B][2][L]");
  std::vector<AudioBuffer> out;
  const auto k = src.shape(0), b = src.shape(1), l = src.shape(3);
  const std::size_t stride = static_cast<std::size_t>(b) * 2 * static_cast<std::size_t>(l);
  for (py::ssize_t i = 0; i < k; ++i) {
    AudioBuffer a(static_cast<int>(b), 2, static_cast<long>(l), fs);
    std::memcpy(a.samples.data(), src.data() + stride * i, sizeof(double) * stride);
    out.push_back(std::move(a));
  }
  return out;
}

Array from_buffers(const std::vector<AudioBuffer>& bufs, int batch, long length) {
  Array a({static_cast<py::ssize_t>(bufs.size()), static_cast<py::ssize_t>(batch), static_cast<py::ssize_t>(2),
           static_cast<py::ssize_t>(length)});
  const std::size_t stride = static_cast<std::size_t>(batch) * 2 * static_cast<std::size_t>(length);
  for (std::size_t i = 0; i < bufs.size(); ++i) std::memcpy(a.mutable_data() + stride * i, bufs[i].samples.data(), sizeof(double) * stride);
  return a;
}

}  // namespace

PYBIND11_MODULE(_core, m) {
  m.doc() = "mixgraph._core: B200-native batched audio-graph renderer (GRAFX) over the C++ API";
  py::register_exception<std::invalid_argument>(m, "InvalidArgument", PyExc_ValueError);

  py::enum_<NodeType>(m, "NodeType")
      .value("In", NodeType::In).value("Out", NodeType::Out).value("Mix", NodeType::Mix)
      .value("Gain", NodeType::Gain).value("Eq", NodeType::Eq).value("Compressor", NodeType::Compressor)
      .value("Noisegate", NodeType::Noisegate).value("Imager", NodeType::Imager)
      .value("Reverb", NodeType::Reverb).value("Delay", NodeType::Delay);
  m.def("param_width", [](const py::handle& t) { return param_width(to_type(t)); });
  m.def("type_code", [](const py::handle& t) { return std::string(1, type_code(to_type(t))); });
  m.def("type_name", [](const py::handle& t) { return std::string(type_name(to_type(t))); });

  py::enum_<Strategy>(m, "Strategy")
      .value("OneByOne", Strategy::OneByOne).value("Greedy", Strategy::Greedy)
      .value("Beam", Strategy::Beam).value("Optimal", Strategy::Optimal);

  py::class_<Edge>(m, "Edge")
      .def(py::init<int, int, int, int>(), py::arg("src"), py::arg("dst"), py::arg("outlet") = 0, py::arg("inlet") = 0)
      .def_readwrite("src", &Edge::src).def_readwrite("dst", &Edge::dst)
      .def_readwrite("outlet", &Edge::outlet).def_readwrite("inlet", &Edge::inlet)
      .def("__eq__", [](const Edge& a, const Edge& b) { return a == b; })
      .def("__repr__", [](const Edge& e) {
        return "Edge(" + std::to_string(e.src) + ", " + std::to_string(e.dst) + ", " + std::to_string(e.outlet) + ", " +
               std::to_string(e.inlet) + ")";
      });

  py::class_<Graph>(m, "Graph")
      .def(py::init<>())
      .def("add_node", [](Graph& g, const py::handle& t) { return g.add_node(to_type(t)); })
      .def("add", [](Graph& g, const py::handle& t) { return g.add_node(to_type(t)); })
      .def("add_serial_chain", [](Graph& g, const py::list& ts) {
        std::vector<NodeType> v;
        for (auto h : ts) v.push_back(to_type(h));
        return g.add_serial_chain(v);
      })
      .def("connect", &Graph::connect, py::arg("src"), py::arg("dst"), py::arg("outlet") = 0, py::arg("inlet") = 0)
      .def("validate", &Graph::validate)
      .def("num_nodes", &Graph::num_nodes)
      .def("node_type", &Graph::node_type)
      .def_property_readonly("node_types", &Graph::node_types)
      .def_property_readonly("edges", &Graph::edges);
  m.def("disjoint_union", &disjoint_union);

  py::class_<FlatGraph>(m, "FlatGraph")
      .def_readonly("node_types", &FlatGraph::node_types)
      .def_readonly("edges", &FlatGraph::edges)
      .def_readonly("num_inputs", &FlatGraph::num_inputs)
      .def_readonly("num_outputs", &FlatGraph::num_outputs)
      .def("num_nodes", &FlatGraph::num_nodes)
      .def_property_readonly("params", [](const FlatGraph& f) { return from_store(f.params); });
  m.def("to_flat", &to_flat);
  m.def("default_params", [](const std::vector<NodeType>& t) { return from_store(default_params(t)); });

  py::class_<ScheduleOptions>(m, "ScheduleOptions")
      .def(py::init([](Strategy s, int beam, int cap) { return ScheduleOptions{s, beam, cap}; }),
           py::arg("strategy") = Strategy::Greedy, py::arg("beam_width") = 32, py::arg("optimal_node_cap") = 256)
      .def_readwrite("strategy", &ScheduleOptions::strategy)
      .def_readwrite("beam_width", &ScheduleOptions::beam_width)
      .def_readwrite("optimal_node_cap", &ScheduleOptions::optimal_node_cap);
  py::class_<Schedule>(m, "Schedule")
      .def_readonly("type_string", &Schedule::type_string)
      .def_readonly("subsets", &Schedule::subsets)
      .def("num_steps", &Schedule::num_steps)
      .def("type_codes", &Schedule::type_codes);
  m.def("make_schedule", py::overload_cast<const FlatGraph&, const ScheduleOptions&>(&make_schedule));
  m.def("validate_schedule", &validate_schedule);
  m.def("optimize_node_order", &optimize_node_order);
  m.def("inverse_permutation", &inverse_permutation);
  m.def("reorder_flat", &reorder_flat);

  py::class_<StepIndex>(m, "StepIndex")
      .def_readonly("type", &StepIndex::type).def_readonly("gather", &StepIndex::gather)
      .def_readonly("aggregate", &StepIndex::aggregate).def_readonly("param_begin", &StepIndex::param_begin)
      .def_readonly("param_end", &StepIndex::param_end).def_readonly("store_begin", &StepIndex::store_begin)
      .def_readonly("store_end", &StepIndex::store_end);
  py::class_<RenderData>(m, "RenderData")
      .def_readonly("schedule", &RenderData::schedule)
      .def_readonly("sigma", &RenderData::sigma)
      .def_readonly("flat", &RenderData::flat)
      .def_readonly("steps", &RenderData::steps)
      .def_readonly("buffer_rows", &RenderData::buffer_rows)
      .def_readonly("num_inputs", &RenderData::num_inputs)
      .def_readonly("output_begin", &RenderData::output_begin)
      .def_readonly("param_source_rows", &RenderData::param_source_rows)
      .def("reorder_params", [](const RenderData& rd, const py::dict& p) { return from_store(rd.reorder_params(to_store(p))); });
  m.def("compute_render_data", &compute_render_data, py::arg("flat"), py::arg("options") = ScheduleOptions{});

  py::class_<ProcessorConfig>(m, "ProcessorConfig")
      .def(py::init([](double fs, std::uint32_t seed, int taps, double floor_) { return ProcessorConfig{fs, seed, taps, floor_}; }),
           py::arg("sample_rate") = 44100.0, py::arg("reverb_seed") = 0, py::arg("envelope_taps") = 32768,
           py::arg("energy_floor") = 1e-7)
      .def_readwrite("sample_rate", &ProcessorConfig::sample_rate)
      .def_readwrite("reverb_seed", &ProcessorConfig::reverb_seed)
      .def_readwrite("envelope_taps", &ProcessorConfig::envelope_taps)
      .def_readwrite("energy_floor", &ProcessorConfig::energy_floor);
  py::class_<ProcessorSet>(m, "ProcessorSet")
      .def(py::init<const ProcessorConfig&>(), py::arg("config") = ProcessorConfig{})
      .def_property_readonly("config", &ProcessorSet::config)
      .def_property_readonly("delay_span", &ProcessorSet::delay_span)
      .def_property_readonly("delay_window", &ProcessorSet::delay_window)
      .def_property_readonly("reverb_length", &ProcessorSet::reverb_length)
      .def("process_node", [](const ProcessorSet& p, const py::handle& t, const Array& input, const Array& params) {
        if (input.ndim() != 3 || input.shape(1) != 2) throw std::invalid_argument("input must be [B][2][L]");
        AudioBuffer a(static_cast<int>(input.shape(0)), 2, static_cast<long>(input.shape(2)), p.config().sample_rate);
        std::memcpy(a.samples.data(), input.data(), sizeof(double) * a.samples.size());
        AudioBuffer y;
        {
          py::gil_scoped_release release;
          y = p.process_node(to_type(t), a, {params.data(), static_cast<std::size_t>(params.size())});
        }
        return from_buffers({y}, y.batch, y.length)[py::int_(0)];
      }, py::arg("type"), py::arg("input"), py::arg("params") = Array())
      .def("reverb_kernel", [](const ProcessorSet& p, const Array& row) {
        return p.reverb_kernel({row.data(), static_cast<std::size_t>(row.size())});
      })
      .def("delay_kernel", [](const ProcessorSet& p, const Array& row, int channel) {
        return p.delay_kernel({row.data(), static_cast<std::size_t>(row.size())}, channel);
      })
      .def("delay_positions", [](const ProcessorSet& p, const Array& row, int channel) {
        return p.delay_positions({row.data(), static_cast<std::size_t>(row.size())}, channel);
      });

  m.def("render", [](const RenderData& rd, const ProcessorSet& procs, const py::dict& params, const Array& sources,
                     bool keep_intermediates) -> py::object {
    const ParamStore store = to_store(params);
    auto bufs = to_buffers(sources, procs.config().sample_rate);
    RenderOptions o;
    o.keep_intermediates = keep_intermediates;
    RenderResult r;
    {
      py::gil_scoped_release release;
      r = render(rd, procs, store, bufs, o);
    }
    const int b = bufs.empty() ? 1 : bufs[0].batch;
    const long l = bufs.empty() ? 0 : bufs[0].length;
    Array out = from_buffers(r.outputs, b, l);
    if (!keep_intermediates) return py::object(out);
    return py::make_tuple(out, from_buffers(r.intermediates, b, l));
  }, py::arg("render_data"), py::arg("processors"), py::arg("params"), py::arg("sources"),
     py::arg("keep_intermediates") = false,
     "render.cpp:14-81: params in RENDER order (RenderData.reorder_params), sources [K][B][2][L]");
}
