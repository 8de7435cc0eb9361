// py_dagplace.cpp — Python bindings (pybind11) of the C++ API `namespace dagplace`
// (/root/reference/proj/include/dagplace/*.hpp, compiled here against those unchanged
// headers) as implemented by the B200 drop-in libdagplace_core_b200.so.  The reference
// wires a python extension module into its build (proj/CMakeLists.txt:14,22-23) whose
// sources are empty (proj/python/CMakeLists.txt); this module is that surface: the same
// types, field names and functions, DagError raised with the reference's kind and message.
// Module name: paper_2208_00184_b200.dagplace.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>

#include "dagplace/estimation.hpp"
#include "dagplace/fusion.hpp"
#include "dagplace/graph.hpp"
#include "dagplace/ordering.hpp"
#include "dagplace/pipeline.hpp"
#include "dagplace/placement.hpp"
#include "dagplace/simulator.hpp"

namespace py = pybind11;
using namespace dagplace;

namespace {

// Bulk construction from numpy arrays (a 1M-node graph as Python objects would dominate).
ComputationGraph graph_from_arrays(py::array_t<int64_t, py::array::c_style | py::array::forcecast> ids,
                                   py::array_t<int64_t, py::array::c_style | py::array::forcecast> compute,
                                   py::array_t<int64_t, py::array::c_style | py::array::forcecast> memory,
                                   py::array_t<int64_t, py::array::c_style | py::array::forcecast> src,
                                   py::array_t<int64_t, py::array::c_style | py::array::forcecast> dst,
                                   py::array_t<int64_t, py::array::c_style | py::array::forcecast> bytes) {
  const auto n = ids.size(), m = src.size();
  if (compute.size() != n || memory.size() != n || dst.size() != m || bytes.size() != m)
    throw std::invalid_argument("node arrays and edge arrays must have matching lengths");
  ComputationGraph g;
  g.nodes.resize(n);
  g.edges.resize(m);
  const int64_t *pi = ids.data(), *pc = compute.data(), *pm = memory.data();
  for (py::ssize_t i = 0; i < n; ++i) {
    g.nodes[i].id = pi[i];
    g.nodes[i].compute_us = pc[i];
    g.nodes[i].memory_bytes = pm[i];
  }
  const int64_t *ps = src.data(), *pd = dst.data(), *pb = bytes.data();
  for (py::ssize_t e = 0; e < m; ++e) g.edges[e] = TensorEdge{ps[e], pd[e], pb[e]};
  return g;
}

py::array_t<int64_t> node_ids(const ComputationGraph& g) {
  py::array_t<int64_t> out(static_cast<py::ssize_t>(g.nodes.size()));
  auto* p = out.mutable_data();
  for (size_t i = 0; i < g.nodes.size(); ++i) p[i] = g.nodes[i].id;
  return out;
}

}  // namespace

PYBIND11_MODULE(dagplace, m) {
  m.doc() = "B200 drop-in of the dagplace C++ API (graph-analysis and placement-evaluation path)";

  static py::exception<DagError> dag_error(m, "DagError", PyExc_RuntimeError);
  py::register_exception_translator([](std::exception_ptr p) {
    try {
      if (p) std::rethrow_exception(p);
    } catch (const DagError& e) {
      // DagError(message) with .kind (the reference's ErrorKind), message = "<Kind>: ..."
      py::object err = py::reinterpret_borrow<py::object>(dag_error.ptr())(e.what());
      err.attr("kind") = py::cast(e.kind());
      PyErr_SetObject(dag_error.ptr(), err.ptr());
    }
  });

  py::enum_<ErrorKind>(m, "ErrorKind")
      .value("CycleDetected", ErrorKind::CycleDetected)
      .value("DanglingEdge", ErrorKind::DanglingEdge)
      .value("DuplicateId", ErrorKind::DuplicateId)
      .value("DuplicateEdge", ErrorKind::DuplicateEdge)
      .value("InvalidValue", ErrorKind::InvalidValue)
      .value("ZeroComputeTime", ErrorKind::ZeroComputeTime)
      .value("NoSuchEdge", ErrorKind::NoSuchEdge)
      .value("NodeExceedsClusterLimit", ErrorKind::NodeExceedsClusterLimit)
      .value("GroupExceedsClusterLimit", ErrorKind::GroupExceedsClusterLimit)
      .value("InfeasiblePartition", ErrorKind::InfeasiblePartition)
      .value("InvalidClusterMap", ErrorKind::InvalidClusterMap)
      .value("InsufficientSamples", ErrorKind::InsufficientSamples)
      .value("UnknownNode", ErrorKind::UnknownNode)
      .value("NodeUniverseMismatch", ErrorKind::NodeUniverseMismatch)
      .value("UnplacedNode", ErrorKind::UnplacedNode)
      .value("InstanceTooLarge", ErrorKind::InstanceTooLarge)
      .value("InstanceInfeasible", ErrorKind::InstanceInfeasible)
      .value("UnreachableTargetCcr", ErrorKind::UnreachableTargetCcr)
      .value("ParseError", ErrorKind::ParseError);
  m.attr("kNever") = kNever;

  // ---------------------------------------------------------------- graph.hpp
  py::class_<OpNode>(m, "OpNode")
      .def(py::init<>())
      .def(py::init([](NodeId id, const std::string& name, Duration c, Bytes mem, std::optional<std::string> grp) {
             return OpNode{id, name, c, mem, std::move(grp)};
           }),
           py::arg("id"), py::arg("name") = "", py::arg("compute_us") = 0, py::arg("memory_bytes") = 0,
           py::arg("colocation_group") = py::none())
      .def_readwrite("id", &OpNode::id)
      .def_readwrite("name", &OpNode::name)
      .def_readwrite("compute_us", &OpNode::compute_us)
      .def_readwrite("memory_bytes", &OpNode::memory_bytes)
      .def_readwrite("colocation_group", &OpNode::colocation_group);
  py::class_<TensorEdge>(m, "TensorEdge")
      .def(py::init<>())
      .def(py::init([](NodeId s, NodeId d, Bytes b) { return TensorEdge{s, d, b}; }), py::arg("src"), py::arg("dst"),
           py::arg("tensor_bytes") = 0)
      .def_readwrite("src", &TensorEdge::src)
      .def_readwrite("dst", &TensorEdge::dst)
      .def_readwrite("tensor_bytes", &TensorEdge::tensor_bytes);
  py::class_<ComputationGraph>(m, "ComputationGraph")
      .def(py::init<>())
      .def(py::init([](std::vector<OpNode> nodes, std::vector<TensorEdge> edges) {
             return ComputationGraph{std::move(nodes), std::move(edges)};
           }),
           py::arg("nodes"), py::arg("edges"))
      .def_readwrite("nodes", &ComputationGraph::nodes)
      .def_readwrite("edges", &ComputationGraph::edges)
      .def_static("from_arrays", &graph_from_arrays, py::arg("ids"), py::arg("compute_us"), py::arg("memory_bytes"),
                  py::arg("edge_src"), py::arg("edge_dst"), py::arg("tensor_bytes"))
      .def("node_ids", &node_ids)
      .def("__len__", [](const ComputationGraph& g) { return g.nodes.size(); });
  py::class_<CommModel>(m, "CommModel")
      .def(py::init<>())
      .def(py::init([](double k, double b) { return CommModel{k, b}; }), py::arg("k_us_per_byte"), py::arg("b_us"))
      .def_readwrite("k_us_per_byte", &CommModel::k_us_per_byte)
      .def_readwrite("b_us", &CommModel::b_us);
  py::class_<DeviceSpec>(m, "DeviceSpec")
      .def(py::init<>())
      .def(py::init([](DeviceId id, Bytes mem) { return DeviceSpec{id, mem}; }), py::arg("id"),
           py::arg("memory_bytes"))
      .def_readwrite("id", &DeviceSpec::id)
      .def_readwrite("memory_bytes", &DeviceSpec::memory_bytes);
  py::class_<NodeLevels>(m, "NodeLevels")
      .def(py::init<>())
      .def_readwrite("tlevel", &NodeLevels::tlevel)
      .def_readwrite("blevel", &NodeLevels::blevel)
      .def_readwrite("cpath", &NodeLevels::cpath);
  py::class_<LevelTable>(m, "LevelTable")
      .def(py::init<>())
      .def_readwrite("levels", &LevelTable::levels)
      .def("at", &LevelTable::at, py::return_value_policy::copy)
      .def("max_cpath", &LevelTable::max_cpath);
  py::class_<Violation>(m, "Violation")
      .def_readwrite("kind", &Violation::kind)
      .def_readwrite("message", &Violation::message)
      .def_readwrite("nodes", &Violation::nodes);
  py::class_<ValidationResult>(m, "ValidationResult")
      .def_readwrite("ok", &ValidationResult::ok)
      .def_readwrite("violations", &ValidationResult::violations);
  m.def("validate", &validate, py::arg("graph"));
  m.def("require_valid", &require_valid, py::arg("graph"));
  m.def("comm_time", &comm_time, py::arg("bytes"), py::arg("model"));
  m.def("ccr", &ccr, py::arg("graph"), py::arg("model"));
  m.def("compute_levels", &compute_levels, py::arg("graph"), py::arg("model"));

  // ---------------------------------------------------------------- ordering.hpp
  py::enum_<TopoPolicy>(m, "TopoPolicy")
      .value("MTopo", TopoPolicy::MTopo)
      .value("DfsTopo", TopoPolicy::DfsTopo)
      .value("CpdTopo", TopoPolicy::CpdTopo);
  py::class_<TopoOrder>(m, "TopoOrder")
      .def(py::init<>())
      .def_readwrite("policy", &TopoOrder::policy)
      .def_readwrite("sequence", &TopoOrder::sequence);
  m.def("topo_policy_from_string", &topo_policy_from_string, py::arg("name"));
  m.def("to_string", py::overload_cast<TopoPolicy>(&dagplace::to_string), py::arg("policy"));
  m.def("m_topo", &m_topo, py::arg("graph"));
  m.def("dfs_topo", &dfs_topo, py::arg("graph"));
  m.def("cpd_topo", &cpd_topo, py::arg("graph"), py::arg("levels"));
  m.def("is_valid_topo_order", &is_valid_topo_order, py::arg("graph"), py::arg("order"));

  // ---------------------------------------------------------------- fusion.hpp
  py::class_<FusionConfig>(m, "FusionConfig")
      .def(py::init<>())
      .def(py::init([](int r, Bytes lim) { return FusionConfig{r, lim}; }), py::arg("range") = 200,
           py::arg("cluster_memory_limit") = 0)
      .def_readwrite("range", &FusionConfig::range)
      .def_readwrite("cluster_memory_limit", &FusionConfig::cluster_memory_limit);
  py::class_<Cluster>(m, "Cluster")
      .def_readwrite("id", &Cluster::id)
      .def_readwrite("members", &Cluster::members)
      .def_readwrite("total_compute_us", &Cluster::total_compute_us)
      .def_readwrite("total_memory_bytes", &Cluster::total_memory_bytes);
  py::class_<ClusterMap>(m, "ClusterMap")
      .def(py::init<>())
      .def_readwrite("node_to_cluster", &ClusterMap::node_to_cluster)
      .def_readwrite("breakpoints", &ClusterMap::breakpoints)
      .def_readwrite("clusters", &ClusterMap::clusters);
  py::class_<GroupContraction>(m, "GroupContraction")
      .def_readwrite("contracted", &GroupContraction::contracted)
      .def_readwrite("members_of", &GroupContraction::members_of);
  py::class_<FusionResult>(m, "FusionResult")
      .def_readwrite("coarse", &FusionResult::coarse)
      .def_readwrite("map", &FusionResult::map);
  m.def("merge_is_safe", &merge_is_safe, py::arg("graph"), py::arg("u"), py::arg("v"));
  m.def("optimal_breakpoints", &optimal_breakpoints, py::arg("graph"), py::arg("order"), py::arg("model"),
        py::arg("config"));
  m.def("build_coarse_graph", &build_coarse_graph, py::arg("graph"), py::arg("order"), py::arg("clusters"));
  m.def("contract_colocation_groups", &contract_colocation_groups, py::arg("graph"));
  m.def("fuse", &fuse, py::arg("graph"), py::arg("model"), py::arg("config"));

  // ---------------------------------------------------------------- placement.hpp
  py::class_<Placement>(m, "Placement")
      .def(py::init<>())
      .def_readwrite("assignment", &Placement::assignment)
      .def_readwrite("per_device_memory", &Placement::per_device_memory);
  py::class_<BusyInterval>(m, "BusyInterval")
      .def_readwrite("start", &BusyInterval::start)
      .def_readwrite("end", &BusyInterval::end);
  py::class_<DeviceTimeline>(m, "DeviceTimeline")
      .def(py::init<>())
      .def("find_slot", &DeviceTimeline::find_slot, py::arg("earliest"), py::arg("duration"))
      .def("reserve", &DeviceTimeline::reserve, py::arg("start"), py::arg("duration"))
      .def("busy", &DeviceTimeline::busy, py::return_value_policy::copy);
  py::class_<SchedulerState>(m, "SchedulerState")
      .def_readwrite("device_ids", &SchedulerState::device_ids)
      .def_readwrite("finish_time", &SchedulerState::finish_time)
      .def_readwrite("timelines", &SchedulerState::timelines)
      .def_readwrite("available_memory", &SchedulerState::available_memory)
      .def_static("for_devices", &SchedulerState::for_devices, py::arg("devices"))
      .def("device_pos", &SchedulerState::device_pos, py::arg("id"));
  py::class_<PlacementDecision>(m, "PlacementDecision")
      .def_readwrite("node", &PlacementDecision::node)
      .def_readwrite("prev_device", &PlacementDecision::prev_device)
      .def_readwrite("back_cost_us", &PlacementDecision::back_cost_us)
      .def_readwrite("est_us", &PlacementDecision::est_us)
      .def_readwrite("chosen", &PlacementDecision::chosen)
      .def_readwrite("relocated", &PlacementDecision::relocated)
      .def_readwrite("best_effort", &PlacementDecision::best_effort);
  py::class_<PlacementResult>(m, "PlacementResult")
      .def_readwrite("placement", &PlacementResult::placement)
      .def_readwrite("oom_risk", &PlacementResult::oom_risk)
      .def_readwrite("decisions", &PlacementResult::decisions);
  m.def("order_place", &order_place, py::arg("coarse"), py::arg("order"), py::arg("devices"));
  m.def("adjusting_placement", &adjusting_placement, py::arg("coarse"), py::arg("order"), py::arg("devices"),
        py::arg("model"));
  m.def("compute_est", &compute_est, py::arg("state"), py::arg("graph"), py::arg("assignment"), py::arg("node"),
        py::arg("device"), py::arg("model"));
  m.def("expand_placement", &expand_placement, py::arg("original"), py::arg("clusters"), py::arg("coarse_placement"));

  // ---------------------------------------------------------------- simulator.hpp
  py::enum_<TaskKind>(m, "TaskKind")
      .value("Compute", TaskKind::Compute)
      .value("Send", TaskKind::Send)
      .value("Receive", TaskKind::Receive);
  py::class_<SimTaskRecord>(m, "SimTaskRecord")
      .def_readwrite("kind", &SimTaskRecord::kind)
      .def_readwrite("node", &SimTaskRecord::node)
      .def_readwrite("edge_src", &SimTaskRecord::edge_src)
      .def_readwrite("edge_dst", &SimTaskRecord::edge_dst)
      .def_readwrite("device", &SimTaskRecord::device)
      .def_readwrite("start", &SimTaskRecord::start)
      .def_readwrite("end", &SimTaskRecord::end);
  py::class_<DeviceReport>(m, "DeviceReport")
      .def_readwrite("compute_busy", &DeviceReport::compute_busy)
      .def_readwrite("send_busy", &DeviceReport::send_busy)
      .def_readwrite("receive_busy", &DeviceReport::receive_busy)
      .def_readwrite("peak_memory_bytes", &DeviceReport::peak_memory_bytes)
      .def_readwrite("memory_capacity_bytes", &DeviceReport::memory_capacity_bytes);
  py::class_<SimulationReport>(m, "SimulationReport")
      .def_readwrite("makespan", &SimulationReport::makespan)
      .def_readwrite("devices", &SimulationReport::devices)
      .def_readwrite("cross_transfer_count", &SimulationReport::cross_transfer_count)
      .def_readwrite("cross_transfer_bytes", &SimulationReport::cross_transfer_bytes)
      .def_readwrite("oom_flag", &SimulationReport::oom_flag)
      .def_readwrite("trace", &SimulationReport::trace);
  m.def("to_string", py::overload_cast<TaskKind>(&dagplace::to_string), py::arg("kind"));
  m.def("simulate", &simulate, py::arg("graph"), py::arg("placement"), py::arg("devices"), py::arg("model"));
  m.def("brute_force_optimal", &brute_force_optimal, py::arg("graph"), py::arg("devices"), py::arg("model"));

  // ---------------------------------------------------------------- estimation.hpp
  py::class_<NodeSample>(m, "NodeSample")
      .def(py::init<>())
      .def_readwrite("memory_bytes", &NodeSample::memory_bytes)
      .def_readwrite("compute_us", &NodeSample::compute_us);
  py::class_<BatchProfile>(m, "BatchProfile")
      .def(py::init<>())
      .def_readwrite("batch_size", &BatchProfile::batch_size)
      .def_readwrite("nodes", &BatchProfile::nodes);
  py::class_<ProfileSet>(m, "ProfileSet")
      .def(py::init<>())
      .def_readwrite("batches", &ProfileSet::batches)
      .def_readwrite("comm_samples", &ProfileSet::comm_samples);
  py::class_<LinearFit>(m, "LinearFit")
      .def_readwrite("slope", &LinearFit::slope)
      .def_readwrite("intercept", &LinearFit::intercept)
      .def_readwrite("residual_norm", &LinearFit::residual_norm)
      .def("predict", &LinearFit::predict);
  py::class_<NodeCostModel>(m, "NodeCostModel")
      .def_readwrite("memory_fit", &NodeCostModel::memory_fit)
      .def_readwrite("time_fit", &NodeCostModel::time_fit);
  py::class_<EdgeScaling>(m, "EdgeScaling")
      .def(py::init<>())
      .def_readwrite("reference_batch", &EdgeScaling::reference_batch)
      .def_readwrite("scale_override", &EdgeScaling::scale_override);
  py::class_<DeviationReport>(m, "DeviationReport")
      .def_readwrite("memory_deviation", &DeviationReport::memory_deviation)
      .def_readwrite("time_deviation", &DeviationReport::time_deviation)
      .def_readwrite("mean_memory_deviation", &DeviationReport::mean_memory_deviation)
      .def_readwrite("mean_time_deviation", &DeviationReport::mean_time_deviation)
      .def_readwrite("zero_memory_nodes", &DeviationReport::zero_memory_nodes)
      .def_readwrite("zero_time_nodes", &DeviationReport::zero_time_nodes);
  m.def("fit_node_models", &fit_node_models, py::arg("profiles"));
  m.def("estimate_graph", &estimate_graph, py::arg("base"), py::arg("models"), py::arg("target_batch"),
        py::arg("scaling"));
  m.def("fit_comm_model", &fit_comm_model, py::arg("samples"));
  m.def("sequential_eval_placement", &sequential_eval_placement, py::arg("estimated"), py::arg("devices"));
  m.def("deviation_report", &deviation_report, py::arg("estimated"), py::arg("measured"));

  // ---------------------------------------------------------------- pipeline.hpp
  py::enum_<PlaceStrategy>(m, "PlaceStrategy")
      .value("Order", PlaceStrategy::Order)
      .value("Adjust", PlaceStrategy::Adjust)
      .value("SequentialEval", PlaceStrategy::SequentialEval);
  py::class_<PipelineConfig>(m, "PipelineConfig")
      .def(py::init<>())
      .def_readwrite("fusion_range", &PipelineConfig::fusion_range)
      .def_readwrite("cluster_mem_fraction", &PipelineConfig::cluster_mem_fraction)
      .def_readwrite("strategy", &PipelineConfig::strategy)
      .def_readwrite("target_batch", &PipelineConfig::target_batch);
  py::class_<StrategyOutcome>(m, "StrategyOutcome")
      .def_readwrite("makespan_us", &StrategyOutcome::makespan_us)
      .def_readwrite("oom_risk", &StrategyOutcome::oom_risk);
  py::class_<PipelineReport>(m, "PipelineReport")
      .def_readwrite("original_nodes", &PipelineReport::original_nodes)
      .def_readwrite("original_edges", &PipelineReport::original_edges)
      .def_readwrite("original_ccr", &PipelineReport::original_ccr)
      .def_readwrite("coarse_nodes", &PipelineReport::coarse_nodes)
      .def_readwrite("coarse_edges", &PipelineReport::coarse_edges)
      .def_readwrite("coarse_ccr", &PipelineReport::coarse_ccr)
      .def_readwrite("node_reduction_factor", &PipelineReport::node_reduction_factor)
      .def_readwrite("ccr_reduction_factor", &PipelineReport::ccr_reduction_factor)
      .def_readwrite("order_place", &PipelineReport::order_place)
      .def_readwrite("adjusting", &PipelineReport::adjusting)
      .def_readwrite("comm_source", &PipelineReport::comm_source)
      .def_readwrite("chosen_strategy", &PipelineReport::chosen_strategy)
      .def_readwrite("chosen_oom_risk", &PipelineReport::chosen_oom_risk)
      .def_readwrite("chosen_placement", &PipelineReport::chosen_placement)
      .def_readwrite("chosen_simulation", &PipelineReport::chosen_simulation)
      .def_readwrite("fusion", &PipelineReport::fusion)
      .def_readwrite("generation_wall_us", &PipelineReport::generation_wall_us);
  m.def("place_strategy_from_string", &place_strategy_from_string, py::arg("name"));
  m.def("to_string", py::overload_cast<PlaceStrategy>(&dagplace::to_string), py::arg("strategy"));
  m.def("evaluate_pipeline", &evaluate_pipeline, py::arg("graph"), py::arg("profiles"), py::arg("devices"),
        py::arg("device_comm"), py::arg("config"), py::call_guard<py::gil_scoped_release>());
}
