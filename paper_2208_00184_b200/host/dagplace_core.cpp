// dagplace_core.cpp — the C++ drop-in for the reference library target `dagplace_core`.
//
// Implements the public API of /root/reference/proj/include/dagplace/*.hpp (namespace
// dagplace, same declarations and types, compiled against those headers) on top of the
// C-ABI of libdagplace_b200.so: every compute entry point converts the STL types to the
// flat SoA of include/dagplace_b200.h, runs the sm_100a kernels, and materialises the
// reference's return types.  Errors come back as the reference's DagError with the same
// kind and message text.  What stays host-side: the tiny value types' methods
// (DeviceTimeline on a caller-owned timeline, SchedulerState bookkeeping, LevelTable
// lookups), input synthesis (gen_graph) and the Standard Evaluation fits (estimation.cpp
// — per-node O(batches) arithmetic, SURVEY §2 keeps it a host drop-in).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <random>
#include <set>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/dagplace_b200.h"
#include "dagplace/estimation.hpp"
#include "dagplace/fusion.hpp"
#include "dagplace/generator.hpp"
#include "dagplace/graph.hpp"
#include "dagplace/graph_index.hpp"
#include "dagplace/ordering.hpp"
#include "dagplace/pipeline.hpp"
#include "dagplace/placement.hpp"
#include "dagplace/simulator.hpp"

namespace dagplace {

namespace {

// ---------------------------------------------------------------- C-ABI plumbing
struct Ctx {
  dp_ctx_t* ctx = nullptr;
  Ctx() {
    const char* dev = std::getenv("DAGPLACE_DEVICE");
    int rc = dp_ctx_create(dev ? std::atoi(dev) : 0, nullptr, &ctx);
    if (rc) throw std::runtime_error(std::string("libdagplace_b200: ") + dp_last_error_message());
  }
  ~Ctx() { dp_ctx_destroy(ctx); }
};

dp_ctx_t* ctx() {
  thread_local std::unique_ptr<Ctx> c;
  if (!c) c = std::make_unique<Ctx>();
  return c->ctx;
}

[[noreturn]] void rethrow(int rc) {
  std::string what = dp_last_error_message();
  if (rc >= 1 && rc <= 19) {
    const ErrorKind kind = static_cast<ErrorKind>(rc - 1);
    const std::string prefix = std::string(to_string(kind)) + ": ";
    std::string body = what.compare(0, prefix.size(), prefix) == 0 ? what.substr(prefix.size()) : what;
    throw DagError(kind, body);
  }
  // size limits of the device path (more than 256 devices, 2^24 or more peel nodes): the
  // reference has no such limit, so they surface as the library's own error type
  if (rc == DP_E_UNSUPPORTED) throw DagError(ErrorKind::InstanceTooLarge, what);
  throw std::runtime_error("libdagplace_b200: " + what);
}

inline void check(int rc) {
  if (rc) rethrow(rc);
}

// ComputationGraph (AoS) -> flat SoA view.
struct Flat {
  std::vector<int64_t> id, w, mem, src, dst, bytes;
  std::vector<int32_t> group;
  dp_graph_t g{};
  explicit Flat(const ComputationGraph& cg) {
    const size_t n = cg.nodes.size(), m = cg.edges.size();
    id.resize(n);
    w.resize(n);
    mem.resize(n);
    group.assign(n, -1);
    std::unordered_map<std::string, int32_t> labels;
    bool any = false;
    for (size_t i = 0; i < n; ++i) {
      const OpNode& nd = cg.nodes[i];
      id[i] = nd.id;
      w[i] = nd.compute_us;
      mem[i] = nd.memory_bytes;
      if (nd.colocation_group) {
        auto it = labels.emplace(*nd.colocation_group, static_cast<int32_t>(labels.size())).first;
        group[i] = it->second;
        any = true;
      }
    }
    src.resize(m);
    dst.resize(m);
    bytes.resize(m);
    for (size_t e = 0; e < m; ++e) {
      src[e] = cg.edges[e].src;
      dst[e] = cg.edges[e].dst;
      bytes[e] = cg.edges[e].tensor_bytes;
    }
    g.n_nodes = static_cast<int64_t>(n);
    g.n_edges = static_cast<int64_t>(m);
    g.node_id = id.data();
    g.compute_us = w.data();
    g.memory_bytes = mem.data();
    g.group = any ? group.data() : nullptr;
    g.edge_src = src.data();
    g.edge_dst = dst.data();
    g.edge_bytes = bytes.data();
  }
};

struct FlatDevices {
  std::vector<int32_t> id;
  std::vector<int64_t> mem;
  dp_devices_t d{};
  explicit FlatDevices(const std::vector<DeviceSpec>& devs) {
    for (const auto& x : devs) {
      id.push_back(x.id);
      mem.push_back(x.memory_bytes);
    }
    d.count = static_cast<int32_t>(devs.size());
    d.id = id.data();
    d.memory_bytes = mem.data();
  }
};

dp_comm_t cm(const CommModel& c) { return dp_comm_t{c.k_us_per_byte, c.b_us}; }

ComputationGraph from_out(const dp_graph_out_t* o, bool cluster_names, const ComputationGraph* names_from) {
  ComputationGraph g;
  g.nodes.resize(static_cast<size_t>(o->n_nodes));
  std::unordered_map<NodeId, const OpNode*> orig;
  if (names_from)
    for (const auto& n : names_from->nodes) orig.emplace(n.id, &n);
  for (int64_t i = 0; i < o->n_nodes; ++i) {
    OpNode& n = g.nodes[i];
    n.id = o->node_id[i];
    n.compute_us = o->compute_us[i];
    n.memory_bytes = o->memory_bytes[i];
    if (cluster_names) {
      n.name = "cluster_" + std::to_string(n.id);  // fusion.cpp:210
    } else if (names_from) {
      auto it = orig.find(n.id);
      if (it != orig.end()) {
        n.name = it->second->name;
        n.colocation_group = it->second->colocation_group;
      }
    }
  }
  g.edges.resize(static_cast<size_t>(o->n_edges));
  for (int64_t e = 0; e < o->n_edges; ++e) g.edges[e] = {o->edge_src[e], o->edge_dst[e], o->edge_bytes[e]};
  return g;
}

ClusterMap map_from(const dp_cluster_map_t* m, const ComputationGraph& g) {
  ClusterMap out;
  out.node_to_cluster.reserve(g.nodes.size());
  for (size_t i = 0; i < g.nodes.size(); ++i)
    if (m->node_cluster[i] >= 0) out.node_to_cluster[g.nodes[i].id] = m->node_cluster[i];
  out.breakpoints.assign(m->breakpoints, m->breakpoints + m->n_breakpoints);
  out.clusters.resize(static_cast<size_t>(m->n_clusters));
  for (int64_t c = 0; c < m->n_clusters; ++c) {
    Cluster& cl = out.clusters[c];
    cl.id = static_cast<int>(c);
    cl.members.assign(m->members + m->member_off[c], m->members + m->member_off[c + 1]);
    cl.total_compute_us = m->total_compute[c];
    cl.total_memory_bytes = m->total_memory[c];
  }
  return out;
}

PlacementResult placement_from(const dp_placement_result_t* p, const ComputationGraph& g) {
  PlacementResult r;
  r.placement.assignment.reserve(g.nodes.size());
  for (size_t i = 0; i < g.nodes.size(); ++i)
    if (p->device[i] != INT32_MIN) r.placement.assignment[g.nodes[i].id] = p->device[i];
  for (int32_t d = 0; d < p->n_devices; ++d)
    if (p->device_present[d]) r.placement.per_device_memory[p->device_ids[d]] = p->per_device_memory[d];
  r.oom_risk = p->oom_risk != 0;
  r.decisions.resize(static_cast<size_t>(p->n_decisions));
  for (int64_t k = 0; k < p->n_decisions; ++k) {
    PlacementDecision& dec = r.decisions[k];
    dec.node = p->dec_node[k];
    dec.prev_device = p->dec_prev[k];
    dec.back_cost_us = p->dec_back_cost[k];
    for (int32_t d = 0; d < p->n_devices; ++d) dec.est_us[p->device_ids[d]] = p->dec_est[k * p->n_devices + d];
    dec.chosen = p->dec_chosen[k];
    dec.relocated = p->dec_relocated[k] != 0;
    dec.best_effort = p->dec_best_effort[k] != 0;
  }
  return r;
}

std::vector<int32_t> device_of_nodes(const ComputationGraph& g, const Placement& p) {
  std::vector<int32_t> dev(g.nodes.size(), INT32_MIN);
  for (size_t i = 0; i < g.nodes.size(); ++i) {
    auto it = p.assignment.find(g.nodes[i].id);
    if (it != p.assignment.end()) dev[i] = it->second;
  }
  return dev;
}

SimulationReport sim_from(const dp_sim_report_t* r) {
  SimulationReport out;
  out.makespan = r->makespan;
  out.cross_transfer_count = r->cross_transfer_count;
  out.cross_transfer_bytes = r->cross_transfer_bytes;
  out.oom_flag = r->oom_flag != 0;
  for (int32_t d = 0; d < r->n_devices; ++d) {
    DeviceReport dr;
    dr.peak_memory_bytes = r->peak_memory[d];
    dr.memory_capacity_bytes = r->capacity[d];
    out.devices[r->device_ids[d]] = dr;
  }
  out.trace.resize(static_cast<size_t>(r->n_trace));
  for (int64_t t = 0; t < r->n_trace; ++t) {
    SimTaskRecord& rec = out.trace[t];
    rec.kind = static_cast<TaskKind>(r->tr_kind[t]);
    rec.node = r->tr_node[t];
    rec.edge_src = r->tr_src[t];
    rec.edge_dst = r->tr_dst[t];
    rec.device = r->tr_device[t];
    rec.start = r->tr_start[t];
    rec.end = r->tr_end[t];
    DeviceReport& dr = out.devices[rec.device];
    const BusyInterval iv{rec.start, rec.end};
    if (rec.kind == TaskKind::Compute) dr.compute_busy.push_back(iv);
    else if (rec.kind == TaskKind::Send) dr.send_busy.push_back(iv);
    else dr.receive_busy.push_back(iv);
  }
  return out;
}

template <typename T, typename F>
struct Owned {
  T* p = nullptr;
  F f;
  explicit Owned(F fn) : f(fn) {}
  ~Owned() {
    if (p) f(p);
  }
};

}  // namespace

// ---------------------------------------------------------------- graph.hpp
std::string_view to_string(ErrorKind kind) {
  static const char* names[] = {"CycleDetected", "DanglingEdge", "DuplicateId", "DuplicateEdge", "InvalidValue",
                                "ZeroComputeTime", "NoSuchEdge", "NodeExceedsClusterLimit",
                                "GroupExceedsClusterLimit", "InfeasiblePartition", "InvalidClusterMap",
                                "InsufficientSamples", "UnknownNode", "NodeUniverseMismatch", "UnplacedNode",
                                "InstanceTooLarge", "InstanceInfeasible", "UnreachableTargetCcr", "ParseError"};
  const int k = static_cast<int>(kind);
  return (k >= 0 && k < 19) ? names[k] : "UnknownError";
}

const NodeLevels& LevelTable::at(NodeId id) const {
  auto it = levels.find(id);
  if (it == levels.end()) throw DagError(ErrorKind::UnknownNode, "no levels for node " + std::to_string(id));
  return it->second;
}

Duration LevelTable::max_cpath() const {
  Duration best = 0;
  for (const auto& kv : levels) best = std::max(best, kv.second.cpath);
  return best;
}

ValidationResult validate(const ComputationGraph& graph) {
  Flat f(graph);
  Owned<dp_violation_list_t, void (*)(dp_violation_list_t*)> v(dp_violation_list_free);
  check(dp_validate(ctx(), &f.g, &v.p));
  ValidationResult r;
  r.ok = v.p->count == 0;
  for (int64_t i = 0; i < v.p->count; ++i) {
    Violation x;
    x.kind = static_cast<ErrorKind>(v.p->kind[i] - 1);
    x.message.assign(v.p->msg + v.p->msg_off[i], v.p->msg + v.p->msg_off[i + 1]);
    x.nodes.assign(v.p->nodes + v.p->node_off[i], v.p->nodes + v.p->node_off[i + 1]);
    r.violations.push_back(std::move(x));
  }
  return r;
}

void require_valid(const ComputationGraph& graph) {
  Flat f(graph);
  check(dp_require_valid(ctx(), &f.g));
}

Duration comm_time(Bytes bytes, const CommModel& model) {
  int64_t out = 0;
  check(dp_comm_time(bytes, cm(model), &out));
  return out;
}

double ccr(const ComputationGraph& graph, const CommModel& model) {
  Flat f(graph);
  double out = 0;
  check(dp_ccr(ctx(), &f.g, cm(model), &out));
  return out;
}

LevelTable compute_levels(const ComputationGraph& graph, const CommModel& model) {
  Flat f(graph);
  const size_t n = graph.nodes.size();
  std::vector<int64_t> t(n), b(n), c(n);
  check(dp_compute_levels(ctx(), &f.g, cm(model), t.data(), b.data(), c.data()));
  LevelTable table;
  table.levels.reserve(n);
  for (size_t i = 0; i < n; ++i) table.levels[graph.nodes[i].id] = {t[i], b[i], c[i]};
  return table;
}

// ---------------------------------------------------------------- graph_index.hpp
GraphIndex::GraphIndex(const ComputationGraph& graph) : graph_(&graph) {
  Flat f(graph);
  const int n = static_cast<int>(graph.nodes.size()), m = static_cast<int>(graph.edges.size());
  edge_src_.resize(m);
  edge_dst_.resize(m);
  out_start_.resize(n + 1);
  in_start_.resize(n + 1);
  out_list_.resize(m);
  in_list_.resize(m);
  check(dp_graph_index(ctx(), &f.g, edge_src_.data(), edge_dst_.data(), out_start_.data(), out_list_.data(),
                       in_start_.data(), in_list_.data()));
  index_.reserve(n);
  for (int v = 0; v < n; ++v) index_.emplace(graph.nodes[v].id, v);
}

int GraphIndex::index_of(NodeId id) const {
  auto it = index_.find(id);
  if (it == index_.end()) throw DagError(ErrorKind::UnknownNode, "node " + std::to_string(id) + " not in graph");
  return it->second;
}

std::span<const int> GraphIndex::out_edges(int v) const {
  return {out_list_.data() + out_start_[v], static_cast<size_t>(out_start_[v + 1] - out_start_[v])};
}

std::span<const int> GraphIndex::in_edges(int v) const {
  return {in_list_.data() + in_start_[v], static_cast<size_t>(in_start_[v + 1] - in_start_[v])};
}

// ---------------------------------------------------------------- ordering.hpp
std::string to_string(TopoPolicy policy) {
  switch (policy) {
    case TopoPolicy::MTopo: return "m-topo";
    case TopoPolicy::DfsTopo: return "dfs-topo";
    case TopoPolicy::CpdTopo: return "cpd-topo";
  }
  return "unknown";
}

TopoPolicy topo_policy_from_string(const std::string& name) {
  if (name == "m-topo" || name == "mtopo" || name == "m") return TopoPolicy::MTopo;
  if (name == "dfs-topo" || name == "dfs") return TopoPolicy::DfsTopo;
  if (name == "cpd-topo" || name == "cpd") return TopoPolicy::CpdTopo;
  throw DagError(ErrorKind::InvalidValue, "unknown topo policy '" + name + "'");
}

namespace {
TopoOrder topo(const ComputationGraph& graph, TopoPolicy policy, const LevelTable* levels) {
  Flat f(graph);
  std::vector<int64_t> cp;
  if (levels) {
    // the peel needs every node's cpath; LevelTable::at throws UnknownNode like cpd_topo
    // would on its first missing lookup — but only after the validity check, so validate
    // first (ordering.cpp:99-100).
    check(dp_require_valid(ctx(), &f.g));
    cp.reserve(graph.nodes.size());
    for (const auto& n : graph.nodes) cp.push_back(levels->at(n.id).cpath);
  }
  TopoOrder o;
  o.policy = policy;
  o.sequence.resize(graph.nodes.size());
  check(dp_topo_order(ctx(), &f.g, static_cast<int32_t>(policy), levels ? cp.data() : nullptr, o.sequence.data()));
  return o;
}
}  // namespace

TopoOrder m_topo(const ComputationGraph& graph) { return topo(graph, TopoPolicy::MTopo, nullptr); }
TopoOrder dfs_topo(const ComputationGraph& graph) { return topo(graph, TopoPolicy::DfsTopo, nullptr); }
TopoOrder cpd_topo(const ComputationGraph& graph, const LevelTable& levels) {
  return topo(graph, TopoPolicy::CpdTopo, &levels);
}

bool is_valid_topo_order(const ComputationGraph& graph, const TopoOrder& order) {
  Flat f(graph);
  int32_t out = 0;
  check(dp_is_valid_topo_order(ctx(), &f.g, order.sequence.data(), static_cast<int64_t>(order.sequence.size()),
                               &out));
  return out != 0;
}

// ---------------------------------------------------------------- fusion.hpp
bool merge_is_safe(const ComputationGraph& graph, NodeId u, NodeId v) {
  Flat f(graph);
  int32_t out = 0;
  check(dp_merge_is_safe(ctx(), &f.g, u, v, &out));
  return out != 0;
}

ClusterMap optimal_breakpoints(const ComputationGraph& graph, const TopoOrder& order, const CommModel& model,
                               const FusionConfig& config) {
  Flat f(graph);
  Owned<dp_cluster_map_t, void (*)(dp_cluster_map_t*)> m(dp_cluster_map_free);
  check(dp_optimal_breakpoints(ctx(), &f.g, order.sequence.data(), static_cast<int64_t>(order.sequence.size()),
                               cm(model), config.range, config.cluster_memory_limit, &m.p));
  return map_from(m.p, graph);
}

CoarseGraph build_coarse_graph(const ComputationGraph& graph, const TopoOrder& order, const ClusterMap& clusters) {
  Flat f(graph);
  std::vector<int64_t> ids;
  std::vector<int32_t> cl;
  ids.reserve(clusters.node_to_cluster.size());
  for (const auto& kv : clusters.node_to_cluster) {
    ids.push_back(kv.first);
    cl.push_back(kv.second);
  }
  std::vector<int32_t> cid;
  std::vector<int64_t> off{0}, mem;
  for (const Cluster& c : clusters.clusters) {
    cid.push_back(c.id);
    mem.insert(mem.end(), c.members.begin(), c.members.end());
    off.push_back(static_cast<int64_t>(mem.size()));
  }
  Owned<dp_graph_out_t, void (*)(dp_graph_out_t*)> o(dp_graph_out_free);
  check(dp_build_coarse_graph(ctx(), &f.g, order.sequence.data(), static_cast<int64_t>(order.sequence.size()),
                              ids.data(), cl.data(), static_cast<int64_t>(ids.size()),
                              static_cast<int64_t>(clusters.clusters.size()), cid.data(), off.data(), mem.data(),
                              &o.p));
  return from_out(o.p, true, nullptr);
}

GroupContraction contract_colocation_groups(const ComputationGraph& graph) {
  Flat f(graph);
  Owned<dp_contraction_t, void (*)(dp_contraction_t*)> c(dp_contraction_free);
  check(dp_contract_colocation_groups(ctx(), &f.g, &c.p));
  GroupContraction r;
  r.contracted = from_out(c.p->contracted, false, &graph);
  for (int64_t i = 0; i < c.p->contracted->n_nodes; ++i)
    r.members_of[c.p->contracted->node_id[i]].assign(c.p->members + c.p->member_off[i],
                                                     c.p->members + c.p->member_off[i + 1]);
  return r;
}

FusionResult fuse(const ComputationGraph& graph, const CommModel& model, const FusionConfig& config) {
  Flat f(graph);
  Owned<dp_fusion_result_t, void (*)(dp_fusion_result_t*)> r(dp_fusion_result_free);
  check(dp_fuse(ctx(), &f.g, cm(model), config.range, config.cluster_memory_limit, &r.p));
  return {from_out(r.p->coarse, true, nullptr), map_from(r.p->map, graph)};
}

// ---------------------------------------------------------------- placement.hpp
// DeviceTimeline is a caller-owned value type; its two methods keep the reference's
// semantics (placement.cpp:13-32) on the host object.  The placement kernels use the
// device timeline of csrc/placement.cu.
Duration DeviceTimeline::find_slot(Duration earliest, Duration duration) const {
  Duration cand = earliest;
  for (const BusyInterval& iv : busy_) {
    if (iv.end <= cand) continue;
    if (iv.start >= cand && iv.start - cand >= duration) break;
    cand = std::max(cand, iv.end);
  }
  return cand;
}

void DeviceTimeline::reserve(Duration start, Duration duration) {
  const BusyInterval iv{start, start + duration};
  auto pos = std::upper_bound(busy_.begin(), busy_.end(), iv,
                              [](const BusyInterval& a, const BusyInterval& b) { return a.start < b.start; });
  busy_.insert(pos, iv);
}

SchedulerState SchedulerState::for_devices(const std::vector<DeviceSpec>& devices) {
  if (devices.empty()) throw DagError(ErrorKind::InvalidValue, "device list is empty");
  std::vector<DeviceSpec> sorted = devices;
  std::sort(sorted.begin(), sorted.end(), [](const DeviceSpec& a, const DeviceSpec& b) { return a.id < b.id; });
  SchedulerState s;
  for (const DeviceSpec& d : sorted) {
    if (d.memory_bytes <= 0)
      throw DagError(ErrorKind::InvalidValue, "device " + std::to_string(d.id) + " has non-positive memory capacity");
    if (!s.device_ids.empty() && s.device_ids.back() == d.id)
      throw DagError(ErrorKind::DuplicateId, "device id " + std::to_string(d.id) + " repeats");
    s.device_ids.push_back(d.id);
    s.available_memory.push_back(d.memory_bytes);
  }
  s.timelines.resize(s.device_ids.size());
  return s;
}

int SchedulerState::device_pos(DeviceId id) const {
  auto it = std::lower_bound(device_ids.begin(), device_ids.end(), id);
  if (it == device_ids.end() || *it != id)
    throw DagError(ErrorKind::InvalidValue, "unknown device id " + std::to_string(id));
  return static_cast<int>(it - device_ids.begin());
}

PlacementResult order_place(const CoarseGraph& coarse, const TopoOrder& order, const std::vector<DeviceSpec>& devices) {
  Flat f(coarse);
  FlatDevices fd(devices);
  Owned<dp_placement_result_t, void (*)(dp_placement_result_t*)> p(dp_placement_result_free);
  check(dp_order_place(ctx(), &f.g, order.sequence.data(), static_cast<int64_t>(order.sequence.size()), &fd.d, &p.p));
  return placement_from(p.p, coarse);
}

PlacementResult adjusting_placement(const CoarseGraph& coarse, const TopoOrder& order,
                                    const std::vector<DeviceSpec>& devices, const CommModel& model) {
  Flat f(coarse);
  FlatDevices fd(devices);
  Owned<dp_placement_result_t, void (*)(dp_placement_result_t*)> p(dp_placement_result_free);
  check(dp_adjusting_placement(ctx(), &f.g, order.sequence.data(), static_cast<int64_t>(order.sequence.size()),
                               &fd.d, cm(model), &p.p));
  return placement_from(p.p, coarse);
}

// compute_est (placement.cpp:220-237): a single-node query against a caller-owned
// SchedulerState; evaluated on that host state (data-ready time + find_slot).
Duration compute_est(const SchedulerState& state, const CoarseGraph& graph,
                     const std::unordered_map<NodeId, DeviceId>& assignment, NodeId node, DeviceId device,
                     const CommModel& model) {
  GraphIndex ix(graph);
  const int v = ix.index_of(node);
  const int d = state.device_pos(device);
  if (state.available_memory[d] < ix.node(v).memory_bytes) return kNever;
  Duration pre = 0;
  for (int e : ix.in_edges(v)) {
    const int p = ix.edge_src(e);
    const NodeId pid = ix.node(p).id;
    auto it = assignment.find(pid);
    if (it == assignment.end())
      throw DagError(ErrorKind::UnplacedNode, "predecessor " + std::to_string(pid) + " not placed yet");
    const int pd = state.device_pos(it->second);
    const Duration finish = state.finish_time.at(pid);
    pre = std::max(pre, finish + (pd == d ? 0 : comm_time(graph.edges[e].tensor_bytes, model)));
  }
  return state.timelines[d].find_slot(pre, ix.node(v).compute_us);
}

Placement expand_placement(const ComputationGraph& original, const ClusterMap& clusters,
                           const Placement& coarse_placement) {
  Flat f(original);
  if (clusters.node_to_cluster.size() != original.nodes.size()) {
    // GraphIndex(original) runs first in the reference (placement.cpp:241-246)
    const size_t n = original.nodes.size(), m = original.edges.size();
    std::vector<int32_t> es(m), ed(m), os(n + 1), ol(m), is(n + 1), il(m);
    check(dp_graph_index(ctx(), &f.g, es.data(), ed.data(), os.data(), ol.data(), is.data(), il.data()));
    throw DagError(ErrorKind::InvalidClusterMap, "cluster map covers " +
                                                     std::to_string(clusters.node_to_cluster.size()) +
                                                     " nodes, graph has " + std::to_string(n));
  }
  std::vector<int32_t> nc(original.nodes.size(), 0);  // count already checked above
  std::vector<int64_t> off{0}, mem;
  std::vector<int32_t> dev;
  std::vector<uint8_t> placed;
  for (const Cluster& c : clusters.clusters) {
    mem.insert(mem.end(), c.members.begin(), c.members.end());
    off.push_back(static_cast<int64_t>(mem.size()));
    auto it = coarse_placement.assignment.find(c.id);
    dev.push_back(it == coarse_placement.assignment.end() ? 0 : it->second);
    placed.push_back(it != coarse_placement.assignment.end());
  }
  Owned<dp_placement_result_t, void (*)(dp_placement_result_t*)> p(dp_placement_result_free);
  check(dp_expand_placement(ctx(), &f.g, nc.data(), static_cast<int64_t>(clusters.clusters.size()), off.data(),
                            mem.data(), dev.data(), placed.data(), &p.p));
  return placement_from(p.p, original).placement;
}

// ---------------------------------------------------------------- simulator.hpp
std::string to_string(TaskKind kind) {
  switch (kind) {
    case TaskKind::Compute: return "compute";
    case TaskKind::Send: return "send";
    case TaskKind::Receive: return "receive";
  }
  return "unknown";
}

SimulationReport simulate(const ComputationGraph& graph, const Placement& placement,
                          const std::vector<DeviceSpec>& devices, const CommModel& model) {
  Flat f(graph);
  FlatDevices fd(devices);
  std::vector<int32_t> dev = device_of_nodes(graph, placement);
  Owned<dp_sim_report_t, void (*)(dp_sim_report_t*)> r(dp_sim_report_free);
  check(dp_simulate(ctx(), &f.g, dev.data(), &fd.d, cm(model), 1, &r.p));
  return sim_from(r.p);
}

std::pair<Placement, Duration> brute_force_optimal(const ComputationGraph& graph,
                                                   const std::vector<DeviceSpec>& devices, const CommModel& model) {
  Flat f(graph);
  FlatDevices fd(devices);
  std::vector<int32_t> best(graph.nodes.size());
  int64_t ms = 0;
  check(dp_brute_force_optimal(ctx(), &f.g, &fd.d, cm(model), best.data(), &ms));
  Placement p;
  std::vector<DeviceSpec> sorted = devices;
  std::sort(sorted.begin(), sorted.end(), [](const DeviceSpec& a, const DeviceSpec& b) { return a.id < b.id; });
  for (const auto& d : sorted) p.per_device_memory[d.id] = 0;
  for (size_t i = 0; i < graph.nodes.size(); ++i) {
    p.assignment[graph.nodes[i].id] = best[i];
    p.per_device_memory[best[i]] += graph.nodes[i].memory_bytes;
  }
  return {std::move(p), ms};
}

// ---------------------------------------------------------------- estimation.hpp
// Standard Evaluation (estimation.cpp) on the GPU (estimation.cu through the C-ABI).
// The profile-universe checks run here first, over the same unordered_maps as the
// reference, so a missing node is named in the reference's (hash) order.
NodeCostModel fit_node_models(const ProfileSet& profiles) {
  std::set<std::int64_t> sizes;
  for (const auto& b : profiles.batches) sizes.insert(b.batch_size);
  if (sizes.size() < 2)
    throw DagError(ErrorKind::InsufficientSamples,
                   "need at least 2 distinct batch sizes, got " + std::to_string(sizes.size()));
  const auto& universe = profiles.batches.front().nodes;
  for (const auto& b : profiles.batches) {
    if (b.nodes.size() != universe.size())
      throw DagError(ErrorKind::NodeUniverseMismatch,
                     "batch " + std::to_string(b.batch_size) + " profiles a different node set");
    for (const auto& kv : universe)
      if (!b.nodes.count(kv.first))
        throw DagError(ErrorKind::NodeUniverseMismatch, "node " + std::to_string(kv.first) + " missing from batch " +
                                                            std::to_string(b.batch_size));
  }
  std::vector<int64_t> bs, off{0}, id, mem, w;
  for (const auto& b : profiles.batches) {
    bs.push_back(b.batch_size);
    for (const auto& kv : b.nodes) {
      id.push_back(kv.first);
      mem.push_back(kv.second.memory_bytes);
      w.push_back(kv.second.compute_us);
    }
    off.push_back(static_cast<int64_t>(id.size()));
  }
  dp_profiles_t pc{static_cast<int32_t>(bs.size()), bs.data(), off.data(), id.data(), mem.data(), w.data()};
  dp_node_models_t* m = nullptr;
  check(dp_fit_node_models(ctx(), &pc, &m));
  NodeCostModel model;
  for (int64_t i = 0; i < m->n; ++i) {
    const double* f = m->fit + 6 * i;
    model.memory_fit[m->node_id[i]] = LinearFit{f[0], f[1], f[2]};
    model.time_fit[m->node_id[i]] = LinearFit{f[3], f[4], f[5]};
  }
  dp_node_models_free(m);
  return model;
}

ComputationGraph estimate_graph(const ComputationGraph& base, const NodeCostModel& models, std::int64_t target_batch,
                                const EdgeScaling& scaling) {
  Flat f(base);
  std::vector<int64_t> mid;
  for (const auto& kv : models.memory_fit)
    if (models.time_fit.count(kv.first)) mid.push_back(kv.first);
  std::sort(mid.begin(), mid.end());
  std::vector<double> fit(mid.size() * 6);
  for (size_t i = 0; i < mid.size(); ++i) {
    const LinearFit& a = models.memory_fit.at(mid[i]);
    const LinearFit& b = models.time_fit.at(mid[i]);
    double* x = fit.data() + 6 * i;
    x[0] = a.slope; x[1] = a.intercept; x[2] = a.residual_norm;
    x[3] = b.slope; x[4] = b.intercept; x[5] = b.residual_norm;
  }
  dp_node_models_t mc{static_cast<int64_t>(mid.size()), mid.data(), fit.data()};
  std::vector<int64_t> os, od;
  std::vector<double> of;
  for (const auto& kv : scaling.scale_override) {
    os.push_back(kv.first.first);
    od.push_back(kv.first.second);
    of.push_back(kv.second);
  }
  dp_graph_out_t* o = nullptr;
  check(dp_estimate_graph(ctx(), &f.g, &mc, target_batch, scaling.reference_batch, static_cast<int64_t>(os.size()),
                          os.data(), od.data(), of.data(), &o));
  ComputationGraph est = base;
  for (size_t i = 0; i < est.nodes.size(); ++i) {
    est.nodes[i].memory_bytes = o->memory_bytes[i];
    est.nodes[i].compute_us = o->compute_us[i];
  }
  for (size_t e = 0; e < est.edges.size(); ++e) est.edges[e].tensor_bytes = o->edge_bytes[e];
  dp_graph_out_free(o);
  return est;
}

CommModel fit_comm_model(const std::vector<std::pair<Bytes, double>>& samples) {
  std::vector<int64_t> b;
  std::vector<double> u;
  for (const auto& s : samples) {
    b.push_back(s.first);
    u.push_back(s.second);
  }
  dp_comm_t c{};
  check(dp_fit_comm_model(ctx(), static_cast<int64_t>(b.size()), b.data(), u.data(), &c));
  return CommModel{c.k_us_per_byte, c.b_us};
}

PlacementResult sequential_eval_placement(const ComputationGraph& estimated, const std::vector<DeviceSpec>& devices) {
  return order_place(estimated, dfs_topo(estimated), devices);  // estimation.cpp:142-146
}

DeviationReport deviation_report(const ComputationGraph& estimated, const ComputationGraph& measured) {
  Flat fe(estimated), fm(measured);
  dp_deviation_t* d = nullptr;
  check(dp_deviation_report(ctx(), &fe.g, &fm.g, &d));
  DeviationReport r;
  for (int64_t i = 0; i < d->n_memory; ++i) r.memory_deviation[d->memory_id[i]] = d->memory_dev[i];
  for (int64_t i = 0; i < d->n_time; ++i) r.time_deviation[d->time_id[i]] = d->time_dev[i];
  r.mean_memory_deviation = d->mean_memory;
  r.mean_time_deviation = d->mean_time;
  r.zero_memory_nodes.assign(d->zero_memory, d->zero_memory + d->n_zero_memory);
  r.zero_time_nodes.assign(d->zero_time, d->zero_time + d->n_zero_time);
  dp_deviation_free(d);
  return r;
}

// ---------------------------------------------------------------- pipeline.hpp
std::string to_string(PlaceStrategy strategy) {
  switch (strategy) {
    case PlaceStrategy::Order: return "order";
    case PlaceStrategy::Adjust: return "adjust";
    case PlaceStrategy::SequentialEval: return "sequential-eval";
  }
  return "unknown";
}

PlaceStrategy place_strategy_from_string(const std::string& name) {
  if (name == "order" || name == "order-place") return PlaceStrategy::Order;
  if (name == "adjust" || name == "adjusting") return PlaceStrategy::Adjust;
  if (name == "sequential-eval" || name == "sequential") return PlaceStrategy::SequentialEval;
  throw DagError(ErrorKind::InvalidValue, "unknown placement strategy '" + name + "'");
}

PipelineReport evaluate_pipeline(const ComputationGraph& graph, const std::optional<ProfileSet>& profiles,
                                 const std::vector<DeviceSpec>& devices, const CommModel& device_comm,
                                 const PipelineConfig& config) {
  if (devices.empty()) throw DagError(ErrorKind::InvalidValue, "device list is empty");
  require_valid(graph);
  PipelineReport report;
  CommModel comm = device_comm;
  report.comm_source = "devices";
  ComputationGraph working = graph;
  if (profiles) {  // pipeline.cpp:40-54
    if (!config.target_batch) throw DagError(ErrorKind::InvalidValue, "profiles given but no target batch");
    NodeCostModel models = fit_node_models(*profiles);
    std::int64_t reference = 0;
    for (const auto& b : profiles->batches) reference = std::max(reference, b.batch_size);
    EdgeScaling scaling;
    scaling.reference_batch = reference;
    working = estimate_graph(graph, models, *config.target_batch, scaling);
    if (profiles->comm_samples.size() >= 2) {
      comm = fit_comm_model(profiles->comm_samples);
      report.comm_source = "fitted";
    }
  }
  Flat f(working);
  FlatDevices fd(devices);
  dp_pipeline_config_t cfg{config.fusion_range, config.cluster_mem_fraction,
                           config.strategy == PlaceStrategy::Order ? 0 : 1, 2};
  Owned<dp_pipeline_result_t, void (*)(dp_pipeline_result_t*)> r(dp_pipeline_result_free);
  check(dp_pipeline(ctx(), &f.g, &fd.d, cm(comm), &cfg, &r.p));
  report.original_nodes = r.p->original_nodes;
  report.original_edges = r.p->original_edges;
  report.original_ccr = r.p->original_ccr;
  report.coarse_nodes = r.p->coarse_nodes;
  report.coarse_edges = r.p->coarse_edges;
  report.coarse_ccr = r.p->coarse_ccr;
  report.node_reduction_factor =
      static_cast<double>(report.original_nodes) / static_cast<double>(report.coarse_nodes);
  report.ccr_reduction_factor = report.coarse_ccr > 0 ? report.original_ccr / report.coarse_ccr : 0.0;
  report.fusion.coarse = from_out(r.p->fusion->coarse, true, nullptr);
  report.fusion.map = map_from(r.p->fusion->map, working);
  report.generation_wall_us = static_cast<Duration>(r.p->generation_ms * 1000.0);
  PlacementResult order_res = placement_from(r.p->coarse_order, report.fusion.coarse);
  PlacementResult adjust_res = placement_from(r.p->coarse_adjust, report.fusion.coarse);
  Placement order_exp = placement_from(r.p->order_expanded, working).placement;
  Placement adjust_exp = placement_from(r.p->adjust_expanded, working).placement;
  report.order_place = {r.p->order_makespan, order_res.oom_risk};
  report.adjusting = {r.p->adjust_makespan, adjust_res.oom_risk};
  report.chosen_strategy = to_string(config.strategy);
  if (config.strategy == PlaceStrategy::SequentialEval) {
    PlacementResult seq = sequential_eval_placement(working, devices);
    report.chosen_oom_risk = seq.oom_risk;
    report.chosen_placement = seq.placement;
    report.chosen_simulation = simulate(working, seq.placement, devices, comm);
  } else if (config.strategy == PlaceStrategy::Order) {  // the report of pipeline.cpp:89, reused (:100-103)
    report.chosen_oom_risk = order_res.oom_risk;
    report.chosen_placement = std::move(order_exp);
    report.chosen_simulation = sim_from(r.p->order_sim);
  } else {  // pipeline.cpp:90, reused (:104-107)
    report.chosen_oom_risk = adjust_res.oom_risk;
    report.chosen_placement = std::move(adjust_exp);
    report.chosen_simulation = sim_from(r.p->adjust_sim);
  }
  return report;
}

// ---------------------------------------------------------------- generator.hpp
// gen_graph: input synthesis (host), the reference generator's documented recipe
// (generator.hpp:14-36): mt19937_64, u(lo,hi) = lo + rng() % (hi-lo+1), CCR bisection.
std::string to_string(GenKind kind) {
  switch (kind) {
    case GenKind::Layered: return "layered";
    case GenKind::RandomDag: return "random-dag";
    case GenKind::ParallelChains: return "parallel-chains";
  }
  return "unknown";
}

GenKind gen_kind_from_string(const std::string& name) {
  if (name == "layered") return GenKind::Layered;
  if (name == "random-dag" || name == "random") return GenKind::RandomDag;
  if (name == "parallel-chains" || name == "chains") return GenKind::ParallelChains;
  throw DagError(ErrorKind::InvalidValue, "unknown generator kind '" + name + "'");
}

namespace {
struct Rng {
  std::mt19937_64 eng;
  explicit Rng(std::uint64_t s) : eng(s) {}
  std::int64_t uniform(std::int64_t lo, std::int64_t hi) {
    if (hi <= lo) return lo;
    return lo + static_cast<std::int64_t>(eng() % (static_cast<std::uint64_t>(hi - lo) + 1));
  }
};
std::int64_t around(Rng& r, std::int64_t mean, std::int64_t spread, std::int64_t floor_v) {
  return std::max(floor_v, r.uniform(mean - spread, mean + spread));
}
OpNode make_node(const SyntheticSpec& s, Rng& r, std::int64_t id, std::string name) {
  OpNode n;
  n.id = id;
  n.name = std::move(name);
  n.compute_us = around(r, s.compute_mean_us, s.compute_spread_us, 1);
  n.memory_bytes = around(r, s.memory_mean_bytes, s.memory_spread_bytes, 1);
  return n;
}
double host_ccr(const ComputationGraph& g, const CommModel& c) {
  Duration tc = 0, tm = 0;
  for (const auto& n : g.nodes) tc += n.compute_us;
  if (tc <= 0) throw DagError(ErrorKind::ZeroComputeTime, "total compute time is zero");
  for (const auto& e : g.edges) tm += comm_time(e.tensor_bytes, c);
  return static_cast<double>(tm) / static_cast<double>(tc);
}
}  // namespace

ComputationGraph gen_graph(const SyntheticSpec& spec) {
  if (spec.node_count < 1) throw DagError(ErrorKind::InvalidValue, "node count must be >= 1");
  Rng rng(spec.seed);
  ComputationGraph g;
  const int n = spec.node_count;
  const Bytes eb = spec.edge_bytes_mean;
  if (spec.kind == GenKind::Layered) {
    const int width = std::max(1, spec.layer_width);
    std::vector<std::vector<NodeId>> layers;
    for (int i = 0; i < n; ++i) {
      if (i / width >= static_cast<int>(layers.size())) layers.emplace_back();
      layers[i / width].push_back(i);
      g.nodes.push_back(make_node(spec, rng, i, "op" + std::to_string(i)));
    }
    for (size_t l = 1; l < layers.size(); ++l) {
      const auto& prev = layers[l - 1];
      for (NodeId v : layers[l]) {
        const int k = static_cast<int>(std::min<std::int64_t>(static_cast<std::int64_t>(prev.size()), rng.uniform(1, 3)));
        std::vector<NodeId> pool = prev;
        for (int t = 0; t < k; ++t) {
          const std::int64_t pick = rng.uniform(0, static_cast<std::int64_t>(pool.size()) - 1);
          const NodeId u = pool[pick];
          pool.erase(pool.begin() + pick);
          g.edges.push_back({u, v, around(rng, eb, eb / 2, 1)});
        }
      }
    }
    std::sort(g.edges.begin(), g.edges.end(), [](const TensorEdge& a, const TensorEdge& b) {
      return a.src != b.src ? a.src < b.src : a.dst < b.dst;
    });
  } else if (spec.kind == GenKind::RandomDag) {
    for (int i = 0; i < n; ++i) g.nodes.push_back(make_node(spec, rng, i, "op" + std::to_string(i)));
    for (int v = 1; v < n; ++v) {
      const int fanin = static_cast<int>(rng.uniform(1, std::min(3, v)));
      std::vector<NodeId> picked;
      while (static_cast<int>(picked.size()) < fanin) {
        const NodeId u = rng.uniform(0, v - 1);
        if (std::find(picked.begin(), picked.end(), u) == picked.end()) picked.push_back(u);
      }
      std::sort(picked.begin(), picked.end());
      for (NodeId u : picked) g.edges.push_back({u, v, around(rng, eb, eb / 2, 1)});
    }
  } else {
    const int chains = std::max(1, spec.layer_width);
    const int per = std::max(1, n / chains);
    int next = 0;
    for (int c = 0; c < chains && next < n; ++c) {
      const int len = (c == chains - 1) ? n - next : per;
      for (int i = 0; i < len; ++i) {
        g.nodes.push_back(make_node(spec, rng, next, "chain" + std::to_string(c) + "_op" + std::to_string(i)));
        if (i > 0) g.edges.push_back({next - 1, next, around(rng, eb, eb / 2, 1)});
        ++next;
      }
    }
  }
  if (spec.target_ccr) {
    const double target = *spec.target_ccr;
    if (target <= 0) throw DagError(ErrorKind::InvalidValue, "target CCR must be > 0");
    if (g.edges.empty()) throw DagError(ErrorKind::UnreachableTargetCcr, "graph has no edges to carry communication");
    std::vector<Bytes> base;
    for (const auto& e : g.edges) base.push_back(e.tensor_bytes);
    auto apply = [&](double factor) {
      for (size_t e = 0; e < g.edges.size(); ++e) {
        const double scaled = static_cast<double>(base[e]) * factor;
        g.edges[e].tensor_bytes = std::max<Bytes>(0, static_cast<Bytes>(std::llround(std::min(scaled, 1.0e15))));
      }
      return host_ccr(g, spec.comm);
    };
    double lo = 0.0, hi = 1.0;
    double achieved = apply(hi);
    int expand = 0;
    while (achieved < target && expand < 60) {
      hi *= 2;
      achieved = apply(hi);
      ++expand;
    }
    if (achieved < target)
      throw DagError(ErrorKind::UnreachableTargetCcr, "cannot raise CCR to " + std::to_string(target));
    for (int it = 0; it < 64; ++it) {
      const double mid = (lo + hi) / 2;
      if (apply(mid) < target) lo = mid; else hi = mid;
    }
    achieved = apply(hi);
    if (std::abs(achieved - target) / target > 0.2)
      throw DagError(ErrorKind::UnreachableTargetCcr, "achieved CCR " + std::to_string(achieved) + " misses target " +
                                                          std::to_string(target) + " by more than 20%");
  }
  require_valid(g);
  return g;
}

}  // namespace dagplace
