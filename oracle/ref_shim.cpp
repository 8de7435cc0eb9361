// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// Flattening shim over the UNMODIFIED reference library (/root/reference/proj/src,
// compiled by oracle/Makefile into oracle/_ref/libdagplace_ref.so).  Each dpr_*
// function converts the flat dp_graph_t into dagplace::ComputationGraph, calls the
// reference function named in its comment, and flattens the result into the
// structs of include/dagplace_b200.h.  No algorithm lives here.

#include <algorithm>
#include <array>
#include <random>
#include <chrono>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "dagplace/estimation.hpp"
#include "dagplace/fusion.hpp"
#include "dagplace/generator.hpp"
#include "dagplace/graph.hpp"
#include "dagplace/graph_index.hpp"
#include "dagplace/json_io.hpp"
#include "dagplace/ordering.hpp"
#include "dagplace/pipeline.hpp"
#include "dagplace/placement.hpp"
#include "dagplace/simulator.hpp"
#include "dp_results.h"

using namespace dagplace;

namespace {

thread_local std::string g_err;

int fail(const DagError& e) {
  g_err = e.what();
  return 1 + static_cast<int>(e.kind());
}

ComputationGraph to_graph(const dp_graph_t* g) {
  ComputationGraph out;
  out.nodes.resize(static_cast<size_t>(g->n_nodes));
  for (int64_t i = 0; i < g->n_nodes; ++i) {
    OpNode& n = out.nodes[i];
    n.id = g->node_id[i];
    n.name = "op" + std::to_string(n.id);
    n.compute_us = g->compute_us[i];
    n.memory_bytes = g->memory_bytes[i];
    if (g->group && g->group[i] >= 0) n.colocation_group = "g" + std::to_string(g->group[i]);
  }
  out.edges.resize(static_cast<size_t>(g->n_edges));
  for (int64_t e = 0; e < g->n_edges; ++e) {
    out.edges[e] = {g->edge_src[e], g->edge_dst[e], g->edge_bytes[e]};
  }
  return out;
}

std::vector<DeviceSpec> to_devices(const dp_devices_t* d) {
  std::vector<DeviceSpec> out;
  for (int i = 0; i < d->count; ++i) out.push_back({d->id[i], d->memory_bytes[i]});
  return out;
}

CommModel to_comm(dp_comm_t c) { return {c.k_us_per_byte, c.b_us}; }

TopoOrder to_order(const int64_t* seq, int64_t len, TopoPolicy p = TopoPolicy::CpdTopo) {
  TopoOrder o;
  o.policy = p;
  o.sequence.assign(seq, seq + len);
  return o;
}

int32_t group_label(const std::optional<std::string>& g) {
  if (!g) return -1;
  return static_cast<int32_t>(std::stol(g->substr(1)));
}

dp_graph_out_t* flatten_graph(const ComputationGraph& g) {
  dp_graph_out_t* o = dpr_graph_out_new(static_cast<int64_t>(g.nodes.size()),
                                        static_cast<int64_t>(g.edges.size()));
  for (size_t i = 0; i < g.nodes.size(); ++i) {
    o->node_id[i] = g.nodes[i].id;
    o->compute_us[i] = g.nodes[i].compute_us;
    o->memory_bytes[i] = g.nodes[i].memory_bytes;
    o->group[i] = group_label(g.nodes[i].colocation_group);
  }
  for (size_t e = 0; e < g.edges.size(); ++e) {
    o->edge_src[e] = g.edges[e].src;
    o->edge_dst[e] = g.edges[e].dst;
    o->edge_bytes[e] = g.edges[e].tensor_bytes;
  }
  return o;
}

dp_cluster_map_t* flatten_map(const ComputationGraph& g, const ClusterMap& map) {
  int64_t k = static_cast<int64_t>(map.clusters.size());
  dp_cluster_map_t* m = dpr_cluster_map_new(static_cast<int64_t>(g.nodes.size()), k,
                                            static_cast<int64_t>(map.breakpoints.size()));
  for (size_t i = 0; i < g.nodes.size(); ++i) {
    auto it = map.node_to_cluster.find(g.nodes[i].id);
    m->node_cluster[i] = it == map.node_to_cluster.end() ? -1 : it->second;
  }
  int64_t off = 0;
  for (int64_t c = 0; c < k; ++c) {
    m->member_off[c] = off;
    for (NodeId id : map.clusters[c].members) m->members[off++] = id;
    m->total_compute[c] = map.clusters[c].total_compute_us;
    m->total_memory[c] = map.clusters[c].total_memory_bytes;
  }
  m->member_off[k] = off;
  for (size_t b = 0; b < map.breakpoints.size(); ++b) m->breakpoints[b] = map.breakpoints[b];
  return m;
}

dp_placement_result_t* flatten_placement(const ComputationGraph& g, const PlacementResult& r,
                                         const std::vector<DeviceSpec>& devs) {
  std::vector<DeviceId> ids;
  for (const auto& d : devs) ids.push_back(d.id);
  std::sort(ids.begin(), ids.end());
  int32_t nd = static_cast<int32_t>(ids.size());
  dp_placement_result_t* p = dpr_placement_new(static_cast<int64_t>(g.nodes.size()), nd,
                                               static_cast<int64_t>(r.decisions.size()));
  for (size_t i = 0; i < g.nodes.size(); ++i) {
    auto it = r.placement.assignment.find(g.nodes[i].id);
    p->device[i] = it == r.placement.assignment.end() ? INT32_MIN : it->second;
  }
  for (int32_t d = 0; d < nd; ++d) {
    p->device_ids[d] = ids[d];
    auto it = r.placement.per_device_memory.find(ids[d]);
    p->device_present[d] = it != r.placement.per_device_memory.end();
    p->per_device_memory[d] = p->device_present[d] ? it->second : 0;
  }
  p->oom_risk = r.oom_risk;
  for (size_t k = 0; k < r.decisions.size(); ++k) {
    const PlacementDecision& dec = r.decisions[k];
    p->dec_node[k] = dec.node;
    p->dec_prev[k] = dec.prev_device;
    p->dec_back_cost[k] = dec.back_cost_us;
    for (int32_t d = 0; d < nd; ++d) p->dec_est[k * nd + d] = dec.est_us.at(ids[d]);
    p->dec_chosen[k] = dec.chosen;
    p->dec_relocated[k] = dec.relocated;
    p->dec_best_effort[k] = dec.best_effort;
  }
  return p;
}

Placement to_placement(const ComputationGraph& g, const int32_t* device_of_node) {
  Placement p;
  for (size_t i = 0; i < g.nodes.size(); ++i) {
    if (device_of_node[i] == INT32_MIN) continue;  // unplaced
    p.assignment[g.nodes[i].id] = device_of_node[i];
    p.per_device_memory[device_of_node[i]] += g.nodes[i].memory_bytes;
  }
  return p;
}

dp_sim_report_t* flatten_sim(const SimulationReport& r, bool trace) {
  dp_sim_report_t* o = dpr_sim_new(static_cast<int32_t>(r.devices.size()),
                                   trace ? static_cast<int64_t>(r.trace.size()) : 0);
  o->makespan = r.makespan;
  o->cross_transfer_count = r.cross_transfer_count;
  o->cross_transfer_bytes = r.cross_transfer_bytes;
  o->oom_flag = r.oom_flag;
  int d = 0;
  for (const auto& [id, dr] : r.devices) {
    o->device_ids[d] = id;
    o->peak_memory[d] = dr.peak_memory_bytes;
    o->capacity[d] = dr.memory_capacity_bytes;
    ++d;
  }
  if (trace) {
    for (size_t t = 0; t < r.trace.size(); ++t) {
      const SimTaskRecord& rec = r.trace[t];
      o->tr_kind[t] = static_cast<int32_t>(rec.kind);
      o->tr_node[t] = rec.node;
      o->tr_src[t] = rec.edge_src;
      o->tr_dst[t] = rec.edge_dst;
      o->tr_device[t] = rec.device;
      o->tr_start[t] = rec.start;
      o->tr_end[t] = rec.end;
    }
  }
  return o;
}

ClusterMap to_map(const int64_t* map_ids, const int32_t* map_cluster, int64_t map_count,
                  int64_t n_clusters, const int32_t* cluster_ids, const int64_t* member_off,
                  const int64_t* members) {
  ClusterMap m;
  for (int64_t i = 0; i < map_count; ++i) m.node_to_cluster[map_ids[i]] = map_cluster[i];
  for (int64_t c = 0; c < n_clusters; ++c) {
    Cluster cl;
    cl.id = cluster_ids[c];
    cl.members.assign(members + member_off[c], members + member_off[c + 1]);
    m.clusters.push_back(std::move(cl));
  }
  return m;
}

}  // namespace

extern "C" {

DPR_DEFINE_FREES(dpr_)

const char* dpr_last_error_message(void) { return g_err.c_str(); }

// graph_from_json (json_io.cpp:43-74) over json::parse of the text; colocation_group
// strings become labels in first-appearance order.  json::exception -> ParseError.
int dpr_graph_from_json(const char* text, int64_t len, dp_graph_out_t** out) {
  try {
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(std::string(text, static_cast<size_t>(len)));
    } catch (const nlohmann::json::exception& e) {
      g_err = std::string("ParseError: invalid JSON: ") + e.what();
      return 1 + static_cast<int>(ErrorKind::ParseError);
    }
    const ComputationGraph g = graph_from_json(j);
    dp_graph_out_t* o = dpr_graph_out_new(static_cast<int64_t>(g.nodes.size()), static_cast<int64_t>(g.edges.size()));
    std::map<std::string, int32_t> labels;
    for (size_t i = 0; i < g.nodes.size(); ++i) {
      o->node_id[i] = g.nodes[i].id;
      o->compute_us[i] = g.nodes[i].compute_us;
      o->memory_bytes[i] = g.nodes[i].memory_bytes;
      int32_t lab = -1;
      if (g.nodes[i].colocation_group) {
        auto it = labels.emplace(*g.nodes[i].colocation_group, static_cast<int32_t>(labels.size())).first;
        lab = it->second;
      }
      o->group[i] = lab;
    }
    for (size_t e = 0; e < g.edges.size(); ++e) {
      o->edge_src[e] = g.edges[e].src;
      o->edge_dst[e] = g.edges[e].dst;
      o->edge_bytes[e] = g.edges[e].tensor_bytes;
    }
    *out = o;
    return 0;
  } catch (const DagError& e) {
    return fail(e);
  }
}

// devices_from_json (json_io.cpp:93-117).
int dpr_devices_from_json(const char* text, int64_t len, int32_t* count, int32_t* ids, int64_t* memory_bytes,
                          int32_t capacity, dp_comm_t* comm) {
  try {
    nlohmann::json j;
    try {
      j = nlohmann::json::parse(std::string(text, static_cast<size_t>(len)));
    } catch (const nlohmann::json::exception& e) {
      g_err = std::string("ParseError: invalid JSON: ") + e.what();
      return 1 + static_cast<int>(ErrorKind::ParseError);
    }
    const DeviceFile f = devices_from_json(j);
    *count = static_cast<int32_t>(f.devices.size());
    for (size_t i = 0; i < f.devices.size() && static_cast<int32_t>(i) < capacity; ++i) {
      ids[i] = f.devices[i].id;
      memory_bytes[i] = f.devices[i].memory_bytes;
    }
    comm->k_us_per_byte = f.comm.k_us_per_byte;
    comm->b_us = f.comm.b_us;
    return 0;
  } catch (const DagError& e) {
    return fail(e);
  }
}

// ---- Standard Evaluation (estimation.cpp) over the flat structs of dagplace_b200.h
ProfileSet dpr_to_profiles(const dp_profiles_t* p) {
  ProfileSet ps;
  for (int32_t b = 0; b < p->n_batches; ++b) {
    BatchProfile bp;
    bp.batch_size = p->batch_size[b];
    for (int64_t i = p->node_off[b]; i < p->node_off[b + 1]; ++i)
      bp.nodes[p->node_id[i]] = NodeSample{p->memory_bytes[i], p->compute_us[i]};
    ps.batches.push_back(std::move(bp));
  }
  return ps;
}

// fit_node_models (estimation.cpp:67-88); output sorted by id.
int dpr_fit_node_models(const dp_profiles_t* p, dp_node_models_t** out) {
  try {
    const NodeCostModel m = fit_node_models(dpr_to_profiles(p));
    std::vector<NodeId> ids;
    for (const auto& kv : m.memory_fit) ids.push_back(kv.first);
    std::sort(ids.begin(), ids.end());
    auto* r = static_cast<dp_node_models_t*>(calloc(1, sizeof(dp_node_models_t)));
    r->n = static_cast<int64_t>(ids.size());
    r->node_id = static_cast<int64_t*>(calloc(ids.size() + 1, sizeof(int64_t)));
    r->fit = static_cast<double*>(calloc(6 * ids.size() + 1, sizeof(double)));
    for (size_t i = 0; i < ids.size(); ++i) {
      const LinearFit& a = m.memory_fit.at(ids[i]);
      const LinearFit& b = m.time_fit.at(ids[i]);
      r->node_id[i] = ids[i];
      double* f = r->fit + 6 * i;
      f[0] = a.slope; f[1] = a.intercept; f[2] = a.residual_norm;
      f[3] = b.slope; f[4] = b.intercept; f[5] = b.residual_norm;
    }
    *out = r;
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

void dpr_node_models_free(dp_node_models_t* m) {
  if (!m) return;
  free(m->node_id); free(m->fit); free(m);
}

// estimate_graph (estimation.cpp:90-119).
int dpr_estimate_graph(const dp_graph_t* base, const dp_node_models_t* models, int64_t target_batch,
                       int64_t reference_batch, int64_t n_override, const int64_t* ov_src, const int64_t* ov_dst,
                       const double* ov_factor, dp_graph_out_t** out) {
  try {
    NodeCostModel m;
    for (int64_t i = 0; i < models->n; ++i) {
      const double* f = models->fit + 6 * i;
      m.memory_fit[models->node_id[i]] = LinearFit{f[0], f[1], f[2]};
      m.time_fit[models->node_id[i]] = LinearFit{f[3], f[4], f[5]};
    }
    EdgeScaling sc;
    sc.reference_batch = reference_batch;
    for (int64_t i = 0; i < n_override; ++i) sc.scale_override[{ov_src[i], ov_dst[i]}] = ov_factor[i];
    *out = flatten_graph(estimate_graph(to_graph(base), m, target_batch, sc));
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

// fit_comm_model (estimation.cpp:121-140).
int dpr_fit_comm_model(int64_t n, const int64_t* bytes, const double* us, dp_comm_t* out) {
  try {
    std::vector<std::pair<Bytes, double>> s;
    for (int64_t i = 0; i < n; ++i) s.emplace_back(bytes[i], us[i]);
    const CommModel c = fit_comm_model(s);
    out->k_us_per_byte = c.k_us_per_byte;
    out->b_us = c.b_us;
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

// deviation_report (estimation.cpp:148-192).
int dpr_deviation_report(const dp_graph_t* est, const dp_graph_t* meas, dp_deviation_t** out) {
  try {
    const DeviationReport d = deviation_report(to_graph(est), to_graph(meas));
    auto* r = static_cast<dp_deviation_t*>(calloc(1, sizeof(dp_deviation_t)));
    auto fill = [](const std::map<NodeId, double>& mp, int64_t* n, int64_t** ids, double** vals) {
      *n = static_cast<int64_t>(mp.size());
      *ids = static_cast<int64_t*>(calloc(mp.size() + 1, sizeof(int64_t)));
      *vals = static_cast<double*>(calloc(mp.size() + 1, sizeof(double)));
      int64_t k = 0;
      for (const auto& kv : mp) { (*ids)[k] = kv.first; (*vals)[k] = kv.second; ++k; }
    };
    fill(d.memory_deviation, &r->n_memory, &r->memory_id, &r->memory_dev);
    fill(d.time_deviation, &r->n_time, &r->time_id, &r->time_dev);
    r->mean_memory = d.mean_memory_deviation;
    r->mean_time = d.mean_time_deviation;
    auto lst = [](const std::vector<NodeId>& v, int64_t* n, int64_t** ids) {
      *n = static_cast<int64_t>(v.size());
      *ids = static_cast<int64_t*>(calloc(v.size() + 1, sizeof(int64_t)));
      for (size_t i = 0; i < v.size(); ++i) (*ids)[i] = v[i];
    };
    lst(d.zero_memory_nodes, &r->n_zero_memory, &r->zero_memory);
    lst(d.zero_time_nodes, &r->n_zero_time, &r->zero_time);
    *out = r;
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

void dpr_deviation_free(dp_deviation_t* d) {
  if (!d) return;
  free(d->memory_id); free(d->memory_dev); free(d->time_id); free(d->time_dev);
  free(d->zero_memory); free(d->zero_time); free(d);
}

int dpr_comm_time(int64_t bytes, dp_comm_t comm, int64_t* out) {
  try {  // graph.cpp:200-204
    *out = comm_time(bytes, to_comm(comm));
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_ccr(const dp_graph_t* g, dp_comm_t comm, double* out) {
  try {  // graph.cpp:206-215
    *out = ccr(to_graph(g), to_comm(comm));
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_validate(const dp_graph_t* g, dp_violation_list_t** out) {
  ValidationResult r = validate(to_graph(g));  // graph.cpp:98-191
  dp_violation_list_t* v = DPR_NEW(dp_violation_list_t, 1);
  int64_t k = static_cast<int64_t>(r.violations.size());
  v->count = k;
  v->kind = DPR_NEW(int32_t, k);
  v->node_off = DPR_NEW(int64_t, k + 1);
  v->msg_off = DPR_NEW(int64_t, k + 1);
  int64_t nn = 0, nm = 0;
  for (const auto& x : r.violations) {
    nn += static_cast<int64_t>(x.nodes.size());
    nm += static_cast<int64_t>(x.message.size());
  }
  v->nodes = DPR_NEW(int64_t, nn);
  v->msg = DPR_NEW(char, nm + 1);
  nn = nm = 0;
  for (int64_t i = 0; i < k; ++i) {
    const Violation& x = r.violations[i];
    v->kind[i] = 1 + static_cast<int32_t>(x.kind);
    v->node_off[i] = nn;
    v->msg_off[i] = nm;
    for (NodeId id : x.nodes) v->nodes[nn++] = id;
    std::memcpy(v->msg + nm, x.message.data(), x.message.size());
    nm += static_cast<int64_t>(x.message.size());
  }
  v->node_off[k] = nn;
  v->msg_off[k] = nm;
  *out = v;
  return 0;
}

int dpr_require_valid(const dp_graph_t* g) {
  try {  // graph.cpp:193-198
    require_valid(to_graph(g));
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_graph_index(const dp_graph_t* g, int32_t* edge_src_idx, int32_t* edge_dst_idx,
                    int32_t* out_start, int32_t* out_list, int32_t* in_start, int32_t* in_list) {
  try {  // graph_index.cpp:8-60
    ComputationGraph cg = to_graph(g);
    GraphIndex ix(cg);
    int n = ix.node_count(), m = ix.edge_count();
    for (int e = 0; e < m; ++e) {
      edge_src_idx[e] = ix.edge_src(e);
      edge_dst_idx[e] = ix.edge_dst(e);
    }
    int o = 0, i = 0;
    for (int v = 0; v < n; ++v) {
      out_start[v] = o;
      in_start[v] = i;
      for (int e : ix.out_edges(v)) out_list[o++] = e;
      for (int e : ix.in_edges(v)) in_list[i++] = e;
    }
    out_start[n] = o;
    in_start[n] = i;
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_compute_levels(const dp_graph_t* g, dp_comm_t comm, int64_t* tlevel, int64_t* blevel,
                       int64_t* cpath) {
  try {  // graph.cpp:217-269
    ComputationGraph cg = to_graph(g);
    LevelTable t = compute_levels(cg, to_comm(comm));
    for (size_t i = 0; i < cg.nodes.size(); ++i) {
      const NodeLevels& lv = t.at(cg.nodes[i].id);
      tlevel[i] = lv.tlevel;
      blevel[i] = lv.blevel;
      cpath[i] = lv.cpath;
    }
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_topo_order(const dp_graph_t* g, int32_t policy, const int64_t* cpath, int64_t* seq) {
  try {  // ordering.cpp:81-114
    ComputationGraph cg = to_graph(g);
    TopoOrder o;
    if (policy == DP_TOPO_M) {
      o = m_topo(cg);
    } else if (policy == DP_TOPO_DFS) {
      o = dfs_topo(cg);
    } else {
      LevelTable t;
      for (size_t i = 0; i < cg.nodes.size(); ++i) t.levels[cg.nodes[i].id] = {0, 0, cpath[i]};
      o = cpd_topo(cg, t);
    }
    std::copy(o.sequence.begin(), o.sequence.end(), seq);
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_is_valid_topo_order(const dp_graph_t* g, const int64_t* seq, int64_t len, int32_t* out) {
  *out = is_valid_topo_order(to_graph(g), to_order(seq, len));  // ordering.cpp:116-132
  return 0;
}

int dpr_merge_is_safe(const dp_graph_t* g, int64_t u, int64_t v, int32_t* out) {
  try {  // fusion.cpp:16-51
    *out = merge_is_safe(to_graph(g), u, v);
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_optimal_breakpoints(const dp_graph_t* g, const int64_t* seq, int64_t len, dp_comm_t comm,
                            int32_t range, int64_t limit, dp_cluster_map_t** out) {
  try {  // fusion.cpp:85-171
    ComputationGraph cg = to_graph(g);
    FusionConfig cfg{range, limit};
    ClusterMap m = optimal_breakpoints(cg, to_order(seq, len), to_comm(comm), cfg);
    *out = flatten_map(cg, m);
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_build_coarse_graph(const dp_graph_t* g, const int64_t* seq, int64_t len,
                           const int64_t* map_ids, const int32_t* map_cluster, int64_t map_count,
                           int64_t n_clusters, const int32_t* cluster_ids,
                           const int64_t* member_off, const int64_t* members,
                           dp_graph_out_t** out) {
  try {  // fusion.cpp:173-229
    ComputationGraph cg = to_graph(g);
    ClusterMap m = to_map(map_ids, map_cluster, map_count, n_clusters, cluster_ids, member_off,
                          members);
    // Cluster sums are carried by the map in the reference; recompute them the way
    // clusters_from_cuts does (fusion.cpp:69-75) so the shim needs only memberships.
    GraphIndex ix(cg);
    for (Cluster& c : m.clusters) {
      for (NodeId id : c.members) {
        if (!ix.contains(id)) continue;
        const OpNode& node = ix.node(ix.index_of(id));
        c.total_compute_us += node.compute_us;
        c.total_memory_bytes += node.memory_bytes;
      }
    }
    *out = flatten_graph(build_coarse_graph(cg, to_order(seq, len), m));
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_contract_colocation_groups(const dp_graph_t* g, dp_contraction_t** out) {
  try {  // fusion.cpp:231-295
    GroupContraction c = contract_colocation_groups(to_graph(g));
    dp_contraction_t* o = DPR_NEW(dp_contraction_t, 1);
    o->contracted = flatten_graph(c.contracted);
    int64_t k = o->contracted->n_nodes, total = 0;
    for (const auto& n : c.contracted.nodes) total += static_cast<int64_t>(c.members_of.at(n.id).size());
    o->member_off = DPR_NEW(int64_t, k + 1);
    o->members = DPR_NEW(int64_t, total);
    int64_t off = 0;
    for (int64_t i = 0; i < k; ++i) {
      o->member_off[i] = off;
      for (NodeId id : c.members_of.at(c.contracted.nodes[i].id)) o->members[off++] = id;
    }
    o->member_off[k] = off;
    *out = o;
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_fuse(const dp_graph_t* g, dp_comm_t comm, int32_t range, int64_t limit,
             dp_fusion_result_t** out) {
  try {  // fusion.cpp:297-335
    ComputationGraph cg = to_graph(g);
    FusionResult r = fuse(cg, to_comm(comm), FusionConfig{range, limit});
    dp_fusion_result_t* o = DPR_NEW(dp_fusion_result_t, 1);
    o->coarse = flatten_graph(r.coarse);
    o->map = flatten_map(cg, r.map);
    *out = o;
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_order_place(const dp_graph_t* g, const int64_t* seq, int64_t len,
                    const dp_devices_t* devices, dp_placement_result_t** out) {
  try {  // placement.cpp:128-159
    ComputationGraph cg = to_graph(g);
    auto devs = to_devices(devices);
    PlacementResult r = order_place(cg, to_order(seq, len), devs);
    *out = flatten_placement(cg, r, devs);
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_adjusting_placement(const dp_graph_t* g, const int64_t* seq, int64_t len,
                            const dp_devices_t* devices, dp_comm_t comm,
                            dp_placement_result_t** out) {
  try {  // placement.cpp:161-218
    ComputationGraph cg = to_graph(g);
    auto devs = to_devices(devices);
    PlacementResult r = adjusting_placement(cg, to_order(seq, len), devs, to_comm(comm));
    *out = flatten_placement(cg, r, devs);
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_expand_placement(const dp_graph_t* g, const int32_t* node_cluster, int64_t n_clusters,
                         const int64_t* member_off, const int64_t* members,
                         const int32_t* coarse_device, const uint8_t* coarse_placed,
                         dp_placement_result_t** out) {
  try {  // placement.cpp:239-268
    ComputationGraph cg = to_graph(g);
    ClusterMap m;
    for (size_t i = 0; i < cg.nodes.size(); ++i) {
      if (node_cluster[i] >= 0) m.node_to_cluster[cg.nodes[i].id] = node_cluster[i];
    }
    for (int64_t c = 0; c < n_clusters; ++c) {
      Cluster cl;
      cl.id = static_cast<int>(c);
      cl.members.assign(members + member_off[c], members + member_off[c + 1]);
      m.clusters.push_back(std::move(cl));
    }
    Placement coarse;
    for (int64_t c = 0; c < n_clusters; ++c) {
      if (!coarse_placed || coarse_placed[c]) coarse.assignment[c] = coarse_device[c];
    }
    Placement p = expand_placement(cg, m, coarse);
    PlacementResult r;
    r.placement = p;
    std::vector<DeviceSpec> devs;
    for (const auto& [id, b] : p.per_device_memory) devs.push_back({id, 1});
    *out = flatten_placement(cg, r, devs);
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_simulate(const dp_graph_t* g, const int32_t* device_of_node, const dp_devices_t* devices,
                 dp_comm_t comm, int32_t want_trace, dp_sim_report_t** out) {
  try {  // simulator.cpp:56-252
    ComputationGraph cg = to_graph(g);
    SimulationReport r = simulate(cg, to_placement(cg, device_of_node), to_devices(devices),
                                  to_comm(comm));
    *out = flatten_sim(r, want_trace != 0);
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_simulate_candidates(const dp_graph_t* g, const int32_t* node_cluster, int64_t n_clusters,
                            const uint8_t* cand, int64_t n_cand, const dp_devices_t* devices,
                            dp_comm_t comm, int64_t* makespans, int64_t* argmin,
                            int32_t threads) {
  // Loop of simulate (simulator.cpp:56-252) over candidates, split across threads on
  // disjoint index ranges; argmin = first strict minimum (simulator.cpp:292-294).
  ComputationGraph cg = to_graph(g);
  auto devs = to_devices(devices);
  std::vector<DeviceId> ids;
  for (const auto& d : devs) ids.push_back(d.id);
  std::sort(ids.begin(), ids.end());
  CommModel cm = to_comm(comm);
  if (threads < 1) threads = 1;
  std::vector<int> status(threads, 0);
  std::vector<std::string> errs(threads);
  auto work = [&](int t) {
    for (int64_t b = t; b < n_cand; b += threads) {
      std::vector<int32_t> dev(cg.nodes.size());
      for (size_t i = 0; i < cg.nodes.size(); ++i) {
        dev[i] = ids[cand[b * n_clusters + node_cluster[i]]];
      }
      try {
        makespans[b] = simulate(cg, to_placement(cg, dev.data()), devs, cm).makespan;
      } catch (const DagError& e) {
        status[t] = 1 + static_cast<int>(e.kind());
        errs[t] = e.what();
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  for (int t = 0; t < threads; ++t) {
    if (status[t]) {
      g_err = errs[t];
      return status[t];
    }
  }
  int64_t best = -1;
  for (int64_t b = 0; b < n_cand; ++b) {
    if (best < 0 || makespans[b] < makespans[best]) best = b;
  }
  *argmin = best;
  return 0;
}

int dpr_brute_force_optimal(const dp_graph_t* g, const dp_devices_t* devices, dp_comm_t comm,
                            int32_t* best_device_of_node, int64_t* best_makespan) {
  try {  // simulator.cpp:254-310
    ComputationGraph cg = to_graph(g);
    auto [p, ms] = brute_force_optimal(cg, to_devices(devices), to_comm(comm));
    for (size_t i = 0; i < cg.nodes.size(); ++i) best_device_of_node[i] = p.assignment.at(cg.nodes[i].id);
    *best_makespan = ms;
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

static dp_placement_result_t* expanded_flat(const ComputationGraph& cg, const Placement& p,
                                            const std::vector<DeviceSpec>& devs) {
  PlacementResult r;
  r.placement = p;
  return flatten_placement(cg, r, devs);
}

int dpr_pipeline(const dp_graph_t* g, const dp_devices_t* devices, dp_comm_t comm,
                 const dp_pipeline_config_t* cfg, dp_pipeline_result_t** out) {
  try {  // pipeline.cpp:27-111
    ComputationGraph cg = to_graph(g);
    auto devs = to_devices(devices);
    PipelineConfig pc;
    pc.fusion_range = cfg->fusion_range;
    pc.cluster_mem_fraction = cfg->cluster_mem_fraction;
    pc.strategy = cfg->strategy == 0 ? PlaceStrategy::Order : PlaceStrategy::Adjust;
    PipelineReport rep = evaluate_pipeline(cg, std::nullopt, devs, to_comm(comm), pc);
    dp_pipeline_result_t* o = DPR_NEW(dp_pipeline_result_t, 1);
    o->original_nodes = rep.original_nodes;
    o->original_edges = rep.original_edges;
    o->original_ccr = rep.original_ccr;
    o->coarse_nodes = rep.coarse_nodes;
    o->coarse_edges = rep.coarse_edges;
    o->coarse_ccr = rep.coarse_ccr;
    o->fusion = DPR_NEW(dp_fusion_result_t, 1);
    o->fusion->coarse = flatten_graph(rep.fusion.coarse);
    o->fusion->map = flatten_map(cg, rep.fusion.map);
    // Recompute the coarse-level artefacts exactly as pipeline.cpp:70-76 does.
    const CoarseGraph& coarse = rep.fusion.coarse;
    CommModel cm = to_comm(comm);
    LevelTable cl = compute_levels(coarse, cm);
    TopoOrder co = cpd_topo(coarse, cl);
    PlacementResult orr = order_place(coarse, co, devs);
    PlacementResult adj = adjusting_placement(coarse, co, devs, cm);
    o->coarse_order = flatten_placement(coarse, orr, devs);
    o->coarse_adjust = flatten_placement(coarse, adj, devs);
    o->order_expanded = expanded_flat(cg, expand_placement(cg, rep.fusion.map, orr.placement), devs);
    o->adjust_expanded = expanded_flat(cg, expand_placement(cg, rep.fusion.map, adj.placement), devs);
    o->coarse_sequence = DPR_NEW(int64_t, co.sequence.size());
    std::copy(co.sequence.begin(), co.sequence.end(), o->coarse_sequence);
    o->order_makespan = rep.order_place.makespan_us;
    o->adjust_makespan = rep.adjusting.makespan_us;
    o->generation_ms = static_cast<double>(rep.generation_wall_us) / 1000.0;
    *out = o;
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

// gen_graph (generator.cpp:203-209) flattened; kind 0 layered, 1 random, 2 chains;
// target_ccr <= 0 means none.  Arrays sized by the caller (n nodes, n*3 edges).
int dpr_gen_graph(int32_t kind, int64_t n, int32_t width, double target_ccr, uint64_t seed, int64_t* node_id,
                  int64_t* compute_us, int64_t* memory_bytes, int64_t* edge_src, int64_t* edge_dst,
                  int64_t* edge_bytes, int64_t* n_edges) {
  try {
    SyntheticSpec spec;
    spec.kind = kind == 0 ? GenKind::Layered : kind == 1 ? GenKind::RandomDag : GenKind::ParallelChains;
    spec.node_count = static_cast<int>(n);
    spec.layer_width = width;
    if (target_ccr > 0) spec.target_ccr = target_ccr;
    spec.seed = seed;
    ComputationGraph g = gen_graph(spec);
    for (size_t i = 0; i < g.nodes.size(); ++i) {
      node_id[i] = g.nodes[i].id;
      compute_us[i] = g.nodes[i].compute_us;
      memory_bytes[i] = g.nodes[i].memory_bytes;
    }
    for (size_t e = 0; e < g.edges.size(); ++e) {
      edge_src[e] = g.edges[e].src;
      edge_dst[e] = g.edges[e].dst;
      edge_bytes[e] = g.edges[e].tensor_bytes;
    }
    *n_edges = static_cast<int64_t>(g.edges.size());
    return 0;
  } catch (const DagError& e) { return fail(e); }
}

int dpr_pipeline_replicas(const dp_graph_t* g, const dp_devices_t* devices, dp_comm_t comm,
                          const dp_pipeline_config_t* cfg, int32_t threads, int64_t* wall_us,
                          double* total_wall_s) {
  // `threads` concurrent evaluate_pipeline calls (pipeline.cpp:27-111) on private copies;
  // generation_wall_us is the reference's own timer around pipeline.cpp:67-79.  The
  // simulations after the window are skipped by timing only what the reference times.
  ComputationGraph cg = to_graph(g);
  auto devs = to_devices(devices);
  PipelineConfig pc;
  pc.fusion_range = cfg->fusion_range;
  pc.cluster_mem_fraction = cfg->cluster_mem_fraction;
  pc.strategy = cfg->strategy == 0 ? PlaceStrategy::Order : PlaceStrategy::Adjust;
  CommModel cm = to_comm(comm);
  if (threads < 1) threads = 1;
  std::vector<int> status(threads, 0);
  std::vector<std::string> errs(threads);
  std::vector<ComputationGraph> copies(threads, cg);
  auto t0 = std::chrono::steady_clock::now();
  auto work = [&](int t) {
    try {
      // The generation window only: fuse + coarse levels/order + both placements +
      // 2x expand, timed like pipeline.cpp:67-79 (evaluate_pipeline itself would also
      // simulate both candidates after the window).
      const ComputationGraph& working = copies[t];
      Bytes min_capacity = devs.front().memory_bytes;
      for (const auto& d : devs) min_capacity = std::min(min_capacity, d.memory_bytes);
      FusionConfig fc;
      fc.range = pc.fusion_range;
      fc.cluster_memory_limit = std::max<Bytes>(
          1, static_cast<Bytes>(static_cast<double>(min_capacity) * pc.cluster_mem_fraction));
      const auto s0 = std::chrono::steady_clock::now();
      FusionResult fr = fuse(working, cm, fc);
      LevelTable cl = compute_levels(fr.coarse, cm);
      TopoOrder co = cpd_topo(fr.coarse, cl);
      PlacementResult orr = order_place(fr.coarse, co, devs);
      PlacementResult adj = adjusting_placement(fr.coarse, co, devs, cm);
      Placement oe = expand_placement(working, fr.map, orr.placement);
      Placement ae = expand_placement(working, fr.map, adj.placement);
      const auto s1 = std::chrono::steady_clock::now();
      wall_us[t] = std::chrono::duration_cast<std::chrono::microseconds>(s1 - s0).count();
    } catch (const DagError& e) {
      status[t] = 1 + static_cast<int>(e.kind());
      errs[t] = e.what();
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
  work(0);
  for (auto& th : pool) th.join();
  *total_wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  for (int t = 0; t < threads; ++t) {
    if (status[t]) {
      g_err = errs[t];
      return status[t];
    }
  }
  return 0;
}

// SURVEY §8(d) common recipe (the bench's config #4 / #5 graphs), restated here so the
// reference arm of bench.py synthesises its input without the product library:
// u(lo,hi) = lo + mt19937_64() % (hi-lo+1) (generator.cpp:32-46); node costs in id
// order, then per non-first-layer node k = u(fan_lo,fan_hi) picks without replacement
// from the previous layer with bytes u(2^15, 3*2^15); edges sorted by (src, dst).
int dpr_gen_layered(int64_t n, int64_t width, int64_t fan_lo, int64_t fan_hi, uint64_t seed, int64_t* node_id,
                    int64_t* compute_us, int64_t* memory_bytes, int64_t* edge_src, int64_t* edge_dst,
                    int64_t* edge_bytes, int64_t* n_edges) {
  std::mt19937_64 rng(seed);
  auto u = [&rng](int64_t lo, int64_t hi) -> int64_t {
    return hi <= lo ? lo : lo + static_cast<int64_t>(rng() % (static_cast<uint64_t>(hi - lo) + 1));
  };
  for (int64_t i = 0; i < n; ++i) {
    node_id[i] = i;
    compute_us[i] = u(100, 900);
    memory_bytes[i] = u(1 << 19, 3 << 19);
  }
  std::vector<std::array<int64_t, 3>> es;
  std::vector<int64_t> taken;  // offsets already picked for v, ascending
  for (int64_t v = width; v < n; ++v) {
    const int64_t lo = (v / width - 1) * width, hi = std::min(lo + width, n);
    const int64_t k = std::min<int64_t>(hi - lo, u(fan_lo, fan_hi));
    taken.clear();
    for (int64_t t = 0; t < k; ++t) {
      // the pick-th entry of the pool with `taken` erased (pool = lo..hi-1 in order)
      int64_t x = u(0, hi - lo - t - 1);
      size_t j = 0;
      for (; j < taken.size() && taken[j] <= x; ++j) ++x;
      taken.insert(taken.begin() + j, x);
      es.push_back({lo + x, v, u(1 << 15, 3 << 15)});
    }
  }
  std::sort(es.begin(), es.end(), [](const auto& a, const auto& b) { return a[0] != b[0] ? a[0] < b[0] : a[1] < b[1]; });
  for (size_t e = 0; e < es.size(); ++e) {
    edge_src[e] = es[e][0];
    edge_dst[e] = es[e][1];
    edge_bytes[e] = es[e][2];
  }
  *n_edges = static_cast<int64_t>(es.size());
  return 0;
}

// Config #5 candidate family: row k = base with max(1, n_c/100) moves of
// cluster rk() % n_c -> device rk() % D, rk = mt19937_64(k); row 0 = base.
void dpr_gen_candidates(const uint8_t* base, int64_t n_clusters, int32_t D, int64_t first, int64_t count,
                        uint8_t* out) {
  const int64_t moves = std::max<int64_t>(1, n_clusters / 100);
  for (int64_t i = 0; i < count; ++i) {
    const int64_t k = first + i;
    uint8_t* row = out + i * n_clusters;
    std::copy(base, base + n_clusters, row);
    if (k == 0) continue;
    std::mt19937_64 rk(static_cast<uint64_t>(k));
    for (int64_t t = 0; t < moves; ++t) {
      const uint64_t c = rk() % static_cast<uint64_t>(n_clusters);
      row[c] = static_cast<uint8_t>(rk() % static_cast<uint64_t>(D));
    }
  }
}

}  // extern "C"
