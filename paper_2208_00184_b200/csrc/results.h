// results.h — host allocation of the C-ABI result structs (include/dagplace_b200.h).
#pragma once

#include <cstdlib>
#include <new>
#include <cstring>

#include "../../include/dagplace_b200.h"

namespace dpb {

template <typename T>
inline T* halloc(int64_t count) {
  void* p = std::calloc(static_cast<size_t>(count > 0 ? count : 1), sizeof(T));
  if (!p) throw std::bad_alloc();
  return static_cast<T*>(p);
}

inline dp_graph_out_t* new_graph_out(int64_t n, int64_t m) {
  auto* g = halloc<dp_graph_out_t>(1);
  g->n_nodes = n;
  g->n_edges = m;
  g->node_id = halloc<int64_t>(n);
  g->compute_us = halloc<int64_t>(n);
  g->memory_bytes = halloc<int64_t>(n);
  g->group = halloc<int32_t>(n);
  g->edge_src = halloc<int64_t>(m);
  g->edge_dst = halloc<int64_t>(m);
  g->edge_bytes = halloc<int64_t>(m);
  return g;
}
inline void free_graph_out(dp_graph_out_t* g) {
  if (!g) return;
  std::free(g->node_id); std::free(g->compute_us); std::free(g->memory_bytes); std::free(g->group);
  std::free(g->edge_src); std::free(g->edge_dst); std::free(g->edge_bytes); std::free(g);
}
inline dp_cluster_map_t* new_cluster_map(int64_t n, int64_t k, int64_t nb) {
  auto* m = halloc<dp_cluster_map_t>(1);
  m->n_nodes = n;
  m->node_cluster = halloc<int32_t>(n);
  m->n_clusters = k;
  m->member_off = halloc<int64_t>(k + 1);
  m->members = halloc<int64_t>(n);
  m->total_compute = halloc<int64_t>(k);
  m->total_memory = halloc<int64_t>(k);
  m->n_breakpoints = nb;
  m->breakpoints = halloc<int32_t>(nb);
  return m;
}
inline void free_cluster_map(dp_cluster_map_t* m) {
  if (!m) return;
  std::free(m->node_cluster); std::free(m->member_off); std::free(m->members);
  std::free(m->total_compute); std::free(m->total_memory); std::free(m->breakpoints); std::free(m);
}
inline dp_placement_result_t* new_placement(int64_t n, int32_t d, int64_t ndec) {
  auto* p = halloc<dp_placement_result_t>(1);
  p->n_nodes = n;
  p->device = halloc<int32_t>(n);
  p->n_devices = d;
  p->device_ids = halloc<int32_t>(d);
  p->per_device_memory = halloc<int64_t>(d);
  p->device_present = halloc<uint8_t>(d);
  p->n_decisions = ndec;
  p->dec_node = halloc<int64_t>(ndec);
  p->dec_prev = halloc<int32_t>(ndec);
  p->dec_back_cost = halloc<int64_t>(ndec);
  p->dec_est = halloc<int64_t>(ndec * (d > 0 ? d : 1));
  p->dec_chosen = halloc<int32_t>(ndec);
  p->dec_relocated = halloc<uint8_t>(ndec);
  p->dec_best_effort = halloc<uint8_t>(ndec);
  return p;
}
inline void free_placement(dp_placement_result_t* p) {
  if (!p) return;
  std::free(p->device); std::free(p->device_ids); std::free(p->per_device_memory);
  std::free(p->device_present); std::free(p->dec_node); std::free(p->dec_prev);
  std::free(p->dec_back_cost); std::free(p->dec_est); std::free(p->dec_chosen);
  std::free(p->dec_relocated); std::free(p->dec_best_effort); std::free(p);
}
inline dp_sim_report_t* new_sim(int32_t d, int64_t ntrace) {
  auto* r = halloc<dp_sim_report_t>(1);
  r->n_devices = d;
  r->device_ids = halloc<int32_t>(d);
  r->peak_memory = halloc<int64_t>(d);
  r->capacity = halloc<int64_t>(d);
  r->n_trace = ntrace;
  r->tr_kind = halloc<int32_t>(ntrace);
  r->tr_node = halloc<int64_t>(ntrace);
  r->tr_src = halloc<int64_t>(ntrace);
  r->tr_dst = halloc<int64_t>(ntrace);
  r->tr_device = halloc<int32_t>(ntrace);
  r->tr_start = halloc<int64_t>(ntrace);
  r->tr_end = halloc<int64_t>(ntrace);
  return r;
}
inline void free_sim(dp_sim_report_t* r) {
  if (!r) return;
  std::free(r->device_ids); std::free(r->peak_memory); std::free(r->capacity);
  std::free(r->tr_kind); std::free(r->tr_node); std::free(r->tr_src); std::free(r->tr_dst);
  std::free(r->tr_device); std::free(r->tr_start); std::free(r->tr_end); std::free(r);
}

}  // namespace dpb
