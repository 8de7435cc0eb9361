/*
 * dp_results.h — TEST INFRASTRUCTURE ONLY: allocation helpers for the result
 * structs of include/dagplace_b200.h, shared by the oracle restatement and the
 * reference shim.  Every array is a separate malloc; free functions tolerate NULL.
 */
#ifndef DP_RESULTS_H_
#define DP_RESULTS_H_

#include <stdlib.h>
#include <string.h>

#include "dp_oracle.h"

#ifdef __cplusplus
#define DPR_CAST(T, x) static_cast<T>(x)
#else
#define DPR_CAST(T, x) (T)(x)
#endif

static inline void* dpr_zalloc(size_t n) {
  void* p = calloc(n ? n : 1, 1);
  return p;
}
#define DPR_NEW(T, count) DPR_CAST(T*, dpr_zalloc(sizeof(T) * (size_t)(count)))

static inline dp_graph_out_t* dpr_graph_out_new(int64_t n, int64_t m) {
  dp_graph_out_t* g = DPR_NEW(dp_graph_out_t, 1);
  g->n_nodes = n;
  g->n_edges = m;
  g->node_id = DPR_NEW(int64_t, n);
  g->compute_us = DPR_NEW(int64_t, n);
  g->memory_bytes = DPR_NEW(int64_t, n);
  g->group = DPR_NEW(int32_t, n);
  g->edge_src = DPR_NEW(int64_t, m);
  g->edge_dst = DPR_NEW(int64_t, m);
  g->edge_bytes = DPR_NEW(int64_t, m);
  return g;
}
static inline void dpr_graph_out_free_(dp_graph_out_t* g) {
  if (!g) return;
  free(g->node_id); free(g->compute_us); free(g->memory_bytes); free(g->group);
  free(g->edge_src); free(g->edge_dst); free(g->edge_bytes); free(g);
}
static inline dp_cluster_map_t* dpr_cluster_map_new(int64_t n, int64_t k, int64_t nb) {
  dp_cluster_map_t* m = DPR_NEW(dp_cluster_map_t, 1);
  m->n_nodes = n;
  m->node_cluster = DPR_NEW(int32_t, n);
  m->n_clusters = k;
  m->member_off = DPR_NEW(int64_t, k + 1);
  m->members = DPR_NEW(int64_t, n);
  m->total_compute = DPR_NEW(int64_t, k);
  m->total_memory = DPR_NEW(int64_t, k);
  m->n_breakpoints = nb;
  m->breakpoints = DPR_NEW(int32_t, nb);
  return m;
}
static inline void dpr_cluster_map_free_(dp_cluster_map_t* m) {
  if (!m) return;
  free(m->node_cluster); free(m->member_off); free(m->members); free(m->total_compute);
  free(m->total_memory); free(m->breakpoints); free(m);
}
static inline dp_placement_result_t* dpr_placement_new(int64_t n, int32_t d, int64_t ndec) {
  dp_placement_result_t* p = DPR_NEW(dp_placement_result_t, 1);
  p->n_nodes = n;
  p->device = DPR_NEW(int32_t, n);
  p->n_devices = d;
  p->device_ids = DPR_NEW(int32_t, d);
  p->per_device_memory = DPR_NEW(int64_t, d);
  p->device_present = DPR_NEW(uint8_t, d);
  p->n_decisions = ndec;
  p->dec_node = DPR_NEW(int64_t, ndec);
  p->dec_prev = DPR_NEW(int32_t, ndec);
  p->dec_back_cost = DPR_NEW(int64_t, ndec);
  p->dec_est = DPR_NEW(int64_t, ndec * d);
  p->dec_chosen = DPR_NEW(int32_t, ndec);
  p->dec_relocated = DPR_NEW(uint8_t, ndec);
  p->dec_best_effort = DPR_NEW(uint8_t, ndec);
  return p;
}
static inline void dpr_placement_free_(dp_placement_result_t* p) {
  if (!p) return;
  free(p->device); free(p->device_ids); free(p->per_device_memory); free(p->device_present);
  free(p->dec_node); free(p->dec_prev); free(p->dec_back_cost); free(p->dec_est);
  free(p->dec_chosen); free(p->dec_relocated); free(p->dec_best_effort); free(p);
}
static inline dp_sim_report_t* dpr_sim_new(int32_t d, int64_t ntrace) {
  dp_sim_report_t* r = DPR_NEW(dp_sim_report_t, 1);
  r->n_devices = d;
  r->device_ids = DPR_NEW(int32_t, d);
  r->peak_memory = DPR_NEW(int64_t, d);
  r->capacity = DPR_NEW(int64_t, d);
  r->n_trace = ntrace;
  r->tr_kind = DPR_NEW(int32_t, ntrace);
  r->tr_node = DPR_NEW(int64_t, ntrace);
  r->tr_src = DPR_NEW(int64_t, ntrace);
  r->tr_dst = DPR_NEW(int64_t, ntrace);
  r->tr_device = DPR_NEW(int32_t, ntrace);
  r->tr_start = DPR_NEW(int64_t, ntrace);
  r->tr_end = DPR_NEW(int64_t, ntrace);
  return r;
}
static inline void dpr_sim_free_(dp_sim_report_t* r) {
  if (!r) return;
  free(r->device_ids); free(r->peak_memory); free(r->capacity); free(r->tr_kind);
  free(r->tr_node); free(r->tr_src); free(r->tr_dst); free(r->tr_device); free(r->tr_start);
  free(r->tr_end); free(r);
}
static inline void dpr_violations_free_(dp_violation_list_t* v) {
  if (!v) return;
  free(v->kind); free(v->node_off); free(v->nodes); free(v->msg_off); free(v->msg); free(v);
}
static inline void dpr_contraction_free_(dp_contraction_t* c) {
  if (!c) return;
  dpr_graph_out_free_(c->contracted); free(c->member_off); free(c->members); free(c);
}
static inline void dpr_fusion_free_(dp_fusion_result_t* f) {
  if (!f) return;
  dpr_graph_out_free_(f->coarse); dpr_cluster_map_free_(f->map); free(f);
}
static inline void dpr_pipeline_free_(dp_pipeline_result_t* r) {
  if (!r) return;
  dpr_fusion_free_(r->fusion);
  dpr_placement_free_(r->coarse_order); dpr_placement_free_(r->coarse_adjust);
  dpr_placement_free_(r->order_expanded); dpr_placement_free_(r->adjust_expanded);
  free(r->coarse_sequence); free(r);
}

#define DPR_DEFINE_FREES(P)                                                             \
  void P##free_violations(dp_violation_list_t* v) { dpr_violations_free_(v); }          \
  void P##free_cluster_map(dp_cluster_map_t* m) { dpr_cluster_map_free_(m); }           \
  void P##free_graph_out(dp_graph_out_t* g) { dpr_graph_out_free_(g); }                 \
  void P##free_contraction(dp_contraction_t* c) { dpr_contraction_free_(c); }           \
  void P##free_fusion(dp_fusion_result_t* f) { dpr_fusion_free_(f); }                   \
  void P##free_placement(dp_placement_result_t* p) { dpr_placement_free_(p); }          \
  void P##free_sim_report(dp_sim_report_t* r) { dpr_sim_free_(r); }                     \
  void P##free_pipeline(dp_pipeline_result_t* r) { dpr_pipeline_free_(r); }

#endif
