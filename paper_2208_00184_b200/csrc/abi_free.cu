// abi_free.cu — release functions of the library-allocated result structs.
#include "results.h"

using namespace dpb;

extern "C" {
void dp_cluster_map_free(dp_cluster_map_t* m) { free_cluster_map(m); }
void dp_graph_out_free(dp_graph_out_t* g) { free_graph_out(g); }
void dp_contraction_free(dp_contraction_t* c) {
  if (!c) return;
  free_graph_out(c->contracted);
  std::free(c->member_off);
  std::free(c->members);
  std::free(c);
}
void dp_fusion_result_free(dp_fusion_result_t* f) {
  if (!f) return;
  free_graph_out(f->coarse);
  free_cluster_map(f->map);
  std::free(f);
}
void dp_placement_result_free(dp_placement_result_t* p) { free_placement(p); }
void dp_sim_report_free(dp_sim_report_t* r) { free_sim(r); }
void dp_pipeline_result_free(dp_pipeline_result_t* r) {
  if (!r) return;
  dp_fusion_result_free(r->fusion);
  free_placement(r->coarse_order);
  free_placement(r->coarse_adjust);
  free_placement(r->order_expanded);
  free_placement(r->adjust_expanded);
  std::free(r->coarse_sequence);
  dp_sim_report_free(r->order_sim);
  dp_sim_report_free(r->adjust_sim);
  std::free(r);
}
}
