// abi_stubs.cu — entry points not implemented yet in this build return DP_E_UNSUPPORTED.
#include "abi_util.cuh"
#include "results.h"

using namespace dpb;

#define DP_STUB(name, ...)                                        \
  int name(__VA_ARGS__) {                                         \
    set_last_error(DP_E_UNSUPPORTED, #name " not available yet"); \
    return DP_E_UNSUPPORTED;                                      \
  }

extern "C" {
DP_STUB(dp_simulate, dp_ctx_t*, const dp_graph_t*, const int32_t*, const dp_devices_t*, dp_comm_t, int32_t,
        dp_sim_report_t**)
DP_STUB(dp_simulate_candidates, dp_ctx_t*, const dp_graph_t*, const int32_t*, int64_t, const uint8_t*, int64_t,
        const dp_devices_t*, dp_comm_t, int64_t*, int64_t*)
DP_STUB(dp_brute_force_optimal, dp_ctx_t*, const dp_graph_t*, const dp_devices_t*, dp_comm_t, int32_t*, int64_t*)
DP_STUB(dp_pipeline, dp_ctx_t*, const dp_graph_t*, const dp_devices_t*, dp_comm_t, const dp_pipeline_config_t*,
        dp_pipeline_result_t**)
DP_STUB(dp_resident_create, dp_ctx_t*, const dp_graph_t*, const dp_devices_t*, dp_comm_t, const dp_pipeline_config_t*,
        dp_resident_t**)
DP_STUB(dp_resident_generate, dp_resident_t*)
DP_STUB(dp_resident_fetch, dp_resident_t*, int32_t*, int32_t*, int64_t*, int64_t*)
void dp_resident_destroy(dp_resident_t*) {}
void dp_cluster_map_free(dp_cluster_map_t* m) { free_cluster_map(m); }
void dp_graph_out_free(dp_graph_out_t* g) { free_graph_out(g); }
void dp_contraction_free(dp_contraction_t* c) {
  if (!c) return;
  free_graph_out(c->contracted); std::free(c->member_off); std::free(c->members); std::free(c);
}
void dp_fusion_result_free(dp_fusion_result_t* f) {
  if (!f) return;
  free_graph_out(f->coarse); free_cluster_map(f->map); std::free(f);
}
void dp_placement_result_free(dp_placement_result_t* p) { free_placement(p); }
void dp_sim_report_free(dp_sim_report_t* r) { free_sim(r); }
void dp_pipeline_result_free(dp_pipeline_result_t* r) {
  if (!r) return;
  dp_fusion_result_free(r->fusion);
  free_placement(r->coarse_order); free_placement(r->coarse_adjust);
  free_placement(r->order_expanded); free_placement(r->adjust_expanded);
  std::free(r->coarse_sequence); std::free(r);
}
DP_STUB(dp_gen_layered, int64_t, int64_t, int64_t, int64_t, uint64_t, int64_t*, int64_t*, int64_t*, int64_t*, int64_t*,
        int64_t*, int64_t*)
}
