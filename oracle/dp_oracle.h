/*
 * dp_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Two CPU checkers with the same flat signatures as the product C-ABI
 * (include/dagplace_b200.h, minus the dp_ctx_t argument):
 *   dpo_*  plain-C restatement of the reference algorithms (oracle/dp_oracle.c),
 *          built into oracle/build/libdp_oracle.so;
 *   dpr_*  the UNMODIFIED reference sources (/root/reference/proj/src) compiled by
 *          oracle/Makefile into oracle/_ref/libdagplace_ref.so, with the thin
 *          flattening shim oracle/ref_shim.cpp.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm
 * may load these libraries.  The product never links or calls them.
 */
#ifndef DP_ORACLE_H_
#define DP_ORACLE_H_

#include "../include/dagplace_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

#define DP_ORACLE_DECLS(P)                                                                    \
  const char* P##last_error_message(void);                                                    \
  int P##comm_time(int64_t bytes, dp_comm_t comm, int64_t* out);                              \
  int P##ccr(const dp_graph_t* g, dp_comm_t comm, double* out);                               \
  int P##validate(const dp_graph_t* g, dp_violation_list_t** out);                            \
  int P##require_valid(const dp_graph_t* g);                                                  \
  int P##graph_index(const dp_graph_t* g, int32_t* edge_src_idx, int32_t* edge_dst_idx,      \
                     int32_t* out_start, int32_t* out_list, int32_t* in_start,                \
                     int32_t* in_list);                                                       \
  int P##compute_levels(const dp_graph_t* g, dp_comm_t comm, int64_t* tlevel, int64_t* blevel, \
                        int64_t* cpath);                                                      \
  int P##topo_order(const dp_graph_t* g, int32_t policy, const int64_t* cpath,                \
                    int64_t* sequence_out);                                                   \
  int P##is_valid_topo_order(const dp_graph_t* g, const int64_t* sequence, int64_t length,    \
                             int32_t* out);                                                   \
  int P##merge_is_safe(const dp_graph_t* g, int64_t u, int64_t v, int32_t* out);              \
  int P##optimal_breakpoints(const dp_graph_t* g, const int64_t* sequence, int64_t length,    \
                             dp_comm_t comm, int32_t range, int64_t limit,                    \
                             dp_cluster_map_t** out);                                         \
  int P##build_coarse_graph(const dp_graph_t* g, const int64_t* sequence, int64_t length,     \
                            const int64_t* map_ids, const int32_t* map_cluster,               \
                            int64_t map_count, int64_t n_clusters, const int32_t* cluster_ids, \
                            const int64_t* member_off, const int64_t* members,                \
                            dp_graph_out_t** out);                                            \
  int P##contract_colocation_groups(const dp_graph_t* g, dp_contraction_t** out);             \
  int P##fuse(const dp_graph_t* g, dp_comm_t comm, int32_t range, int64_t limit,              \
              dp_fusion_result_t** out);                                                      \
  int P##order_place(const dp_graph_t* coarse, const int64_t* sequence, int64_t length,       \
                     const dp_devices_t* devices, dp_placement_result_t** out);               \
  int P##adjusting_placement(const dp_graph_t* coarse, const int64_t* sequence,               \
                             int64_t length, const dp_devices_t* devices, dp_comm_t comm,     \
                             dp_placement_result_t** out);                                    \
  int P##expand_placement(const dp_graph_t* original, const int32_t* node_cluster,            \
                          int64_t n_clusters, const int64_t* member_off,                      \
                          const int64_t* members, const int32_t* coarse_device,               \
                          const uint8_t* coarse_placed, dp_placement_result_t** out);         \
  int P##simulate(const dp_graph_t* g, const int32_t* device_of_node,                         \
                  const dp_devices_t* devices, dp_comm_t comm, int32_t want_trace,            \
                  dp_sim_report_t** out);                                                     \
  int P##simulate_candidates(const dp_graph_t* g, const int32_t* node_cluster,                \
                             int64_t n_clusters, const uint8_t* cand_dev_pos,                 \
                             int64_t n_candidates, const dp_devices_t* devices,               \
                             dp_comm_t comm, int64_t* makespans, int64_t* argmin,             \
                             int32_t threads);                                                \
  int P##brute_force_optimal(const dp_graph_t* g, const dp_devices_t* devices,                \
                             dp_comm_t comm, int32_t* best_device_of_node,                    \
                             int64_t* best_makespan);                                         \
  int P##pipeline(const dp_graph_t* g, const dp_devices_t* devices, dp_comm_t comm,           \
                  const dp_pipeline_config_t* cfg, dp_pipeline_result_t** out);               \
  void P##free_violations(dp_violation_list_t* v);                                            \
  void P##free_cluster_map(dp_cluster_map_t* m);                                              \
  void P##free_graph_out(dp_graph_out_t* g);                                                  \
  void P##free_contraction(dp_contraction_t* c);                                              \
  void P##free_fusion(dp_fusion_result_t* f);                                                 \
  void P##free_placement(dp_placement_result_t* p);                                           \
  void P##free_sim_report(dp_sim_report_t* r);                                                \
  void P##free_pipeline(dp_pipeline_result_t* r);

DP_ORACLE_DECLS(dpo_)
DP_ORACLE_DECLS(dpr_)

/* Reference-only: run evaluate_pipeline on `threads` independent copies of g at once
 * (one std::thread each; the reference functions are pure) and return
 * the per-copy generation_wall_us (pipeline.cpp:77-79) in wall_us[threads]. */
int dpr_pipeline_replicas(const dp_graph_t* g, const dp_devices_t* devices, dp_comm_t comm,
                          const dp_pipeline_config_t* cfg, int32_t threads, int64_t* wall_us,
                          double* total_wall_s);

/* Reference-only: gen_graph (generator.cpp:203-209). */
int dpr_gen_graph(int32_t kind, int64_t n, int32_t width, double target_ccr, uint64_t seed, int64_t* node_id,
                  int64_t* compute_us, int64_t* memory_bytes, int64_t* edge_src, int64_t* edge_dst,
                  int64_t* edge_bytes, int64_t* n_edges);

#ifdef __cplusplus
}
#endif
#endif
