/*
 * dagplace_b200.h — C-ABI of the B200-native graph-analysis / placement-evaluation
 * path (libdagplace_b200.so).
 *
 * The reference (`/root/reference/proj`, C++ library `dagplace_core`) exposes a C++
 * API of free functions in `namespace dagplace` and no FFI of its own.  This header
 * is the plain-C boundary a binding (ctypes / cgo / JNI / the C++ drop-in host layer
 * in paper_2208_00184_b200/host/) calls.  Every entry point names the reference
 * function it replaces (file:line, relative to /root/reference/proj).
 *
 * Conventions
 *  - Graph inputs are host SoA arrays (dp_graph_t).  "node index" = position in the
 *    node arrays (GraphIndex semantics, include/dagplace/graph_index.hpp:15-17);
 *    "edge index" = position in the edge arrays.
 *  - Every function returns DP_OK (0) or a status code.  Codes 1..19 mirror
 *    dagplace::ErrorKind (include/dagplace/error.hpp:12-32) as 1 + ordinal; the
 *    message text (same wording as the reference's DagError) is available through
 *    dp_last_error_message() on the calling thread.  No C++ exception crosses the ABI.
 *  - Variable-size results are returned as library-allocated structs released with
 *    the matching *_free function.  The library never frees caller memory.
 *  - All compute runs on the GPU of the dp_ctx_t (one context per device/stream; no
 *    global mutable state besides the thread-local last error).  There is no CPU
 *    fallback: without a usable sm_100 device dp_ctx_create fails with DP_E_CUDA.
 */
#ifndef DAGPLACE_B200_H_
#define DAGPLACE_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* ---------------------------------------------------------------- status codes */
enum {
  DP_OK = 0,
  /* 1 + dagplace::ErrorKind ordinal (error.hpp:12-32) */
  DP_E_CYCLE_DETECTED = 1,
  DP_E_DANGLING_EDGE = 2,
  DP_E_DUPLICATE_ID = 3,
  DP_E_DUPLICATE_EDGE = 4,
  DP_E_INVALID_VALUE = 5,
  DP_E_ZERO_COMPUTE_TIME = 6,
  DP_E_NO_SUCH_EDGE = 7,
  DP_E_NODE_EXCEEDS_CLUSTER_LIMIT = 8,
  DP_E_GROUP_EXCEEDS_CLUSTER_LIMIT = 9,
  DP_E_INFEASIBLE_PARTITION = 10,
  DP_E_INVALID_CLUSTER_MAP = 11,
  DP_E_INSUFFICIENT_SAMPLES = 12,
  DP_E_UNKNOWN_NODE = 13,
  DP_E_NODE_UNIVERSE_MISMATCH = 14,
  DP_E_UNPLACED_NODE = 15,
  DP_E_INSTANCE_TOO_LARGE = 16,
  DP_E_INSTANCE_INFEASIBLE = 17,
  DP_E_UNREACHABLE_TARGET_CCR = 18,
  DP_E_PARSE_ERROR = 19,
  /* ABI-level failures (no reference counterpart) */
  DP_E_CUDA = 100,
  DP_E_ARGUMENT = 101,
  DP_E_OUT_OF_MEMORY = 102,
  DP_E_UNSUPPORTED = 103
};

/* Topological policies, ordering.hpp:13 (TopoPolicy). */
enum { DP_TOPO_M = 0, DP_TOPO_DFS = 1, DP_TOPO_CPD = 2 };

/* Simulator task kinds, simulator.hpp:16 (TaskKind). */
enum { DP_TASK_COMPUTE = 0, DP_TASK_SEND = 1, DP_TASK_RECEIVE = 2 };

/* kNever (graph.hpp:23). */
#define DP_NEVER INT64_MAX

/* ---------------------------------------------------------------- plain inputs */
/* ComputationGraph (graph.hpp:42-45) as SoA.  group[i] < 0 means "no
 * colocation_group"; equal non-negative labels are one co-location group
 * (OpNode::colocation_group, graph.hpp:31).  group may be NULL. */
typedef struct dp_graph {
  int64_t n_nodes;
  int64_t n_edges;
  const int64_t* node_id;
  const int64_t* compute_us;
  const int64_t* memory_bytes;
  const int32_t* group;
  const int64_t* edge_src; /* node ids */
  const int64_t* edge_dst; /* node ids */
  const int64_t* edge_bytes;
} dp_graph_t;

/* CommModel (graph.hpp:48-52). */
typedef struct dp_comm {
  double k_us_per_byte;
  double b_us;
} dp_comm_t;

/* std::vector<DeviceSpec> (graph.hpp:54-57), any order. */
typedef struct dp_devices {
  int32_t count;
  const int32_t* id;
  const int64_t* memory_bytes;
} dp_devices_t;

/* ---------------------------------------------------------------- results */
/* ValidationResult (graph.hpp:79-87). */
typedef struct dp_violation_list {
  int64_t count;
  int32_t* kind;     /* status code (1 + ErrorKind) per violation */
  int64_t* node_off; /* [count+1] */
  int64_t* nodes;    /* witness ids */
  int64_t* msg_off;  /* [count+1] */
  char* msg;         /* concatenated messages (no separators) */
} dp_violation_list_t;

/* A graph produced by the library (coarse graph, contracted graph). */
typedef struct dp_graph_out {
  int64_t n_nodes;
  int64_t n_edges;
  int64_t* node_id;
  int64_t* compute_us;
  int64_t* memory_bytes;
  int32_t* group; /* copied label of the representative, or -1 */
  int64_t* edge_src;
  int64_t* edge_dst;
  int64_t* edge_bytes;
} dp_graph_out_t;

/* ClusterMap (fusion.hpp:32-37): clusters in sequence order, clusters[k].id == k. */
typedef struct dp_cluster_map {
  int64_t n_nodes;          /* size of node_to_cluster */
  int32_t* node_cluster;    /* [n_nodes] cluster id by node index of the input graph */
  int64_t n_clusters;
  int64_t* member_off;      /* [n_clusters+1] */
  int64_t* members;         /* [n_nodes] member ids, cluster by cluster */
  int64_t* total_compute;   /* [n_clusters] */
  int64_t* total_memory;    /* [n_clusters] */
  int64_t n_breakpoints;
  int32_t* breakpoints;     /* [n_breakpoints] */
} dp_cluster_map_t;

/* GroupContraction (fusion.hpp:41-45). */
typedef struct dp_contraction {
  dp_graph_out_t* contracted;
  int64_t* member_off; /* [contracted->n_nodes+1], by contracted node index */
  int64_t* members;    /* ascending original ids per contracted node */
} dp_contraction_t;

/* FusionResult (fusion.hpp:47-50). */
typedef struct dp_fusion_result {
  dp_graph_out_t* coarse;
  dp_cluster_map_t* map; /* over original node ids / indices */
} dp_fusion_result_t;

/* PlacementResult (placement.hpp:60-64) + Placement (placement.hpp:16-19). */
typedef struct dp_placement_result {
  int64_t n_nodes;
  int32_t* device;              /* [n_nodes] device id by node index */
  int32_t n_devices;            /* devices sorted by id */
  int32_t* device_ids;          /* [n_devices] */
  int64_t* per_device_memory;   /* [n_devices] */
  uint8_t* device_present;      /* [n_devices] key present in per_device_memory */
  int32_t oom_risk;
  int64_t n_decisions;          /* adjusting_placement only, else 0 */
  int64_t* dec_node;            /* [n_decisions] */
  int32_t* dec_prev;            /* device id */
  int64_t* dec_back_cost;
  int64_t* dec_est;             /* [n_decisions * n_devices], by device position */
  int32_t* dec_chosen;          /* device id */
  uint8_t* dec_relocated;
  uint8_t* dec_best_effort;
} dp_placement_result_t;

/* SimulationReport (simulator.hpp:39-46). */
typedef struct dp_sim_report {
  int64_t makespan;
  int64_t cross_transfer_count;
  int64_t cross_transfer_bytes;
  int32_t oom_flag;
  int32_t n_devices;            /* sorted by id */
  int32_t* device_ids;
  int64_t* peak_memory;
  int64_t* capacity;
  int64_t n_trace;              /* 0 unless the trace was requested */
  int32_t* tr_kind;
  int64_t* tr_node;
  int64_t* tr_src;
  int64_t* tr_dst;
  int32_t* tr_device;
  int64_t* tr_start;
  int64_t* tr_end;
} dp_sim_report_t;

/* PipelineConfig (pipeline.hpp:21-26) without profiles (Standard Evaluation inputs). */
typedef struct dp_pipeline_config {
  int32_t fusion_range;          /* default 200 */
  double cluster_mem_fraction;   /* default 0.25 */
  int32_t strategy;              /* 0 Order, 1 Adjust (default) */
  int32_t simulate;              /* 1: run pipeline.cpp:89-90 simulations (makespans);
                                    2: also return both full SimulationReports (trace) */
} dp_pipeline_config_t;

/* Output of the generation window (pipeline.cpp:67-79) and the report fields. */
typedef struct dp_pipeline_result {
  int64_t original_nodes, original_edges;
  double original_ccr;
  int64_t coarse_nodes, coarse_edges;
  double coarse_ccr;
  dp_fusion_result_t* fusion;
  dp_placement_result_t* coarse_order;    /* order_place on the coarse graph */
  dp_placement_result_t* coarse_adjust;   /* adjusting_placement on the coarse graph */
  dp_placement_result_t* order_expanded;  /* expand_placement(order) */
  dp_placement_result_t* adjust_expanded; /* expand_placement(adjust) */
  int64_t* coarse_sequence;               /* [coarse_nodes] cpd_topo of the coarse graph */
  int64_t order_makespan, adjust_makespan; /* -1 unless simulate */
  double generation_ms;                   /* device time of the window */
  dp_sim_report_t* order_sim;             /* simulate == 2: simulate(order_expanded), */
  dp_sim_report_t* adjust_sim;            /* simulate(adjust_expanded) with trace; else NULL */
} dp_pipeline_result_t;

/* ---------------------------------------------------------------- context */
typedef struct dp_ctx dp_ctx_t;

/* stream: a cudaStream_t (NULL = legacy default stream of `device`). */
int dp_ctx_create(int device, void* stream, dp_ctx_t** out);
void dp_ctx_destroy(dp_ctx_t* ctx);
int dp_ctx_set_stream(dp_ctx_t* ctx, void* stream);
int dp_ctx_synchronize(dp_ctx_t* ctx);
/* Number of kernels this context launched so far (bench/profiling evidence). */
int64_t dp_ctx_launch_count(const dp_ctx_t* ctx);
/* Per-stage device timing (CUDA events on the context stream) of the last
 * pipeline / batch call; names are static strings. */
int dp_ctx_enable_stage_timing(dp_ctx_t* ctx, int32_t on);
int32_t dp_ctx_stage_count(const dp_ctx_t* ctx);
const char* dp_ctx_stage_name(const dp_ctx_t* ctx, int32_t i);
double dp_ctx_stage_ms(const dp_ctx_t* ctx, int32_t i);
double dp_ctx_stage_bytes(const dp_ctx_t* ctx, int32_t i); /* algorithmic bytes */
/* Outcomes of the tree peel (csrc/fixpoint.cu) counted while DP_DEBUG_FIXPOINT is set
 * (diagnostic): out[0] first tree proven, [1] converged by fixed-point rounds, [2] gave up
 * (chain-like), [3] not a DAG, [4] round budget exhausted (the one-warp peel ran). */
int dp_ctx_peel_stats(const dp_ctx_t* ctx, int64_t* out5);

const char* dp_last_error_message(void);
int32_t dp_last_error_code(void);

/* ---------------------------------------------------------------- graph core */
/* comm_time, graph.cpp:200-204 (fp64 mul then add, no FMA; llround). */
int dp_comm_time(int64_t bytes, dp_comm_t comm, int64_t* out);
/* ccr, graph.cpp:206-215. */
int dp_ccr(dp_ctx_t* ctx, const dp_graph_t* g, dp_comm_t comm, double* out);
/* validate, graph.cpp:98-191 (every violation, detection order). */
int dp_validate(dp_ctx_t* ctx, const dp_graph_t* g, dp_violation_list_t** out);
void dp_violation_list_free(dp_violation_list_t* v);
/* require_valid, graph.cpp:193-198: status of the first violation. */
int dp_require_valid(dp_ctx_t* ctx, const dp_graph_t* g);
/* GraphIndex, graph_index.cpp:8-42: endpoints by index and CSR/CSC edge-index
 * lists, stable in input edge order.  Arrays: [m],[m],[n+1],[m],[n+1],[m]. */
int dp_graph_index(dp_ctx_t* ctx, const dp_graph_t* g, int32_t* edge_src_idx,
                   int32_t* edge_dst_idx, int32_t* out_start, int32_t* out_list,
                   int32_t* in_start, int32_t* in_list);
/* compute_levels, graph.cpp:217-269: t/b-level and cpath by node index. */
int dp_compute_levels(dp_ctx_t* ctx, const dp_graph_t* g, dp_comm_t comm, int64_t* tlevel,
                      int64_t* blevel, int64_t* cpath);

/* ---------------------------------------------------------------- ordering */
/* m_topo / dfs_topo / cpd_topo, ordering.cpp:81-114.  cpath (by node index) is
 * the LevelTable's cpath and is required for DP_TOPO_CPD only. */
int dp_topo_order(dp_ctx_t* ctx, const dp_graph_t* g, int32_t policy, const int64_t* cpath,
                  int64_t* sequence_out);
/* is_valid_topo_order, ordering.cpp:116-132. */
int dp_is_valid_topo_order(dp_ctx_t* ctx, const dp_graph_t* g, const int64_t* sequence,
                           int64_t length, int32_t* out);

/* ---------------------------------------------------------------- fusion */
/* merge_is_safe, fusion.cpp:16-51. */
int dp_merge_is_safe(dp_ctx_t* ctx, const dp_graph_t* g, int64_t u, int64_t v, int32_t* out);
/* optimal_breakpoints, fusion.cpp:85-171. */
int dp_optimal_breakpoints(dp_ctx_t* ctx, const dp_graph_t* g, const int64_t* sequence,
                           int64_t length, dp_comm_t comm, int32_t range, int64_t limit,
                           dp_cluster_map_t** out);
void dp_cluster_map_free(dp_cluster_map_t* m);
/* build_coarse_graph, fusion.cpp:173-229.  The ClusterMap is passed as its
 * node_to_cluster entries (ids/cluster, map_count of them) and its clusters
 * (ids 0..n_clusters-1 expected, member lists). */
int dp_build_coarse_graph(dp_ctx_t* ctx, const dp_graph_t* g, const int64_t* sequence,
                          int64_t length, const int64_t* map_ids, const int32_t* map_cluster,
                          int64_t map_count, int64_t n_clusters, const int32_t* cluster_ids,
                          const int64_t* member_off, const int64_t* members,
                          dp_graph_out_t** out);
void dp_graph_out_free(dp_graph_out_t* g);
/* contract_colocation_groups, fusion.cpp:231-295. */
int dp_contract_colocation_groups(dp_ctx_t* ctx, const dp_graph_t* g, dp_contraction_t** out);
void dp_contraction_free(dp_contraction_t* c);
/* fuse, fusion.cpp:297-335. */
int dp_fuse(dp_ctx_t* ctx, const dp_graph_t* g, dp_comm_t comm, int32_t range, int64_t limit,
            dp_fusion_result_t** out);
void dp_fusion_result_free(dp_fusion_result_t* f);

/* ---------------------------------------------------------------- placement */
/* order_place, placement.cpp:128-159. */
int dp_order_place(dp_ctx_t* ctx, const dp_graph_t* coarse, const int64_t* sequence,
                   int64_t length, const dp_devices_t* devices, dp_placement_result_t** out);
/* adjusting_placement, placement.cpp:161-218 (with the decision log). */
int dp_adjusting_placement(dp_ctx_t* ctx, const dp_graph_t* coarse, const int64_t* sequence,
                           int64_t length, const dp_devices_t* devices, dp_comm_t comm,
                           dp_placement_result_t** out);
/* expand_placement, placement.cpp:239-268.  coarse_device: device id per cluster id. */
int dp_expand_placement(dp_ctx_t* ctx, const dp_graph_t* original, const int32_t* node_cluster,
                        int64_t n_clusters, const int64_t* member_off, const int64_t* members,
                        const int32_t* coarse_device, const uint8_t* coarse_placed,
                        dp_placement_result_t** out);
void dp_placement_result_free(dp_placement_result_t* p);

/* ---------------------------------------------------------------- simulator */
/* simulate, simulator.cpp:56-252.  device_of_node: device id by node index. */
int dp_simulate(dp_ctx_t* ctx, const dp_graph_t* g, const int32_t* device_of_node,
                const dp_devices_t* devices, dp_comm_t comm, int32_t want_trace,
                dp_sim_report_t** out);
void dp_sim_report_free(dp_sim_report_t* r);
/* Batched candidates (no reference entry point; semantic template is the candidate
 * loop + first-strict-minimum argmin of brute_force_optimal, simulator.cpp:278-304).
 * Candidate b assigns cluster c to device position cand_dev_pos[b*n_clusters + c]
 * (positions in the id-sorted device list); node v inherits node_cluster[v].
 * makespans[b] = simulate(...).makespan.  *argmin = lowest b with the minimum. */
int dp_simulate_candidates(dp_ctx_t* ctx, const dp_graph_t* g, const int32_t* node_cluster,
                           int64_t n_clusters, const uint8_t* cand_dev_pos, int64_t n_candidates,
                           const dp_devices_t* devices, dp_comm_t comm, int64_t* makespans,
                           int64_t* argmin);
/* brute_force_optimal, simulator.cpp:254-310 (every candidate simulated on the GPU). */
int dp_brute_force_optimal(dp_ctx_t* ctx, const dp_graph_t* g, const dp_devices_t* devices,
                           dp_comm_t comm, int32_t* best_device_of_node, int64_t* best_makespan);

/* ---------------------------------------------------------------- pipeline */
/* evaluate_pipeline, pipeline.cpp:27-111 (no profiles).  Host buffers in and out;
 * the H2D upload and D2H result copies are part of the call. */
int dp_pipeline(dp_ctx_t* ctx, const dp_graph_t* g, const dp_devices_t* devices, dp_comm_t comm,
                const dp_pipeline_config_t* cfg, dp_pipeline_result_t** out);
/* evaluate_pipeline over `count` independent graphs with the same devices and config
 * (out[i] for graphs[i], each freed with dp_pipeline_result_free).  The graphs share one
 * stream; their sequential peel + DP cores run in one launch (4 graphs per launch), so a
 * caller with many graphs keeps more of the GPU busy per stream.  generation_ms is the
 * window of the whole call.  New surface: the reference evaluates one graph per call. */
int dp_pipeline_batch(dp_ctx_t* ctx, int32_t count, const dp_graph_t* const* graphs,
                      const dp_devices_t* devices, dp_comm_t comm, const dp_pipeline_config_t* cfg,
                      dp_pipeline_result_t** out);
void dp_pipeline_result_free(dp_pipeline_result_t* r);

/* ---------------------------------------------------------------- Standard Evaluation
 * (estimation.cpp, estimation.hpp:13-86), bit-exact fp64 on the GPU (estimation.cu). */
/* ProfileSet (estimation.hpp:25-28): batch b's samples are [node_off[b], node_off[b+1]). */
typedef struct dp_profiles {
  int32_t n_batches;
  const int64_t* batch_size;    /* [n_batches] */
  const int64_t* node_off;      /* [n_batches + 1] */
  const int64_t* node_id;
  const int64_t* memory_bytes;
  const int64_t* compute_us;
} dp_profiles_t;
/* NodeCostModel (estimation.hpp:37-40), ascending id; fit[6k..6k+5] = memory {slope,
 * intercept, residual_norm}, compute {slope, intercept, residual_norm} (LinearFit). */
typedef struct dp_node_models {
  int64_t n;
  int64_t* node_id;
  double* fit;
} dp_node_models_t;
/* DeviationReport (estimation.hpp:44-53): maps as ascending-id arrays. */
typedef struct dp_deviation {
  int64_t n_memory;
  int64_t* memory_id;
  double* memory_dev;
  int64_t n_time;
  int64_t* time_id;
  double* time_dev;
  double mean_memory, mean_time;
  int64_t n_zero_memory;
  int64_t* zero_memory;
  int64_t n_zero_time;
  int64_t* zero_time;
} dp_deviation_t;
/* fit_node_models (estimation.cpp:67-88).  A batch listing a node twice (not
 * representable in the reference's unordered_map) is DP_E_INVALID_VALUE; a missing node
 * is reported as the smallest missing id (the reference names the first in hash order). */
int dp_fit_node_models(dp_ctx_t* ctx, const dp_profiles_t* profiles, dp_node_models_t** out);
void dp_node_models_free(dp_node_models_t* m);
/* estimate_graph (estimation.cpp:90-119): EdgeScaling as reference_batch + overrides
 * (src, dst, factor); the last of repeated override pairs wins. */
int dp_estimate_graph(dp_ctx_t* ctx, const dp_graph_t* base, const dp_node_models_t* models, int64_t target_batch,
                      int64_t reference_batch, int64_t n_override, const int64_t* ov_src, const int64_t* ov_dst,
                      const double* ov_factor, dp_graph_out_t** out);
/* fit_comm_model (estimation.cpp:121-140). */
int dp_fit_comm_model(dp_ctx_t* ctx, int64_t n, const int64_t* bytes, const double* us, dp_comm_t* out);
/* deviation_report (estimation.cpp:148-192). */
int dp_deviation_report(dp_ctx_t* ctx, const dp_graph_t* estimated, const dp_graph_t* measured,
                        dp_deviation_t** out);
void dp_deviation_free(dp_deviation_t* d);

/* Graph / device documents parsed straight into SoA arrays (host code,
 * json_load.cu): replaces graph_from_json (json_io.cpp:43-74) + the AoS
 * ComputationGraph, so a document feeds dp_* calls directly (the result casts to the
 * dp_graph_t view: same field order).  colocation_group strings become labels in
 * first-appearance order (-1 = none); node names are not kept.  Errors: DP_E_PARSE_ERROR
 * with the reference's message for schema errors; syntax errors (which json::parse
 * rejects) are "invalid JSON: <what>".  Free with dp_graph_out_free. */
int dp_graph_from_json(const char* text, int64_t len, dp_graph_out_t** out);
/* devices_from_json (json_io.cpp:93-117): writes min(count, capacity) devices. */
int dp_devices_from_json(const char* text, int64_t len, int32_t* count, int32_t* ids, int64_t* memory_bytes,
                         int32_t capacity, dp_comm_t* comm);

/* Device-resident variant for throughput measurement: upload once, then run the
 * generation window (pipeline.cpp:67-79) with every intermediate kept in HBM.
 * dp_resident_generate writes only device buffers; dp_resident_fetch copies the two
 * expanded placements (device id by node index) to host. */
typedef struct dp_resident dp_resident_t;
int dp_resident_create(dp_ctx_t* ctx, const dp_graph_t* g, const dp_devices_t* devices,
                       dp_comm_t comm, const dp_pipeline_config_t* cfg, dp_resident_t** out);
int dp_resident_generate(dp_resident_t* r);
/* The windows of `count` residents of ONE context, peel + DP cores in one launch. */
int dp_resident_generate_batch(dp_resident_t* const* rs, int32_t count);
int dp_resident_fetch(dp_resident_t* r, int32_t* order_device, int32_t* adjust_device,
                      int64_t* coarse_nodes, int64_t* coarse_edges);
void dp_resident_destroy(dp_resident_t* r);

/* ---------------------------------------------------------------- input synthesis */
/* Deterministic generators (host code; not on the measured path).  Layered recipe of
 * mt19937_64(seed), compute u(100,900), memory u(2^19,3*2^19), fan-in
 * u(fan_lo,fan_hi) distinct picks from the previous layer, bytes u(2^15,3*2^15), edges
 * sorted by (src,dst).  Arrays must hold n nodes and n*fan_hi edges. */
int dp_gen_layered(int64_t n, int64_t width, int64_t fan_lo, int64_t fan_hi, uint64_t seed,
                   int64_t* node_id, int64_t* compute_us, int64_t* memory_bytes,
                   int64_t* edge_src, int64_t* edge_dst, int64_t* edge_bytes, int64_t* n_edges);

/* Config #2 GNMT-like chains and config #3 BERT-like skip-layered graphs. */
int dp_gen_gnmt(int64_t chains, int64_t T, uint64_t seed, int64_t* node_id, int64_t* compute_us,
                int64_t* memory_bytes, int64_t* edge_src, int64_t* edge_dst, int64_t* edge_bytes, int64_t* n_edges);
int dp_gen_bert(int64_t n, int64_t width, int64_t skip, uint64_t seed, int64_t* node_id, int64_t* compute_us,
                int64_t* memory_bytes, int64_t* edge_src, int64_t* edge_dst, int64_t* edge_bytes, int64_t* n_edges);

/* Config #5 candidate family: candidate 0 = base (device position per
 * cluster); candidate k > 0 applies max(1, n_clusters/100) moves drawn from
 * std::mt19937_64(k): cluster rk() % n_clusters -> device rk() % D.  Writes candidates
 * first .. first+count-1 into out[count * n_clusters]. */
int dp_gen_candidates(const uint8_t* base, int64_t n_clusters, int32_t D, int64_t first, int64_t count,
                      uint8_t* out);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* DAGPLACE_B200_H_ */
