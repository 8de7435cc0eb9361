// graph.cuh — device-resident ComputationGraph (SoA in HBM) and the graph-core stages.
#pragma once

#include "common.cuh"

namespace dpb {

// Layout in HBM (n nodes, m edges; indices are int32, ids/costs int64):
//   nodes:  id[n] w[n] mem[n] (+ group[n])                 24-28 B/node
//   edges:  src_id[m] dst_id[m] bytes[m] -> esrc[m] edst[m] cost[m]
//   CSR:    out_off[n+1] out_eid[m] out_dst[m] out_cost[m]  (stable in edge order)
//   CSC:    in_off[n+1]  in_eid[m]  in_src[m]  in_cost[m]
struct DevGraph {
  dp_ctx* ctx = nullptr;
  int32_t n = 0, m = 0;
  DevBuf<int64_t> id, w, mem;
  DevBuf<int32_t> group;
  bool has_group = false;
  DevBuf<int64_t> src_id, dst_id, bytes;
  DevBuf<int32_t> esrc, edst;         // -1 when the endpoint id is not a node
  bool dense_ids = false;             // id[i] == i for all i
  DevBuf<uint64_t> sorted_key;        // sign-flipped ids, ascending (when !dense_ids)
  DevBuf<int32_t> sorted_idx;         // node index per sorted key (ascending idx on ties)
  // adjacency over edges whose endpoints both resolve
  bool has_adj = false;
  bool big_rows = false;  // some CSR row is longer than 64 (duplicate-edge check sorts)
  int32_t m_ok = 0;
  bool topo_known = false;          // index_topo / span_sum set by graph_adjacency
  bool index_topo = false;          // every resolved edge u -> v has u < v
  unsigned long long span_sum = 0;  // sum of v - u over the resolved edges
  DevBuf<int32_t> out_off, out_eid, in_off, in_eid, out_dst, in_src;
  // costs
  bool has_cost = false;
  double ck = 0, cb = 0;
  DevBuf<int64_t> cost, out_cost, in_cost;
  // Kahn levels (filled by kahn())
  int32_t processed = 0, num_levels = 0;
  DevBuf<int32_t> order, level_off;
};

struct Validation {
  // first violation, detection order of graph.cpp:98-191
  int code = 0;                       // 0 = valid
  std::string message;
  std::vector<int64_t> nodes;
  // full list (when requested)
  std::vector<int32_t> kinds;
  std::vector<std::string> messages;
  std::vector<std::vector<int64_t>> witnesses;
};

// Host SoA -> HBM (async on ctx->stream).
// Uploads on ctx->stream, or (copy != null) on `copy` with `done` recorded after the
// copies: the caller makes ctx->stream wait on `done` before using the graph.
void graph_upload(DevGraph& g, dp_ctx* ctx, const dp_graph_t* h, cudaStream_t copy = nullptr,
                  cudaEvent_t done = nullptr);
// Adopt device arrays of a graph with dense ids 0..n-1 (coarse graph).
void graph_adopt_dense(DevGraph& g, dp_ctx* ctx, int32_t n, int32_t m, DevBuf<int64_t>&& w,
                       DevBuf<int64_t>&& mem, DevBuf<int32_t>&& esrc, DevBuf<int32_t>&& edst,
                       DevBuf<int64_t>&& bytes);
// id -> index map and edge endpoint resolution.
void graph_resolve(DevGraph& g);
struct ResolveState {
  DevBuf<int> flag;
  int dense = 0;
};
void graph_resolve_begin(DevGraph& g, ResolveState& st);  // caller syncs between
void graph_resolve_end(DevGraph& g, ResolveState& st);
// CSR/CSC over resolvable edges (stable in edge order).
void graph_adjacency(DevGraph& g);
// ... split around its one host round trip (the caller syncs between the two; several
// graphs may share that sync).
struct AdjState {
  DevBuf<int32_t> cnt, vals;
  DevBuf<uint32_t> keys, keys_out;
  DevBuf<int> flags;
  DevBuf<unsigned long long> span;
  int hs[4] = {0, 0, 0, 0};
  unsigned long long hspan = 0;
};
void graph_adjacency_begin(DevGraph& g, AdjState& st);
void graph_adjacency_end(DevGraph& g, AdjState& st);
// Per-edge comm_time and the CSR/CSC-ordered copies.
void graph_costs(DevGraph& g, dp_comm_t comm);
// validate(): needs host arrays for message text.  all=false stops at the first.
// cycle_check=false skips the Kahn pass (callers that run graph_kahn with levels right
// after check g.processed themselves and call graph_cycle_witness).
Validation graph_validate(DevGraph& g, const dp_graph_t* h, bool all, bool cycle_check = true);
// ... split around its first host round trip (several graphs may share it).
struct ValState {
  DevBuf<int32_t> dupcount;
  DevBuf<uint8_t> nflags, eflags, dupflag;
  DevBuf<int> first;
  int fh[2] = {0, 0};
};
void graph_validate_begin(DevGraph& g, ValState& vs);
Validation graph_validate_end(DevGraph& g, const dp_graph_t* h, ValState& vs, bool all, bool cycle_check);
// Kahn frontier (level-synchronous, persistent cooperative kernel): fills order /
// level_off / processed, and when requested tlevel / blevel (graph.cpp:228-261).
bool graph_levels_indexorder(DevGraph& g, int64_t* tlevel, int64_t* blevel, bool chainlike);
// a coarse (chain-like) graph of n nodes takes the dataflow kernel instead of the sweep
bool coarse_flow_wanted(int32_t n);
void graph_kahn(DevGraph& g, int64_t* tlevel, int64_t* blevel, int32_t* level_of);
// Batched building blocks of the chain-like (coarse) levels of several graphs.
void levels_sweep_launch(DevGraph* const* gs, int64_t* const* tlevel, int64_t* const* blevel, int count);
std::vector<char> graphs_index_topological(DevGraph* const* gs, int count,
                                           std::vector<unsigned long long>* spans = nullptr);
// graph_levels_indexorder(chainlike = false) of several graphs with shared launches.
std::vector<char> graphs_levels_indexorder(DevGraph* const* gs, int count, int64_t* const* tlevel,
                                           int64_t* const* blevel);
// CycleDetected witness after an incomplete Kahn pass (graph.cpp:71-94).
std::vector<int64_t> graph_cycle_witness(DevGraph& g);
// Node index of an id (UnknownNode when absent); host lookup helper via device search.
int32_t graph_index_of(DevGraph& g, int64_t id);
// Translate node ids (device array, count k) into indices (-1 when absent).
void graph_ids_to_index(DevGraph& g, const int64_t* ids, int32_t* out, int64_t k);

std::string join_ids(const std::vector<int64_t>& ids);

}  // namespace dpb
