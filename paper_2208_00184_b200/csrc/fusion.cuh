// fusion.cuh — optimal breakpoints, clusters, coarse graph, co-location contraction
// (fusion.cpp:55-335, /root/reference/proj/src).
#pragma once

#include "graph.cuh"
#include "peel_dp.cuh"

namespace dpb {

// Clusters of a sequence: contiguous runs of positions (clusters_from_cuts, fusion.cpp:61-81).
struct Clusters {
  int32_t n = 0, k = 0;
  DevBuf<int32_t> cl_of_pos;   // [n]
  DevBuf<int32_t> cut_pos;     // [k+1] start position of each cluster, then n
  DevBuf<int64_t> tot_w, tot_mem;
};

// optimal_breakpoints core (fusion.cpp:95-170) on a validated device graph with costs.
// seq/pos_of: node index by position and its inverse.  Throws NodeExceedsClusterLimit /
// InfeasiblePartition like the reference.
void breakpoints_dev(DevGraph& g, const int32_t* seq, const int32_t* pos_of, int32_t range, int64_t limit,
                     Clusters& out);

// Traceback of prev_cut[1..n] and the clusters of the sequence.
void clusters_from_prev_cut(DevGraph& g, const int32_t* seq, const int32_t* prev_cut, Clusters& out);

// Coarse graph (build_coarse_graph, fusion.cpp:205-225): cluster nodes and crossing
// edges aggregated by byte sum in (cu, cv) order.  cl_of_node: cluster by node index.
void coarse_graph_dev(DevGraph& g, const int32_t* cl_of_node, int32_t k, const int64_t* tot_w,
                      const int64_t* tot_mem, DevGraph& coarse);

// Co-location contraction (fusion.cpp:231-295) into `work`; member lists of each
// contracted node (ascending original ids) in mem_off/mem_ids; rep_cidx: contracted
// index of every original node.  Throws CycleDetected for inconsistent groups.
struct Contraction {
  DevGraph work;
  DevBuf<int64_t> mem_off;  // [nw+1]
  DevBuf<int64_t> mem_ids;  // [n]
  DevBuf<int32_t> cidx_of;  // [n] contracted index of each original node
  bool identity = true;
};
void contract_dev(DevGraph& g, Contraction& c, bool materialize_identity);

// fuse (fusion.cpp:297-335) on a validated graph: contraction, limit check, levels,
// cpd_topo, breakpoints, coarse graph.  node_cluster: by ORIGINAL node index.
struct FuseOut {
  Contraction con;
  Clusters cl;
  DevBuf<int32_t> seq, pos_of;     // work sequence
  DevBuf<int32_t> node_cluster;    // by original node index
  DevGraph coarse;
};
void fuse_dev(DevGraph& g, dp_comm_t comm, int32_t range, int64_t limit, FuseOut& out);

// fuse_dev split around the streamed peel + DP launch, so that several independent graphs
// can share it: fuse_begin (contraction, levels, job preparation — or, off the streamed
// path, the whole peel and DP), peel_dp_launch over the jobs, fuse_end (limit check,
// traceback, coarse graph).
struct FuseStage {
  DevBuf<int64_t> t, b, c;
  DevBuf<int32_t> prev_cut;
  DevBuf<int> first;
  PeelDpHandle job;
  bool streamed = false;
  int64_t limit = 0;
};
void fuse_begin(DevGraph& g, dp_comm_t comm, int32_t range, int64_t limit, FuseOut& out, FuseStage& fs);
// fuse_begin of several graphs (same comm model and range) with their levels batched.
void fuse_begin_batch(DevGraph* const* gs, int count, dp_comm_t comm, int32_t range, const int64_t* limit,
                      FuseOut* const* out, FuseStage* const* fs);
void fuse_end(DevGraph& g, FuseOut& out, FuseStage& fs);
// fuse_end of several graphs sharing three host round trips (streamed graphs only; others
// run fuse_end one by one).
void fuse_end_batch(DevGraph* const* gs, int count, FuseOut* const* outs, FuseStage* const* fss);

// ClusterMap re-expressed over original ids (fusion.cpp:317-333) into host buffers.
dp_cluster_map_t* fuse_map_to_host(DevGraph& g, FuseOut& f);
// ... enqueueing its downloads; the map is complete after sync(ctx) and `fin`.
dp_cluster_map_t* fuse_map_to_host_async(DevGraph& g, FuseOut& f, Finalizers& fin);

}  // namespace dpb
