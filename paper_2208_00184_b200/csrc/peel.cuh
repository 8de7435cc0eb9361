// peel.cuh — topological orders (ordering.cpp:40-114).
#pragma once
#include <vector>
#include "graph.cuh"

namespace dpb {
// Node indices sorted by id ascending (identity for dense ids).
void node_order_by_id(DevGraph& g, DevBuf<int32_t>& by_id);
// Emits the policy's order as node indices into seq[n] (+ pos_of[v]); returns the
// number of emitted nodes (< n means a cycle).  cpath (by node index) for CPD only.
int32_t topo_order(DevGraph& g, int policy, const int64_t* cpath, int32_t* seq, int32_t* pos_of);
// The same for several graphs, one peel launch (one CTA per graph); emitted count per graph.
// tree = false: chain-like graphs (the coarse graphs of fuse) skip the tree peel attempt.
std::vector<int32_t> topo_order_batch(DevGraph* const* gs, int count, int policy, const int64_t* const* cpath,
                                      int32_t* const* seq, int32_t* const* pos_of, bool tree = true);
}  // namespace dpb
