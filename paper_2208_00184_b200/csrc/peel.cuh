// peel.cuh — topological orders (ordering.cpp:40-114).
#pragma once
#include "graph.cuh"

namespace dpb {
// Node indices sorted by id ascending (identity for dense ids).
void node_order_by_id(DevGraph& g, DevBuf<int32_t>& by_id);
// Emits the policy's order as node indices into seq[n] (+ pos_of[v]); returns the
// number of emitted nodes (< n means a cycle).  cpath (by node index) for CPD only.
int32_t topo_order(DevGraph& g, int policy, const int64_t* cpath, int32_t* seq, int32_t* pos_of);
}  // namespace dpb
