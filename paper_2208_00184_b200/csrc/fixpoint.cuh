// fixpoint.cuh — the stack peel as a level-parallel tree construction plus a parallel proof.
#pragma once
#include "graph.cuh"

namespace dpb {

// The tree peel is tried for stack policies on graphs of at least 2,048 nodes (it gives up
// by itself on chain-like graphs: more levels than n / 40).
bool fixpoint_wanted(const DevGraph& g);

// Enqueues the tree peel of g (ranks from peel_prepare: by_rank, rank, source flags and
// their scan).  When its proof holds within the round budget it writes seq/pos_of, sets
// *skip = 1 and the peel counters (*progress = *emitted = n); otherwise it leaves them and
// the one-warp peel launched next does the work.  No host round trip.
void fixpoint_launch(DevGraph& g, const int32_t* by_rank, const int32_t* rank, const int32_t* flag,
                     const int32_t* fpos, int32_t* seq, int32_t* pos_of, int* skip, int* progress, int* emitted);

}  // namespace dpb
