// fixpoint.cuh — the stack peel as a level-parallel tree construction plus a parallel proof.
#pragma once
#include <memory>

#include "graph.cuh"

namespace dpb {

struct TreeArgs {
  int32_t n;
  const int32_t* nsrc;  // device: number of sources
  const int32_t* in_off;
  const int32_t* in_src;
  const int32_t* out_off;
  const int32_t* rowc;   // CSR children, each row sorted by rank (best first)
  const int32_t* roots;  // sources by rank
  int32_t* seq0;         // breadth-first order s0 (level-major)
  int2* bi;              // per node {s0 position of the T0 parent, remaining in-degree}: the
                         // numbering step reads both with one 8-byte load
  int32_t* size;
  int32_t* pre;          // preorder positions
  int32_t* pre2;         // general rounds: second buffer
  int32_t* par;          // general rounds: T(s) parent
  int32_t* lvl_off;      // [n + 1]
  int32_t* cs;           // [n + 1] s0 position of each position's first T0 child (cs[n] = n)
  int32_t* psize;        // T0 subtree size by s0 position
  int32_t* ppre;         // T0 preorder position by s0 position
  int32_t max_levels;    // more levels than this: give up (chain-like graph)
  int32_t max_rounds;    // general rounds after a failed proof (-1: from the cost model)
  int32_t* seq;
  int32_t* pos_of;
  int* skip;
  int* progress;
  int* emitted;
  int* info;             // [0] status (1 ok, 2 too deep, 3 not a DAG, 4 budget, 5 proof pending),
                         // [1] levels, [2] rounds, [3..6] phase clocks, [7] proof failed (split)
  int split;             // 1: the proof and the emission run as grid kernels (k_tree_proof / _emit)
};

constexpr int kTreeBatch = 8;

struct TreeJob {
  dp_ctx* ctx = nullptr;
  DevBuf<int32_t> rowc, roots, seq0, size, pre, pre2, par, lvl_off, cs, psize, ppre;
  DevBuf<int2> bi;
  DevBuf<int> info;
  TreeArgs a{};
  double bytes = 0.0;  // algorithmic bytes (stage timing)
  bool wide = false;   // mean edge span >= kTreeWideSpan: levels wide enough for a cluster
};

// The tree peel is tried for stack policies on graphs of at least 2,048 nodes (it gives up
// by itself on chain-like graphs: more levels than n / 40).
bool fixpoint_wanted(const DevGraph& g);

// Builds the tree peel's inputs for g (ranks from peel_prepare_begin: by_rank, rank,
// source flags and their scan) on the context stream.  The job must outlive its launch.
std::unique_ptr<TreeJob> fixpoint_prepare(DevGraph& g, const int32_t* by_rank, const int32_t* rank,
                                          const int32_t* flag, const int32_t* fpos, int32_t* seq, int32_t* pos_of,
                                          int* skip, int* progress, int* emitted);

// One CTA per graph, up to kTreeBatch graphs per launch.  A graph whose proof holds within
// the round budget gets seq/pos_of, *skip = 1 and the peel counters (*progress = *emitted
// = n); otherwise they are left alone and the one-warp peel does the work.
void fixpoint_launch_batch(dp_ctx* ctx, TreeJob* const* jobs, int count);

}  // namespace dpb
