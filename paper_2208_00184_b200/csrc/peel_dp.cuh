// peel_dp.cuh — latency-engineered peel and the streamed breakpoint DP.
#pragma once
#include "fixpoint.cuh"
#include "graph.cuh"

namespace dpb {

struct PeelState {
  bool stack_mode = true;
  DevBuf<int4> gstack, slot;
  DevBuf<int2> nr2, gstack2;
  DevBuf<int32_t> ell;
  int32_t ellw = 8;
  DevBuf<int32_t> indeg;
  DevBuf<int64_t> spill;
  DevBuf<int> counters;  // [0] progress, [1] emitted, [2] number of sources
  // peel v6
  bool v6 = false;
  DevBuf<int4> ell6;
  DevBuf<int2> cmeta;
  DevBuf<int32_t> gsid;
  DevBuf<int32_t> gover;
  DevBuf<uint32_t> dense16;  // v6 dense mode: 16-bit in-degrees, two per word (small graphs)
  DevBuf<int> dense_bad;     // set when some in-degree does not fit 16 bits
  // ranks and sources (peel_prepare_begin)
  DevBuf<int32_t> by_rank, rank, flag, fpos;
  // tree peel (fixpoint.cu): the job until tree_run launched it; skip = 1 on the device and
  // tree_ok on the host once its proof held (seq/pos_of and the counters are then final)
  std::unique_ptr<TreeJob> tree;
  bool tree_ok = false;
  DevBuf<int> skip;
};

// Ranks, sources, counters; with seq/pos_of and tree (stack policies) the tree peel's job.
void peel_prepare_begin(DevGraph& g, int policy, const int64_t* cpath, PeelState& st, int32_t* seq,
                        int32_t* pos_of, bool tree);
// The one-warp peel's inputs (needed unless the tree peel's proof held).
void peel_prepare_end(DevGraph& g, PeelState& st, bool force_v5);
// begin + end without a tree peel.
void peel_prepare(DevGraph& g, int policy, const int64_t* cpath, PeelState& st, bool force_v5 = false);
// Launches the tree peels of the given states together and waits for their verdicts.
void tree_run(dp_ctx* ctx, PeelState* const* sts, int count);

// CPD peel of g streamed into the breakpoint DP (R <= 256); writes seq/pos_of and
// prev_cut[1..n]; *first_exceed = first position whose node exceeds `limit` (or
// INT_MAX).  Returns the number of emitted nodes.
int32_t peel_dp_stream(DevGraph& g, const int64_t* cpath, int32_t range, int64_t limit, int32_t* seq, int32_t* pos_of,
                       int32_t* prev_cut, int* first_exceed);

// The same, split so that several independent graphs share one launch: prepare each
// graph's job, launch them together (up to 4 graphs per cooperative launch, 2 CTAs each),
// release after the outputs have been consumed.
struct PeelDpJob;
PeelDpJob* peel_dp_prepare(DevGraph& g, const int64_t* cpath, int32_t range, int64_t limit, int32_t* seq,
                           int32_t* pos_of, int32_t* prev_cut, int* first_exceed);
// ... split around its one host round trip (several graphs may share it): begin enqueues,
// finish runs after a sync of the context stream.
PeelDpJob* peel_dp_prepare_begin(DevGraph& g, const int64_t* cpath, int32_t range, int64_t limit, int32_t* seq,
                                 int32_t* pos_of, int32_t* prev_cut, int* first_exceed);
void peel_dp_prepare_finish(PeelDpJob* j);
void peel_dp_launch(dp_ctx* ctx, PeelDpJob* const* jobs, int count);
void peel_dp_release(PeelDpJob* j);
struct PeelDpHandle {
  PeelDpJob* j = nullptr;
  PeelDpHandle() = default;
  explicit PeelDpHandle(PeelDpJob* x) : j(x) {}
  PeelDpHandle(const PeelDpHandle&) = delete;
  PeelDpHandle& operator=(const PeelDpHandle&) = delete;
  ~PeelDpHandle() { peel_dp_release(j); }
};

}  // namespace dpb
