// placement.cuh — order_place / adjusting_placement / expand_placement
// (placement.cpp:13-268, /root/reference/proj/src) on the GPU.
#pragma once

#include "graph.cuh"

namespace dpb {

struct Devices {
  int32_t D = 0;
  std::vector<int32_t> ids;   // ascending
  std::vector<int64_t> cap;
};
// SchedulerState::for_devices checks (placement.cpp:34-53).
Devices devices_sorted(const dp_devices_t* d);

struct PlaceOut {
  DevBuf<int32_t> dev;          // device position by node index
  DevBuf<int64_t> per_dev_mem;  // [D]
  DevBuf<int32_t> flags;        // [0] oom_risk
  // decision log (adjusting only), by order position
  DevBuf<int32_t> dec_prev, dec_chosen;
  DevBuf<int64_t> dec_back, dec_est;
  DevBuf<uint8_t> dec_reloc, dec_be;
};

// Both heuristics over one order; either output may be null.  `seq`: node indices in
// order (a valid topological order); graph with adjacency and costs (for adjusting).
void place_dev(DevGraph& g, const int32_t* seq, const Devices& devs, PlaceOut* order_out, PlaceOut* adjust_out,
               bool want_decisions);

// place_dev split so that independent graphs share one launch (2 CTAs per graph, up to 8
// graphs per launch): prepare each job, launch them together, release after the outputs
// have been consumed.
struct PlaceJob;
PlaceJob* place_prepare(DevGraph& g, const int32_t* seq, const Devices& devs, PlaceOut* order_out,
                        PlaceOut* adjust_out, bool want_decisions);
void place_launch(dp_ctx* ctx, PlaceJob* const* jobs, int count);
void place_release(PlaceJob* j);
struct PlaceHandle {
  PlaceJob* j = nullptr;
  PlaceHandle() = default;
  explicit PlaceHandle(PlaceJob* x) : j(x) {}
  PlaceHandle(const PlaceHandle&) = delete;
  PlaceHandle& operator=(const PlaceHandle&) = delete;
  ~PlaceHandle() { place_release(j); }
};

// expand_placement (placement.cpp:239-268) as a gather: dev_node[v] = coarse_dev[cl[v]],
// per-device memory sums.
void expand_dev(DevGraph& g, const int32_t* node_cluster, const int32_t* coarse_dev, int32_t D, int32_t* dev_node,
                int64_t* per_dev_mem);

}  // namespace dpb
