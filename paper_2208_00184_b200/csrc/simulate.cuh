// simulate.cuh — discrete-event makespan simulation (simulator.cpp:56-252).
#pragma once

#include "graph.cuh"

namespace dpb {

struct SimInput {
  // one of: node_dev (device position per node) for a single placement, or
  // cand (B x n_clusters device positions) + node_cluster for a candidate batch
  const int32_t* node_dev = nullptr;
  const uint8_t* cand = nullptr;
  const int32_t* node_cluster = nullptr;
  int32_t n_clusters = 0;
  int64_t n_candidates = 1;
  int32_t D = 0;
  bool trace = false;
};

struct SimOutput {
  DevBuf<int64_t> makespan;  // [B]; -1 marks a candidate whose engine queue overflowed
  DevBuf<int64_t> tstart, tend;  // [n + m] per task (trace mode)
};

// Requires adjacency + costs on g.  queue_cap: ring capacity per engine (power of 2).
void simulate_dev(DevGraph& g, const SimInput& in, SimOutput& out, int32_t queue_cap);

// First-pass ring capacity (1024, or DP_SIM_QUEUE for tests).
int32_t sim_queue_cap();
// The next ring capacity after an overflow at Q: 16 Q, at most the exact bound.
int32_t sim_queue_grow(const DevGraph& g, int32_t Q);

// Batch with automatic re-run of overflowed candidates at a larger queue capacity.
void simulate_batch_dev(DevGraph& g, const SimInput& in, SimOutput& out);

}  // namespace dpb
