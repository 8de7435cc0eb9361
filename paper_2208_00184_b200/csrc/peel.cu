// peel.cu — M-TOPO / DFS-TOPO / CPD-TOPO (ATO) on the GPU, bit-exact with
// ordering.cpp:40-114 (/root/reference/proj/src).
//
// The reference peel is a deque used as a stack for DFS/CPD (freed children pushed to
// the head, so the highest-priority freed child is emitted right after its parent —
// pinned by test_ordering.cpp:104-135) and as a FIFO for M-TOPO.  Both comparators of a
// policy are one static total order, so each node gets a 32-bit rank (lower = emitted
// first among simultaneously available nodes):
//   CPD: (cpath desc, id asc)    DFS / M: (id asc)
// The peel itself is inherently sequential (a stack discipline); it runs as one warp:
// per popped node the lanes stride its CSR row, decrement the in-degree counters,
// ballot the freed children and place them on the stack ordered by rank.
#include "graph.cuh"
#include "peel.cuh"

namespace dpb {
namespace {

__global__ void k_iota32(int32_t* a, int32_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = static_cast<int32_t>(i);
}

}  // namespace

void node_order_by_id(DevGraph& g, DevBuf<int32_t>& by_id) {
  dp_ctx* ctx = g.ctx;
  by_id.alloc(ctx, g.n > 0 ? g.n : 1);
  if (g.dense_ids) {
    DP_LAUNCH(ctx, k_iota32, grid_for(g.n, 256), 256, 0, by_id.p, g.n);
  } else if (g.n) {
    DP_CUDA(cudaMemcpyAsync(by_id.p, g.sorted_idx.p, sizeof(int32_t) * g.n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
}

}  // namespace dpb
