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

__global__ void k_rank_keys(const int64_t* cpath, const int32_t* by_id, int32_t n, uint64_t* keys,
                            int32_t* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = by_id ? by_id[i] : static_cast<int32_t>(i);
    // descending signed cpath -> ascending unsigned key
    keys[i] = ~(static_cast<uint64_t>(cpath[v]) ^ (1ull << 63));
    vals[i] = v;
  }
}

__global__ void k_iota32(int32_t* a, int32_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = static_cast<int32_t>(i);
}

__global__ void k_rank_of(const int32_t* by_rank, int32_t n, int32_t* rank) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    rank[by_rank[r]] = static_cast<int32_t>(r);
}

__global__ void k_source_flags(const int32_t* by_rank, const int32_t* in_off, int32_t n, int32_t* flag) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = by_rank[r];
    flag[r] = (in_off[v + 1] - in_off[v]) == 0 ? 1 : 0;
  }
}

// Sources in ascending rank.  Stack mode stores them reversed (top = lowest rank).
__global__ void k_source_place(const int32_t* by_rank, const int32_t* flag, const int32_t* pos, int32_t n,
                               int32_t nsrc, bool stack, int32_t* buf) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[r]) continue;
    int32_t p = pos[r];
    buf[stack ? nsrc - 1 - p : p] = by_rank[r];
  }
}

__global__ void k_indeg_init(const int32_t* in_off, int32_t n, int32_t* indeg) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    indeg[v] = in_off[v + 1] - in_off[v];
}

__global__ void k_slot_rank(const int32_t* out_dst, const int32_t* rank, int32_t m, int64_t* packed) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = out_dst[k];
    packed[k] = (static_cast<int64_t>(rank[c]) << 32) | static_cast<uint32_t>(c);
  }
}

constexpr int kFreedCap = 4096;

// One warp.  buf: stack (stack mode, top = buf[top]) or ring-less queue (queue mode:
// head..tail, never wraps since every node is enqueued once).  slot[k] packs
// (rank(dst) << 32 | dst) for CSR slot k so one load yields both.
__global__ void __launch_bounds__(32) k_peel(const int32_t* out_off, const int64_t* slot, int32_t* indeg,
                                             int32_t* buf, int32_t nsrc, int32_t n, bool stack,
                                             int32_t* seq, int32_t* pos_of, int32_t* emitted,
                                             int64_t* spill) {
  __shared__ int64_t freed[kFreedCap];
  const int lane = threadIdx.x;
  int32_t top = nsrc - 1;  // stack mode
  int32_t head = 0, tail = nsrc;  // queue mode
  int32_t p = 0;
  for (;;) {
    int32_t v;
    if (stack) {
      if (top < 0) break;
      v = buf[top--];
    } else {
      if (head == tail) break;
      v = buf[head++];
    }
    if (lane == 0) {
      seq[p] = v;
      pos_of[v] = p;
    }
    ++p;
    int32_t kb = out_off[v], ke = out_off[v + 1];
    int32_t nf = 0;
    for (int32_t base = kb; base < ke; base += 32) {
      int32_t k = base + lane;
      bool act = k < ke;
      int64_t s = act ? slot[k] : 0;
      int32_t c = static_cast<int32_t>(s & 0xffffffff);
      bool fr = false;
      if (act) {
        int32_t d = indeg[c] - 1;
        indeg[c] = d;
        fr = d == 0;
      }
      unsigned mask = __ballot_sync(0xffffffffu, fr);
      if (fr) {
        int32_t at = nf + __popc(mask & ((1u << lane) - 1));
        if (at < kFreedCap) freed[at] = s; else spill[at - kFreedCap] = s;
      }
      nf += __popc(mask);
    }
    __syncwarp();
    if (nf == 0) continue;
    if (nf == 1) {
      int32_t c = static_cast<int32_t>(freed[0] & 0xffffffff);
      if (lane == 0) {
        if (stack) buf[top + 1] = c; else buf[tail] = c;
      }
      if (stack) ++top; else ++tail;
      __syncwarp();
      continue;
    }
    // order freed children by rank: position = #(others that go below/before it)
    for (int32_t i = lane; i < nf; i += 32) {
      int64_t si = i < kFreedCap ? freed[i] : spill[i - kFreedCap];
      int32_t ri = static_cast<int32_t>(si >> 32);
      int32_t cnt = 0;
      for (int32_t j = 0; j < nf; ++j) {
        int64_t sj = j < kFreedCap ? freed[j] : spill[j - kFreedCap];
        int32_t rj = static_cast<int32_t>(sj >> 32);
        cnt += stack ? (rj > ri) : (rj < ri);  // ranks are distinct
      }
      int32_t c = static_cast<int32_t>(si & 0xffffffff);
      if (stack) buf[top + 1 + cnt] = c; else buf[tail + cnt] = c;
    }
    if (stack) top += nf; else tail += nf;
    __syncwarp();
  }
  if (lane == 0) *emitted = p;
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

int32_t topo_order(DevGraph& g, int policy, const int64_t* cpath, int32_t* seq, int32_t* pos_of) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  int32_t n = g.n;
  if (n == 0) return 0;
  DevBuf<int32_t> by_id;
  node_order_by_id(g, by_id);
  DevBuf<int32_t> by_rank(ctx, n), rank(ctx, n);
  if (policy == DP_TOPO_CPD) {
    DevBuf<uint64_t> keys(ctx, n), keys_out(ctx, n);
    DevBuf<int32_t> vals(ctx, n);
    DP_LAUNCH(ctx, k_rank_keys, grid_for(n, B), B, 0, cpath, by_id.p, n, keys.p, vals.p);
    sort_pairs_u64(ctx, keys.p, keys_out.p, vals.p, by_rank.p, n, 0, 64);
  } else {
    DP_CUDA(cudaMemcpyAsync(by_rank.p, by_id.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  DP_LAUNCH(ctx, k_rank_of, grid_for(n, B), B, 0, by_rank.p, n, rank.p);
  DevBuf<int32_t> flag(ctx, (size_t)n + 1), fpos(ctx, (size_t)n + 1);
  flag.zero();
  DP_LAUNCH(ctx, k_source_flags, grid_for(n, B), B, 0, by_rank.p, g.in_off.p, n, flag.p);
  exclusive_scan_i32(ctx, flag.p, fpos.p, (int64_t)n + 1);
  int32_t nsrc = scalar_to_host(ctx, fpos.p + n);
  bool stack = policy != DP_TOPO_M;
  DevBuf<int32_t> buf(ctx, (size_t)n + 1), indeg(ctx, n), emitted(ctx, 1);
  DP_LAUNCH(ctx, k_source_place, grid_for(n, B), B, 0, by_rank.p, flag.p, fpos.p, n, nsrc, stack, buf.p);
  DP_LAUNCH(ctx, k_indeg_init, grid_for(n, B), B, 0, g.in_off.p, n, indeg.p);
  int32_t m = g.m_ok;
  DevBuf<int64_t> slot(ctx, m > 0 ? m : 1), spill(ctx, m > 0 ? m : 1);
  DP_LAUNCH(ctx, k_slot_rank, grid_for(m, B), B, 0, g.out_dst.p, rank.p, m, slot.p);
  {
    StageScope st(ctx, policy == DP_TOPO_CPD ? "cpd_peel" : "peel", 0.0);
    DP_LAUNCH(ctx, k_peel, 1, 32, 0, g.out_off.p, slot.p, indeg.p, buf.p, nsrc, n, stack, seq, pos_of,
              emitted.p, spill.p);
  }
  return scalar_to_host(ctx, emitted.p);
}

}  // namespace dpb
