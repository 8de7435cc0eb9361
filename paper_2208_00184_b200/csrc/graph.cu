// graph.cu — graph core on the GPU: upload, id->index, CSR/CSC, validation flags,
// comm costs, Kahn frontier levels with t/b-level max-plus relaxation.
//
// Reference behaviour followed (paths relative to /root/reference/proj):
//   GraphIndex::GraphIndex        src/graph_index.cpp:8-42  (stable CSR/CSC of edge ids)
//   validate / require_valid      src/graph.cpp:98-198      (detection order + messages)
//   find_cycle_witness            src/graph.cpp:71-94
//   comm_time                     src/graph.cpp:200-204     (no FMA; llround)
//   compute_levels                src/graph.cpp:217-269     (int64 max-plus; any topo order)
#include <algorithm>
#include <climits>
#include <cstring>
#include <sstream>

#include "graph.cuh"

namespace dpb {

std::string join_ids(const std::vector<int64_t>& ids) {
  std::ostringstream out;
  for (size_t i = 0; i < ids.size(); ++i) {
    if (i) out << ",";
    out << ids[i];
  }
  return out.str();
}

// ------------------------------------------------------------------ kernels
namespace {

__global__ void k_dense_check(const int64_t* id, int32_t n, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (id[i] != i) atomicExch(flag, 0);
}

__global__ void k_id_keys(const int64_t* id, int32_t n, uint64_t* keys, int32_t* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = static_cast<uint64_t>(id[i]) ^ (1ull << 63);
    vals[i] = static_cast<int32_t>(i);
  }
}

__device__ __forceinline__ int32_t find_sorted(const uint64_t* keys, const int32_t* idx, int32_t n,
                                               int64_t id) {
  uint64_t k = static_cast<uint64_t>(id) ^ (1ull << 63);
  int32_t lo = 0, hi = n;
  while (lo < hi) {
    int32_t mid = lo + ((hi - lo) >> 1);
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  return (lo < n && keys[lo] == k) ? idx[lo] : -1;
}

__global__ void k_resolve(const int64_t* src_id, const int64_t* dst_id, int32_t m, int32_t n, bool dense,
                          const uint64_t* keys, const int32_t* idx, int32_t* esrc, int32_t* edst) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = src_id[e], d = dst_id[e];
    if (dense) {
      esrc[e] = (s >= 0 && s < n) ? static_cast<int32_t>(s) : -1;
      edst[e] = (d >= 0 && d < n) ? static_cast<int32_t>(d) : -1;
    } else {
      esrc[e] = find_sorted(keys, idx, n, s);
      edst[e] = find_sorted(keys, idx, n, d);
    }
  }
}

__global__ void k_ids_to_index(const int64_t* ids, int64_t k, int32_t n, bool dense, const uint64_t* keys,
                               const int32_t* idx, int32_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = ids[i];
    out[i] = dense ? ((s >= 0 && s < n) ? static_cast<int32_t>(s) : -1) : find_sorted(keys, idx, n, s);
  }
}

// Row keys for the stable CSR/CSC sorts; edges with an unresolved endpoint go to row n.
__global__ void k_row_keys(const int32_t* esrc, const int32_t* edst, int32_t m, int32_t n, bool by_src,
                           uint32_t* keys, int32_t* vals, int32_t* counts) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = esrc[e], d = edst[e];
    bool ok = s >= 0 && d >= 0;
    int32_t r = by_src ? s : d;
    keys[e] = ok ? static_cast<uint32_t>(r) : static_cast<uint32_t>(n);
    vals[e] = static_cast<int32_t>(e);
    if (ok) atomicAdd(&counts[r], 1);
  }
}

// 1 when every edge resolves and esrc is non-decreasing (generator output order), so the
// CSR permutation is the identity and the sort can be skipped.
// flag[0]: edges sorted by source with both endpoints resolved; flag[2]: every resolved
// edge u -> v has u < v (the index order is topological), *span += v - u over them (the
// dataflow level kernel's launch plan) -- the level pass needs no host round trip of its own.
__global__ void k_sorted_check(const int32_t* esrc, const int32_t* edst, int32_t m, int* flag,
                               unsigned long long* span) {
  unsigned long long sp = 0;
  bool unsorted = false, cyclic = false;  // one atomic per warp at the end, not per edge
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = esrc[e], d = edst[e];
    unsorted |= !(s >= 0 && d >= 0 && (e == 0 || esrc[e - 1] <= s));
    if (s >= 0 && d >= 0) {
      if (s >= d) cyclic = true;
      else sp += static_cast<unsigned long long>(d - s);
    }
  }
  for (int o = 16; o; o >>= 1) sp += __shfl_xor_sync(0xffffffffu, sp, o);
  unsorted = __any_sync(0xffffffffu, unsorted);
  cyclic = __any_sync(0xffffffffu, cyclic);
  if ((threadIdx.x & 31) == 0) {
    if (sp) atomicAdd(span, sp);
    if (unsorted) atomicExch(flag, 0);
    if (cyclic) atomicExch(flag + 2, 0);
  }
}

__global__ void k_iota(int32_t* a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = static_cast<int32_t>(i);
}

__global__ void k_gather_i32(const int32_t* src, const int32_t* perm, int32_t* dst, int64_t k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}

__global__ void k_gather_i64(const int64_t* src, const int32_t* perm, int64_t* dst, int64_t k) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}

__global__ void k_costs(const int64_t* bytes, int32_t m, double k, double b, int64_t* cost) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
    cost[e] = comm_cost_dev(bytes[e], k, b);
}

// Duplicate ids: runs of equal keys in the sorted id table; the first index of a run
// (smallest node index) carries the count (graph.cpp:105-113).
__global__ void k_dup_runs(const uint64_t* keys, const int32_t* idx, int32_t n, int32_t* dupcount) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    if (s > 0 && keys[s] == keys[s - 1]) continue;
    int64_t t = s + 1;
    while (t < n && keys[t] == keys[s]) ++t;
    if (t - s > 1) dupcount[idx[s]] = static_cast<int32_t>(t - s);
  }
}

// Node flags: bit0 duplicate id (first occurrence), bit1 negative compute, bit2 negative memory.
__global__ void k_node_flags(const int64_t* w, const int64_t* mem, const int32_t* dupcount, int32_t n,
                             uint8_t* flags, int* first) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint8_t f = (dupcount && dupcount[i] > 1 ? 1 : 0) | (w[i] < 0 ? 2 : 0) | (mem[i] < 0 ? 4 : 0);
    flags[i] = f;
    if (f) atomicMin(first, static_cast<int>(i));
  }
}

// Duplicate edges among edges with ok endpoints (resolved, not a self-loop): an edge is
// a duplicate when an earlier edge of the same row (stable CSR = earlier edge index) has
// the same destination (graph.cpp:122,149-154).  Rows longer than 64 are left to the
// sort-based pass.
__global__ void k_dup_edges(const int32_t* out_off, const int32_t* out_eid, const int32_t* out_dst,
                            int32_t n, uint8_t* dupflag, int* big) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    int32_t b = out_off[u], e = out_off[u + 1];
    if (e - b > 64) {
      atomicExch(big, 1);
      continue;
    }
    for (int32_t k = b + 1; k < e; ++k) {
      int32_t x = out_dst[k];
      if (x == u) continue;
      for (int32_t q = b; q < k; ++q) {
        if (out_dst[q] == x) {
          dupflag[out_eid[k]] = 1;
          break;
        }
      }
    }
  }
}

__global__ void k_big_rows(const int32_t* out_off, int32_t n, int* big) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    if (out_off[u + 1] - out_off[u] > 64) atomicExch(big, 1);
}

__global__ void k_pair_keys(const int32_t* esrc, const int32_t* edst, int32_t m, uint64_t* keys,
                            int32_t* vals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = esrc[e], d = edst[e];
    bool ok = s >= 0 && d >= 0 && s != d;
    keys[e] = ok ? ((static_cast<uint64_t>(s) << 32) | static_cast<uint32_t>(d)) : ~0ull;
    vals[e] = static_cast<int32_t>(e);
  }
}

__global__ void k_pair_dups(const uint64_t* keys, const int32_t* vals, int32_t m, uint8_t* dupflag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    if (i > 0 && keys[i] != ~0ull && keys[i] == keys[i - 1]) dupflag[vals[i]] = 1;
}

// Edge flags: bit0 dangling src, bit1 dangling dst, bit2 self-loop, bit3 negative bytes,
// bit4 duplicate (graph.cpp:124-156 order).
__global__ void k_edge_flags(const int64_t* src_id, const int64_t* dst_id, const int64_t* bytes,
                             const int32_t* esrc, const int32_t* edst, const uint8_t* dupflag, int32_t m,
                             uint8_t* flags, int* first) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    bool ds = esrc[e] < 0, dd = edst[e] < 0, sl = src_id[e] == dst_id[e];
    bool ok = !ds && !dd && !sl;
    uint8_t f = (ds ? 1 : 0) | (dd ? 2 : 0) | (sl ? 4 : 0) | (bytes[e] < 0 ? 8 : 0) |
                (ok && dupflag[e] ? 16 : 0);
    flags[e] = f;
    if (f) atomicMin(first, static_cast<int>(e));
  }
}

struct KahnArgs {
  int32_t n;
  const int32_t* out_off;
  const int32_t* out_dst;
  const int64_t* out_cost;
  const int64_t* w;
  int32_t* indeg;
  int32_t* order;
  int32_t* level_off;
  int64_t* tlevel;
  int64_t* blevel;
  int32_t* level_of;
  int* counters;  // [0] tail, [1] level, [2] lb (start of the current frontier), [3] max width
  unsigned* bar;
  int32_t narrow_max;  // narrow kernel hands over when a frontier exceeds this
};

// Level-synchronous Kahn frontier (graph.cpp:228-244 emits the same node set per
// level; any topological order gives the same levels).  Each frontier node relaxes the
// tlevel of its children with atomicMax (int64 max-plus is order-insensitive) and
// releases them when their remaining in-degree reaches zero; released nodes are
// appended to `order`, which therefore lists the nodes level by level.
__device__ __forceinline__ void kahn_relax_edge(const KahnArgs& a, int32_t k, int64_t t, bool* freed, int32_t* v) {
  *v = a.out_dst[k];
  if (a.tlevel) atomic_max_i64(&a.tlevel[*v], t + a.out_cost[k]);
  *freed = atomicSub(&a.indeg[*v], 1) == 1;
}

// Frontier node u (or none when u < 0): short rows are handled by the owning thread with
// up to 8 in-degree atomics in flight; rows longer than 8 are taken by the whole warp,
// lanes striding the row.  Every lane of the warp must call this together.
__device__ __forceinline__ void kahn_relax_warp(const KahnArgs& a, int32_t u, int32_t level, int* tail) {
  const int lane = threadIdx.x & 31;
  int32_t kb = 0, ke = 0;
  int64_t t = 0;
  if (u >= 0) {
    if (a.level_of) a.level_of[u] = level;
    t = a.tlevel ? a.tlevel[u] + a.w[u] : 0;
    kb = a.out_off[u];
    ke = a.out_off[u + 1];
  }
  const bool small = u >= 0 && ke - kb <= 8;
  int32_t fv[8];
  bool ff[8];
  // Phases (all loads, then all relaxations, then all in-degree decrements, then the
  // checks) so the up-to-8 independent atomics of a row are in flight together instead
  // of one round trip each.
  int64_t cv[8];
  int32_t old[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const bool act = small && kb + q < ke;
    fv[q] = act ? a.out_dst[kb + q] : 0;
    cv[q] = act && a.tlevel ? a.out_cost[kb + q] : 0;
  }
  // predicated PTX atomics: no branch around each one, so all issue back to back
  if (a.tlevel) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int on = small && kb + q < ke;
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0; @p red.global.max.s64 [%0], %1; }" ::"l"(
                       a.tlevel + fv[q]),
                   "l"(t + cv[q]), "r"(on)
                   : "memory");
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int on = small && kb + q < ke;
    int r = 0;
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %2, 0; @p atom.global.add.s32 %0, [%1], -1; }"
                 : "+r"(r)
                 : "l"(a.indeg + fv[q]), "r"(on)
                 : "memory");
    old[q] = r;
  }
  // one append per warp for all its lanes' freed children (one atomic on the shared tail
  // instead of eight)
  int nf = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    ff[q] = old[q] == 1;
    nf += ff[q] ? 1 : 0;
  }
  {
    int incl = nf;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    int base = 0;
    if (lane == 31 && incl) base = atomicAdd(tail, incl);
    base = __shfl_sync(0xffffffffu, base, 31) + incl - nf;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (ff[q]) a.order[base++] = fv[q];
  }
  unsigned big = __ballot_sync(0xffffffffu, u >= 0 && !small);
  while (big) {
    const int src = __ffs(big) - 1;
    big &= big - 1;
    const int32_t bkb = __shfl_sync(0xffffffffu, kb, src), bke = __shfl_sync(0xffffffffu, ke, src);
    const int64_t bt = __shfl_sync(0xffffffffu, t, src);
    for (int32_t k0 = bkb; k0 < bke; k0 += 32) {
      bool fr = false;
      int32_t v = 0;
      if (k0 + lane < bke) kahn_relax_edge(a, k0 + lane, bt, &fr, &v);
      const int slot = warp_append(tail, fr);
      if (fr) a.order[slot] = v;
    }
  }
}

// blevel(v) = w(v) + max_s(blevel(s) + c(v,s)) pulled over CSR (graph.cpp:253-261);
// long rows are reduced by the whole warp.  Warp-collective like kahn_relax_warp.
__device__ __forceinline__ void kahn_pull_warp(const KahnArgs& a, int32_t v) {
  const int lane = threadIdx.x & 31;
  int32_t kb = 0, ke = 0;
  if (v >= 0) {
    kb = a.out_off[v];
    ke = a.out_off[v + 1];
  }
  const bool small = v >= 0 && ke - kb <= 8;
  if (small) {
    int32_t x[8];
    int64_t c[8], bl[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      x[q] = kb + q < ke ? a.out_dst[kb + q] : -1;
      c[q] = kb + q < ke ? a.out_cost[kb + q] : 0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) bl[q] = x[q] >= 0 ? a.blevel[x[q]] : 0;
    int64_t best = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (x[q] >= 0) best = bl[q] + c[q] > best ? bl[q] + c[q] : best;
    a.blevel[v] = best + a.w[v];
  }
  unsigned big = __ballot_sync(0xffffffffu, v >= 0 && !small);
  while (big) {
    const int src = __ffs(big) - 1;
    big &= big - 1;
    const int32_t bkb = __shfl_sync(0xffffffffu, kb, src), bke = __shfl_sync(0xffffffffu, ke, src);
    const int32_t bv = __shfl_sync(0xffffffffu, v, src);
    int64_t best = 0;
    for (int32_t k = bkb + lane; k < bke; k += 32) {
      const int64_t c = a.blevel[a.out_dst[k]] + a.out_cost[k];
      best = c > best ? c : best;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const int64_t y = __shfl_xor_sync(0xffffffffu, best, o);
      best = y > best ? y : best;
    }
    if (lane == 0) a.blevel[bv] = best + a.w[bv];
  }
}


// ---- levels in index order (graphs whose node index order is topological, e.g. the
// coarse graph of fuse(), whose clusters are runs of a topological order).  Such graphs
// are chain-like (depth ~ n), where the level-synchronous frontier pays one grid-wide
// step per node.  Here one CTA sweeps the nodes in index order: all warps stage a tile of
// rows (CSC for tlevel, CSR backwards for blevel) into shared memory, then warp 0 walks
// the tile with the running finish/blevel values in shared memory: per node one gather
// per in-edge and a two-step 64-bit max (redux.sync on high then low words).
constexpr int kSeqMaxN = 16384;  // graphs up to this size always take the one-CTA sweep
constexpr int kSeqRing = 8192;   // power of two: sweep values kept in shared memory
constexpr int kSeqTile = 8192;   // edges staged per tile
constexpr int kSeqTileN = 2048;  // nodes staged per tile

// ok = 0 unless every edge u->v has u < v; span += sum of (v - u) (how far ahead of a node
// its inputs lie in index order, sizing the dataflow kernel's lookahead)
__global__ void k_index_topo(const int32_t* in_off, const int32_t* in_src, int32_t n, int* ok,
                             unsigned long long* span) {
  unsigned long long s = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    for (int32_t k = in_off[v]; k < in_off[v + 1]; ++k) {
      const int32_t u = in_src[k];
      if (u >= v) atomicExch(ok, 0);
      else s += static_cast<unsigned long long>(v - u);
    }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(span, s);
}

__device__ __forceinline__ int64_t warp_max_nonneg(int64_t x) {
  const uint32_t hi = static_cast<uint32_t>(static_cast<uint64_t>(x) >> 32);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t lo = hi == mh ? static_cast<uint32_t>(x) : 0u;
  const uint32_t ml = __reduce_max_sync(0xffffffffu, lo);
  return static_cast<int64_t>((static_cast<uint64_t>(mh) << 32) | ml);
}

// forward: tlevel[v] = max(0, max_{u->v} f[u] + c), f[u] = tlevel[u] + w[u]
// backward (rev): blevel[v] = w[v] + max(0, max_{v->s} blevel[s] + c)
// Values of the last kSeqRing sweep positions live in a shared-memory ring; older ones
// (graphs larger than the ring) are read from `gval` in HBM/L2 with ld.global.cg (the
// sweep writes them there too), so any n works and chain-like graphs hit the ring.
// One CTA per graph (independent graphs of a batched call share the launch).
struct SeqArgs {
  int32_t n;
  const int32_t* off;
  const int32_t* nbr;
  const int64_t* cost;
  const int64_t* w;
  int64_t* out;
  int64_t* gval;
};
constexpr int kSeqBatch = 8;
struct SeqBatch {
  SeqArgs a[2][kSeqBatch];  // [0] forward (t-levels), [1] backward (b-levels)
};

// blockIdx.y = direction: the two passes are independent and run on two SMs at once.
__global__ void __launch_bounds__(1024) k_levels_seq(const __grid_constant__ SeqBatch batch) {
  const bool rev = blockIdx.y != 0;
  const SeqArgs& A = batch.a[blockIdx.y][blockIdx.x];
  const int32_t n = A.n;
  const int32_t* off = A.off;
  const int32_t* nbr = A.nbr;
  const int64_t* cost = A.cost;
  const int64_t* w = A.w;
  int64_t* out = A.out;
  int64_t* gval = A.gval;
  extern __shared__ int64_t sm64[];
  int64_t* val = sm64;                                         // ring [kSeqRing]: f (fwd) or blevel (bwd)
  int64_t* ec = val + kSeqRing;                                // [kSeqTile]
  int64_t* wt = ec + kSeqTile;                                 // [kSeqTileN]
  int64_t* bmax = wt + kSeqTileN;                              // [kSeqTileN]
  int32_t* en = reinterpret_cast<int32_t*>(bmax + kSeqTileN);  // [kSeqTile]
  int32_t* ot = en + kSeqTile;                                 // [kSeqTileN + 1]
  int32_t* icnt = ot + kSeqTileN + 1;                          // [kSeqTileN]
  __shared__ int32_t tile_hi;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int32_t done = 0;  // nodes processed (in sweep order)
  while (done < n) {
    // tile: sweep positions [done, hi) with at most kSeqTile edges (at least one node)
    if (threadIdx.x == 0) {
      const int32_t v0 = rev ? n - 1 - done : done;
      const int32_t base = rev ? off[v0 + 1] : off[v0];
      int32_t lo = done + 1, hi = min(n, done + kSeqTileN);  // largest end with edge span <= kSeqTile
      while (lo < hi) {
        const int32_t mid = (lo + hi + 1) >> 1;
        const int32_t span = rev ? base - off[n - mid] : off[mid] - base;
        if (span <= kSeqTile) lo = mid; else hi = mid - 1;
      }
      tile_hi = lo;
    }
    __syncthreads();
    const int32_t hi = tile_hi;
    const int32_t e0 = rev ? off[n - hi] : off[done];
    const int32_t e1 = rev ? off[n - done] : off[hi];
    const bool fits = e1 - e0 <= kSeqTile;
    if (fits) {
      // a source swept before this tile has its value already: stage f[u] + c with en = -1,
      // so the walk only chains through in-tile sources (en = u, ec = c)
      for (int32_t k = threadIdx.x; k < e1 - e0; k += blockDim.x) {
        const int32_t u = nbr[e0 + k];
        const int64_t c = cost[e0 + k];
        const int32_t pu = rev ? n - 1 - u : u;
        const bool before = pu < done;
        en[k] = before ? -1 : u;
        ec[k] = before ? (done - pu <= kSeqRing ? val[pu & (kSeqRing - 1)] : __ldcg(gval + u)) + c : c;
      }
    }
    for (int32_t i = done + threadIdx.x; i <= hi; i += blockDim.x) {
      const int32_t v = rev ? n - 1 - i : i;  // sweep position i -> row start of node v (i < hi)
      if (i < hi) {
        wt[i - done] = w[v];
        ot[i - done] = rev ? off[v + 1] : off[v];  // row end (bwd) / start (fwd)
      } else {
        ot[i - done] = rev ? off[n - hi] : off[hi];
      }
    }
    __syncthreads();
    if (fits) {
      // per node (one warp each): the max over sources swept before the tile, and the
      // in-tile sources compacted to the row's front -- the walk below then touches only
      // the chain it depends on (one shared read per in-tile source, none otherwise)
      for (int32_t i = done + warp; i < hi; i += nwarps) {
        const int32_t rb = (rev ? ot[i + 1 - done] : ot[i - done]) - e0;
        const int32_t re = (rev ? ot[i - done] : ot[i + 1 - done]) - e0;
        int64_t bm = 0;
        int32_t cnt = 0;
        for (int32_t k0 = rb; k0 < re; k0 += 32) {
          const int32_t k = k0 + lane;
          const bool act = k < re;
          const int32_t u = act ? en[k] : -1;
          const int64_t x = act ? ec[k] : 0;
          if (act && u < 0) bm = max(bm, x);
          const unsigned intra = __ballot_sync(0xffffffffu, u >= 0);
          __syncwarp();  // every lane read its slot before the compacted writes below
          if (u >= 0) {
            const int32_t p = rb + cnt + __popc(intra & ((1u << lane) - 1u));
            en[p] = u;
            ec[p] = x;
          }
          cnt += __popc(intra);
          __syncwarp();
        }
        bm = warp_max_nonneg(bm);
        if (lane == 0) {
          bmax[i - done] = bm;
          icnt[i - done] = cnt;
        }
      }
      __syncthreads();
    }
    if (warp == 0) {
      for (int32_t i = done; i < hi; ++i) {
        const int32_t v = rev ? n - 1 - i : i;
        const int32_t b = rev ? ot[i + 1 - done] : ot[i - done], e = rev ? ot[i - done] : ot[i + 1 - done];
        int64_t mx = 0;
        if (fits) {
          const int32_t cnt = icnt[i - done];
          mx = bmax[i - done];
          if (cnt > 0) {
            int64_t m = lane == 0 ? mx : 0;
            for (int32_t k = lane; k < cnt; k += 32) {
              const int32_t u = en[b - e0 + k];
              const int32_t pu = rev ? n - 1 - u : u;  // in this tile: the ring holds it
              m = max(m, val[pu & (kSeqRing - 1)] + ec[b - e0 + k]);
            }
            mx = warp_max_nonneg(m);
          }
        } else {
          for (int32_t k = b + lane; k < e; k += 32) {
            const int32_t u = nbr[k];
            const int64_t c = cost[k];
            const int32_t pu = rev ? n - 1 - u : u;  // sweep position of u (< i)
            const int64_t fu = i - pu <= kSeqRing ? val[pu & (kSeqRing - 1)] : __ldcg(gval + u);
            mx = max(mx, fu + c);
          }
          mx = warp_max_nonneg(mx);
        }
        if (lane == 0) {
          const int64_t vv = mx + wt[i - done];  // f[v] = tlevel + w (fwd); blevel (bwd)
          val[i & (kSeqRing - 1)] = vv;
          if (gval) __stcg(gval + v, vv);
          out[v] = rev ? vv : mx;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    done = hi;
  }
}

// ---- dataflow levels (graphs whose index order is topological, any width).  No level
// barriers: warps take 32-node chunks in sweep order from a ticket counter, and a node's
// value is published in HBM/L2 as soon as its last input is known (-1 = not yet), so the
// critical path is the DAG's depth x one L2 round trip instead of depth x (frontier
// kernel step + barrier).  A chunk waits only on lower tickets, which are held by running
// warps, so there is no deadlock; a second counter (chunks finished) keeps the ticket
// holders within `ahead` chunks of the finished ones, which bounds the number of warps
// polling at once (the wavefront of a deep graph is narrow).  Each lane keeps up to 8 of
// its in-edges in flight; the warp loop is uniform, so lanes of one warp may depend on
// each other.
__device__ __forceinline__ int64_t ld_relaxed_i64(const int64_t* p) {
  int64_t x;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(x) : "l"(p) : "memory");
  return x;
}
__device__ __forceinline__ void st_relaxed_i64(int64_t* p, int64_t x) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(x) : "memory");
}
__device__ __forceinline__ int ld_relaxed_i32(const int* p) {
  int x;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
  return x;
}

constexpr int kFlowFin = 32;  // finished counter one L2 line (128 B) away from the ticket
constexpr int kFlowCtr = 64;  // ints of counters per pass

// forward (rev = false): in-CSC rows, val = tlevel + w, out = tlevel
// backward (rev = true): out-CSR rows, val = out = blevel
__device__ __forceinline__ void levels_flow_body(int32_t n, const int32_t* off, const int32_t* nbr,
                                                 const int64_t* cost, const int64_t* w, int64_t* val, int64_t* out,
                                                 bool rev, int* ctr, int32_t ahead, int32_t grain,
                                                 unsigned sleep_cap, int prefetch) {
  const int lane = threadIdx.x & 31;
  const int32_t nchunks = (n + 31) >> 5;
  // Software pipeline over a warp's chunks: the next ticket is taken when the current chunk
  // starts and its row bounds / weight are loaded while the current chunk waits on its
  // inputs, so a chunk's chain is rows -> inputs -> publish instead of ticket -> bounds ->
  // rows -> inputs -> publish.  A warp's current chunk is always its lowest ticket, so the
  // lowest unfinished chunk is always being worked on (no deadlock).  A ticket is `grain`
  // consecutive chunks (one atomic per grain: on a wide graph thousands of warps share the
  // ticket counter, whose same-address atomics serialise in L2); ctr[0] = next ticket,
  // ctr[kFlowFin] = chunks finished (the lookahead throttle; skipped when unthrottled).
  int c = 0;
  if (lane == 0) c = atomicAdd(&ctr[0], grain);
  c = __shfl_sync(0xffffffffu, c, 0);
  int rem = grain - 1;  // chunks of the current ticket after c
  const bool throttled = ahead < nchunks;
  int fin_seen = 0;  // lane 0: last value read from ctr[kFlowFin] (re-read only when needed)
  int32_t k = 0, e = 0;
  int64_t wv = 0;
  if (c < nchunks) {
    const int32_t i = c * 32 + lane;
    if (i < n) {
      const int32_t v = rev ? n - 1 - i : i;
      k = off[v];
      e = off[v + 1];
      wv = w[v];
    }
  }
  while (c < nchunks) {
    int cn = 0;
    if (lane == 0) {
      if (rem == 0) cn = atomicAdd(&ctr[0], grain);
      if (c - ahead > fin_seen)
        while ((fin_seen = ld_relaxed_i32(&ctr[kFlowFin])) < c - ahead) __nanosleep(128);
    }
    const int32_t i = c * 32 + lane;
    const bool valid = i < n;
    const int32_t v = valid ? (rev ? n - 1 - i : i) : 0;
    int32_t kn = 0, en = 0;
    int64_t wvn = 0;
    bool fetched = false;  // next chunk's bounds requested
    bool pf = prefetch != 0;  // next chunk's rows still to be prefetched into L2
    int64_t mx = 0;
    bool done = !valid;
    unsigned pend = 0;
    int32_t u[8];
    int64_t cc[8];
    unsigned sleep_ns = 0;
    for (;;) {
      bool progress = false;
      if (!done) {
        if (pend == 0 && k < e) {
          const int cnt = min(8, e - k);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            u[q] = q < cnt ? nbr[k + q] : 0;
            cc[q] = q < cnt ? cost[k + q] : 0;
          }
          pend = (1u << cnt) - 1u;
          k += cnt;
        }
      }
      if (!fetched) {  // first pass: the rows are requested, now the next chunk's bounds
        fetched = true;
        cn = rem > 0 ? c + 1 : __shfl_sync(0xffffffffu, cn, 0);
        const int32_t in = cn * 32 + lane;
        if (cn < nchunks && in < n) {
          const int32_t vn = rev ? n - 1 - in : in;
          kn = off[vn];
          en = off[vn + 1];
          wvn = w[vn];
        }
      }
      if (!done) {
        if (pend) {
          int64_t x[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) x[q] = (pend >> q) & 1u ? ld_relaxed_i64(val + u[q]) : -1;
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (x[q] >= 0) {
              mx = max(mx, x[q] + cc[q]);
              pend &= ~(1u << q);
              progress = true;
            }
        }
        if (pend == 0 && k == e) {
          const int64_t vv = mx + wv;
          st_relaxed_i64(val + v, vv);
          out[v] = rev ? vv : mx;
          done = true;
          progress = true;
        }
      }
      if (pf) {
        // the first poll's values are back, so the next chunk's bounds (requested before
        // them) are too: one bulk L2 prefetch of its whole row span per array (the rows of
        // 32 consecutive nodes are contiguous), so its row loads hit L2 instead of HBM
        pf = false;
        const bool has = kn < en;
        const int32_t lo = __reduce_min_sync(0xffffffffu, has ? kn : INT_MAX);
        const int32_t hi = __reduce_max_sync(0xffffffffu, has ? en : 0);
        if (lane == 0 && lo < hi) {
          const int32_t lo4 = lo & ~3, hi4 = (hi + 3) & ~3;  // 16-byte aligned spans
          const int32_t lo2 = lo & ~1, hi2 = (hi + 1) & ~1;
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nbr + lo4),
                       "r"(static_cast<unsigned>(4 * (hi4 - lo4))) : "memory");
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(cost + lo2),
                       "r"(static_cast<unsigned>(8 * (hi2 - lo2))) : "memory");
        }
      }
      if (__all_sync(0xffffffffu, done)) break;
      if (__any_sync(0xffffffffu, progress)) {
        sleep_ns = 0;
      } else {
        sleep_ns = sleep_ns ? min(sleep_ns * 2, sleep_cap) : 32u;
        if (sleep_cap) __nanosleep(sleep_ns);
      }
    }
    if (throttled && lane == 0) atomicAdd(&ctr[kFlowFin], 1);
    rem = rem > 0 ? rem - 1 : grain - 1;
    c = cn;
    k = kn;
    e = en;
    wv = wvn;
  }
}

// Both directions of several graphs in one launch (blockIdx.y = pass): the t and b passes
// are independent, and the graphs of a batched call stop waiting on each other's level
// kernels (each pass keeps its own ticket counters and warp count).
struct FlowPass {
  int32_t n;
  const int32_t* off;
  const int32_t* nbr;
  const int64_t* cost;
  const int64_t* w;
  int64_t* val;
  int64_t* out;
  bool rev;
  int* ctr;  // kFlowCtr ints, zeroed
  int32_t ahead, grain, blocks;
};
constexpr int kFlowBatch = 16;
struct FlowBatch {
  FlowPass p[kFlowBatch];
  unsigned sleep_cap;
  int prefetch;  // bulk L2 prefetch of the next chunk's rows (DP_FLOW_NO_PREFETCH: off)
};
__global__ void __launch_bounds__(128) k_levels_flow_batch(const __grid_constant__ FlowBatch b) {
  const FlowPass& P = b.p[blockIdx.y];
  if (static_cast<int32_t>(blockIdx.x) >= P.blocks) return;
  levels_flow_body(P.n, P.off, P.nbr, P.cost, P.w, P.val, P.out, P.rev, P.ctr, P.ahead, P.grain, b.sleep_cap,
                   b.prefetch);
}

__global__ void k_kahn_init(KahnArgs a) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < a.n; v += (int64_t)gridDim.x * blockDim.x) {
    const bool src = a.indeg[v] == 0;
    if (a.tlevel) a.tlevel[v] = 0;
    const int slot = warp_append(&a.counters[0], src);
    if (src) a.order[slot] = static_cast<int32_t>(v);
  }
}

// One CTA, __syncthreads between levels (deep DAGs: hundreds to thousands of narrow
// levels, where a grid barrier per level would dominate).
__global__ void __launch_bounds__(1024) k_kahn_fwd_narrow(KahnArgs a) {
  __shared__ int tail;
  __shared__ int maxw;
  __shared__ int s_le;
  if (threadIdx.x == 0) {
    tail = a.counters[0];
    maxw = a.counters[3];
  }
  int32_t lb = a.counters[2], level = a.counters[1];
  for (;;) {
    __syncthreads();  // every append of the previous level is done
    if (threadIdx.x == 0) s_le = tail;
    __syncthreads();  // frontier end snapshot taken before anyone appends again
    const int32_t le = s_le;
    if (le == lb || le - lb > a.narrow_max) break;
    if (threadIdx.x == 0) {
      a.level_off[level] = lb;
      if (le - lb > maxw) maxw = le - lb;
    }
    for (int32_t i0 = lb; i0 < le; i0 += blockDim.x) {
      const int32_t i = i0 + threadIdx.x;
      kahn_relax_warp(a, i < le ? a.order[i] : -1, level, &tail);
    }
    lb = le;
    ++level;
  }
  if (threadIdx.x == 0) {
    a.counters[0] = tail;
    a.counters[1] = level;
    a.counters[2] = lb;
    a.counters[3] = maxw;
    __threadfence();
  }
}

// Persistent multi-CTA variant (cooperative launch) for wide frontiers.
__global__ void __launch_bounds__(512) k_kahn_fwd_wide(KahnArgs a) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  int32_t lb = a.counters[2], level = a.counters[1], maxw = a.counters[3];
  int32_t le = a.counters[0];  // nobody appends before every CTA has read this (no relax yet)
  grid_barrier(a.bar, gridDim.x);
  for (;;) {
    if (le == lb) break;
    if (le - lb > maxw) maxw = le - lb;
    if (tid == 0) a.level_off[level] = lb;
    for (int64_t i0 = lb + (tid - (tid & 31)); i0 < le; i0 += nth) {
      const int64_t i = i0 + (tid & 31);
      kahn_relax_warp(a, i < le ? a.order[i] : -1, level, &a.counters[0]);
    }
    grid_barrier(a.bar, gridDim.x, &a.counters[0], &a.counters[4]);
    lb = le;
    le = *((volatile int*)&a.counters[4]);
    ++level;
  }
  if (tid == 0) {
    a.counters[1] = level;
    a.counters[2] = lb;
    a.counters[3] = maxw;
  }
}

__global__ void __launch_bounds__(1024) k_kahn_bwd_narrow(KahnArgs a, int32_t levels) {
  for (int32_t L = levels - 1; L >= 0; --L) {
    const int32_t b = a.level_off[L], e = a.level_off[L + 1];
    for (int32_t i0 = b; i0 < e; i0 += blockDim.x) {
      const int32_t i = i0 + threadIdx.x;
      kahn_pull_warp(a, i < e ? a.order[i] : -1);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(512) k_kahn_bwd_wide(KahnArgs a, int32_t levels) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int32_t L = levels - 1; L >= 0; --L) {
    const int32_t b = a.level_off[L], e = a.level_off[L + 1];
    for (int64_t i0 = b + (tid - (tid & 31)); i0 < e; i0 += nth) {
      const int64_t i = i0 + (tid & 31);
      kahn_pull_warp(a, i < e ? a.order[i] : -1);
    }
    grid_barrier(a.bar, gridDim.x);
  }
}

__global__ void k_indeg(const int32_t* in_off, int32_t n, int32_t* indeg) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    indeg[v] = in_off[v + 1] - in_off[v];
}

__global__ void k_min_remaining_id(const int32_t* indeg, const int64_t* id, int32_t n,
                                   unsigned long long* best) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    if (indeg[v] > 0) atomicMin(best, static_cast<unsigned long long>(id[v]) ^ (1ull << 63));
}

// find_cycle_witness (graph.cpp:71-94), single thread: from the smallest remaining id,
// follow the smallest-id successor inside the remaining set until an id repeats.
__global__ void k_witness(const int32_t* indeg, const int64_t* id, const int32_t* out_off,
                          const int32_t* out_dst, int32_t n, int32_t start, int32_t* pos_in_path,
                          int32_t* path, int32_t* result) {
  if (threadIdx.x || blockIdx.x) return;
  int32_t len = 0, cur = start;
  for (;;) {
    if (pos_in_path[cur] >= 0) {
      result[0] = pos_in_path[cur];
      result[1] = len;
      return;
    }
    pos_in_path[cur] = len;
    path[len++] = cur;
    int32_t best = -1;
    for (int32_t k = out_off[cur]; k < out_off[cur + 1]; ++k) {
      int32_t x = out_dst[k];
      if (indeg[x] > 0 && (best < 0 || id[x] < id[best])) best = x;
    }
    if (best < 0) {
      result[0] = 0;
      result[1] = len;
      return;
    }
    cur = best;
  }
}

int coop_grid(const void* kernel, int block, int64_t work, int num_sms) {
  int per_sm = 0;
  DP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0));
  if (per_sm < 1) per_sm = 1;
  int64_t want = (work + block - 1) / block;
  int64_t cap = static_cast<int64_t>(per_sm) * num_sms;
  if (cap > 2 * num_sms) cap = 2 * num_sms;  // barrier cost grows with CTA count
  if (want < 1) want = 1;
  return static_cast<int>(want < cap ? want : cap);
}

}  // namespace

// ------------------------------------------------------------------ host orchestration
void graph_upload(DevGraph& g, dp_ctx* ctx, const dp_graph_t* h, cudaStream_t copy, cudaEvent_t done) {
  if (h->n_nodes < 0 || h->n_edges < 0 || h->n_nodes > INT32_MAX - 2 || h->n_edges > INT32_MAX - 2)
    fail(DP_E_ARGUMENT, "graph sizes out of range (n=%lld, m=%lld)", (long long)h->n_nodes,
         (long long)h->n_edges);
  g.ctx = ctx;
  g.n = static_cast<int32_t>(h->n_nodes);
  g.m = static_cast<int32_t>(h->n_edges);
  g.id.alloc(ctx, g.n);
  g.w.alloc(ctx, g.n);
  g.mem.alloc(ctx, g.n);
  g.has_group = false;
  if (h->group) {
    for (int64_t i = 0; i < h->n_nodes; ++i) {
      if (h->group[i] >= 0) { g.has_group = true; break; }
    }
  }
  if (g.has_group) g.group.alloc(ctx, g.n);
  g.src_id.alloc(ctx, g.m);
  g.dst_id.alloc(ctx, g.m);
  g.bytes.alloc(ctx, g.m);
  cudaStream_t s = ctx->stream;
  if (copy) {  // the buffers were allocated on ctx->stream: the copy stream waits for that
    DP_CUDA(cudaEventRecord(done, ctx->stream));
    DP_CUDA(cudaStreamWaitEvent(copy, done, 0));
    s = copy;
  }
  auto up = [&](void* d, const void* hsrc, size_t bytes) {
    if (bytes) DP_CUDA(cudaMemcpyAsync(d, hsrc, bytes, cudaMemcpyHostToDevice, s));
  };
  up(g.id.p, h->node_id, sizeof(*h->node_id) * g.n);
  up(g.w.p, h->compute_us, sizeof(*h->compute_us) * g.n);
  up(g.mem.p, h->memory_bytes, sizeof(*h->memory_bytes) * g.n);
  if (g.has_group) up(g.group.p, h->group, sizeof(*h->group) * g.n);
  up(g.src_id.p, h->edge_src, sizeof(*h->edge_src) * g.m);
  up(g.dst_id.p, h->edge_dst, sizeof(*h->edge_dst) * g.m);
  up(g.bytes.p, h->edge_bytes, sizeof(*h->edge_bytes) * g.m);
  if (copy) DP_CUDA(cudaEventRecord(done, copy));
}

void graph_adopt_dense(DevGraph& g, dp_ctx* ctx, int32_t n, int32_t m, DevBuf<int64_t>&& w,
                       DevBuf<int64_t>&& mem, DevBuf<int32_t>&& esrc, DevBuf<int32_t>&& edst,
                       DevBuf<int64_t>&& bytes) {
  g = DevGraph();
  g.ctx = ctx;
  g.n = n;
  g.m = m;
  g.w = std::move(w);
  g.mem = std::move(mem);
  g.esrc = std::move(esrc);
  g.edst = std::move(edst);
  g.bytes = std::move(bytes);
  g.dense_ids = true;
  g.has_group = false;
}

void graph_resolve_begin(DevGraph& g, ResolveState& st) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  st.flag.alloc(ctx, 1);
  const int one = 1;
  st.flag.upload(&one, 1);
  DP_LAUNCH(ctx, k_dense_check, grid_for(g.n, B), B, 0, g.id.p, g.n, st.flag.p);
  download_bytes(ctx, &st.dense, st.flag.p, sizeof(int));
}

void graph_resolve(DevGraph& g) {
  ResolveState st;
  graph_resolve_begin(g, st);
  sync(g.ctx);
  graph_resolve_end(g, st);
}

void graph_resolve_end(DevGraph& g, ResolveState& st) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  g.dense_ids = st.dense == 1;
  if (!g.dense_ids) {
    DevBuf<uint64_t> keys(ctx, g.n);
    DevBuf<int32_t> vals(ctx, g.n);
    g.sorted_key.alloc(ctx, g.n);
    g.sorted_idx.alloc(ctx, g.n);
    DP_LAUNCH(ctx, k_id_keys, grid_for(g.n, B), B, 0, g.id.p, g.n, keys.p, vals.p);
    sort_pairs_u64(ctx, keys.p, g.sorted_key.p, vals.p, g.sorted_idx.p, g.n, 0, 64);
  }
  g.esrc.alloc(ctx, g.m);
  g.edst.alloc(ctx, g.m);
  DP_LAUNCH(ctx, k_resolve, grid_for(g.m, B), B, 0, g.src_id.p, g.dst_id.p, g.m, g.n, g.dense_ids,
            g.sorted_key.p, g.sorted_idx.p, g.esrc.p, g.edst.p);
}

void graph_ids_to_index(DevGraph& g, const int64_t* ids, int32_t* out, int64_t k) {
  DP_LAUNCH(g.ctx, k_ids_to_index, grid_for(k, 256), 256, 0, ids, k, g.n, g.dense_ids, g.sorted_key.p,
            g.sorted_idx.p, out);
}

int32_t graph_index_of(DevGraph& g, int64_t id) {
  DevBuf<int64_t> d(g.ctx, 1);
  DevBuf<int32_t> o(g.ctx, 1);
  d.upload(&id, 1);
  graph_ids_to_index(g, d.p, o.p, 1);
  return scalar_to_host(g.ctx, o.p);
}

// graph_adjacency split around its one host round trip, so several graphs share it.
void graph_adjacency_begin(DevGraph& g, AdjState& st) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  int32_t n = g.n, m = g.m;
  g.out_off.alloc(ctx, (size_t)n + 1);
  g.in_off.alloc(ctx, (size_t)n + 1);
  g.out_eid.alloc(ctx, m);
  g.in_eid.alloc(ctx, m);
  st.cnt.alloc(ctx, (size_t)n + 1);
  st.keys.alloc(ctx, m);
  st.keys_out.alloc(ctx, m);
  st.vals.alloc(ctx, m);
  // CSR by source
  st.flags.alloc(ctx, 4);  // [0] sorted by source, [1] some row longer than 64, [2] index order topological
  const int init[4] = {1, 0, 1, 0};
  st.flags.upload(init, 4);
  st.span.alloc(ctx, 1);
  st.span.zero();
  DP_LAUNCH(ctx, k_sorted_check, grid_for(m, B), B, 0, g.esrc.p, g.edst.p, m, st.flags.p, st.span.p);
  st.cnt.zero();
  DP_LAUNCH(ctx, k_row_keys, grid_for(m, B), B, 0, g.esrc.p, g.edst.p, m, n, true, st.keys.p, st.vals.p, st.cnt.p);
  exclusive_scan_i32(ctx, st.cnt.p, g.out_off.p, (int64_t)n + 1);
  DP_LAUNCH(ctx, k_big_rows, grid_for(n, B), B, 0, g.out_off.p, n, st.flags.p + 1);
  // the three facts the host needs: already sorted by source, edges with resolved
  // endpoints, some row longer than 64 (valid after the caller's sync)
  download_bytes(ctx, &st.hs[0], st.flags.p, sizeof(int));
  download_bytes(ctx, &st.hs[1], g.out_off.p + n, sizeof(int32_t));
  download_bytes(ctx, &st.hs[2], st.flags.p + 1, sizeof(int));
  download_bytes(ctx, &st.hs[3], st.flags.p + 2, sizeof(int));
  download_bytes(ctx, &st.hspan, st.span.p, sizeof(unsigned long long));
}

void graph_adjacency_end(DevGraph& g, AdjState& st) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  int32_t n = g.n, m = g.m;
  int endbit = bits_for(static_cast<uint64_t>(n));
  g.m_ok = st.hs[1];
  g.big_rows = st.hs[2] != 0;
  g.topo_known = true;
  g.index_topo = st.hs[3] == 1 && n > 0;
  g.span_sum = st.hspan;
  if (st.hs[0] == 1) {
    DP_LAUNCH(ctx, k_iota, grid_for(m, B), B, 0, g.out_eid.p, (int64_t)m);
  } else {
    sort_pairs_u32(ctx, st.keys.p, st.keys_out.p, st.vals.p, g.out_eid.p, m, endbit);
  }
  // CSC by destination
  st.cnt.zero();
  DP_LAUNCH(ctx, k_row_keys, grid_for(m, B), B, 0, g.esrc.p, g.edst.p, m, n, false, st.keys.p, st.vals.p, st.cnt.p);
  exclusive_scan_i32(ctx, st.cnt.p, g.in_off.p, (int64_t)n + 1);
  sort_pairs_u32(ctx, st.keys.p, st.keys_out.p, st.vals.p, g.in_eid.p, m, endbit);
  g.out_dst.alloc(ctx, g.m_ok);
  g.in_src.alloc(ctx, g.m_ok);
  DP_LAUNCH(ctx, k_gather_i32, grid_for(g.m_ok, B), B, 0, g.edst.p, g.out_eid.p, g.out_dst.p, (int64_t)g.m_ok);
  DP_LAUNCH(ctx, k_gather_i32, grid_for(g.m_ok, B), B, 0, g.esrc.p, g.in_eid.p, g.in_src.p, (int64_t)g.m_ok);
  g.has_adj = true;
  g.has_cost = false;  // CSR/CSC-ordered cost copies must follow the new permutation
}

void graph_adjacency(DevGraph& g) {
  AdjState st;
  graph_adjacency_begin(g, st);
  sync(g.ctx);
  graph_adjacency_end(g, st);
}

void graph_costs(DevGraph& g, dp_comm_t comm) {
  dp_ctx* ctx = g.ctx;
  if (g.has_cost && g.ck == comm.k_us_per_byte && g.cb == comm.b_us) return;
  const int B = 256;
  g.cost.alloc(ctx, g.m);
  DP_LAUNCH(ctx, k_costs, grid_for(g.m, B), B, 0, g.bytes.p, g.m, comm.k_us_per_byte, comm.b_us, g.cost.p);
  if (g.has_adj) {
    g.out_cost.alloc(ctx, g.m_ok);
    g.in_cost.alloc(ctx, g.m_ok);
    DP_LAUNCH(ctx, k_gather_i64, grid_for(g.m_ok, B), B, 0, g.cost.p, g.out_eid.p, g.out_cost.p, (int64_t)g.m_ok);
    DP_LAUNCH(ctx, k_gather_i64, grid_for(g.m_ok, B), B, 0, g.cost.p, g.in_eid.p, g.in_cost.p, (int64_t)g.m_ok);
  }
  g.has_cost = true;
  g.ck = comm.k_us_per_byte;
  g.cb = comm.b_us;
}

// The one-CTA index-order sweep of several graphs (index order topological, checked by the
// caller), one launch per direction.
void levels_sweep_launch(DevGraph* const* gs, int64_t* const* tlevel, int64_t* const* blevel, int count) {
  dp_ctx* ctx = gs[0]->ctx;
  const size_t sm =
      sizeof(int64_t) * (kSeqRing + kSeqTile + 2 * kSeqTileN) + sizeof(int32_t) * (kSeqTile + 2 * kSeqTileN + 1);
  static bool attr = false;
  if (!attr) {
    DP_CUDA(cudaFuncSetAttribute(k_levels_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    attr = true;
  }
  std::vector<DevBuf<int64_t>> gval(2 * static_cast<size_t>(count));  // per direction (they run at once)
  for (int b0 = 0; b0 < count; b0 += kSeqBatch) {
    const int k = std::min(kSeqBatch, count - b0);
    SeqBatch sb{};
    for (int q = 0; q < k; ++q) {
      DevGraph& g = *gs[b0 + q];
      if (g.n > kSeqRing) {
        gval[2 * (b0 + q)].alloc(ctx, g.n);
        gval[2 * (b0 + q) + 1].alloc(ctx, g.n);
      }
      sb.a[0][q] = SeqArgs{g.n, g.in_off.p, g.in_src.p, g.in_cost.p, g.w.p, tlevel[b0 + q], gval[2 * (b0 + q)].p};
      sb.a[1][q] =
          SeqArgs{g.n, g.out_off.p, g.out_dst.p, g.out_cost.p, g.w.p, blevel[b0 + q], gval[2 * (b0 + q) + 1].p};
    }
    k_levels_seq<<<dim3(k, 2), 1024, sm, ctx->stream>>>(sb);
    ++ctx->launches;
    DP_CUDA(cudaGetLastError());
  }
}

// Index-order check of several graphs with one host sync; ok[i] = index order topological.
std::vector<char> graphs_index_topological(DevGraph* const* gs, int count, std::vector<unsigned long long>* spans) {
  dp_ctx* ctx = gs[0]->ctx;
  bool known = true;  // all facts from graph_adjacency's round trip: no launch, no sync
  for (int i = 0; i < count; ++i) known = known && gs[i]->topo_known;
  if (known) {
    std::vector<char> ok(count);
    if (spans) spans->resize(count);
    for (int i = 0; i < count; ++i) {
      ok[i] = gs[i]->index_topo;
      if (spans) (*spans)[i] = gs[i]->span_sum;
    }
    return ok;
  }
  DevBuf<unsigned long long> chk(ctx, 2 * (size_t)count);
  std::vector<unsigned long long> init(2 * (size_t)count, 0ull);
  for (int i = 0; i < count; ++i) init[2 * i] = 1ull;
  chk.upload(init.data(), init.size());
  for (int i = 0; i < count; ++i) {
    DevGraph& g = *gs[i];
    if (g.n > 0)
      DP_LAUNCH(ctx, k_index_topo, grid_for(g.n, 256), 256, 0, g.in_off.p, g.in_src.p, g.n,
                reinterpret_cast<int*>(chk.p + 2 * i), chk.p + 2 * i + 1);
  }
  std::vector<unsigned long long> h = to_host(ctx, chk.p, 2 * (size_t)count);
  std::vector<char> ok(count);
  for (int i = 0; i < count; ++i) ok[i] = gs[i]->n > 0 && static_cast<int>(h[2 * i]) == 1;
  if (spans) {
    spans->resize(count);
    for (int i = 0; i < count; ++i) (*spans)[i] = h[2 * i + 1];
  }
  return ok;
}

bool coarse_flow_wanted(int32_t n) { return n > kSeqMaxN && getenv("DP_COARSE_FLOW") != nullptr; }

// Levels when the node index order is topological (every edge u->v has u < v): the
// one-CTA sweep for small or chain-like graphs (the coarse graph of fuse), the dataflow
// kernel otherwise.  Returns false when the index order is not topological (caller uses
// graph_kahn).
// Dataflow launch plan of one graph from its summed edge span (u -> v: v - u).
// Narrow wavefront (mean span under kFlowWideChunks chunks; config #4 deep): lookahead of
// two mean spans, at least 64 chunks (more polling warps only cost when many graphs run
// at once: 64 vs 256 chunks = 2.47 vs 2.33 ms alone, 707 vs 730 ms per 128-graph step),
// one chunk per ticket, up to 32 warps per SM.  Wide wavefront (config #4 wide: 16 levels
// of 65,536): no lookahead limit, so warps run far ahead and their rows load early, and
// 8 warps per SM per pass -- measured on the B200 (tools/levels_probe.py, both passes):
// 0.36 ms with the narrow plan, 0.10-0.12 ms with 8 warps per SM and no limit (fewer
// polling warps, less L2 contention; 4 / 16 / 24 warps: 0.19 / 0.13 / 0.14 ms; a lookahead
// of 128 chunks: 0.92 ms).  Tickets of more than one chunk measured slower (4 chunks: 0.16
// ms).  DP_FLOW_AHEAD / _GRAIN / _WARPS (per SM) override.
constexpr double kFlowWideChunks = 256.0;
struct FlowPlan {
  int32_t ahead, grain;
  int blocks;
};
FlowPlan flow_plan(dp_ctx* ctx, const DevGraph& g, unsigned long long span_sum) {
  const double mean_span = g.m_ok > 0 ? static_cast<double>(span_sum) / g.m_ok : 32.0;
  FlowPlan pl{};
  const bool wide = mean_span / 32.0 >= kFlowWideChunks;
  pl.ahead = wide ? (1 << 30) : static_cast<int32_t>(std::max(64.0, 2.0 * mean_span / 32.0));
  if (const char* s = getenv("DP_FLOW_AHEAD")) pl.ahead = atoi(s);
  pl.grain = 1;
  if (const char* s = getenv("DP_FLOW_GRAIN")) pl.grain = std::max(1, atoi(s));
  const int32_t nchunks = (g.n + 31) / 32;
  int32_t per_sm = wide ? 8 : 32;
  if (const char* s = getenv("DP_FLOW_WARPS")) per_sm = atoi(s);
  const int32_t warps =
      std::max(1, std::min({nchunks, static_cast<int32_t>(std::min<int64_t>(pl.ahead + 32LL, 1 << 30)),
                            ctx->num_sms * per_sm}));
  pl.blocks = (warps + 3) / 4;
  if (getenv("DP_DEBUG_FLOW"))
    fprintf(stderr, "[flow] n=%d m=%d mean_span=%.1f wide=%d ahead=%d grain=%d warps=%d\n", g.n, g.m_ok, mean_span,
            static_cast<int>(wide), pl.ahead, pl.grain, warps);
  return pl;
}
unsigned flow_sleep_cap() {
  unsigned sleep_cap = 256;
  if (const char* s = getenv("DP_FLOW_SLEEP")) sleep_cap = static_cast<unsigned>(atoi(s));
  return sleep_cap;
}

bool graph_levels_indexorder(DevGraph& g, int64_t* tlevel, int64_t* blevel, bool chainlike) {
  dp_ctx* ctx = g.ctx;
  const int32_t n = g.n;
  if (n == 0 || getenv("DP_LEVELS_KAHN")) return false;
  unsigned long long h[2];  // [0] ok flag, [1] span sum
  if (g.topo_known) {  // from graph_adjacency's round trip
    h[0] = g.index_topo ? 1ull : 0ull;
    h[1] = g.span_sum;
  } else {
    DevBuf<unsigned long long> chk(ctx, 2);
    const unsigned long long init[2] = {1ull, 0ull};
    chk.upload(init, 2);
    DP_LAUNCH(ctx, k_index_topo, grid_for(n, 256), 256, 0, g.in_off.p, g.in_src.p, n, reinterpret_cast<int*>(chk.p),
              chk.p + 1);
    chk.download(h, 2);
    sync(ctx);
  }
  if (static_cast<int>(h[0]) != 1) return false;
  const bool sweep = (n <= kSeqMaxN || (chainlike && !coarse_flow_wanted(n))) && getenv("DP_LEVELS_FLOW") == nullptr;

  if (sweep) {
    DevGraph* gs[1] = {&g};
    int64_t* t1[1] = {tlevel};
    int64_t* b1[1] = {blevel};
    levels_sweep_launch(gs, t1, b1, 1);
    g.processed = n;
    return true;
  }
  FlowBatch fb{};
  fb.sleep_cap = flow_sleep_cap();
  fb.prefetch = getenv("DP_FLOW_NO_PREFETCH") == nullptr;
  const FlowPlan pl = flow_plan(ctx, g, h[1]);
  DevBuf<int64_t> f(ctx, n);
  DevBuf<int> ctr(ctx, 2 * kFlowCtr);
  f.fill_bytes(0xff);
  ctr.zero();
  DP_CUDA(cudaMemsetAsync(blevel, 0xff, sizeof(int64_t) * n, ctx->stream));
  fb.p[0] = FlowPass{n, g.in_off.p, g.in_src.p, g.in_cost.p, g.w.p, f.p, tlevel, false, ctr.p, pl.ahead, pl.grain,
                     pl.blocks};
  fb.p[1] = FlowPass{n, g.out_off.p, g.out_dst.p, g.out_cost.p, g.w.p, blevel, blevel, true, ctr.p + kFlowCtr, pl.ahead,
                     pl.grain,
                     pl.blocks};
  k_levels_flow_batch<<<dim3(pl.blocks, 2), 128, 0, ctx->stream>>>(fb);
  ++ctx->launches;
  DP_CUDA(cudaGetLastError());
  g.processed = n;
  return true;
}

// graph_levels_indexorder (chainlike = false) for several graphs: one index-order check (one
// host round trip), one sweep launch per direction for the small ones, ONE launch for both
// dataflow passes of all the others.  ok[i] = false: not topological in index order (the
// caller runs graph_kahn).
std::vector<char> graphs_levels_indexorder(DevGraph* const* gs, int count, int64_t* const* tlevel,
                                           int64_t* const* blevel) {
  std::vector<char> ok(count, 0);
  if (count == 0 || getenv("DP_LEVELS_KAHN")) return ok;
  dp_ctx* ctx = gs[0]->ctx;
  std::vector<unsigned long long> spans;
  ok = graphs_index_topological(gs, count, &spans);
  std::vector<DevGraph*> sg;
  std::vector<int64_t*> st, sb;
  std::vector<int> flow;
  for (int i = 0; i < count; ++i) {
    if (!ok[i]) continue;
    gs[i]->processed = gs[i]->n;
    if (gs[i]->n <= kSeqMaxN && getenv("DP_LEVELS_FLOW") == nullptr) {
      sg.push_back(gs[i]);
      st.push_back(tlevel[i]);
      sb.push_back(blevel[i]);
    } else {
      flow.push_back(i);
    }
  }
  if (!sg.empty()) levels_sweep_launch(sg.data(), st.data(), sb.data(), static_cast<int>(sg.size()));
  if (flow.empty()) return ok;
  const unsigned sleep_cap = flow_sleep_cap();
  std::vector<DevBuf<int64_t>> fval(flow.size());
  DevBuf<int> ctr(ctx, 2 * kFlowCtr * flow.size());
  ctr.zero();
  for (size_t q0 = 0; q0 < flow.size(); q0 += kFlowBatch / 2) {
    const size_t k = std::min<size_t>(kFlowBatch / 2, flow.size() - q0);
    FlowBatch b{};
    b.sleep_cap = sleep_cap;
    b.prefetch = getenv("DP_FLOW_NO_PREFETCH") == nullptr;
    int gridx = 1;
    for (size_t q = 0; q < k; ++q) {
      const int i = flow[q0 + q];
      DevGraph& g = *gs[i];
      const int32_t n = g.n;
      const FlowPlan pl = flow_plan(ctx, g, spans[i]);
      const int blocks = pl.blocks, ahead = pl.ahead;
      gridx = std::max(gridx, blocks);
      fval[q0 + q].alloc(ctx, n);
      fval[q0 + q].fill_bytes(0xff);
      DP_CUDA(cudaMemsetAsync(blevel[i], 0xff, sizeof(int64_t) * n, ctx->stream));
      int* c = ctr.p + 2 * kFlowCtr * (q0 + q);
      b.p[2 * q] = FlowPass{n, g.in_off.p, g.in_src.p, g.in_cost.p, g.w.p, fval[q0 + q].p, tlevel[i], false, c, ahead,
                            pl.grain, blocks};
      b.p[2 * q + 1] = FlowPass{n, g.out_off.p, g.out_dst.p, g.out_cost.p, g.w.p, blevel[i], blevel[i], true,
                                c + kFlowCtr, ahead, pl.grain, blocks};
    }
    k_levels_flow_batch<<<dim3(gridx, 2 * static_cast<unsigned>(k)), 128, 0, ctx->stream>>>(b);
    ++ctx->launches;
    DP_CUDA(cudaGetLastError());
  }
  return ok;
}

void graph_kahn(DevGraph& g, int64_t* tlevel, int64_t* blevel, int32_t* level_of) {
  dp_ctx* ctx = g.ctx;
  const int32_t n = g.n;
  g.order.alloc(ctx, n > 0 ? n : 1);
  g.level_off.alloc(ctx, (size_t)n + 2);
  if (n == 0) {
    g.processed = 0;
    g.num_levels = 0;
    return;
  }
  DevBuf<int32_t> indeg(ctx, n);
  DP_LAUNCH(ctx, k_indeg, grid_for(n, 256), 256, 0, g.in_off.p, n, indeg.p);
  DevBuf<int> counters(ctx, 5);
  DevBuf<unsigned> bar(ctx, 2);
  counters.zero();
  bar.zero();
  KahnArgs a;
  a.n = n;
  a.out_off = g.out_off.p;
  a.out_dst = g.out_dst.p;
  a.out_cost = (tlevel || blevel) ? g.out_cost.p : nullptr;
  a.w = g.w.p;
  a.indeg = indeg.p;
  a.order = g.order.p;
  a.level_off = g.level_off.p;
  a.tlevel = tlevel;
  a.blevel = blevel;
  a.level_of = level_of;
  a.counters = counters.p;
  a.bar = bar.p;
  a.narrow_max = 16384;
  DP_LAUNCH(ctx, k_kahn_init, grid_for(n, 256), 256, 0, a);
  DP_LAUNCH(ctx, k_kahn_fwd_narrow, 1, 1024, 0, a);
  int host[4];
  counters.download(host, 4);
  sync(ctx);
  if (host[2] != host[0]) {  // a wide frontier remains: continue with the whole GPU
    const int B = 512;
    int grid = coop_grid(reinterpret_cast<const void*>(k_kahn_fwd_wide), B, n, ctx->num_sms);
    void* args[] = {&a};
    DP_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_kahn_fwd_wide), grid, B, args, 0,
                                        ctx->stream));
    ++ctx->launches;
    counters.download(host, 4);
    sync(ctx);
  }
  g.processed = host[0];
  g.num_levels = host[1];
  if (g.processed == n) {
    int32_t last = n;
    DP_CUDA(cudaMemcpyAsync(g.level_off.p + g.num_levels, &last, sizeof(int32_t), cudaMemcpyHostToDevice,
                            ctx->stream));
    if (blevel) {
      if (host[3] <= a.narrow_max) {
        DP_LAUNCH(ctx, k_kahn_bwd_narrow, 1, 1024, 0, a, g.num_levels);
      } else {
        bar.zero();
        const int B = 512;
        int grid = coop_grid(reinterpret_cast<const void*>(k_kahn_bwd_wide), B, n, ctx->num_sms);
        int32_t lv = g.num_levels;
        void* args[] = {&a, &lv};
        DP_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_kahn_bwd_wide), grid, B, args, 0,
                                            ctx->stream));
        ++ctx->launches;
      }
    }
    sync(ctx);
  } else {
    // keep the residual in-degrees for the witness
    g.level_off.release();
    g.level_off.alloc(ctx, n);
    DP_CUDA(cudaMemcpyAsync(g.level_off.p, indeg.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
}

std::vector<int64_t> graph_cycle_witness(DevGraph& g) {
  dp_ctx* ctx = g.ctx;
  int32_t n = g.n;
  const int32_t* indeg = g.level_off.p;  // residual in-degrees (graph_kahn)
  DevBuf<unsigned long long> best(ctx, 1);
  best.fill_bytes(0xff);
  DP_LAUNCH(ctx, k_min_remaining_id, grid_for(n, 256), 256, 0, indeg, g.id.p, n, best.p);
  unsigned long long key = scalar_to_host(ctx, best.p);
  int64_t start_id = static_cast<int64_t>(key ^ (1ull << 63));
  int32_t start = graph_index_of(g, start_id);
  DevBuf<int32_t> pos(ctx, n), path(ctx, (size_t)n + 1), res(ctx, 2);
  pos.fill_bytes(0xff);
  DP_LAUNCH(ctx, k_witness, 1, 1, 0, indeg, g.id.p, g.out_off.p, g.out_dst.p, n, start, pos.p, path.p, res.p);
  int32_t r[2];
  res.download(r, 2);
  sync(ctx);
  std::vector<int32_t> idx = to_host(ctx, path.p + r[0], static_cast<size_t>(r[1] - r[0]));
  std::vector<int64_t> ids = to_host(ctx, g.id.p, n);
  std::vector<int64_t> out;
  for (int32_t v : idx) out.push_back(ids[v]);
  return out;
}

void graph_validate_begin(DevGraph& g, ValState& vs) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  int32_t n = g.n, m = g.m;
  DevBuf<int32_t>& dupcount = vs.dupcount;
  if (!g.dense_ids && n > 0) {
    dupcount.alloc(ctx, n);
    dupcount.zero();
    DP_LAUNCH(ctx, k_dup_runs, grid_for(n, B), B, 0, g.sorted_key.p, g.sorted_idx.p, n, dupcount.p);
  }
  if (!g.has_adj) graph_adjacency(g);
  DevBuf<uint8_t>& nflags = vs.nflags;
  DevBuf<uint8_t>& eflags = vs.eflags;
  DevBuf<uint8_t>& dupflag = vs.dupflag;
  DevBuf<int>& first = vs.first;
  nflags.alloc(ctx, n > 0 ? n : 1);
  eflags.alloc(ctx, m > 0 ? m : 1);
  dupflag.alloc(ctx, m > 0 ? m : 1);
  dupflag.zero();
  first.alloc(ctx, 3);
  const int init[3] = {INT32_MAX, INT32_MAX, 0};
  first.upload(init, 3);
  DP_LAUNCH(ctx, k_dup_edges, grid_for(n, B), B, 0, g.out_off.p, g.out_eid.p, g.out_dst.p, n, dupflag.p,
            first.p + 2);
  if (g.big_rows) {  // rows longer than 64 (known from graph_adjacency): sort-based pass
    DevBuf<uint64_t> k(ctx, m), ko(ctx, m);
    DevBuf<int32_t> v(ctx, m), vo(ctx, m);
    DP_LAUNCH(ctx, k_pair_keys, grid_for(m, B), B, 0, g.esrc.p, g.edst.p, m, k.p, v.p);
    sort_pairs_u64(ctx, k.p, ko.p, v.p, vo.p, m, 0, 64);
    DP_LAUNCH(ctx, k_pair_dups, grid_for(m, B), B, 0, ko.p, vo.p, m, dupflag.p);
  }
  DP_LAUNCH(ctx, k_node_flags, grid_for(n, B), B, 0, g.w.p, g.mem.p, dupcount.p, n, nflags.p, first.p);
  DP_LAUNCH(ctx, k_edge_flags, grid_for(m, B), B, 0, g.src_id.p, g.dst_id.p, g.bytes.p, g.esrc.p, g.edst.p,
            dupflag.p, m, eflags.p, first.p + 1);
  first.download(vs.fh, 2);  // read after the caller's sync
}

Validation graph_validate(DevGraph& g, const dp_graph_t* h, bool all, bool cycle_check) {
  ValState vs;
  graph_validate_begin(g, vs);
  sync(g.ctx);
  return graph_validate_end(g, h, vs, all, cycle_check);
}

Validation graph_validate_end(DevGraph& g, const dp_graph_t* h, ValState& vs, bool all, bool cycle_check) {
  dp_ctx* ctx = g.ctx;
  int32_t n = g.n, m = g.m;
  Validation out;
  const int* fh = vs.fh;
  DevBuf<int32_t>& dupcount = vs.dupcount;
  DevBuf<uint8_t>& nflags = vs.nflags;
  DevBuf<uint8_t>& eflags = vs.eflags;
  auto add = [&](int code, std::string msg, std::vector<int64_t> nodes) {
    if (!out.code) {
      out.code = code;
      out.message = msg;
      out.nodes = nodes;
    }
    if (all) {
      out.kinds.push_back(code);
      out.messages.push_back(std::move(msg));
      out.witnesses.push_back(std::move(nodes));
    }
  };
  auto S = [](int64_t v) { return std::to_string(v); };
  std::vector<uint8_t> nf, ef;
  std::vector<int32_t> dc;
  bool any_dup = false, edges_resolvable = true;
  if (all || fh[0] != INT32_MAX || fh[1] != INT32_MAX) {
    nf = to_host(ctx, nflags.p, n);
    ef = to_host(ctx, eflags.p, m);
    if (dupcount.p) dc = to_host(ctx, dupcount.p, n);
  }
  int32_t nb = all ? 0 : (fh[0] == INT32_MAX ? n : fh[0]);
  for (int32_t i = nb; i < n; ++i) {
    uint8_t f = nf[i];
    if (!f) continue;
    int64_t id = h->node_id[i];
    if (f & 1) {
      any_dup = true;
      add(DP_E_DUPLICATE_ID, "node id " + S(id) + " appears " + S(dc[i]) + " times", {id});
    }
    if (f & 2) add(DP_E_INVALID_VALUE, "node " + S(id) + " has negative compute_us", {id});
    if (f & 4) add(DP_E_INVALID_VALUE, "node " + S(id) + " has negative memory_bytes", {id});
    if (!all) break;
  }
  if (!all && out.code) return out;
  int32_t eb = all ? 0 : (fh[1] == INT32_MAX ? m : fh[1]);
  for (int32_t e = eb; e < m; ++e) {
    uint8_t f = ef[e];
    if (!f) continue;
    int64_t s = h->edge_src[e], d = h->edge_dst[e];
    std::string pair = "(" + S(s) + "," + S(d) + ")";
    if (f & 1) add(DP_E_DANGLING_EDGE, "edge " + pair + " references missing node " + S(s), {s, d});
    if (f & 2) add(DP_E_DANGLING_EDGE, "edge " + pair + " references missing node " + S(d), {s, d});
    if (f & 4) add(DP_E_CYCLE_DETECTED, "self-loop on node " + S(s), {s});
    if (f & 8) add(DP_E_INVALID_VALUE, "edge " + pair + " has negative tensor_bytes", {s, d});
    if (f & 16)
      add(DP_E_DUPLICATE_EDGE, "parallel edge " + pair + "; aggregate tensor bytes upstream", {s, d});
    if (f & 7) edges_resolvable = false;
    if (!all) break;
  }
  if (!all && out.code) return out;
  if (cycle_check && edges_resolvable && !any_dup && n > 0) {
    graph_kahn(g, nullptr, nullptr, nullptr);
    if (g.processed != n) {
      std::vector<int64_t> wit = graph_cycle_witness(g);
      add(DP_E_CYCLE_DETECTED, "cycle: [" + join_ids(wit) + "]", wit);
    }
  }
  return out;
}

}  // namespace dpb
