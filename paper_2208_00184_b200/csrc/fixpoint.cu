// fixpoint.cu — the stack peel (ordering.cpp:40-77: cpd_topo :98-114, dfs_topo :88-96) as a
// level-parallel tree construction plus a parallel proof, instead of a one-warp chain.
//
// Characterisation: for a topological order s let T(s) be the forest in
// which parent(v) is v's predecessor emitted last in s; children, and the roots (the
// sources), are visited by rank (cpath desc, id asc for CPD; id asc for DFS).  The peel's
// order is the unique topological s with s = preorder(T(s)): the peel pops a node, then
// the best child it freed (a node is freed by its last predecessor), and when a subtree is
// exhausted it resumes with the stack top, which is the next unvisited child of the nearest
// ancestor.  Any topological s with T(preorder(T(s))) = T(s) is therefore the peel order.
//
// The start that makes this cheap: s0 = the Kahn order built level by level where level
// l+1 lists the nodes freed by level l grouped by their last-processed predecessor (in s0
// order) and, within a group, by rank.  Then T0 = T(s0) is exactly that freeing forest, a
// node's T0-parent lies on the level just above it, so the depth of a node in T0 is its hop
// level, and within one depth the preorder of T0 lists nodes in the same order as the
// breadth-first order s0 does.  When every edge joins consecutive levels (layered DAGs,
// config #4 deep and wide) T(preorder(T0)) = T0 follows, i.e. one tree construction is the
// answer; the proof runs anyway and is cheap.  Otherwise the iteration s <- preorder(T(s))
// continues from there (it converges: agreement with the peel on a prefix of length P
// implies agreement on P + 1 after one more step), under a round budget; past it the
// one-warp peel runs (PeelArgs.skip stays 0).
//
// One CTA per graph, __syncthreads between levels (no grid barrier, no cooperative launch,
// one SM per graph like the one-warp peel):
//   1  Kahn by levels: A relaxes level l (atomicMax of the parent position, in-degree
//      decrement), B numbers level l+1 from level l's rows in rank order (block scan)
//   2  subtree sizes of T0, deepest level first
//   3  preorder positions, shallowest level first (roots by a block scan)
//   4  proof: for every node the predecessor with the largest preorder position is its T0
//      parent; writes seq / pos_of
// Algorithmic bytes per node and edge: 1 reads the rows twice and relaxes each edge once,
// 2 and 3 read the rows once more, 4 reads the CSC once (fixpoint_launch).
#include <algorithm>

#include <cooperative_groups.h>

#include "fixpoint.cuh"
#include "graph.cuh"

namespace dpb {
namespace {
namespace cg = cooperative_groups;

// CTAs per cluster of a single graph's tree peel.  A cluster pays three cluster barriers per
// level, so it only helps wide levels: measured (profiles/r2cc_*) the Kahn phase at config #4
// wide (16 levels of 65,536) 16.5 ms on one CTA -> 2.6 ms on 8 -> 1.4 ms on 16; at deep (977
// levels of 1,024) 15.8 -> 20.1 / 20.7 ms.  Wide = mean edge span (index order) of at least
// kTreeWideSpan nodes.  DP_TREE_CLUSTER = 1 / 4 / 8 / 16 forces the size for every graph.
constexpr double kTreeWideSpan = 8192.0;
int tree_cluster(bool wide) {
  const char* e = getenv("DP_TREE_CLUSTER");
  if (!e) return wide ? 16 : 1;
  const int v = atoi(e);
  return v == 4 || v == 8 || v == 16 ? v : 1;
}

// One graph alone: 1,024 threads (a level of the deep config is one node per thread).  Several
// graphs per call: 512 threads per CTA, which leaves room on the SM for other graphs'
// kernels (throughput mode).
template <int T>
struct TreeCfg {
  static constexpr int kThreads = T, kWarps = T / 32;
};

struct TreeBatch {
  TreeArgs a[kTreeBatch];
};

__device__ __forceinline__ int32_t ldcg(const int32_t* p) { return __ldcg(p); }
// child c is freed by this level and its T0 parent is position i
__device__ __forceinline__ bool claimed(const int2* p, int32_t i) {
  const int2 x = __ldcg(p);
  return x.x == i && x.y == 0;
}

// Exclusive block scan over TT::kThreads threads; *total = sum.  All threads call.
template <typename TT>
__device__ __forceinline__ int32_t block_scan(int32_t x, int32_t* total, int32_t* ws) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int32_t s = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += y;
  }
  if (lane == 31) ws[warp] = s;
  __syncthreads();
  if (warp == 0) {
    int32_t t = lane < TT::kWarps ? ws[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    ws[lane] = t;
  }
  __syncthreads();
  const int32_t r = (warp ? ws[warp - 1] : 0) + s - x;
  *total = ws[TT::kWarps - 1];
  __syncthreads();
  return r;
}

// pre[roots in s0 level 0 order] = exclusive scan of their subtree sizes
template <typename TT>
__device__ void roots_scan(const TreeArgs& a, int32_t nsrc, const int32_t* size, int32_t* pre, int32_t* ws) {
  int32_t carry = 0;
  for (int32_t i0 = 0; i0 < nsrc; i0 += TT::kThreads) {
    const int32_t i = i0 + threadIdx.x;
    const int32_t v = i < nsrc ? a.seq0[i] : -1;
    const int32_t s = v >= 0 ? size[v] : 0;
    int32_t tot;
    const int32_t ex = block_scan<TT>(s, &tot, ws);
    if (v >= 0) pre[v] = carry + ex;
    carry += tot;
  }
}

// CL > 1 (one graph alone): phase 1 runs on a thread-block cluster of CL CTAs (CL SMs'
// load/store and atomic throughput: phase 1 is ~2 global atomics + 2 L2 loads per edge,
// which one SM issues at ~1 per cycle) with cluster barriers between its steps; the
// per-CTA totals of the next-level numbering meet in CTA 0's shared memory (DSMEM).
// Phases 2-4 stay on CTA 0 (rank != 0 exits after phase 1).  Values written by other CTAs
// are read through L2 (ld.cg); the cluster barrier orders them (release / acquire).
// Fixed-point rounds after a failed proof (any_bad), then the emission of seq / pos_of and
// the verdict; one CTA.  Called at the end of k_treepeel, or by its continuation launch
// (mode 1) when the proof ran as a grid kernel and failed.
template <typename TT, typename Phase>
__device__ void tree_finish(const TreeArgs& a, int32_t L, int32_t nsrc, bool any_bad, int32_t* ws, Phase&& phase) {
  const int tid = threadIdx.x;
  const int32_t n = a.n;
  int32_t* pos = a.pre;
  int rounds = 1;
  if (any_bad) {
    // general rounds s <- preorder(T(s)) on the same levels (a T(s) parent is a
    // predecessor, so it sits on a shallower level)
    int32_t budget = a.max_rounds;
    if (budget < 0) budget = max(0, (n / 8) / (6 * L + 8));
    int32_t* nxt = a.pre2;
    bool done = false;
    for (int r = 0; r < budget && !done; ++r) {
      ++rounds;
      for (int32_t v = tid; v < n; v += TT::kThreads) {
        int32_t bp = -1, bu = -1;
        for (int32_t k = a.in_off[v]; k < a.in_off[v + 1]; ++k) {
          const int32_t u = a.in_src[k];
          const int32_t q = pos[u];
          if (q > bp) {
            bp = q;
            bu = u;
          }
        }
        a.par[v] = bu;
      }
      __syncthreads();
      for (int32_t l = L - 1; l >= 0; --l) {
        const int32_t b = a.lvl_off[l], e = a.lvl_off[l + 1];
        for (int32_t i = b + tid; i < e; i += TT::kThreads) {
          const int32_t v = a.seq0[i];
          int32_t s = 1;
          for (int32_t k = a.out_off[v]; k < a.out_off[v + 1]; ++k) {
            const int32_t c = a.rowc[k];
            if (a.par[c] == v) s += a.size[c];
          }
          a.size[v] = s;
        }
        __syncthreads();
      }
      roots_scan<TT>(a, nsrc, a.size, nxt, ws);
      __syncthreads();
      for (int32_t l = 0; l + 1 < L; ++l) {
        const int32_t b = a.lvl_off[l], e = a.lvl_off[l + 1];
        for (int32_t i = b + tid; i < e; i += TT::kThreads) {
          const int32_t v = a.seq0[i];
          int32_t acc = nxt[v] + 1;
          for (int32_t k = a.out_off[v]; k < a.out_off[v + 1]; ++k) {
            const int32_t c = a.rowc[k];
            if (a.par[c] == v) {
              nxt[c] = acc;
              acc += a.size[c];
            }
          }
        }
        __syncthreads();
      }
      bool chg = false;
      for (int32_t v = tid; v < n; v += TT::kThreads) chg |= nxt[v] != pos[v];
      done = !__syncthreads_or(chg);
      int32_t* t = pos;
      pos = nxt;
      nxt = t;
    }
    if (!done) {
      if (tid == 0) {
        a.info[0] = 4;
        a.info[1] = L;
        a.info[2] = rounds;
      }
      return;
    }
  }
  for (int32_t v = tid; v < n; v += TT::kThreads) {
    const int32_t p = pos[v];
    a.seq[p] = v;
    a.pos_of[v] = p;
  }
  __syncthreads();
  phase(3);
  if (tid == 0) {
    __threadfence();
    a.info[0] = 1;
    a.info[1] = L;
    a.info[2] = rounds;
    *a.skip = 1;
    *a.emitted = n;
    *a.progress = n;
  }
}

template <typename TT, int CL>
__global__ void __launch_bounds__(TT::kThreads, 1024 / TT::kThreads) k_treepeel(const __grid_constant__ TreeBatch batch,
                                                                                      int mode) {
  const TreeArgs& a = batch.a[blockIdx.x / CL];
  __shared__ int32_t ws[32];
  __shared__ int32_t ctot[2][CL];  // cluster: per-CTA totals of one numbering step (CTA 0's copy)
  __shared__ int32_t cloc[CL];
  const int tid = threadIdx.x;
  if (mode == 1) {  // continuation after the grid proof / emission (one CTA per graph)
    if (a.info[0] != 5) return;
    if (a.info[7] == 0) {  // proof held: the emission kernel wrote seq / pos_of
      if (tid == 0) {
        a.info[0] = 1;
        a.info[2] = 1;
        *a.skip = 1;
        *a.emitted = a.n;
        *a.progress = a.n;
      }
      return;
    }
    auto nophase = [](int) {};
    tree_finish<TT>(a, a.info[1], *a.nsrc, true, ws, nophase);
    return;
  }
  int rank = 0;
  if constexpr (CL > 1) rank = static_cast<int>(cg::this_cluster().block_rank());
  constexpr int32_t SPAN = CL * TT::kThreads;
  auto csync = [&]() {
    if constexpr (CL > 1) cg::this_cluster().sync();
    else __syncthreads();
  };
  const int32_t n = a.n;
  const int32_t nsrc = *a.nsrc;
  for (int32_t v = rank * TT::kThreads + tid; v < n; v += SPAN) {
    a.bi[v] = make_int2(-1, a.in_off[v + 1] - a.in_off[v]);
  }
  for (int32_t i = rank * TT::kThreads + tid; i < nsrc; i += SPAN) a.seq0[i] = a.roots[i];
  if (tid == 0 && rank == 0) {
    a.lvl_off[0] = 0;
    a.info[7] = 0;
  }
  csync();
  // ---- 1: breadth-first order s0 and the freeing forest T0
  long long clk = clock64();  // phase clocks (DP_DEBUG_FIXPOINT): info[3..6], in 1,024 cycles
  auto phase = [&](int i) {
    if (tid == 0) {
      const long long c = clock64();
      a.info[3 + i] = static_cast<int>((c - clk) >> 10);
      clk = c;
    }
  };
  int32_t lb = 0, le = nsrc, L = 0;
  while (lb < le) {
    if (tid == 0 && rank == 0) a.lvl_off[L + 1] = le;
    if (L >= a.max_levels) {
      if (tid == 0 && rank == 0) a.info[0] = 2;
      return;
    }
    // a level that fits one sweep of the CTA(s) keeps each thread's row (node, bounds, up to
    // 8 children) in registers from the relaxation to the numbering step
    const bool one = le - lb <= SPAN;
    int32_t rkb = 0, rke = 0;
    int32_t cc[8];
    for (int32_t i = lb + rank * TT::kThreads + tid; i < le; i += SPAN) {
      const int32_t v = ldcg(a.seq0 + i);
      const int32_t kb = a.out_off[v], ke = a.out_off[v + 1];
      if (ke - kb <= 8) {  // the row's loads first, then its atomics (no load between them)
#pragma unroll
        for (int q = 0; q < 8; ++q) cc[q] = kb + q < ke ? a.rowc[kb + q] : 0;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (kb + q < ke) {
            atomicMax(&a.bi[cc[q]].x, i);
            atomicSub(&a.bi[cc[q]].y, 1);
          }
      } else {
        for (int32_t k = kb; k < ke; ++k) {
          const int32_t c = a.rowc[k];
          atomicMax(&a.bi[c].x, i);
          atomicSub(&a.bi[c].y, 1);
        }
      }
      rkb = kb;
      rke = ke;
    }
    csync();
    int32_t carry = 0, par = 0;
    for (int32_t i0 = lb; i0 < le; i0 += SPAN) {
      const int32_t i = i0 + rank * TT::kThreads + tid;
      int32_t kb = 0, ke = 0, cnt = 0;
      // (the T0 children of position i will be positions [cs[i], cs[i + 1]) of s0)
      unsigned hit = 0;
      if (i < le) {
        if (one) {
          kb = rkb;
          ke = rke;
        } else {
          const int32_t v = ldcg(a.seq0 + i);
          kb = a.out_off[v];
          ke = a.out_off[v + 1];
        }
        if (ke - kb <= 8) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            if (!one) cc[q] = kb + q < ke ? a.rowc[kb + q] : 0;
            if (kb + q < ke && claimed(a.bi + cc[q], i)) hit |= 1u << q;
          }
          cnt = __popc(hit);
        } else {
          for (int32_t k = kb; k < ke; ++k) {
            const int32_t c = a.rowc[k];
            cnt += claimed(a.bi + c, i) ? 1 : 0;
          }
        }
      }
      int32_t tot;
      const int32_t ex = block_scan<TT>(cnt, &tot, ws);
      int32_t before = 0, all = tot;  // numbering of the CTAs of lower rank; of the whole step
      if constexpr (CL > 1) {
        int32_t* slot0 = cg::this_cluster().map_shared_rank(&ctot[par][0], 0);
        if (tid == 0) slot0[rank] = tot;
        cg::this_cluster().sync();
        if (tid < CL) cloc[tid] = slot0[tid];
        __syncthreads();
        all = 0;
#pragma unroll
        for (int r = 0; r < CL; ++r) {
          before += r < rank ? cloc[r] : 0;
          all += cloc[r];
        }
        __syncthreads();  // cloc is rewritten by the next step
        par ^= 1;
      }
      if (i < le) a.cs[i] = le + carry + before + ex;
      if (cnt) {
        int32_t o = le + carry + before + ex;
        if (ke - kb <= 8) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (hit >> q & 1u) a.seq0[o++] = cc[q];
        } else {
          for (int32_t k = kb; k < ke; ++k) {
            const int32_t c = a.rowc[k];
            if (claimed(a.bi + c, i)) a.seq0[o++] = c;
          }
        }
      }
      carry += all;
    }
    csync();
    lb = le;
    le += carry;
    ++L;
  }
  if (le != n) {  // not a DAG: the one-warp peel reports it
    if (tid == 0 && rank == 0) a.info[0] = 3;
    return;
  }
  if (rank != 0) return;  // phases 2-4 on CTA 0
  if (tid == 0) a.cs[n] = n;
  __syncthreads();
  phase(0);
  // ---- 2: subtree sizes of T0, by s0 position: position i's children are the contiguous
  // positions [cs[i], cs[i + 1]) of the next level (phase 1 numbered them so)
  int32_t* psize = a.psize;
  int32_t* ppre = a.ppre;
  for (int32_t l = L - 1; l >= 0; --l) {
    const int32_t b = a.lvl_off[l], e = a.lvl_off[l + 1];
    for (int32_t i = b + tid; i < e; i += TT::kThreads) {
      int32_t s = 1;
      for (int32_t q = a.cs[i]; q < a.cs[i + 1]; ++q) s += psize[q];
      psize[i] = s;
    }
    __syncthreads();
  }
  // ---- 3: preorder positions of T0 (roots: level 0 in rank order)
  {
    int32_t carry = 0;
    for (int32_t i0 = 0; i0 < nsrc; i0 += TT::kThreads) {
      const int32_t i = i0 + tid;
      const int32_t sz = i < nsrc ? psize[i] : 0;
      int32_t tot;
      const int32_t ex = block_scan<TT>(sz, &tot, ws);
      if (i < nsrc) ppre[i] = carry + ex;
      carry += tot;
    }
  }
  __syncthreads();
  for (int32_t l = 0; l + 1 < L; ++l) {
    const int32_t b = a.lvl_off[l], e = a.lvl_off[l + 1];
    for (int32_t i = b + tid; i < e; i += TT::kThreads) {
      int32_t acc = ppre[i] + 1;
      for (int32_t q = a.cs[i]; q < a.cs[i + 1]; ++q) {
        ppre[q] = acc;
        acc += psize[q];
      }
    }
    __syncthreads();
  }
  for (int32_t i = tid; i < n; i += TT::kThreads) a.pre[a.seq0[i]] = ppre[i];
  __syncthreads();
  phase(1);
  if (a.split && mode == 0) {  // proof and emission by the grid kernels below
    if (tid == 0 && rank == 0) {
      a.info[0] = 5;
      a.info[1] = L;
    }
    return;
  }
  // ---- 4: proof T(preorder(T0)) = T0
  bool bad = false;
  for (int32_t v = tid; v < n; v += TT::kThreads) {
    const int32_t b = a.in_off[v], e = a.in_off[v + 1];
    if (b == e) continue;
    int32_t mx = -1;
    for (int32_t k = b; k < e; ++k) mx = max(mx, a.pre[a.in_src[k]]);
    bad |= mx != ppre[__ldcg(&a.bi[v].x)];
  }
  const bool any_bad = __syncthreads_or(bad);
  phase(2);
  tree_finish<TT>(a, L, nsrc, any_bad, ws, phase);
}

// Split proof (TreeArgs.split): every node's predecessor with the largest preorder position
// must be its T0 parent -- a flat pass over the CSC, on the whole GPU instead of one CTA;
// blockIdx.y = graph.  Then the emission seq[pre[v]] = v when no node failed.
__global__ void k_tree_proof(const __grid_constant__ TreeBatch batch) {
  const TreeArgs& a = batch.a[blockIdx.y];
  if (a.info[0] != 5) return;
  bool bad = false;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < a.n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = a.in_off[v], e = a.in_off[v + 1];
    if (b == e) continue;
    int32_t mx = -1;
    for (int32_t k = b; k < e; ++k) mx = max(mx, __ldcg(a.pre + a.in_src[k]));
    bad |= mx != __ldcg(a.ppre + __ldcg(&a.bi[v].x));
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(a.info + 7, 1);
}
__global__ void k_tree_emit(const __grid_constant__ TreeBatch batch) {
  const TreeArgs& a = batch.a[blockIdx.y];
  if (a.info[0] != 5 || __ldcg(a.info + 7) != 0) return;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < a.n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = __ldcg(a.pre + v);
    a.seq[p] = static_cast<int32_t>(v);
    a.pos_of[v] = p;
  }
}

// Rows of at most 64 children sorted by rank, one thread per row (insertion sort in place).
__global__ void k_rows_by_rank(const int32_t* out_off, const int32_t* out_dst, const int32_t* rank, int32_t n,
                               int32_t* rowc, int* long_rows) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = out_off[v], d = out_off[v + 1] - b;
    if (d > 64) {
      atomicExch(long_rows, 1);
      continue;
    }
    for (int32_t q = 0; q < d; ++q) {
      const int32_t c = out_dst[b + q];
      const int32_t rc = rank[c];
      int32_t j = q;
      while (j > 0 && rank[rowc[b + j - 1]] > rc) {
        rowc[b + j] = rowc[b + j - 1];
        --j;
      }
      rowc[b + j] = c;
    }
  }
}

__global__ void k_row_rank_keys(const int32_t* out_off, const int32_t* out_dst, const int32_t* rank, int32_t n,
                                uint64_t* keys, int32_t* vals) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    for (int32_t k = out_off[v]; k < out_off[v + 1]; ++k) {
      keys[k] = (static_cast<uint64_t>(v) << 32) | static_cast<uint32_t>(rank[out_dst[k]]);
      vals[k] = out_dst[k];
    }
}

__global__ void k_roots(const int32_t* by_rank, const int32_t* flag, const int32_t* fpos, int32_t n, int32_t* roots) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    if (flag[r]) roots[fpos[r]] = by_rank[r];
}

}  // namespace

bool fixpoint_wanted(const DevGraph& g) {
  if (getenv("DP_PEEL_NO_FIXPOINT")) return false;
  return g.n >= (getenv("DP_PEEL_FIXPOINT") ? 1 : 2048) && g.m_ok > 0;
}

std::unique_ptr<TreeJob> fixpoint_prepare(DevGraph& g, const int32_t* by_rank, const int32_t* rank,
                                          const int32_t* flag, const int32_t* fpos, int32_t* seq, int32_t* pos_of,
                                          int* skip, int* progress, int* emitted) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  const int32_t n = g.n, m = g.m_ok;
  std::unique_ptr<TreeJob> j(new TreeJob);
  j->ctx = ctx;
  j->wide = g.topo_known && m > 0 && static_cast<double>(g.span_sum) / m >= kTreeWideSpan;
  j->rowc.alloc(ctx, m > 0 ? m : 1);
  DevBuf<int> flags(ctx, 1);
  flags.zero();
  DP_LAUNCH(ctx, k_rows_by_rank, grid_for(n, B), B, 0, g.out_off.p, g.out_dst.p, rank, n, j->rowc.p, flags.p);
  if (g.big_rows && scalar_to_host(ctx, flags.p)) {  // some row > 64: one global sort of (row, rank)
    DevBuf<uint64_t> keys(ctx, m), keys_out(ctx, m);
    DevBuf<int32_t> vals(ctx, m);
    DP_LAUNCH(ctx, k_row_rank_keys, grid_for(n, B), B, 0, g.out_off.p, g.out_dst.p, rank, n, keys.p, vals.p);
    int bits = 1;
    while ((1ll << bits) < n) ++bits;
    sort_pairs_u64(ctx, keys.p, keys_out.p, vals.p, j->rowc.p, m, 0, 32 + bits);
  }
  j->roots.alloc(ctx, n);
  DP_LAUNCH(ctx, k_roots, grid_for(n, B), B, 0, by_rank, flag, fpos, n, j->roots.p);
  j->seq0.alloc(ctx, n);
  j->bi.alloc(ctx, n);
  j->size.alloc(ctx, n);
  j->pre.alloc(ctx, n);
  j->pre2.alloc(ctx, n);
  j->par.alloc(ctx, n);
  j->lvl_off.alloc(ctx, (size_t)n + 1);
  j->cs.alloc(ctx, (size_t)n + 1);
  j->psize.alloc(ctx, n);
  j->ppre.alloc(ctx, n);
  j->info.alloc(ctx, 8);
  j->info.zero();
  TreeArgs& a = j->a;
  a.split = getenv("DP_TREE_FUSED_PROOF") ? 0 : 1;
  a.n = n;
  a.nsrc = fpos + n;
  a.in_off = g.in_off.p;
  a.in_src = g.in_src.p;
  a.out_off = g.out_off.p;
  a.rowc = j->rowc.p;
  a.roots = j->roots.p;
  a.seq0 = j->seq0.p;
  a.bi = j->bi.p;
  a.size = j->size.p;
  a.pre = j->pre.p;
  a.pre2 = j->pre2.p;
  a.par = j->par.p;
  a.lvl_off = j->lvl_off.p;
  a.cs = j->cs.p;
  a.psize = j->psize.p;
  a.ppre = j->ppre.p;
  // ~8 us per level (all phases) against ~0.4 us per node for the one-warp peel
  a.max_levels = getenv("DP_PEEL_FIXPOINT") ? n + 1 : std::max(64, n / 40);
  a.max_rounds = getenv("DP_PEEL_FIXPOINT") ? 4096 : -1;
  if (const char* e = getenv("DP_FIXPOINT_ROUNDS")) a.max_rounds = std::max(0, atoi(e));
  a.seq = seq;
  a.pos_of = pos_of;
  a.skip = skip;
  a.progress = progress;
  a.emitted = emitted;
  a.info = j->info.p;
  j->bytes = 40.0 * n + 20.0 * m;
  return j;
}

void fixpoint_launch_batch(dp_ctx* ctx, TreeJob* const* jobs, int count) {
  for (int b0 = 0; b0 < count; b0 += kTreeBatch) {
    const int k = std::min(kTreeBatch, count - b0);
    TreeBatch b{};
    double bytes = 0.0;
    for (int q = 0; q < k; ++q) {
      b.a[q] = jobs[b0 + q]->a;
      bytes += jobs[b0 + q]->bytes;
    }
    StageScope s(ctx, "peel (tree)", bytes);
    if (count == 1 && tree_cluster(jobs[b0]->wide) > 1) {
      const int cl = tree_cluster(jobs[b0]->wide);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(static_cast<unsigned>(k * cl));
      cfg.blockDim = dim3(1024);
      cfg.stream = ctx->stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = static_cast<unsigned>(cl);
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      if (cl == 16) {
        static bool np = false;
        if (!np) {
          DP_CUDA(cudaFuncSetAttribute(k_treepeel<TreeCfg<1024>, 16>,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
          np = true;
        }
        DP_CUDA(cudaLaunchKernelEx(&cfg, k_treepeel<TreeCfg<1024>, 16>, b, 0));
      } else if (cl == 4) {
        DP_CUDA(cudaLaunchKernelEx(&cfg, k_treepeel<TreeCfg<1024>, 4>, b, 0));
      } else {
        DP_CUDA(cudaLaunchKernelEx(&cfg, k_treepeel<TreeCfg<1024>, 8>, b, 0));
      }
      ++ctx->launches;
    } else if (count == 1) {
      k_treepeel<TreeCfg<1024>, 1><<<k, 1024, 0, ctx->stream>>>(b, 0);
      ++ctx->launches;
      DP_CUDA(cudaGetLastError());
    } else {
      k_treepeel<TreeCfg<512>, 1><<<k, 512, 0, ctx->stream>>>(b, 0);
      ++ctx->launches;
      DP_CUDA(cudaGetLastError());
    }
    if (b.a[0].split) {  // grid proof, grid emission, then the one-CTA continuation
      int32_t maxn = 1;
      for (int q = 0; q < k; ++q) maxn = std::max(maxn, b.a[q].n);
      const dim3 grid(static_cast<unsigned>(grid_for(maxn, 256)), static_cast<unsigned>(k));
      k_tree_proof<<<grid, 256, 0, ctx->stream>>>(b);
      k_tree_emit<<<grid, 256, 0, ctx->stream>>>(b);
      if (count == 1) k_treepeel<TreeCfg<1024>, 1><<<k, 1024, 0, ctx->stream>>>(b, 1);
      else k_treepeel<TreeCfg<512>, 1><<<k, 512, 0, ctx->stream>>>(b, 1);
      ctx->launches += 3;
      DP_CUDA(cudaGetLastError());
    }
  }
  if (getenv("DP_DEBUG_FIXPOINT")) {
    std::vector<int> h(8 * (size_t)count);
    for (int q = 0; q < count; ++q) jobs[q]->info.download(h.data() + 8 * q, 8);
    sync(ctx);
    for (int q = 0; q < count; ++q) {
      const int* x = h.data() + 8 * q;
      fprintf(stderr,
              "[treepeel] n=%d status=%d levels=%d rounds=%d; ms: kahn %.2f, sizes+preorder %.2f, proof %.2f, "
              "rounds+emit %.2f (at 1.965 GHz)\n",
              jobs[q]->a.n, x[0], x[1], x[2], x[3] * 1024 / 1.965e6, x[4] * 1024 / 1.965e6, x[5] * 1024 / 1.965e6,
              x[6] * 1024 / 1.965e6);
      const int slot = x[0] == 1 ? (x[2] == 1 ? 0 : 1) : x[0];
      if (slot >= 0 && slot < 5) ++ctx->tree_stats[slot];
    }
  }
}

}  // namespace dpb
