// fusion.cu — coarsening on the GPU, bit-exact with fusion.cpp (/root/reference/proj/src):
//   optimal_breakpoints  :85-171  windowed min-plus DP over the CPD-TOPO sequence
//   clusters_from_cuts   :61-81   cut traceback -> contiguous clusters
//   build_coarse_graph   :173-229 crossing edges aggregated in (cu, cv) order
//   contract_colocation_groups :231-295, fuse :297-335
//
// The DP recurrence is sequential in the cut position j.  With D_j(i) = best[i] + C(i,j)
// (C = transfer time of edges leaving window [i,j) to positions >= j) the reference's
// incremental forward[] update becomes, per step,
//   D_{j+1}(i) = D_j(i) + out(j) - sum{c(a->j) : a >= i}      and     D_{j+1}(j) = best[j] + out(j)
// so one warp keeps the whole window (R <= 256 candidates) in registers — 8 slots per
// lane, slot = i mod 256 — and per step does the in-edge updates, an (value, -i)
// argmin (strict '<' scanning i downward == ties go to the largest i) and one insert.
#include <algorithm>

#include "fusion.cuh"
#include "peel.cuh"
#include "peel_dp.cuh"
#include "results.h"

namespace dpb {

void levels_dev(DevGraph& g, dp_comm_t comm, DevBuf<int64_t>& t, DevBuf<int64_t>& b, DevBuf<int64_t>& c,
                bool chainlike);
void levels_dev_batch(DevGraph* const* gs, int count, dp_comm_t comm, DevBuf<int64_t>* const* t,
                      DevBuf<int64_t>* const* b, DevBuf<int64_t>* const* c);

namespace {

constexpr int64_t kInf = INT64_MAX;

__global__ void k_dp_prep(const int32_t* seq, int32_t n, const int64_t* mem, const int32_t* out_off,
                          const int64_t* out_cost, const int32_t* in_off, int64_t limit, int64_t* mem_pos,
                          int64_t* out_sum, int32_t* in_cnt, int* first_exceed) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = seq[p];
    int64_t mv = mem[v];
    mem_pos[p] = mv;
    if (mv > limit) atomicMin(first_exceed, static_cast<int>(p));
    int64_t s = 0;
    for (int32_t k = out_off[v]; k < out_off[v + 1]; ++k) s += out_cost[k];
    out_sum[p] = s;
    in_cnt[p] = in_off[v + 1] - in_off[v];
  }
}

__global__ void k_in_fill(const int32_t* seq, const int32_t* pos_of, int32_t n, const int32_t* in_off,
                          const int32_t* in_src, const int64_t* in_cost, const int32_t* in_off_pos,
                          int32_t* in_pos, int64_t* in_c) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = seq[p];
    int32_t o = in_off_pos[p];
    for (int32_t k = in_off[v]; k < in_off[v + 1]; ++k, ++o) {
      in_pos[o] = pos_of[in_src[k]];
      in_c[o] = in_cost[k];
    }
  }
}

// lo[j] = max(j - R, smallest i with prefix[j] - prefix[i] <= limit)  (fusion.cpp:145-148)
__global__ void k_lo(const int64_t* prefix, int32_t n, int32_t range, int64_t limit, int32_t* lo) {
  for (int64_t j = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= n; j += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = static_cast<int32_t>(j > range ? j - range : 0), b = static_cast<int32_t>(j - 1);
    int64_t pj = prefix[j];
    while (a < b) {  // first i in [a, b] with pj - prefix[i] <= limit (monotone)
      int32_t mid = (a + b) >> 1;
      if (pj - prefix[mid] <= limit) b = mid; else a = mid + 1;
    }
    lo[j] = a;
  }
}

__device__ __forceinline__ void argmin_reduce(int64_t& v, int32_t& d) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    int64_t ov = __shfl_xor_sync(0xffffffffu, v, o);
    int32_t od = __shfl_xor_sync(0xffffffffu, d, o);
    if (ov < v || (ov == v && od < d)) {
      v = ov;
      d = od;
    }
  }
}

constexpr int kChunk = 256;   // steps staged per smem refill
constexpr int kInCap = 2048;  // in-edges staged per refill

// Register-window DP, R <= 32*SPL.  One warp.  prev_cut[j] for j = 1..n.
template <int SPL>
__global__ void __launch_bounds__(32) k_dp_window(int32_t n, const int32_t* lo, const int64_t* out_sum,
                                                  const int32_t* in_off, const int32_t* in_pos,
                                                  const int64_t* in_c, int32_t* prev_cut) {
  constexpr int W = 32 * SPL;
  __shared__ int32_t s_lo[kChunk + 1];
  __shared__ int64_t s_out[kChunk + 1];
  __shared__ int32_t s_off[kChunk + 2];
  __shared__ int32_t s_pos[kInCap];
  __shared__ int64_t s_c[kInCap];
  const int lane = threadIdx.x;
  int64_t D[SPL];
#pragma unroll
  for (int r = 0; r < SPL; ++r) D[r] = 0;
  if (lane == 0) D[0] = out_sum[0];  // candidate i = 0 for j = 1: best[0] + C(0,1)
  for (int32_t j0 = 1; j0 <= n; j0 += kChunk) {
    const int32_t j1 = min(n, j0 + kChunk - 1);
    // stage lo[j], out_sum[j], in_off[j..j+1] for j in [j0, j1]
    for (int32_t t = lane; t <= j1 - j0; t += 32) {
      s_lo[t] = lo[j0 + t];
      s_out[t] = j0 + t < n ? out_sum[j0 + t] : 0;
    }
    for (int32_t t = lane; t <= j1 - j0 + 1; t += 32) s_off[t] = in_off[min(j0 + t, n)];
    __syncwarp();
    const int32_t ib = s_off[0];
    const int32_t in_end = s_off[j1 - j0 + 1];
    const bool staged = in_end - ib <= kInCap;
    if (staged) {
      for (int32_t t = ib + lane; t < in_end; t += 32) {
        s_pos[t - ib] = in_pos[t];
        s_c[t - ib] = in_c[t];
      }
    }
    __syncwarp();
    for (int32_t j = j0; j <= j1; ++j) {
      const int32_t loj = s_lo[j - j0];
      int64_t bv = kInf;
      int32_t bd = INT32_MAX;
#pragma unroll
      for (int r = 0; r < SPL; ++r) {
        const int32_t s = lane * SPL + r;
        const int32_t d = (j - 1 - s) & (W - 1);
        if (j - 1 - d >= loj) {
          if (D[r] < bv || (D[r] == bv && d < bd)) {
            bv = D[r];
            bd = d;
          }
        }
      }
      argmin_reduce(bv, bd);
      if (lane == 0) prev_cut[j] = j - 1 - bd;
      if (j == n) break;
      const int64_t o = s_out[j - j0];
#pragma unroll
      for (int r = 0; r < SPL; ++r) D[r] += o;
      // in-edges of position j (sources a < j); candidates i <= a lose c
      const int32_t kb = s_off[j - j0];
      const int32_t ke = s_off[j - j0 + 1];
      for (int32_t base = kb; base < ke; base += 32) {
        int32_t a = -1;
        int64_t c = 0;
        if (base + lane < ke) {
          if (staged) {
            a = s_pos[base + lane - ib];
            c = s_c[base + lane - ib];
          } else {
            a = in_pos[base + lane];
            c = in_c[base + lane];
          }
        }
        const int cnt = min(32, ke - base);
        for (int t = 0; t < cnt; ++t) {
          const int32_t at = __shfl_sync(0xffffffffu, a, t);
          const int64_t ct = __shfl_sync(0xffffffffu, c, t);
          if (at <= j - W) continue;  // source left the window
#pragma unroll
          for (int r = 0; r < SPL; ++r) {
            const int32_t s = lane * SPL + r;
            const int32_t i2 = j - ((j - s) & (W - 1));
            if (i2 <= at) D[r] -= ct;
          }
        }
      }
      // new candidate i = j: best[j] + out(j)
      const int32_t sl = j & (W - 1);
#pragma unroll
      for (int r = 0; r < SPL; ++r)
        if (lane * SPL + r == sl) D[r] = bv + o;
    }
    __syncwarp();
  }
}

// Generic DP for any R: the reference loop (fusion.cpp:133-162) with the downward scan
// over i done 32 candidates at a time (warp scan of forward[] + argmin).
__global__ void __launch_bounds__(32) k_dp_generic(int32_t n, const int32_t* lo, const int64_t* out_sum,
                                                   const int32_t* in_off, const int32_t* in_pos,
                                                   const int64_t* in_c, int64_t* forward, int64_t* best,
                                                   int32_t* prev_cut) {
  const int lane = threadIdx.x;
  if (lane == 0) best[0] = 0;
  __syncwarp();
  for (int32_t j = 1; j <= n; ++j) {
    const int32_t fp = j - 1;
    if (lane == 0) forward[fp] = out_sum[fp];
    __syncwarp();
    for (int32_t k = in_off[fp] + lane; k < in_off[fp + 1]; k += 32) forward[in_pos[k]] -= in_c[k];
    __syncwarp();
    const int32_t loj = lo[j];
    int64_t carry = 0, bv = kInf;
    int32_t bi = -1;
    for (int32_t top = j - 1; top >= loj; top -= 32) {
      const int32_t i = top - lane;
      const bool act = i >= loj;
      int64_t f = act ? forward[i] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int64_t x = __shfl_up_sync(0xffffffffu, f, o);
        if (lane >= o) f += x;
      }
      int64_t cand = act ? best[i] + carry + f : kInf;
      int32_t ci = act ? i : -1;
      // min value, largest i on ties (= smallest lane)
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        int64_t ov = __shfl_xor_sync(0xffffffffu, cand, o);
        int32_t oi = __shfl_xor_sync(0xffffffffu, ci, o);
        if (ov < cand || (ov == cand && oi > ci)) {
          cand = ov;
          ci = oi;
        }
      }
      if (cand < bv) {
        bv = cand;
        bi = ci;
      }
      carry += __shfl_sync(0xffffffffu, f, 31);
    }
    if (lane == 0) {
      best[j] = bv;
      prev_cut[j] = bi;
    }
    __syncwarp();
  }
}

// Cut traceback from n (fusion.cpp:164-169).  prev_cut is read in fixed windows of
// kTbWin positions, double-buffered in shared memory: while thread 0 chases the cuts down
// window k (one shared load per cut, ~n / 140 cuts at config #4), warps 1.. load window
// k + 1.  A cut is at most R <= 256 positions below the previous one, so the chase always
// continues in the next window.
constexpr int32_t kTbWin = 24576;
constexpr size_t kTbSmem = 2 * sizeof(int32_t) * kTbWin;
__global__ void __launch_bounds__(1024) k_traceback(const int32_t* prev_cut, int32_t n, uint8_t* is_cut) {
  extern __shared__ int32_t tbuf[];  // [2][kTbWin]
  __shared__ int32_t cur_s;
  if (threadIdx.x == 0) {
    is_cut[n] = 1;
    is_cut[0] = 1;
    cur_s = n;
  }
  // window k covers positions [max(1, n - (k + 1) W + 1), n - k W]
  auto load = [&](int32_t k, int32_t* dst, int32_t t0, int32_t nt) {
    const int32_t hi = n - k * kTbWin, lo = max(1, hi - kTbWin + 1);
    for (int32_t i = t0; i <= hi - lo; i += nt) dst[i] = prev_cut[lo + i];
  };
  if (n > 0) load(0, tbuf, threadIdx.x, blockDim.x);
  __syncthreads();
  for (int32_t k = 0;; ++k) {
    const int32_t hi = n - k * kTbWin, lo = max(1, hi - kTbWin + 1);
    int32_t* cur = tbuf + (k & 1) * kTbWin;
    if (threadIdx.x == 0) {
      int32_t c = cur_s;
      while (c >= lo && c > 0) {
        const int32_t p = cur[c - lo];
        is_cut[p] = 1;
        c = p;
      }
      cur_s = c;
    } else if (threadIdx.x >= 32 && lo > 1) {
      load(k + 1, tbuf + ((k + 1) & 1) * kTbWin, threadIdx.x - 32, blockDim.x - 32);
    }
    __syncthreads();
    if (cur_s <= 0 || lo <= 1) break;
  }
}

void traceback_launch(dp_ctx* ctx, const int32_t* prev_cut, int32_t n, uint8_t* is_cut) {
  static bool attr = false;
  if (!attr) {
    DP_CUDA(cudaFuncSetAttribute(k_traceback, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTbSmem)));
    attr = true;
  }
  DP_LAUNCH(ctx, k_traceback, 1, 1024, kTbSmem, prev_cut, n, is_cut);
}

__global__ void k_cut_scan_in(const uint8_t* is_cut, int32_t n, int32_t* f) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    f[p] = (p > 0 && is_cut[p]) ? 1 : 0;
}

__global__ void k_clusters(const int32_t* cl_excl, const uint8_t* is_cut, const int32_t* seq, int32_t n,
                           const int64_t* w, const int64_t* mem, int32_t* cl_of_pos, int32_t* cut_pos,
                           int64_t* tot_w, int64_t* tot_mem) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    // inclusive count of interior cuts at positions 1..p
    int32_t c = cl_excl[p] + ((p > 0 && is_cut[p]) ? 1 : 0);
    cl_of_pos[p] = c;
    if (p == 0 || is_cut[p]) cut_pos[c] = static_cast<int32_t>(p);
    int32_t v = seq[p];
    atomic_add_i64(&tot_w[c], w[v]);
    atomic_add_i64(&tot_mem[c], mem[v]);
  }
}

__global__ void k_cl_of_node(const int32_t* cl_of_pos, const int32_t* pos_of, int32_t n, int32_t* cl_of_node) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    cl_of_node[v] = cl_of_pos[pos_of[v]];
}

__global__ void k_coarse_keys(const int32_t* esrc, const int32_t* edst, const int64_t* bytes, int32_t m,
                              const int32_t* cl, int bits, uint64_t* keys, int64_t* vals) {
  const uint64_t sentinel = (bits >= 32) ? ~0ull : ((1ull << (2 * bits)) - 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t s = esrc[e], d = edst[e];
    int32_t cu = s >= 0 ? cl[s] : -1, cv = d >= 0 ? cl[d] : -1;
    if (cu >= 0 && cv >= 0 && cu != cv) {
      keys[e] = (static_cast<uint64_t>(cu) << bits) | static_cast<uint64_t>(cv);
      vals[e] = bytes[e];
    } else {
      keys[e] = sentinel;
      vals[e] = 0;
    }
  }
}

__global__ void k_coarse_decode(const uint64_t* uniq, const int64_t* sums, int32_t mc, int bits, int32_t* esrc,
                                int32_t* edst, int64_t* bytes) {
  const uint64_t mask = (1ull << bits) - 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mc; e += (int64_t)gridDim.x * blockDim.x) {
    esrc[e] = static_cast<int32_t>(uniq[e] >> bits);
    edst[e] = static_cast<int32_t>(uniq[e] & mask);
    bytes[e] = sums[e];
  }
}

// coarse edge count: reduce-by-key runs minus the sentinel run (dropped edges), if present
__global__ void k_coarse_count(const int64_t* runs, const uint64_t* uniq, uint64_t sentinel, int32_t* mc) {
  const int64_t nr = *runs;
  *mc = static_cast<int32_t>(nr) - ((nr > 0 && uniq[nr - 1] == sentinel) ? 1 : 0);
}

__global__ void k_fill_dense_ids(int64_t* id, int32_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    id[i] = i;
}

// ---- co-location contraction
__global__ void k_idrank(const int32_t* by_id, int32_t n, int32_t* idrank) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    idrank[by_id[r]] = static_cast<int32_t>(r);
}

__global__ void k_group_keys(const int32_t* group, const int32_t* idrank, int32_t n, uint64_t* keys, int32_t* vals) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    int32_t gl = group[v];
    keys[v] = gl >= 0 ? ((static_cast<uint64_t>(gl) << 32) | static_cast<uint32_t>(idrank[v])) : ~0ull;
    vals[v] = static_cast<int32_t>(v);
  }
}

__global__ void k_group_runs(const uint64_t* keys, const int32_t* vals, int32_t n, int32_t* rep_of,
                             int32_t* run_len, int32_t* pos_in_run) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    if (keys[s] == ~0ull) continue;
    if (s > 0 && (keys[s] >> 32) == (keys[s - 1] >> 32)) continue;
    int64_t t = s;
    while (t < n && keys[t] != ~0ull && (keys[t] >> 32) == (keys[s] >> 32)) ++t;
    int32_t rep = vals[s];
    for (int64_t q = s; q < t; ++q) {
      rep_of[vals[q]] = rep;
      pos_in_run[vals[q]] = static_cast<int32_t>(q - s);
    }
    run_len[rep] = static_cast<int32_t>(t - s);
  }
}

__global__ void k_rep_init(int32_t* rep_of, int32_t* run_len, int32_t* pos_in_run, int32_t n) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    rep_of[v] = static_cast<int32_t>(v);
    run_len[v] = 1;
    pos_in_run[v] = 0;
  }
}

__global__ void k_keep(const int32_t* rep_of, int32_t n, int32_t* keep) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    keep[v] = rep_of[v] == v ? 1 : 0;
}

__global__ void k_contract_nodes(const int32_t* rep_of, const int32_t* keep, const int32_t* cpos, const int32_t* run_len,
                                 const int64_t* id, const int32_t* group, int32_t n, int32_t* cidx_of, int64_t* cid,
                                 int32_t* cgroup, int64_t* cnt) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = cpos[rep_of[v]];
    cidx_of[v] = c;
    if (keep[v]) {
      cid[c] = id[v];
      cgroup[c] = group ? group[v] : -1;
      cnt[c] = run_len[v];
    }
  }
}

__global__ void k_contract_sums(const int32_t* cidx_of, const int64_t* w, const int64_t* mem, const int64_t* id,
                                const int32_t* pos_in_run, const int64_t* moff, int32_t n, int64_t* cw, int64_t* cmem,
                                int64_t* mem_ids) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    int32_t c = cidx_of[v];
    atomic_add_i64(&cw[c], w[v]);
    atomic_add_i64(&cmem[c], mem[v]);
    mem_ids[moff[c] + pos_in_run[v]] = id[v];
  }
}

__global__ void k_contract_edge_keys(const int32_t* esrc, const int32_t* edst, const int64_t* bytes, int32_t m,
                                     const int32_t* rep_of, const int32_t* idrank, uint64_t* keys, int64_t* vals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t u = rep_of[esrc[e]], v = rep_of[edst[e]];
    if (u != v) {
      keys[e] = (static_cast<uint64_t>(idrank[u]) << 32) | static_cast<uint32_t>(idrank[v]);
      vals[e] = bytes[e];
    } else {
      keys[e] = ~0ull;
      vals[e] = 0;
    }
  }
}

__global__ void k_contract_edge_decode(const uint64_t* uniq, const int64_t* sums, int32_t mc, const int32_t* by_id,
                                       const int32_t* cidx_of, const int64_t* cid, int32_t* esrc, int32_t* edst,
                                       int64_t* bytes, int64_t* src_id, int64_t* dst_id) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < mc; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t u = cidx_of[by_id[uniq[e] >> 32]], v = cidx_of[by_id[uniq[e] & 0xffffffffull]];
    esrc[e] = u;
    edst[e] = v;
    bytes[e] = sums[e];
    src_id[e] = cid[u];
    dst_id[e] = cid[v];
  }
}

__global__ void k_kept_by_id(const int32_t* by_id, const int32_t* keep, const int32_t* cpos, int32_t n,
                             int32_t* sorted_idx_c, uint64_t* sorted_key_c, const int64_t* id, const int32_t* kpos) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = by_id[r];
    if (!keep[v]) continue;
    int32_t o = kpos[r];
    sorted_idx_c[o] = cpos[v];
    sorted_key_c[o] = static_cast<uint64_t>(id[v]) ^ (1ull << 63);
  }
}

__global__ void k_keep_by_rank(const int32_t* by_id, const int32_t* keep, int32_t n, int32_t* f) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    f[r] = keep[by_id[r]];
}

__global__ void k_group_limit(const int64_t* moff, const int64_t* cmem, int32_t nc, int64_t limit, int* first) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < nc; c += (int64_t)gridDim.x * blockDim.x)
    if (moff[c + 1] - moff[c] > 1 && cmem[c] > limit) atomicMin(first, static_cast<int>(c));
}

// members re-expressed over original ids: per position p of the work sequence the member
// list of work node seq[p] (fusion.cpp:326-331).
__global__ void k_member_counts(const int32_t* seq, int32_t n, const int64_t* moff, int64_t* cnt) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = seq[p];
    cnt[p] = moff ? moff[v + 1] - moff[v] : 1;
  }
}
__global__ void k_member_fill(const int32_t* seq, int32_t n, const int64_t* moff, const int64_t* mids,
                              const int64_t* wid, const int64_t* poff, int64_t* out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    int32_t v = seq[p];
    if (!moff) {
      out[poff[p]] = wid ? wid[v] : v;
    } else {
      for (int64_t q = moff[v]; q < moff[v + 1]; ++q) out[poff[p] + (q - moff[v])] = mids[q];
    }
  }
}
__global__ void k_node_cluster_orig(const int32_t* cidx_of, const int32_t* cl_work, int32_t n, int32_t* out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[v] = cl_work[cidx_of ? cidx_of[v] : v];
}

}  // namespace

void breakpoints_dev(DevGraph& g, const int32_t* seq, const int32_t* pos_of, int32_t range, int64_t limit,
                     Clusters& out) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  const int32_t n = g.n;
  out.n = n;
  if (n == 0) {
    out.k = 0;
    out.cut_pos.alloc(ctx, 1);
    int32_t z = 0;
    out.cut_pos.upload(&z, 1);
    return;
  }
  DevBuf<int64_t> mem_pos(ctx, (size_t)n + 1), prefix(ctx, (size_t)n + 1), out_sum(ctx, n);
  DevBuf<int32_t> in_cnt(ctx, (size_t)n + 1), in_off_pos(ctx, (size_t)n + 1), lo(ctx, (size_t)n + 1);
  DevBuf<int> first(ctx, 1);
  int big = INT32_MAX;
  first.upload(&big, 1);
  mem_pos.zero();
  in_cnt.zero();
  DP_LAUNCH(ctx, k_dp_prep, grid_for(n, B), B, 0, seq, n, g.mem.p, g.out_off.p, g.out_cost.p, g.in_off.p, limit,
            mem_pos.p, out_sum.p, in_cnt.p, first.p);
  int fe = scalar_to_host(ctx, first.p);
  if (fe != INT32_MAX) {  // fusion.cpp:110-115, first position in sequence order
    int32_t v;
    DP_CUDA(cudaMemcpyAsync(&v, seq + fe, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
    int64_t id = g.dense_ids ? v : scalar_to_host(ctx, g.id.p + v);
    int64_t mv = scalar_to_host(ctx, g.mem.p + v);
    fail(DP_E_NODE_EXCEEDS_CLUSTER_LIMIT, "node %lld needs %lld bytes, cluster limit is %lld", (long long)id,
         (long long)mv, (long long)limit);
  }
  exclusive_scan_i64(ctx, mem_pos.p, prefix.p, (int64_t)n + 1);
  exclusive_scan_i32(ctx, in_cnt.p, in_off_pos.p, (int64_t)n + 1);
  const int32_t mi = g.m_ok;
  DevBuf<int32_t> in_pos(ctx, mi > 0 ? mi : 1);
  DevBuf<int64_t> in_c(ctx, mi > 0 ? mi : 1);
  DP_LAUNCH(ctx, k_in_fill, grid_for(n, B), B, 0, seq, pos_of, n, g.in_off.p, g.in_src.p, g.in_cost.p,
            in_off_pos.p, in_pos.p, in_c.p);
  DP_LAUNCH(ctx, k_lo, grid_for(n, B), B, 0, prefix.p, n, range, limit, lo.p);
  DevBuf<int32_t> prev_cut(ctx, (size_t)n + 1);
  {
    StageScope st(ctx, "breakpoint_dp", 0.0);
    if (range <= 256) {
      DP_LAUNCH(ctx, k_dp_window<8>, 1, 32, 0, n, lo.p, out_sum.p, in_off_pos.p, in_pos.p, in_c.p, prev_cut.p);
    } else if (range <= 1024) {
      DP_LAUNCH(ctx, k_dp_window<32>, 1, 32, 0, n, lo.p, out_sum.p, in_off_pos.p, in_pos.p, in_c.p, prev_cut.p);
    } else {
      DevBuf<int64_t> fwd(ctx, n), best(ctx, (size_t)n + 1);
      DP_LAUNCH(ctx, k_dp_generic, 1, 32, 0, n, lo.p, out_sum.p, in_off_pos.p, in_pos.p, in_c.p, fwd.p, best.p,
                prev_cut.p);
    }
  }
  clusters_from_prev_cut(g, seq, prev_cut.p, out);
}

// Cut traceback and clusters_from_cuts (fusion.cpp:61-81, 164-170) on the device.
void clusters_from_prev_cut(DevGraph& g, const int32_t* seq, const int32_t* prev_cut, Clusters& out) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  const int32_t n = g.n;
  out.n = n;
  DevBuf<uint8_t> is_cut(ctx, (size_t)n + 1);
  is_cut.zero();
  traceback_launch(ctx, prev_cut, n, is_cut.p);
  DevBuf<int32_t> f(ctx, (size_t)n + 1), fx(ctx, (size_t)n + 1);
  f.zero();
  DP_LAUNCH(ctx, k_cut_scan_in, grid_for(n, B), B, 0, is_cut.p, n, f.p);
  exclusive_scan_i32(ctx, f.p, fx.p, (int64_t)n + 1);
  int32_t interior = scalar_to_host(ctx, fx.p + n);
  out.k = interior + 1;
  out.cl_of_pos.alloc(ctx, n);
  out.cut_pos.alloc(ctx, (size_t)out.k + 1);
  out.tot_w.alloc(ctx, out.k);
  out.tot_mem.alloc(ctx, out.k);
  out.tot_w.zero();
  out.tot_mem.zero();
  DP_LAUNCH(ctx, k_clusters, grid_for(n, B), B, 0, fx.p, is_cut.p, seq, n, g.w.p, g.mem.p, out.cl_of_pos.p,
            out.cut_pos.p, out.tot_w.p, out.tot_mem.p);
  DP_CUDA(cudaMemcpyAsync(out.cut_pos.p + out.k, &out.n, sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
  sync(ctx);
}

void coarse_graph_dev(DevGraph& g, const int32_t* cl_of_node, int32_t k, const int64_t* tot_w, const int64_t* tot_mem,
                      DevGraph& coarse) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  const int32_t m = g.m;
  int bits = bits_for(static_cast<uint64_t>(k));
  DevBuf<uint64_t> keys(ctx, m > 0 ? m : 1), ko(ctx, m > 0 ? m : 1), uniq(ctx, m > 0 ? m : 1);
  DevBuf<int64_t> vals(ctx, m > 0 ? m : 1), vo(ctx, m > 0 ? m : 1), sums(ctx, m > 0 ? m : 1);
  DevBuf<int64_t> runs(ctx, 1);
  DP_LAUNCH(ctx, k_coarse_keys, grid_for(m, B), B, 0, g.esrc.p, g.edst.p, g.bytes.p, m, cl_of_node, bits, keys.p,
            vals.p);
  {
    StageScope st(ctx, "coarse_aggregate", 24.0 * m);
    sort_pairs_u64_i64(ctx, keys.p, ko.p, vals.p, vo.p, m, 2 * bits);
    reduce_by_key_u64(ctx, ko.p, uniq.p, vo.p, sums.p, runs.p, m);
  }
  int64_t nr = scalar_to_host(ctx, runs.p);
  int32_t mc = static_cast<int32_t>(nr);
  if (nr > 0) {
    uint64_t last = scalar_to_host(ctx, uniq.p + nr - 1);
    const uint64_t sentinel = (bits >= 32) ? ~0ull : ((1ull << (2 * bits)) - 1);
    if (last == sentinel) --mc;
  }
  DevBuf<int64_t> cw(ctx, k > 0 ? k : 1), cm(ctx, k > 0 ? k : 1), cb(ctx, mc > 0 ? mc : 1);
  DevBuf<int32_t> cs(ctx, mc > 0 ? mc : 1), cd(ctx, mc > 0 ? mc : 1);
  if (k) {
    DP_CUDA(cudaMemcpyAsync(cw.p, tot_w, sizeof(int64_t) * k, cudaMemcpyDeviceToDevice, ctx->stream));
    DP_CUDA(cudaMemcpyAsync(cm.p, tot_mem, sizeof(int64_t) * k, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  DP_LAUNCH(ctx, k_coarse_decode, grid_for(mc, B), B, 0, uniq.p, sums.p, mc, bits, cs.p, cd.p, cb.p);
  graph_adopt_dense(coarse, ctx, k, mc, std::move(cw), std::move(cm), std::move(cs), std::move(cd), std::move(cb));
  coarse.id.alloc(ctx, k > 0 ? k : 1);
  DP_LAUNCH(ctx, k_fill_dense_ids, grid_for(k, B), B, 0, coarse.id.p, k);
  graph_adjacency(coarse);
}

void contract_dev(DevGraph& g, Contraction& c, bool materialize_identity) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  const int32_t n = g.n, m = g.m;
  c.identity = !g.has_group;
  if (c.identity && !materialize_identity) return;
  DevBuf<int32_t> by_id, idrank(ctx, n > 0 ? n : 1);
  node_order_by_id(g, by_id);
  DP_LAUNCH(ctx, k_idrank, grid_for(n, B), B, 0, by_id.p, n, idrank.p);
  DevBuf<int32_t> rep_of(ctx, n > 0 ? n : 1), run_len(ctx, n > 0 ? n : 1), pos_in_run(ctx, n > 0 ? n : 1);
  DP_LAUNCH(ctx, k_rep_init, grid_for(n, B), B, 0, rep_of.p, run_len.p, pos_in_run.p, n);
  if (g.has_group) {
    DevBuf<uint64_t> keys(ctx, n), ko(ctx, n);
    DevBuf<int32_t> vals(ctx, n), vo(ctx, n);
    DP_LAUNCH(ctx, k_group_keys, grid_for(n, B), B, 0, g.group.p, idrank.p, n, keys.p, vals.p);
    sort_pairs_u64(ctx, keys.p, ko.p, vals.p, vo.p, n, 0, 64);
    DP_LAUNCH(ctx, k_group_runs, grid_for(n, B), B, 0, ko.p, vo.p, n, rep_of.p, run_len.p, pos_in_run.p);
  }
  DevBuf<int32_t> keep(ctx, (size_t)n + 1), cpos(ctx, (size_t)n + 1);
  keep.zero();
  DP_LAUNCH(ctx, k_keep, grid_for(n, B), B, 0, rep_of.p, n, keep.p);
  exclusive_scan_i32(ctx, keep.p, cpos.p, (int64_t)n + 1);
  const int32_t nc = scalar_to_host(ctx, cpos.p + n);
  DevGraph& w = c.work;
  w.ctx = ctx;
  w.n = nc;
  w.id.alloc(ctx, nc > 0 ? nc : 1);
  w.w.alloc(ctx, nc > 0 ? nc : 1);
  w.mem.alloc(ctx, nc > 0 ? nc : 1);
  w.group.alloc(ctx, nc > 0 ? nc : 1);
  w.has_group = g.has_group;
  w.w.zero();
  w.mem.zero();
  c.cidx_of.alloc(ctx, n > 0 ? n : 1);
  DevBuf<int64_t> cnt(ctx, (size_t)nc + 1);
  cnt.zero();
  DP_LAUNCH(ctx, k_contract_nodes, grid_for(n, B), B, 0, rep_of.p, keep.p, cpos.p, run_len.p, g.id.p,
            g.has_group ? g.group.p : nullptr, n, c.cidx_of.p, w.id.p, w.group.p, cnt.p);
  c.mem_off.alloc(ctx, (size_t)nc + 1);
  exclusive_scan_i64(ctx, cnt.p, c.mem_off.p, (int64_t)nc + 1);
  c.mem_ids.alloc(ctx, n > 0 ? n : 1);
  DP_LAUNCH(ctx, k_contract_sums, grid_for(n, B), B, 0, c.cidx_of.p, g.w.p, g.mem.p, g.id.p, pos_in_run.p,
            c.mem_off.p, n, w.w.p, w.mem.p, c.mem_ids.p);
  // edges: representatives' ids, merged by (u id, v id) via std::map order (fusion.cpp:277-286)
  DevBuf<uint64_t> keys(ctx, m > 0 ? m : 1), ko(ctx, m > 0 ? m : 1), uniq(ctx, m > 0 ? m : 1);
  DevBuf<int64_t> vals(ctx, m > 0 ? m : 1), vo(ctx, m > 0 ? m : 1), sums(ctx, m > 0 ? m : 1), runs(ctx, 1);
  DP_LAUNCH(ctx, k_contract_edge_keys, grid_for(m, B), B, 0, g.esrc.p, g.edst.p, g.bytes.p, m, rep_of.p, idrank.p,
            keys.p, vals.p);
  sort_pairs_u64_i64(ctx, keys.p, ko.p, vals.p, vo.p, m, 64);
  reduce_by_key_u64(ctx, ko.p, uniq.p, vo.p, sums.p, runs.p, m);
  int64_t nr = scalar_to_host(ctx, runs.p);
  int32_t mc = static_cast<int32_t>(nr);
  if (nr > 0 && scalar_to_host(ctx, uniq.p + nr - 1) == ~0ull) --mc;
  w.m = mc;
  w.esrc.alloc(ctx, mc > 0 ? mc : 1);
  w.edst.alloc(ctx, mc > 0 ? mc : 1);
  w.bytes.alloc(ctx, mc > 0 ? mc : 1);
  w.src_id.alloc(ctx, mc > 0 ? mc : 1);
  w.dst_id.alloc(ctx, mc > 0 ? mc : 1);
  DP_LAUNCH(ctx, k_contract_edge_decode, grid_for(mc, B), B, 0, uniq.p, sums.p, mc, by_id.p, c.cidx_of.p, w.id.p,
            w.esrc.p, w.edst.p, w.bytes.p, w.src_id.p, w.dst_id.p);
  // id order of the contracted nodes (for DFS/CPD ranks and id lookups)
  DevBuf<int32_t> f(ctx, (size_t)n + 1), fpos(ctx, (size_t)n + 1);
  f.zero();
  DP_LAUNCH(ctx, k_keep_by_rank, grid_for(n, B), B, 0, by_id.p, keep.p, n, f.p);
  exclusive_scan_i32(ctx, f.p, fpos.p, (int64_t)n + 1);
  w.dense_ids = false;
  w.sorted_idx.alloc(ctx, nc > 0 ? nc : 1);
  w.sorted_key.alloc(ctx, nc > 0 ? nc : 1);
  DP_LAUNCH(ctx, k_kept_by_id, grid_for(n, B), B, 0, by_id.p, keep.p, cpos.p, n, w.sorted_idx.p, w.sorted_key.p,
            g.id.p, fpos.p);
  graph_adjacency(w);
}

// fuse_begin = fuse_contract + levels (levels_dev) + fuse_order; the batched pipeline runs
// the levels of all its graphs together between the two.
DevGraph& fuse_contract(DevGraph& g, int64_t limit, FuseOut& out, FuseStage& fs) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  fs.limit = limit;
  contract_dev(g, out.con, false);
  DevGraph& work = out.con.identity ? g : out.con.work;
  if (!out.con.identity) {
    // validate(contracted): only a cycle can appear (fusion.cpp:288-293)
    graph_kahn(work, nullptr, nullptr, nullptr);
    if (work.processed != work.n) {
      std::vector<int64_t> wit = graph_cycle_witness(work);
      fail(DP_E_CYCLE_DETECTED, "co-location groups are inconsistent with a DAG: cycle: [%s]", join_ids(wit).c_str());
    }
    DevBuf<int> first(ctx, 1);
    int big = INT32_MAX;
    first.upload(&big, 1);
    DP_LAUNCH(ctx, k_group_limit, grid_for(work.n, B), B, 0, out.con.mem_off.p, work.mem.p, work.n, limit, first.p);
    int fc = scalar_to_host(ctx, first.p);
    if (fc != INT32_MAX) {
      fail(DP_E_GROUP_EXCEEDS_CLUSTER_LIMIT, "co-location group of node %lld needs %lld bytes, cluster limit is %lld",
           (long long)scalar_to_host(ctx, work.id.p + fc), (long long)scalar_to_host(ctx, work.mem.p + fc),
           (long long)limit);
    }
  }
  return work;
}

void fuse_order(DevGraph& g, int32_t range, int64_t limit, FuseOut& out, FuseStage& fs, bool defer = false) {
  dp_ctx* ctx = g.ctx;
  DevGraph& work = out.con.identity ? g : out.con.work;
  const int32_t n = work.n;
  out.seq.alloc(ctx, n > 0 ? n : 1);
  out.pos_of.alloc(ctx, n > 0 ? n : 1);
  fs.streamed = range >= 1 && range <= 256 && limit > 0 && n > 0;
  if (fs.streamed) {
    // cpd_topo streamed into optimal_breakpoints (peel_dp.cu); launched by the caller
    fs.prev_cut.alloc(ctx, (size_t)n + 1);
    fs.first.alloc(ctx, 1);
    int big = INT32_MAX;
    fs.first.upload(&big, 1);
    // defer: the caller syncs once for several graphs, then runs peel_dp_prepare_finish
    fs.job.j = defer ? peel_dp_prepare_begin(work, fs.c.p, range, limit, out.seq.p, out.pos_of.p, fs.prev_cut.p,
                                             fs.first.p)
                     : peel_dp_prepare(work, fs.c.p, range, limit, out.seq.p, out.pos_of.p, fs.prev_cut.p, fs.first.p);
  } else {
    topo_order(work, DP_TOPO_CPD, fs.c.p, out.seq.p, out.pos_of.p);
    if (range < 1) fail(DP_E_INVALID_VALUE, "exploration range must be >= 1");
    if (limit <= 0) fail(DP_E_INVALID_VALUE, "cluster memory limit must be > 0");
    breakpoints_dev(work, out.seq.p, out.pos_of.p, range, limit, out.cl);
  }
}

void fuse_begin(DevGraph& g, dp_comm_t comm, int32_t range, int64_t limit, FuseOut& out, FuseStage& fs) {
  DevGraph& work = fuse_contract(g, limit, out, fs);
  levels_dev(work, comm, fs.t, fs.b, fs.c, false);
  fuse_order(g, range, limit, out, fs);
}

void fuse_begin_batch(DevGraph* const* gs, int count, dp_comm_t comm, int32_t range, const int64_t* limit,
                      FuseOut* const* out, FuseStage* const* fs) {
  // errors in graph order, as if each graph ran fuse_begin alone: a graph whose contraction
  // fails is reported after the levels of the graphs before it (cycles) are checked
  std::vector<DevGraph*> work(count);
  std::vector<DevBuf<int64_t>*> t(count), b(count), c(count);
  for (int i = 0; i < count; ++i) {
    try {
      work[i] = &fuse_contract(*gs[i], limit[i], *out[i], *fs[i]);
    } catch (DpFail&) {
      for (int q = 0; q < i; ++q) levels_dev(*work[q], comm, fs[q]->t, fs[q]->b, fs[q]->c, false);
      throw;
    }
    t[i] = &fs[i]->t;
    b[i] = &fs[i]->b;
    c[i] = &fs[i]->c;
  }
  levels_dev_batch(work.data(), count, comm, t.data(), b.data(), c.data());
  for (int i = 0; i < count; ++i) fuse_order(*gs[i], range, limit[i], *out[i], *fs[i], true);
  sync(gs[0]->ctx);  // one round trip for every graph's DP key width
  for (int i = 0; i < count; ++i)
    if (fs[i]->streamed) peel_dp_prepare_finish(fs[i]->job.j);
}

void fuse_end(DevGraph& g, FuseOut& out, FuseStage& fs) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  DevGraph& work = out.con.identity ? g : out.con.work;
  const int32_t n = work.n;
  if (fs.streamed) {
    const int fe = scalar_to_host(ctx, fs.first.p);
    if (fe != INT32_MAX) {  // fusion.cpp:110-115, first position in sequence order
      const int32_t v = scalar_to_host(ctx, out.seq.p + fe);
      fail(DP_E_NODE_EXCEEDS_CLUSTER_LIMIT, "node %lld needs %lld bytes, cluster limit is %lld",
           (long long)scalar_to_host(ctx, work.id.p + v), (long long)scalar_to_host(ctx, work.mem.p + v),
           (long long)fs.limit);
    }
    clusters_from_prev_cut(work, out.seq.p, fs.prev_cut.p, out.cl);
  }
  DevBuf<int32_t> cl_work(ctx, n > 0 ? n : 1);
  DP_LAUNCH(ctx, k_cl_of_node, grid_for(n, B), B, 0, out.cl.cl_of_pos.p, out.pos_of.p, n, cl_work.p);
  coarse_graph_dev(work, cl_work.p, out.cl.k, out.cl.tot_w.p, out.cl.tot_mem.p, out.coarse);
  out.node_cluster.alloc(ctx, g.n > 0 ? g.n : 1);
  DP_LAUNCH(ctx, k_node_cluster_orig, grid_for(g.n, B), B, 0, out.con.identity ? nullptr : out.con.cidx_of.p,
            cl_work.p, g.n, out.node_cluster.p);
}

// fuse_end of several streamed graphs with three host round trips in all (cut counts and
// limit checks; coarse edge counts; coarse adjacency) instead of about six per graph.
// Errors surface graph by graph in order, as from fuse_end.
void fuse_end_batch(DevGraph* const* gs, int count, FuseOut* const* outs, FuseStage* const* fss) {
  bool all = count > 1;
  for (int i = 0; i < count; ++i) all = all && fss[i]->streamed;
  if (!all) {
    for (int i = 0; i < count; ++i) fuse_end(*gs[i], *outs[i], *fss[i]);
    return;
  }
  dp_ctx* ctx = gs[0]->ctx;
  const int B = 256;
  struct Tmp {
    DevBuf<uint8_t> is_cut;
    DevBuf<int32_t> f, fx, cl_work, mcd;
    DevBuf<uint64_t> keys, ko, uniq;
    DevBuf<int64_t> vals, vo, sums, runs;
    int h[2] = {0, 0};
    int32_t mc = 0;
    int bits = 1;
    AdjState adj;
  };
  std::vector<std::unique_ptr<Tmp>> T(count);
  auto work_of = [&](int i) -> DevGraph& { return outs[i]->con.identity ? *gs[i] : outs[i]->con.work; };
  // 1: traceback and cut counts; the first-exceed flags ride along
  for (int i = 0; i < count; ++i) {
    T[i].reset(new Tmp);
    Tmp& t = *T[i];
    const int32_t n = work_of(i).n;
    t.is_cut.alloc(ctx, (size_t)n + 1);
    t.is_cut.zero();
    traceback_launch(ctx, fss[i]->prev_cut.p, n, t.is_cut.p);
    t.f.alloc(ctx, (size_t)n + 1);
    t.fx.alloc(ctx, (size_t)n + 1);
    t.f.zero();
    DP_LAUNCH(ctx, k_cut_scan_in, grid_for(n, B), B, 0, t.is_cut.p, n, t.f.p);
    exclusive_scan_i32(ctx, t.f.p, t.fx.p, (int64_t)n + 1);
    download_bytes(ctx, &t.h[0], fss[i]->first.p, sizeof(int));
    download_bytes(ctx, &t.h[1], t.fx.p + n, sizeof(int32_t));
  }
  sync(ctx);
  // 2: limit checks in graph order (fusion.cpp:110-115), clusters, coarse edge aggregation
  for (int i = 0; i < count; ++i) {
    Tmp& t = *T[i];
    DevGraph& work = work_of(i);
    FuseOut& out = *outs[i];
    const int32_t n = work.n;
    if (t.h[0] != INT32_MAX) {
      const int32_t v = scalar_to_host(ctx, out.seq.p + t.h[0]);
      fail(DP_E_NODE_EXCEEDS_CLUSTER_LIMIT, "node %lld needs %lld bytes, cluster limit is %lld",
           (long long)scalar_to_host(ctx, work.id.p + v), (long long)scalar_to_host(ctx, work.mem.p + v),
           (long long)fss[i]->limit);
    }
    Clusters& cl = out.cl;
    cl.n = n;
    cl.k = t.h[1] + 1;
    const int32_t k = cl.k;
    cl.cl_of_pos.alloc(ctx, n);
    cl.cut_pos.alloc(ctx, (size_t)k + 1);
    cl.tot_w.alloc(ctx, k);
    cl.tot_mem.alloc(ctx, k);
    cl.tot_w.zero();
    cl.tot_mem.zero();
    DP_LAUNCH(ctx, k_clusters, grid_for(n, B), B, 0, t.fx.p, t.is_cut.p, out.seq.p, n, work.w.p, work.mem.p,
              cl.cl_of_pos.p, cl.cut_pos.p, cl.tot_w.p, cl.tot_mem.p);
    DP_CUDA(cudaMemcpyAsync(cl.cut_pos.p + k, &cl.n, sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
    t.cl_work.alloc(ctx, n > 0 ? n : 1);
    DP_LAUNCH(ctx, k_cl_of_node, grid_for(n, B), B, 0, cl.cl_of_pos.p, out.pos_of.p, n, t.cl_work.p);
    const int32_t m = work.m;
    t.bits = bits_for(static_cast<uint64_t>(k));
    t.keys.alloc(ctx, m > 0 ? m : 1);
    t.ko.alloc(ctx, m > 0 ? m : 1);
    t.uniq.alloc(ctx, m > 0 ? m : 1);
    t.vals.alloc(ctx, m > 0 ? m : 1);
    t.vo.alloc(ctx, m > 0 ? m : 1);
    t.sums.alloc(ctx, m > 0 ? m : 1);
    t.runs.alloc(ctx, 1);
    t.mcd.alloc(ctx, 1);
    DP_LAUNCH(ctx, k_coarse_keys, grid_for(m, B), B, 0, work.esrc.p, work.edst.p, work.bytes.p, m, t.cl_work.p,
              t.bits, t.keys.p, t.vals.p);
    {
      StageScope st(ctx, "coarse_aggregate", 24.0 * m);
      sort_pairs_u64_i64(ctx, t.keys.p, t.ko.p, t.vals.p, t.vo.p, m, 2 * t.bits);
      reduce_by_key_u64(ctx, t.ko.p, t.uniq.p, t.vo.p, t.sums.p, t.runs.p, m);
    }
    const uint64_t sentinel = (t.bits >= 32) ? ~0ull : ((1ull << (2 * t.bits)) - 1);
    DP_LAUNCH(ctx, k_coarse_count, 1, 1, 0, t.runs.p, t.uniq.p, sentinel, t.mcd.p);
    download_bytes(ctx, &t.mc, t.mcd.p, sizeof(int32_t));
  }
  sync(ctx);
  // 3: coarse graphs (cluster k: id k, summed compute / memory; fusion.cpp:173-229)
  for (int i = 0; i < count; ++i) {
    Tmp& t = *T[i];
    FuseOut& out = *outs[i];
    const int32_t k = out.cl.k, mc = t.mc;
    DevBuf<int64_t> cw(ctx, k > 0 ? k : 1), cm(ctx, k > 0 ? k : 1), cb(ctx, mc > 0 ? mc : 1);
    DevBuf<int32_t> cs(ctx, mc > 0 ? mc : 1), cd(ctx, mc > 0 ? mc : 1);
    if (k) {
      DP_CUDA(cudaMemcpyAsync(cw.p, out.cl.tot_w.p, sizeof(int64_t) * k, cudaMemcpyDeviceToDevice, ctx->stream));
      DP_CUDA(cudaMemcpyAsync(cm.p, out.cl.tot_mem.p, sizeof(int64_t) * k, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    DP_LAUNCH(ctx, k_coarse_decode, grid_for(mc, B), B, 0, t.uniq.p, t.sums.p, mc, t.bits, cs.p, cd.p, cb.p);
    graph_adopt_dense(out.coarse, ctx, k, mc, std::move(cw), std::move(cm), std::move(cs), std::move(cd),
                      std::move(cb));
    out.coarse.id.alloc(ctx, k > 0 ? k : 1);
    DP_LAUNCH(ctx, k_fill_dense_ids, grid_for(k, B), B, 0, out.coarse.id.p, k);
    graph_adjacency_begin(out.coarse, t.adj);
  }
  sync(ctx);
  for (int i = 0; i < count; ++i) {
    FuseOut& out = *outs[i];
    graph_adjacency_end(out.coarse, T[i]->adj);
    DevGraph& g = *gs[i];
    out.node_cluster.alloc(ctx, g.n > 0 ? g.n : 1);
    DP_LAUNCH(ctx, k_node_cluster_orig, grid_for(g.n, B), B, 0, out.con.identity ? nullptr : out.con.cidx_of.p,
              T[i]->cl_work.p, g.n, out.node_cluster.p);
  }
}

void fuse_dev(DevGraph& g, dp_comm_t comm, int32_t range, int64_t limit, FuseOut& out) {
  FuseStage fs;
  fuse_begin(g, comm, range, limit, out, fs);
  if (fs.streamed) peel_dp_launch(g.ctx, &fs.job.j, 1);
  fuse_end(g, out, fs);
}

dp_cluster_map_t* fuse_map_to_host_async(DevGraph& g, FuseOut& f, Finalizers& fin) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  DevGraph& work = f.con.identity ? g : f.con.work;
  const int32_t nw = work.n, k = f.cl.k;
  DevBuf<int64_t> cnt(ctx, (size_t)nw + 1), poff(ctx, (size_t)nw + 1), members(ctx, g.n > 0 ? g.n : 1);
  cnt.zero();
  const int64_t* moff = f.con.identity ? nullptr : f.con.mem_off.p;
  DP_LAUNCH(ctx, k_member_counts, grid_for(nw, B), B, 0, f.seq.p, nw, moff, cnt.p);
  exclusive_scan_i64(ctx, cnt.p, poff.p, (int64_t)nw + 1);
  DP_LAUNCH(ctx, k_member_fill, grid_for(nw, B), B, 0, f.seq.p, nw, moff, f.con.mem_ids.p,
            (f.con.identity && g.dense_ids) ? nullptr : work.id.p, poff.p, members.p);
  dp_cluster_map_t* m = new_cluster_map(g.n, k, k > 0 ? k - 1 : 0);
  f.node_cluster.download(m->node_cluster, g.n);
  members.download(m->members, g.n);  // stream-ordered: the buffers are freed after the copies
  f.cl.tot_w.download(m->total_compute, k);
  f.cl.tot_mem.download(m->total_memory, k);
  auto cuts = std::make_shared<std::vector<int32_t>>((size_t)k + 1);
  auto po = std::make_shared<std::vector<int64_t>>((size_t)nw + 1);
  download_bytes(ctx, cuts->data(), f.cl.cut_pos.p, sizeof(int32_t) * ((size_t)k + 1));
  download_bytes(ctx, po->data(), poff.p, sizeof(int64_t) * ((size_t)nw + 1));
  fin.push_back([m, cuts, po, k] {
    for (int32_t c = 0; c <= k; ++c) m->member_off[c] = (*po)[(*cuts)[c]];
    for (int32_t c = 1; c < k; ++c) m->breakpoints[c - 1] = (*cuts)[c];
  });
  return m;
}

dp_cluster_map_t* fuse_map_to_host(DevGraph& g, FuseOut& f) {
  Finalizers fin;
  dp_cluster_map_t* m = fuse_map_to_host_async(g, f, fin);
  sync(g.ctx);
  for (auto& x : fin) x();
  return m;
}

}  // namespace dpb
