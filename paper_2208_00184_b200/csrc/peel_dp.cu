// peel_dp.cu — latency-engineered topological peel (ordering.cpp:40-114) and the
// streaming breakpoint DP (fusion.cpp:126-162) that consumes its output.
//
// The reference peel is a deque used as a stack for DFS/CPD (freed children pushed to the
// head, so the highest-priority freed child is emitted right after its parent — pinned by
// test_ordering.cpp:104-135) and as a FIFO for M-TOPO.  Both comparators of a policy are
// one static total order, so each node gets a 32-bit rank (lower = emitted first among
// simultaneously available nodes): CPD (cpath desc, id asc), DFS / M (id asc).
//
// Peel (one warp).  Per CSR slot the warp loads one 16-byte record
//   { child, rank(child), row_start(child), out_degree(child) }
// so a popped stack entry already names its own row and a freed child can be pushed
// with its row descriptor without another dependent load.  The stack top lives in a
// shared-memory window (spilled to / refilled from HBM in halves when deep).  While the
// in-degree decrements of a node's children are in flight, the rows of all children are
// prefetched into L1, so when the next popped node is a just-freed child its record
// load is already close.  Dependent HBM/L2 round trips per node: ~2 -> ~1.
//
// Streaming DP (second CTA of the same cooperative launch).  The peel publishes its
// progress (positions emitted); the DP warp follows it in chunks of 256 positions: it
// stages position data (node, memory prefix, lo[j], out-cost sum, in-edges as source
// positions) into shared memory with coalesced loads, then runs the register-window
// recurrence of fusion.cu on shared-memory operands.  Peel and DP overlap, so the
// sequential part of fuse() costs max(peel, DP) instead of their sum.
#include <algorithm>
#include <cstddef>
#include <cstdlib>
#include <memory>
#include <vector>

#include "fusion.cuh"
#include "graph.cuh"
#include "peel.cuh"
#include "peel_dp.cuh"
#include "fixpoint.cuh"

namespace dpb {
namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kStackCache = 4096;  // stack entries in shared memory (power of 2)
constexpr int kFreedCap = 2048;

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct PeelArgs {
  int32_t n;
  const int4* slot;     // per CSR slot: child, rank(child), row_start(child), deg(child)
  int32_t* indeg;       // working in-degrees
  int4* gstack;         // global stack backing store (n entries), initial sources at [0, nsrc)
  const int32_t* nsrc;  // number of sources (device: no host round trip before the launch)
  bool stack_mode;      // false: FIFO (M-TOPO)
  int32_t* seq;         // node index by position
  int32_t* pos_of;
  int* progress;        // positions emitted (published with release semantics)
  int* emitted;         // final count
  int64_t* freed_spill; // rank<<32|slot-index spill for huge fan-outs
  // stack-mode layout (peel_warp_v5)
  int2* nr2;             // { remaining in-degree, rank | min(out-degree, 255) << 24 }
  const int32_t* ell;    // padded rows, -1 past the degree
  int32_t ellw;
  const int32_t* out_off;
  const int32_t* out_dst;
  int2* gstack2;         // { node, min(out-degree, 255) }
  // stack-mode layout (peel_warp_v6)
  bool v6;
  const int4* ell6;      // 8 slots {child, rank | min(indeg,127) << 24 | (deg > 8) << 31} per node
  const int2* cmeta;     // the same records over the CSR (rows longer than 8)
  int32_t* rem_big;      // remaining in-degree of nodes with in-degree >= 127
  int32_t* gsid;         // global stack of {node | long flag}
  int32_t* gover;        // remaining in-degree of keys spilled from full buckets (0 = absent)
  long long* debug;      // optional: peel warp cycles
  bool prefetch;         // v6: prefetch the rows of a pushed child's children to L2
  const int* skip;       // *skip != 0: the order was produced by the fixed-point peel (fixpoint.cu)
  const uint32_t* dense16;  // v6 dense mode (nullptr: off): initial in-degrees, 16 bits each
  const int* dense_bad;     // *dense_bad != 0: an in-degree >= 65,535 (dense mode off)
};

// The peel warp.  Shared memory: stack cache (kStackCache int4) + freed buffer.
__device__ void peel_warp(const PeelArgs& a, int4* sstack, int64_t* sfreed) {
  const int lane = threadIdx.x & 31;
  const int32_t SC = kStackCache;
  // ---------------- stack (stack mode): logical entries [0, top]; [base, top] cached
  const int32_t nsrc = *a.nsrc;
  int32_t top = nsrc - 1, base = 0;
  // ---------------- queue (FIFO mode): entries [head, tail) in gstack
  int32_t head = 0, tail = nsrc;
  if (a.stack_mode) {
    base = max(0, nsrc - SC / 2);
    for (int32_t i = base + lane; i <= top; i += 32) sstack[i & (SC - 1)] = a.gstack[i];
  }
  __syncwarp();
  int32_t p = 0;
  for (;;) {
    int4 e;
    if (a.stack_mode) {
      if (top < 0) break;
      if (top < base) {  // refill the cache from HBM
        base = max(0, top + 1 - SC / 2);
        for (int32_t i = base + lane; i <= top; i += 32) sstack[i & (SC - 1)] = a.gstack[i];
        __syncwarp();
      }
      e = sstack[top & (SC - 1)];
      --top;
    } else {
      if (head == tail) break;
      e = a.gstack[head++];
    }
    const int32_t v = e.x, rs = e.y, deg = e.z;
    if (lane == 0) {
      a.seq[p] = v;
      a.pos_of[v] = p;
    }
    ++p;
    if (a.progress && (p & 63) == 0) {
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        st_release(a.progress, p);
      }
    }
    int32_t nf = 0;
    for (int32_t b0 = 0; b0 < deg; b0 += 32) {
      const int32_t k = b0 + lane;
      const bool act = k < deg;
      int4 s = make_int4(0, 0, 0, 0);
      if (act) s = a.slot[rs + k];
      if (act) prefetch_l1(a.slot + s.z);  // child's row, in case it is popped next
      bool fr = false;
      if (act) {
        const int32_t d = a.indeg[s.x] - 1;
        a.indeg[s.x] = d;
        fr = d == 0;
      }
      const unsigned m = __ballot_sync(FULL, fr);
      if (deg <= 32) {
        // fast path: freed children are in registers
        nf = __popc(m);
        if (nf == 0) break;
        if (!a.stack_mode) {
          // FIFO: append in ascending rank
          int32_t cnt = 0;
          for (unsigned mm = m; mm; mm &= mm - 1) {
            const int32_t rb = __shfl_sync(FULL, s.y, __ffs(mm) - 1);
            cnt += rb < s.y;
          }
          if (fr) a.gstack[tail + cnt] = make_int4(s.x, s.z, s.w, 0);
          tail += nf;
          __syncwarp();
          break;
        }
        if (top + nf - base >= SC - 1) {  // spill the lower half of the cache
          const int32_t half = SC / 2;
          for (int32_t i = base + lane; i < base + half; i += 32) a.gstack[i] = sstack[i & (SC - 1)];
          __syncwarp();
          base += half;
        }
        int32_t cnt = 0;  // pushed in descending rank: lowest rank ends on top
        for (unsigned mm = m; mm; mm &= mm - 1) {
          const int32_t rb = __shfl_sync(FULL, s.y, __ffs(mm) - 1);
          cnt += rb > s.y;
        }
        if (fr) sstack[(top + 1 + cnt) & (SC - 1)] = make_int4(s.x, s.z, s.w, 0);
        top += nf;
        __syncwarp();
        break;
      }
      // general path (rows longer than 32): collect (rank, child entry index) first
      if (fr) {
        const int32_t at = nf + __popc(m & ((1u << lane) - 1));
        const int64_t rec = (static_cast<int64_t>(s.y) << 32) | static_cast<uint32_t>(rs + k);
        if (at < kFreedCap) sfreed[at] = rec; else a.freed_spill[at - kFreedCap] = rec;
      }
      nf += __popc(m);
    }
    if (deg > 32 && nf > 0) {
      __syncwarp();
      if (a.stack_mode && top + nf - base >= SC - 1) {
        // make room: flush the whole cache window, keep nothing cached
        for (int32_t i = base + lane; i <= top; i += 32) a.gstack[i] = sstack[i & (SC - 1)];
        __syncwarp();
        base = top + 1;
      }
      const bool big = a.stack_mode && (nf >= SC - 1);
      for (int32_t i = lane; i < nf; i += 32) {
        const int64_t ri = i < kFreedCap ? sfreed[i] : a.freed_spill[i - kFreedCap];
        const int32_t rk = static_cast<int32_t>(ri >> 32);
        int32_t cnt = 0;
        for (int32_t j = 0; j < nf; ++j) {
          const int64_t rj = j < kFreedCap ? sfreed[j] : a.freed_spill[j - kFreedCap];
          const int32_t r2 = static_cast<int32_t>(rj >> 32);
          cnt += a.stack_mode ? (r2 > rk) : (r2 < rk);
        }
        const int4 s = a.slot[static_cast<int32_t>(ri & 0xffffffff)];
        const int4 ent = make_int4(s.x, s.z, s.w, 0);
        if (!a.stack_mode) a.gstack[tail + cnt] = ent;
        else if (big) a.gstack[top + 1 + cnt] = ent;
        else sstack[(top + 1 + cnt) & (SC - 1)] = ent;
      }
      if (!a.stack_mode) {
        tail += nf;
      } else {
        top += nf;
        if (big) base = top + 1;  // everything lives in HBM; the next pop refills
      }
      __syncwarp();
    }
  }
  if (lane == 0) {
    *a.emitted = p;
    if (a.progress) {
      __threadfence();
      st_release(a.progress, p);
    }
  }
}

// Stack-mode peel (DFS/CPD), lean version.  Data (peel_prepare):
//   nr2[v] = { remaining in-degree, rank | min(deg,255) << 24 }   8 B / node
//   ell[v] = first EW children, -1 padded (address = v * EW)    4*EW B / node
// Stack entries are {node, deg}.  While lane k's nr2[c_k] is in flight the lane also
// loads ell[c_k]; the warp loads the stack top's row.  After the freed decision the row
// of whichever node is popped next (min-rank freed child, or the old top) is kept in
// shared memory, so each node costs one dependent L2 round trip.  The emitted sequence
// is buffered and stored 32 ids at a time; pos_of is scattered by the consumer.
template <int EW>
__device__ void peel_warp_v5(const PeelArgs& a, int2* sstack, int64_t* sfreed, int32_t* srow, int32_t* stop,
                             int32_t* seqbuf) {
  const int lane = threadIdx.x & 31;
  const int32_t SC = 2 * kStackCache;
  const int32_t nsrc = *a.nsrc;
  int32_t top = nsrc - 1;
  int32_t base = max(0, nsrc - SC / 2);
  for (int32_t i = base + lane; i <= top; i += 32) sstack[i & (SC - 1)] = a.gstack2[i];
  __syncwarp();
  int32_t p = 0;
  int32_t exp_idx = -1;
  int exp_src = 0;
  while (top >= 0) {
    if (top < base) {
      base = max(0, top + 1 - SC / 2);
      for (int32_t i = base + lane; i <= top; i += 32) sstack[i & (SC - 1)] = a.gstack2[i];
      __syncwarp();
    }
    const int32_t my_idx = top;
    const int2 e = sstack[top & (SC - 1)];
    --top;
    const int32_t v = e.x, deg = e.y;
    if (lane == 0) {
      seqbuf[p & 31] = v;
      a.pos_of[v] = p;
    }
    ++p;
    if ((p & 31) == 0) {
      __syncwarp();
      a.seq[p - 32 + lane] = seqbuf[lane];
      if (a.progress && lane == 0) {
        __threadfence();
        st_release(a.progress, p);
      }
    }
    if (deg > EW) {
      // ---- long row (CSR), children's rows not prefetched
      const int32_t rs = a.out_off[v], dg = a.out_off[v + 1] - rs;
      int32_t nf = 0;
      for (int32_t b0 = 0; b0 < dg; b0 += 32) {
        const int32_t k = b0 + lane;
        const bool act = k < dg;
        int32_t c = 0;
        int2 r2 = make_int2(1, 0);
        if (act) {
          c = a.out_dst[rs + k];
          r2 = a.nr2[c];
        }
        bool fr = false;
        if (act) {
          const int32_t d = r2.x - 1;
          a.nr2[c].x = d;
          fr = d == 0;
        }
        const unsigned m = __ballot_sync(FULL, fr);
        if (fr) {
          const int32_t at = nf + __popc(m & ((1u << lane) - 1));
          const int64_t r = (static_cast<int64_t>(r2.y) << 32) | static_cast<uint32_t>(c);
          if (at < kFreedCap) sfreed[at] = r; else a.freed_spill[at - kFreedCap] = r;
        }
        nf += __popc(m);
      }
      __syncwarp();
      if (nf > 0) {
        if (top + nf - base >= SC - 1) {
          for (int32_t i = base + lane; i <= top; i += 32) a.gstack2[i] = sstack[i & (SC - 1)];
          __syncwarp();
          base = top + 1;
        }
        const bool big = nf >= SC - 1;
        for (int32_t i = lane; i < nf; i += 32) {
          const int64_t ri = i < kFreedCap ? sfreed[i] : a.freed_spill[i - kFreedCap];
          const int32_t rk = static_cast<int32_t>(ri >> 32) & 0xffffff;
          int32_t cnt = 0;
          for (int32_t j = 0; j < nf; ++j) {
            const int64_t rj = j < kFreedCap ? sfreed[j] : a.freed_spill[j - kFreedCap];
            cnt += (static_cast<int32_t>(rj >> 32) & 0xffffff) > rk;
          }
          const int2 ent = make_int2(static_cast<int32_t>(ri & 0xffffffff),
                                     static_cast<int32_t>(static_cast<uint32_t>(ri >> 32) >> 24));
          if (big) a.gstack2[top + 1 + cnt] = ent; else sstack[(top + 1 + cnt) & (SC - 1)] = ent;
        }
        top += nf;
        if (big) base = top + 1;
        __syncwarp();
      }
      exp_idx = -1;
      continue;
    }
    const int src = (my_idx == exp_idx) ? exp_src : 0;
    int32_t c = -1;
    if (lane < EW) c = src == 1 ? srow[lane] : (src == 2 ? stop[lane] : a.ell[static_cast<int64_t>(v) * EW + lane]);
    const bool act = c >= 0;
    int2 r2 = make_int2(1, 0);
    int4 crow[EW / 4];
    if (act) {
      r2 = a.nr2[c];
      const int4* rp = reinterpret_cast<const int4*>(a.ell + static_cast<int64_t>(c) * EW);
#pragma unroll
      for (int q = 0; q < EW / 4; ++q) crow[q] = rp[q];
    }
    const bool have_top = top >= base;
    int32_t trow = -1;
    if (have_top && lane < EW) {
      const int2 te = sstack[top & (SC - 1)];
      if (te.y <= EW) trow = a.ell[static_cast<int64_t>(te.x) * EW + lane];
    }
    bool fr = false;
    if (act) {
      const int32_t d = r2.x - 1;
      a.nr2[c].x = d;
      fr = d == 0;
    }
    const unsigned m = __ballot_sync(FULL, fr);
    if (m == 0) {
      if (have_top && lane < EW) stop[lane] = trow;
      exp_idx = have_top ? top : -1;
      exp_src = 2;
      __syncwarp();
      continue;
    }
    const int nf = __popc(m);
    if (top + nf - base >= SC - 1) {
      const int32_t half = SC / 2;
      for (int32_t i = base + lane; i < base + half; i += 32) a.gstack2[i] = sstack[i & (SC - 1)];
      __syncwarp();
      base += half;
    }
    const int32_t rk = r2.y & 0xffffff;
    int32_t cnt = 0;  // pushed in descending rank: the lowest rank ends on top
    if (nf > 1) {
      for (unsigned mm = m; mm; mm &= mm - 1) {
        const int32_t rb = __shfl_sync(FULL, rk, __ffs(mm) - 1);
        cnt += rb > rk;
      }
    }
    if (fr) {
      sstack[(top + 1 + cnt) & (SC - 1)] = make_int2(c, static_cast<int32_t>(static_cast<uint32_t>(r2.y) >> 24));
      if (cnt == nf - 1) {
        int4* dst = reinterpret_cast<int4*>(srow);
#pragma unroll
        for (int q = 0; q < EW / 4; ++q) dst[q] = crow[q];
      }
    }
    top += nf;
    exp_idx = top;
    exp_src = 1;
    __syncwarp();
  }
  __syncwarp();
  if (lane < (p & 31)) a.seq[(p & ~31) + lane] = seqbuf[lane];
  __syncwarp();
  if (lane == 0) {
    *a.emitted = p;
    if (a.progress) {
      __threadfence();
      st_release(a.progress, p);
    }
  }
}

// ---------------------------------------------------------------- peel v6
// Stack-mode peel (DFS/CPD) with the remaining in-degrees on chip.
//  * Remaining in-degrees of OPEN nodes (some but not all predecessors emitted) live in a
//    2-way bucketed hash table in shared memory (one 8-byte load answers a lookup);
//    a bucket whose two ways are taken spills further keys to a global counter array
//    and counts them, so lookups only touch HBM in buckets that actually overflowed.
//    A node's first decrement needs no lookup: its initial in-degree rides in its
//    parent's row.
//  * Rows hold 8 slots {child, rank | min(indeg,127) << 24 | (deg > 8) << 31} sorted by
//    rank, so the push order of the freed children is a popcount of the freed mask.
//  * Every cached stack entry carries its node's 64-byte row: a popped node's row is on
//    chip.  The only global load of a step — the rows of the popped node's children, any
//    of which may be pushed — is issued first and overlaps the table work; when a child
//    is pushed, its children's rows are prefetched to L2.
//  * Rows longer than 8 take a CSR path; in-degrees >= 127 use global counters.
constexpr int kV6Stack = 512;
// hash buckets (log2): 16,384 x 2 ways (128 KB) when the peel has its SM alone, 8,192 when
// it shares it with the DP (k_peel_dp_shared)
constexpr int kV6BucketBits = 14;
constexpr int kV6BucketBitsShared = 13;
constexpr uint32_t kV6Empty = 0xffffffffu;
constexpr int32_t kV6Long = 1 << 30;  // sid flag: out-degree > 8 (CSR path)
constexpr int kV6FreedCap = 1024;

template <int BB>
struct V6Smem {
  int4 row[kV6Stack][4];
  int32_t sid[kV6Stack];
  uint32_t ht[2 << BB];      // way 0 / way 1 of bucket b at [2b], [2b+1]
  uint32_t ovc[1 << (BB - 1)];  // 16-bit overflow counts, two per word
  int64_t freed[kV6FreedCap];
  int32_t seqbuf[32];
};

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <int BB>
__device__ __forceinline__ uint32_t v6_bucket(int32_t c) {
  return (static_cast<uint32_t>(c) * 0x9E3779B1u) >> (32 - BB);
}

// One decrement of child c (initial in-degree `code`, 2..126).  Returns true when c is freed.
template <int BB>
__device__ __forceinline__ bool v6_dec(V6Smem<BB>& S, int32_t* gover, int32_t c, int code) {
  const uint32_t b = v6_bucket<BB>(c), uc = static_cast<uint32_t>(c);
  const uint2 w = *reinterpret_cast<const uint2*>(&S.ht[2 * b]);
  const uint32_t sh = (b & 1u) * 16;
  const uint32_t ov = S.ovc[b >> 1];
  const bool h0 = (w.x >> 7) == uc, h1 = (w.y >> 7) == uc;
  if (h0 | h1) {
    const uint32_t e = h0 ? w.x : w.y;
    const bool fr = (e & 127u) == 1u;
    S.ht[2 * b + (h0 ? 0 : 1)] = fr ? kV6Empty : e - 1;
    return fr;
  }
  if ((ov >> sh) & 0xffffu) {
    const int32_t g = gover[c];
    if (g > 0) {
      gover[c] = g - 1;
      if (g == 1) atomicSub(&S.ovc[b >> 1], 1u << sh);
      return g == 1;
    }
  }
  const uint32_t nv = (uc << 7) | static_cast<uint32_t>(code - 1);
  if (w.x == kV6Empty && atomicCAS(&S.ht[2 * b], kV6Empty, nv) == kV6Empty) return false;
  if (w.y == kV6Empty && atomicCAS(&S.ht[2 * b + 1], kV6Empty, nv) == kV6Empty) return false;
  gover[c] = code - 1;
  atomicAdd(&S.ovc[b >> 1], 1u << sh);
  return false;
}

// Dense mode (graphs of at most 2 x (2^(BB+1) + 2^(BB-1)) nodes, every in-degree < 65,535):
// the remaining in-degree of EVERY node lives in shared memory as a 16-bit counter (two per
// word, over the hash table's and overflow counts' storage), so a decrement is one shared
// atomic -- no bucket probe, no global counter for in-degrees >= 127 or spilled buckets.
// Parallel edges are rejected by validation, so a row decrements each child once and a
// counter never goes below zero (no borrow into its neighbour).
template <int BB>
constexpr int32_t v6_dense_cap() {
  return 2 * ((2 << BB) + (1 << (BB - 1)));
}
__device__ __forceinline__ uint32_t v6_dense_dec(uint32_t* dw, int32_t c) {
  const uint32_t sh = (static_cast<uint32_t>(c) & 1u) * 16u;
  return (atomicSub(&dw[c >> 1], 1u << sh) >> sh) & 0xffffu;  // remaining before this decrement
}

// Loads stack entries [lo, hi] (ids from the global stack, rows from the ELL) into the cache.
template <int BB>
__device__ void v6_fill(const PeelArgs& a, V6Smem<BB>& S, int32_t lo, int32_t hi, int lane) {
  for (int32_t idx = lane; idx < (hi - lo + 1) * 4; idx += 32) {
    const int32_t i = lo + (idx >> 2);
    const int32_t sv = a.gsid[i];
    if ((idx & 3) == 0) S.sid[i & (kV6Stack - 1)] = sv;
    S.row[i & (kV6Stack - 1)][idx & 3] = a.ell6[static_cast<int64_t>(sv & 0xffffff) * 4 + (idx & 3)];
  }
}

__device__ __forceinline__ void v6_publish(const PeelArgs& a, int32_t p) {
  if (a.progress) {
    __threadfence();
    st_release(a.progress, p);
  }
}

template <int BB>
__device__ void peel_warp_v6(const PeelArgs& a, V6Smem<BB>& S) {
  const int lane = threadIdx.x & 31;
  const long long t_start = clock64();
  constexpr int32_t SC = kV6Stack;
  static_assert(offsetof(V6Smem<BB>, ovc) == offsetof(V6Smem<BB>, ht) + sizeof(uint32_t) * (2 << BB),
                "dense counters span ht and ovc");
  const bool dense = a.dense16 != nullptr && a.n <= v6_dense_cap<BB>() && *a.dense_bad == 0;
  uint32_t* const dw = S.ht;  // dense mode: counters over ht + ovc
  if (dense) {
    for (int i = lane; i < (a.n + 1) / 2; i += 32) dw[i] = a.dense16[i];
  } else {
    for (int i = lane; i < (2 << BB); i += 32) S.ht[i] = kV6Empty;
    for (int i = lane; i < (1 << (BB - 1)); i += 32) S.ovc[i] = 0;
  }
  const int32_t nsrc = *a.nsrc;
  int32_t top = nsrc - 1;
  int32_t base = max(0, nsrc - SC / 2);
  v6_fill(a, S, base, top, lane);
  __syncwarp();
  int32_t p = 0, held = 0;
  int32_t* const seq = a.seq;
  int32_t* const pos_of = a.pos_of;
  // per-lane row base kept in a register (not re-read from the parameter bank each step)
  const int4* ell6l = a.ell6 + (lane & 3);
  const int4* ell6 = a.ell6;
  asm volatile("" : "+l"(ell6l), "+l"(ell6));
  const bool pf = a.prefetch;
  while (top >= 0) {
    if (top < base) {
      base = max(0, top + 1 - SC / 2);
      v6_fill(a, S, base, top, lane);
      __syncwarp();
    }
    const int32_t slot = top & (SC - 1);
    const int32_t sv = S.sid[slot];
    const int2* rowp = reinterpret_cast<const int2*>(S.row[slot]);
    const int2 cq = rowp[lane >> 2];  // child whose row this lane fetches
    const int2 my = rowp[lane & 7];   // child this lane decrements (lanes 0..7)
    --top;
    const int32_t v = sv & 0xffffff;
    if (lane == (p & 31)) held = v;  // lane k holds the node of position 32i + k
    ++p;
    if ((p & 31) == 0) {
      seq[p - 32 + lane] = held;
      pos_of[held] = p - 32 + lane;
      if ((p & 255) == 0) {
        __syncwarp();
        if (lane == 0) v6_publish(a, p);
      }
    }
    if (sv & kV6Long) {
      // ---- CSR path: rows longer than 8
      const int32_t rs = a.out_off[v], dg = a.out_off[v + 1] - rs;
      int32_t nf = 0;
      for (int32_t b0 = 0; b0 < dg; b0 += 32) {
        const int32_t k = b0 + lane;
        int2 cm = make_int2(-1, 0);
        if (k < dg) cm = a.cmeta[rs + k];
        bool fr = false;
        if (cm.x >= 0) {
          const int code = (cm.y >> 24) & 127;
          if (code == 1) fr = true;
          else if (dense) fr = v6_dense_dec(dw, cm.x) == 1u;
          else if (code == 127) fr = atomicSub(a.rem_big + cm.x, 1) == 1;
          else fr = v6_dec(S, a.gover, cm.x, code);
        }
        const unsigned m = __ballot_sync(FULL, fr);
        if (fr) {
          const int32_t at = nf + __popc(m & ((1u << lane) - 1));
          const int64_t rec = (static_cast<int64_t>(cm.y & 0xffffff) << 32) |
                              static_cast<uint32_t>(cm.x | (cm.y < 0 ? kV6Long : 0));
          if (at < kV6FreedCap) S.freed[at] = rec; else a.freed_spill[at - kV6FreedCap] = rec;
        }
        nf += __popc(m);
      }
      __syncwarp();
      if (nf > 0) {
        if (top + nf - base >= SC - 1) {
          for (int32_t i = base + lane; i <= top; i += 32) a.gsid[i] = S.sid[i & (SC - 1)];
          __syncwarp();
          base = top + 1;
        }
        const bool big = nf >= SC - 1;
        for (int32_t i = lane; i < nf; i += 32) {
          const int64_t ri = i < kV6FreedCap ? S.freed[i] : a.freed_spill[i - kV6FreedCap];
          const int32_t rk = static_cast<int32_t>(ri >> 32);
          int32_t cnt = 0;
          for (int32_t j = 0; j < nf; ++j) {
            const int64_t rj = j < kV6FreedCap ? S.freed[j] : a.freed_spill[j - kV6FreedCap];
            cnt += static_cast<int32_t>(rj >> 32) > rk;
          }
          const int32_t sidv = static_cast<int32_t>(ri & 0xffffffff);
          if (big) a.gsid[top + 1 + cnt] = sidv; else S.sid[(top + 1 + cnt) & (SC - 1)] = sidv;
        }
        __syncwarp();
        if (!big) {
          for (int32_t idx = lane; idx < nf * 4; idx += 32) {
            const int32_t e = (top + 1 + (idx >> 2)) & (SC - 1);
            const int32_t c = S.sid[e] & 0xffffff;
            S.row[e][idx & 3] = a.ell6[static_cast<int64_t>(c) * 4 + (idx & 3)];
          }
        }
        top += nf;
        if (big) base = top + 1;
        __syncwarp();
      }
      continue;
    }
    // ---- 8-slot row on chip (slots sorted by rank)
    const int q = lane >> 2;
    int4 crow = make_int4(-1, 0, -1, 0);
    if (cq.x >= 0) crow = ell6l[static_cast<int64_t>(cq.x) * 4];
    bool fr = false;
    if (dense) {
      if (lane < 8 && my.x >= 0) {
        const uint32_t code = (static_cast<uint32_t>(my.y) >> 24) & 127u;
        const uint32_t rem = code == 1u ? 1u : v6_dense_dec(dw, my.x);
        fr = rem == 1u;
        if (pf && rem == 2u) prefetch_l2(ell6 + static_cast<int64_t>(my.x) * 4);
      }
    } else if (lane < 8 && my.x >= 0) {
      // branch-light table step: one bucket load; remaining = table value on a hit, the
      // initial in-degree on a first touch (code == 1 frees without touching the table)
      const uint32_t code = (static_cast<uint32_t>(my.y) >> 24) & 127u, uc = static_cast<uint32_t>(my.x);
      const uint32_t b = v6_bucket<BB>(my.x), sh = (b & 1u) * 16;
      const uint2 w = *reinterpret_cast<const uint2*>(&S.ht[2 * b]);
      const uint32_t ov = (S.ovc[b >> 1] >> sh) & 0xffffu;
      const bool h0 = (w.x >> 7) == uc, h1 = (w.y >> 7) == uc, hit = h0 | h1;
      const uint32_t e = h0 ? w.x : w.y;
      if (code == 127u || (!hit && ov != 0u)) {
        fr = code == 127u ? atomicSub(a.rem_big + my.x, 1) == 1 : v6_dec(S, a.gover, my.x, static_cast<int>(code));
      } else {
        const uint32_t rem = hit ? (e & 127u) : code;
        fr = rem == 1u;
        // armed: one predecessor left, so this child is freed (and, if it is the best freed
        // child, popped next) when that predecessor is popped — usually many steps later.
        // Its row goes to L2 now, off the chain.
        if (pf && rem == 2u) prefetch_l2(ell6 + static_cast<int64_t>(my.x) * 4);
        if (hit) {
          S.ht[2 * b + (h0 ? 0 : 1)] = fr ? kV6Empty : e - 1;
        } else if (!fr) {  // first touch: insert (ways taken by concurrent lanes -> spill)
          const uint32_t nv = (uc << 7) | (code - 1);
          bool ok = w.x == kV6Empty && atomicCAS(&S.ht[2 * b], kV6Empty, nv) == kV6Empty;
          if (!ok) ok = w.y == kV6Empty && atomicCAS(&S.ht[2 * b + 1], kV6Empty, nv) == kV6Empty;
          if (!ok) {
            a.gover[my.x] = static_cast<int32_t>(code - 1);
            atomicAdd(&S.ovc[b >> 1], 1u << sh);
          }
        }
      }
    }
    const unsigned m = __ballot_sync(FULL, fr);
    if (m) {
      const int nf = __popc(m);
      if (top + nf - base >= SC - 1) {  // spill the lower half of the cache (rows are dropped)
        for (int32_t i = base + lane; i < base + SC / 2; i += 32) a.gsid[i] = S.sid[i & (SC - 1)];
        __syncwarp();
        base += SC / 2;
      }
      // pushed in descending rank: slot k lands above every freed slot of higher rank
      if ((m >> q) & 1u) {
        S.row[(top + 1 + __popc(m >> q >> 1)) & (SC - 1)][lane & 3] = crow;
        if (pf) {
          if (crow.x >= 0) prefetch_l2(ell6 + static_cast<int64_t>(crow.x) * 4);
          if (crow.z >= 0) prefetch_l2(ell6 + static_cast<int64_t>(crow.z) * 4);
        }
      }
      if (fr) S.sid[(top + 1 + __popc(m >> lane >> 1)) & (SC - 1)] = my.x | (my.y < 0 ? kV6Long : 0);
      top += nf;
    }
    __syncwarp();
  }
  __syncwarp();
  if (lane < (p & 31)) {
    seq[(p & ~31) + lane] = held;
    pos_of[held] = (p & ~31) + lane;
  }
  __syncwarp();
  if (lane == 0) {
    *a.emitted = p;
    v6_publish(a, p);
    if (a.debug) *a.debug = clock64() - t_start;
  }
}

template <int BB>
__device__ __forceinline__ void peel_dispatch(const PeelArgs& a, int4* smem4) {
  if (a.skip && *a.skip) return;
  if (a.v6) {
    peel_warp_v6(a, *reinterpret_cast<V6Smem<BB>*>(smem4));
    return;
  }
  int64_t* sfreed = reinterpret_cast<int64_t*>(smem4 + kStackCache);
  int32_t* srow = reinterpret_cast<int32_t*>(sfreed + kFreedCap);
  int32_t* stop = srow + 32;
  int32_t* seqbuf = stop + 32;
  if (!a.stack_mode) peel_warp(a, smem4, sfreed);
  else if (a.ellw == 8) peel_warp_v5<8>(a, reinterpret_cast<int2*>(smem4), sfreed, srow, stop, seqbuf);
  else peel_warp_v5<32>(a, reinterpret_cast<int2*>(smem4), sfreed, srow, stop, seqbuf);
}

// One CTA (one warp) per graph: independent graphs of a batched call share the launch.
constexpr int kPeelBatch = 8;
struct PeelBatch {
  PeelArgs a[kPeelBatch];
};

__global__ void __launch_bounds__(32) k_peel2(const __grid_constant__ PeelBatch b) {
  extern __shared__ int4 smem4[];
  peel_dispatch<kV6BucketBits>(b.a[blockIdx.x], smem4);
}

// ---------------------------------------------------------------- streaming DP
constexpr int kCh = 256;      // positions per staged chunk
constexpr int kInCap = 2048;  // staged in-edges per chunk
constexpr int kRing = 1024;   // memory-prefix ring (>= R + kCh + 2)

struct DpArgs {
  int32_t n, range;
  int64_t limit;
  const int32_t* seq;
  int32_t* pos_of;
  const int64_t* mem;
  const int64_t* out_sum;   // by node index
  const int32_t* in_off;    // CSC
  const int32_t* in_src;
  const int64_t* in_cost;
  const int* progress;
  int32_t* prev_cut;        // [n+1]
  int* first_exceed;
  bool keys32;              // window values fit 32-bit keys (see peel_dp_stream)
  bool block32;             // ... with 32 steps of drift headroom: 32-step block recurrence
  bool v3;                  // block32 and R <= 225: multi-warp age-ordered recurrence
  long long* debug;         // optional: [total, waiting, staging] cycles of the DP warp
  // DP v5: per-position records built by k_dp_records (order known before the DP)
  const int4* rec01;        // first two in-window in-edges {pos, cost << 8, pos, cost << 8}
  const int4* rec23;        // third and fourth
  const int4* recz;         // {lo, index of the fifth in ovf, number beyond four, 0}
  const int32_t* bext;      // per 32 positions: some position has more than four
  const int2* ovf;          // in-window in-edges beyond the fourth
};

__device__ __forceinline__ void argmin_reduce(int64_t& v, int32_t& d) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t ov = __shfl_xor_sync(FULL, v, o);
    const int32_t od = __shfl_xor_sync(FULL, d, o);
    if (ov < v || (ov == v && od < d)) {
      v = ov;
      d = od;
    }
  }
}

struct DpSmem {
  int32_t lo[kCh];
  int64_t out[kCh];
  int32_t off[kCh + 1];
  int32_t ipos[kInCap];
  int64_t ic[kInCap];
  int64_t pref[kRing];
  int32_t node[kCh];
  int32_t ioff[kCh];
  int32_t mt[32][33];  // block recurrence: per step, per lane minimum over old candidates
  int32_t ct[32][33];  // block recurrence: per step, placeholder key of block candidate k
};

__device__ void dp_warp(const DpArgs& a, DpSmem& S) {
  constexpr int SPL = 8, W = 256;
  const int lane = threadIdx.x & 31;
  const int32_t n = a.n;
  int64_t D[SPL];
#pragma unroll
  for (int r = 0; r < SPL; ++r) D[r] = 0;
  constexpr int32_t kUnfilled = 0x3f000000;
  int32_t K[SPL];
#pragma unroll
  for (int r = 0; r < SPL; ++r) K[r] = kUnfilled;
  int64_t off = 0;     // D = (K >> 8) + off
  int32_t bvr = 0;     // best of the last query, relative to off
  int64_t carry = 0;  // prefix[j0]
  long long wait_cycles = 0, stage_cycles = 0;
  const long long t_start = clock64();
  if (lane == 0) S.pref[0] = 0;
  int avail = 0;
  for (int32_t j0 = 0; j0 < n; j0 += kCh) {
    // positions [j0, j1] staged; steps j in [max(1,j0), j1+1] use them
    const int32_t j1 = min(n - 1, j0 + kCh - 1);
    const int32_t cnt = j1 - j0 + 1;
    const long long tw0 = clock64();
    while (avail < j1 + 1) {
      avail = ld_acquire(a.progress);
        if (avail < j1 + 1) __nanosleep(200);
    }
    wait_cycles += clock64() - tw0;
    // node, memory, out-cost, in-degree per position
    int32_t my_in = 0;
    for (int32_t t = lane; t < kCh; t += 32) {
      if (t < cnt) {
        const int32_t v = a.seq[j0 + t];
        S.node[t] = v;
        S.out[t] = a.out_sum[v];
        a.pos_of[v] = j0 + t;  // the peel does not write pos_of; in-edge sources read it below
      }
    }
    __syncwarp();
    __threadfence_block();
    // memory prefix (warp scan in 32-wide pieces) + exceed check
    for (int32_t t0 = 0; t0 < cnt; t0 += 32) {
      const int32_t t = t0 + lane;
      int64_t mv = t < cnt ? a.mem[S.node[t]] : 0;
      if (t < cnt && mv > a.limit) atomicMin(a.first_exceed, j0 + t);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t x = __shfl_up_sync(FULL, mv, o);
        if (lane >= o) mv += x;
      }
      if (t < cnt) S.pref[(j0 + t + 1) & (kRing - 1)] = carry + mv;
      carry += __shfl_sync(FULL, mv, 31);
    }
    // in-edge offsets (per position) and each row's CSC start
    for (int32_t t0 = 0; t0 < kCh; t0 += 32) {
      const int32_t t = t0 + lane;
      int32_t c = 0;
      if (t < cnt) {
        const int32_t v = S.node[t];
        const int32_t b = a.in_off[v];
        S.ioff[t] = b;
        c = a.in_off[v + 1] - b;
      }
      int32_t x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, x, o);
        if (lane >= o) x += y;
      }
      if (t < kCh) S.off[t + 1] = my_in + x;
      my_in += __shfl_sync(FULL, x, 31);
    }
    if (lane == 0) S.off[0] = 0;
    __syncwarp();
    const bool staged = my_in <= kInCap;
    if (staged) {
      // flattened over the chunk's in-edges, 4 independent gathers in flight per lane
      for (int32_t o0 = 0; o0 < my_in; o0 += 128) {
        int32_t src[4], oo[4];
        int64_t cc[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int32_t o = o0 + u * 32 + lane;
          oo[u] = o;
          src[u] = 0;
          cc[u] = 0;
          if (o < my_in) {
            int32_t lo = 0, hi = cnt - 1;  // last t with off[t] <= o
            while (lo < hi) {
              const int32_t mid = (lo + hi + 1) >> 1;
              if (S.off[mid] <= o) lo = mid; else hi = mid - 1;
            }
            const int32_t k = S.ioff[lo] + (o - S.off[lo]);
            src[u] = a.in_src[k];
            cc[u] = a.in_cost[k];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (oo[u] < my_in) {
            S.ipos[oo[u]] = a.pos_of[src[u]];
            S.ic[oo[u]] = cc[u];
          }
        }
      }
    }
    __syncwarp();
    // lo[j] for the steps of this chunk that produce best[j]: j = j0+t+1?  Steps use
    // lo[j] with j in [j0+1, j1+1] -> prefix indices up to j1+1 (staged above).
    for (int32_t t = lane; t < cnt; t += 32) {
      const int32_t j = j0 + t + 1;
      int32_t lo = j > a.range ? j - a.range : 0, hi = j - 1;
      const int64_t pj = S.pref[j & (kRing - 1)];
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (pj - S.pref[mid & (kRing - 1)] <= a.limit) hi = mid; else lo = mid + 1;
      }
      S.lo[t] = lo;
    }
    __syncwarp();
    stage_cycles += clock64() - tw0;
    if (a.keys32 && a.block32) {
      // ---- 32-step blocks, 32-bit keys K = (D - off) * 256 + distance, slot of candidate
      // i = lane (i & 31), register (i >> 5) & 7.  Per block [P, P+32):
      //  A. lanes advance all window slots through the 32 transitions (independent work):
      //     the minimum over the block's OLD candidates (i <= P, value known) per step goes
      //     to S.mt[step][lane]; block candidate P+k lives in lane k's register Kn, entered
      //     with a placeholder value 0 instead of best[P+k] (unknown yet), and its key per
      //     step goes to S.ct[step][k].  All later updates are additive, so its real key is
      //     placeholder + (best[P+k] - off_{P+k-1}) * 256.
      //  B. lane t: R = min_q mt[t][q], then k = 1..31 in order: best[P+k] = lane k-1's R
      //     (final once candidates < P+k are in), candidate key ct[t][k] + bestrel * 256.
      //  Ties: the smaller key has the smaller distance = the larger i (fusion.cpp:152).
      if (j0 == 0) {
        off = S.out[0];  // candidate 0: D_1(0) = out(0)
        if (lane == 0) K[0] = 0;
      }
      for (int32_t tb = 0; tb < cnt; tb += 32) {
        const int32_t P = j0 + tb;
        const int32_t nb = min(32, cnt - tb);
        const int rb = (P >> 5) & (SPL - 1);
        int32_t Kn = 0;
        for (int32_t u = 0; u < nb; ++u) {
          const int32_t t = tb + u, p = P + u;
          if (p > 0) {
#pragma unroll
            for (int r = 0; r < SPL; ++r) K[r] += 1;
            Kn += 1;
            if (u == 0) {
              if (lane == 0) {
#pragma unroll
                for (int r = 0; r < SPL; ++r)
                  if (r == rb) K[r] = bvr * 256;
              }
            } else if (lane == u) {
              Kn = 0;
            }
            const bool live_n = lane >= 1 && lane <= u;
            const int32_t kb = S.off[t], ke = S.off[t + 1];
            for (int32_t k = kb; k < ke; ++k) {
              int32_t av;
              int64_t cv;
              if (staged) {
                av = S.ipos[k];
                cv = S.ic[k];
              } else {
                av = a.pos_of[a.in_src[S.ioff[t] - kb + k]];
                cv = a.in_cost[S.ioff[t] - kb + k];
              }
              if (av <= p - W) continue;
              const int32_t thr = p - av;
              const int32_t sub = static_cast<int32_t>(cv) << 8;
#pragma unroll
              for (int r = 0; r < SPL; ++r)
                if ((K[r] & 255) >= thr) K[r] -= sub;
              if (live_n && (Kn & 255) >= thr) Kn -= sub;
            }
            off += S.out[t];
          }
          // minimum over the old candidates: u <= distance <= p - lo[p+1]
          const int32_t span = p - S.lo[t] - u;
          int32_t mk = INT32_MAX;
          if (span >= 0) {
#pragma unroll
            for (int r = 0; r < SPL; ++r)
              if (static_cast<uint32_t>((K[r] & 255) - u) <= static_cast<uint32_t>(span) && K[r] < mk) mk = K[r];
          }
          S.mt[u][lane] = mk;
          if (lane >= 1 && lane <= u) S.ct[u][lane] = Kn;
        }
        __syncwarp();
        int32_t R = INT32_MAX, maxd = -1;
        if (lane < nb) {
#pragma unroll 8
          for (int q = 0; q < 32; ++q) R = min(R, S.mt[lane][q]);
          maxd = P + lane - S.lo[tb + lane];
        }
        for (int k = 1; k < nb; ++k) {
          const int32_t b = __shfl_sync(FULL, R, k - 1) >> 8;
          const int32_t c = S.ct[lane][k];
          if (lane >= k && lane - k <= maxd) R = min(R, c + b * 256);
        }
        if (lane < nb) a.prev_cut[P + lane + 1] = P + lane - (R & 255);
        const int32_t bk = __shfl_up_sync(FULL, R, 1) >> 8;
        if (lane >= 1 && lane < nb) {
#pragma unroll
          for (int r = 0; r < SPL; ++r)
            if (r == rb) K[r] = Kn + bk * 256;
        }
        bvr = __shfl_sync(FULL, R, nb - 1) >> 8;
        if (bvr > (1 << 20) || bvr < -(1 << 20)) {
#pragma unroll
          for (int r = 0; r < SPL; ++r)
            if (K[r] < kUnfilled) K[r] -= bvr * 256;
          off += bvr;
          bvr = 0;
        }
        __syncwarp();
      }
      continue;
    }
    if (a.keys32) {
      // ---- 32-bit keys: K = (D - OFFSET) * 256 + distance; argmin = one redux.sync
      if (j0 == 0) {
        off = S.out[0];  // candidate 0: D_1(0) = out(0)
        if (lane == 0) K[0] = 0;
      }
      for (int32_t t = 0; t < cnt; ++t) {
        const int32_t p = j0 + t;
        if (p > 0) {
          // transition into position p: distances +1, candidate p enters, in-edges of p
#pragma unroll
          for (int r = 0; r < SPL; ++r) K[r] += 1;
          const int32_t sl = p & (W - 1);
#pragma unroll
          for (int r = 0; r < SPL; ++r)
            if (lane * SPL + r == sl) K[r] = bvr * 256;
          const int32_t kb = S.off[t], ke = S.off[t + 1];
          for (int32_t k = kb; k < ke; ++k) {
            int32_t av;
            int64_t cv;
            if (staged) {
              av = S.ipos[k];
              cv = S.ic[k];
            } else {
              av = a.pos_of[a.in_src[S.ioff[t] - kb + k]];
              cv = a.in_cost[S.ioff[t] - kb + k];
            }
            if (av <= p - W) continue;  // source outside the window: no candidate moves
            const int32_t thr = p - av;  // candidates i <= av  <=>  distance >= p - av
            const int32_t sub = static_cast<int32_t>(cv) << 8;
#pragma unroll
            for (int r = 0; r < SPL; ++r)
              if ((K[r] & 255) >= thr) K[r] -= sub;
          }
          off += S.out[t];
        }
        // best[p+1]
        const int32_t maxd = p - S.lo[t];
        int32_t mk = INT32_MAX;
#pragma unroll
        for (int r = 0; r < SPL; ++r)
          if ((K[r] & 255) <= maxd && K[r] < mk) mk = K[r];
        mk = __reduce_min_sync(FULL, mk);
        bvr = mk >> 8;
        if (lane == 0) a.prev_cut[p + 1] = p - (mk & 255);
        if (bvr > (1 << 20) || bvr < -(1 << 20)) {  // rebase the relative values
#pragma unroll
          for (int r = 0; r < SPL; ++r)
            if (K[r] < kUnfilled) K[r] -= bvr * 256;
          off += bvr;
          bvr = 0;
        }
      }
      __syncwarp();
      continue;
    }
    if (j0 == 0 && lane == 0) D[0] = S.out[0];  // candidate i = 0 for j = 1
    // steps: for position p = j0+t, first compute best[j] for j = p+1?  Layout: the
    // transition after best[p] uses position p's out-sum and in-edges; best[p+1] uses lo.
    for (int32_t t = 0; t < cnt; ++t) {
      const int32_t p = j0 + t;
      if (p > 0) {
        // transition from step p to p+1: position p enters (out-sum, in-edges)
        const int64_t o = S.out[t];
#pragma unroll
        for (int r = 0; r < SPL; ++r) D[r] += o;
        const int32_t kb = S.off[t], ke = S.off[t + 1];
        const int32_t gkb = S.ioff[t] - kb;
        for (int32_t base = kb; base < ke; base += 32) {
          int32_t av = -1;
          int64_t cv = 0;
          if (base + lane < ke) {
            if (staged) {
              av = S.ipos[base + lane];
              cv = S.ic[base + lane];
            } else {
              av = a.pos_of[a.in_src[gkb + base + lane]];
              cv = a.in_cost[gkb + base + lane];
            }
          }
          const int c = min(32, ke - base);
          for (int q = 0; q < c; ++q) {
            const int32_t at = __shfl_sync(FULL, av, q);
            const int64_t ct = __shfl_sync(FULL, cv, q);
            if (at <= p - W) continue;
#pragma unroll
            for (int r = 0; r < SPL; ++r) {
              const int32_t s = lane * SPL + r;
              const int32_t i2 = p - ((p - s) & (W - 1));
              if (i2 <= at) D[r] -= ct;
            }
          }
        }
        // new candidate i = p: best[p] + out(p) — best[p] was broadcast as `bestp`
      }
      // best[p+1]
      const int32_t j = p + 1;
      const int32_t loj = S.lo[t];
      int64_t bv = INT64_MAX;
      int32_t bd = INT32_MAX;
#pragma unroll
      for (int r = 0; r < SPL; ++r) {
        const int32_t s = lane * SPL + r;
        const int32_t d = (j - 1 - s) & (W - 1);
        if (j - 1 - d >= loj && (D[r] < bv || (D[r] == bv && d < bd))) {
          bv = D[r];
          bd = d;
        }
      }
      argmin_reduce(bv, bd);
      if (lane == 0) a.prev_cut[j] = j - 1 - bd;
      // candidate i = j enters with best[j] + out(j); out(j) is added at the next
      // transition, so store best[j] now
      if (j < n) {
        const int32_t sl = j & (W - 1);
#pragma unroll
        for (int r = 0; r < SPL; ++r)
          if (lane * SPL + r == sl) D[r] = bv;
      }
    }
    __syncwarp();
  }
  if (lane == 0 && a.debug) {
    a.debug[0] = clock64() - t_start;
    a.debug[1] = wait_cycles;
    a.debug[2] = stage_cycles - wait_cycles;
  }
}


// ---------------------------------------------------------------- DP v3 (R <= 225)
// One compute warp plus kDpProducers staging warps per DP CTA.  Producer k stages chunks
// k, k + P, ... (256 positions each) into its own buffer — node, out-cost sum, lo[j] from a
// local memory prefix, in-edges as (source position, cost) — so staging latency is off
// the recurrence's path.  The compute warp keeps the window in AGE order: lane l holds
// old candidates i = B - 224 + 32r + l (r = 0..6, B = block start) in K[r] and the block's
// own candidate B + l in Kn; keys are (value - off) * 256 + (255 - (i - (B - 224))), so the
// tie-break byte is fixed inside a block (no per-step increments), "i <= a" is r <= a
// shifted by 5, and each block ends with one register rotation.  Blocks run the two-phase
// recurrence of the block32 path (independent slot updates, then a 31-step chain over the
// block's own candidates).
constexpr int kDpProducers = 3;
constexpr int kLpMax = 256 + kCh + 1;
// compacted in-edges per staged chunk (more: the chunk is read from HBM); 1,024 when the DP
// shares its SM with the peel (k_peel_dp_shared)
constexpr int kE2Cap = 4096;
constexpr int kE2CapShared = 1024;

template <int E2, bool REC = false>
struct DpBuf {
  int32_t lo[kCh];   // lo[j] for j = j0 + t + 1 (absolute position)
  int64_t out[kCh];
  int32_t off[kCh + 1];   // all in-edges of position t: [off[t], off[t+1])
  int32_t off2[kCh + 1];  // in-window in-edges of position t in e2
  int32_t cnt2[kCh];
  int2 e2[E2 + 2];    // {source position, cost << 8}, sources >= block start - 224
  int32_t ioff[kCh];
  int64_t lp[kLpMax];
  int32_t node[kCh];
  int32_t cnt, n2;        // n2 > kE2Cap: the compute warp reads in-edges from HBM
  // DP v5: per position the first four in-window in-edges {pos, cost << 8} (cost 0 past
  // the count) and {lo, index of the fifth, number beyond four, 0}, read with broadcast
  // loads; per 32-position block whether any position has more than four
  int4 r01[REC ? kCh : 1];
  int4 r23[REC ? kCh : 1];
  int4 rz[REC ? kCh : 1];
  int32_t bext[REC ? kCh / 32 : 1];
};

template <int E2>
struct DpSmem3 {
  DpBuf<E2> buf[kDpProducers];
  int32_t mt[32][33];
  int32_t ct[32][33];
  int ready[kDpProducers];
  int consumed;
};

__device__ __forceinline__ int ld_volatile_shared(const int* p) { return *reinterpret_cast<const volatile int*>(p); }

template <int E2, bool REC>
__device__ void dp_stage(const DpArgs& a, DpBuf<E2, REC>& B, int32_t j0, int32_t cnt, int lane) {
  for (int32_t t = lane; t < cnt; t += 32) {
    const int32_t v = a.seq[j0 + t];
    B.node[t] = v;
    B.out[t] = a.out_sum[v];
  }
  // memory prefix over positions [b0, j0 + cnt): the window of every j in the chunk
  const int32_t b0 = max(0, j0 - a.range);
  const int32_t L = j0 + cnt - b0;
  int64_t carry = 0;
  if (lane == 0) B.lp[0] = 0;
  for (int32_t x0 = 0; x0 < L; x0 += 32) {
    const int32_t x = x0 + lane;
    int64_t mv = 0;
    if (x < L) {
      const int32_t pos = b0 + x;
      mv = a.mem[a.seq[pos]];
      if (pos >= j0 && mv > a.limit) atomicMin(a.first_exceed, pos);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(FULL, mv, o);
      if (lane >= o) mv += y;
    }
    if (x < L) B.lp[x + 1] = carry + mv;
    carry += __shfl_sync(FULL, mv, 31);
  }
  __syncwarp();
  for (int32_t t = lane; t < cnt; t += 32) {
    const int32_t j = j0 + t + 1;
    int32_t lo = max(0, j - a.range), hi = j - 1;
    const int64_t pj = B.lp[j - b0];
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (pj - B.lp[mid - b0] <= a.limit) hi = mid; else lo = mid + 1;
    }
    B.lo[t] = lo;
  }
  // in-edge offsets per position
  int32_t my_in = 0;
  for (int32_t t0 = 0; t0 < kCh; t0 += 32) {
    const int32_t t = t0 + lane;
    int32_t c = 0;
    if (t < cnt) {
      const int32_t v = B.node[t];
      const int32_t b = a.in_off[v];
      B.ioff[t] = b;
      c = a.in_off[v + 1] - b;
    }
    if (t < kCh) B.cnt2[t] = 0;
    int32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    if (t < kCh) B.off[t + 1] = my_in + x;
    my_in += __shfl_sync(FULL, x, 31);
  }
  if (lane == 0) B.off[0] = 0;
  __syncwarp();
  // gather (source position, cost) of every in-edge; keep those whose source can still
  // be a candidate in the edge's block (>= block start - 224), compacted in edge order
  int32_t n2 = 0;
  for (int32_t o0 = 0; o0 < my_in; o0 += 128) {
    int32_t src[4], tt[4];
    int64_t cc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int32_t o = o0 + u * 32 + lane;
      src[u] = -1;
      cc[u] = 0;
      tt[u] = 0;
      if (o < my_in) {
        int32_t lo = 0, hi = cnt - 1;  // last t with off[t] <= o
        while (lo < hi) {
          const int32_t mid = (lo + hi + 1) >> 1;
          if (B.off[mid] <= o) lo = mid; else hi = mid - 1;
        }
        const int32_t k = B.ioff[lo] + (o - B.off[lo]);
        tt[u] = lo;
        src[u] = a.in_src[k];
        cc[u] = a.in_cost[k];
      }
    }
    int32_t av[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) av[u] = src[u] >= 0 ? a.pos_of[src[u]] : -1;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool keep = src[u] >= 0 && av[u] >= j0 + (tt[u] & ~31) - 224;
      const unsigned m = __ballot_sync(FULL, keep);
      if (keep) {
        const int32_t idx = n2 + __popc(m & ((1u << lane) - 1));
        if (idx < E2) B.e2[idx] = make_int2(av[u], static_cast<int32_t>(cc[u]) << 8);
        atomicAdd(&B.cnt2[tt[u]], 1);
      }
      n2 += __popc(m);
    }
  }
  __syncwarp();
  int32_t run = 0;
  for (int32_t t0 = 0; t0 < kCh; t0 += 32) {
    const int32_t t = t0 + lane;
    int32_t x = B.cnt2[t];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, x, o);
      if (lane >= o) x += y;
    }
    B.off2[t + 1] = run + x;
    run += __shfl_sync(FULL, x, 31);
  }
  if (lane == 0) {
    B.off2[0] = 0;
    B.cnt = cnt;
    B.n2 = n2;
  }
  if constexpr (REC) {
    __syncwarp();
    if (n2 <= E2) {
      for (int32_t t0 = 0; t0 < cnt; t0 += 32) {
        const int32_t t = t0 + lane;
        int32_t ex = 0;
        if (t < cnt) {
          const int32_t eb = B.off2[t], ee = B.off2[t + 1];
          int2 x[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) x[q] = eb + q < ee ? B.e2[eb + q] : make_int2(0, 0);
          B.r01[t] = make_int4(x[0].x, x[0].y, x[1].x, x[1].y);
          B.r23[t] = make_int4(x[2].x, x[2].y, x[3].x, x[3].y);
          ex = max(0, ee - eb - 4);
          B.rz[t] = make_int4(B.lo[t], eb + 4, ex, 0);
        }
        const unsigned any = __ballot_sync(FULL, ex > 0);
        if (lane == 0) B.bext[t0 >> 5] = any != 0;
      }
    }
  }
}

template <typename SmemT>
__device__ void dp_producer(const DpArgs& a, SmemT& S, int k, int lane) {
  int avail = 0;
  for (int32_t c = k;; c += kDpProducers) {
    const int32_t j0 = c * kCh;
    if (j0 >= a.n) break;
    const int32_t j1 = min(a.n - 1, j0 + kCh - 1);
    while (ld_volatile_shared(&S.consumed) < c - kDpProducers + 1) __nanosleep(1000);
    while (avail < j1 + 1) {
      avail = ld_acquire(a.progress);
      if (avail < j1 + 1) __nanosleep(200);
    }
    dp_stage(a, S.buf[k], j0, j1 - j0 + 1, lane);
    __syncwarp();
    __threadfence_block();
    if (lane == 0) *reinterpret_cast<volatile int*>(&S.ready[k]) = c;
  }
}

template <int E2>
__device__ void dp_compute_v3(const DpArgs& a, DpSmem3<E2>& S) {
  constexpr int NR = 7;
  const int lane = threadIdx.x & 31;
  const int32_t n = a.n;
  constexpr int32_t kUnfilled = 0x3f000000;
  int32_t K[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) K[r] = kUnfilled;
  int32_t Kn = kUnfilled;
  int64_t off = 0;   // candidate 0 enters with best[0] = 0 relative to off = 0
  int32_t bvr = 0;
  long long wait_cycles = 0;
  const long long t_start = clock64();
  for (int32_t c = 0;; ++c) {
    const int32_t j0 = c * kCh;
    if (j0 >= n) break;
    const int kb = c % kDpProducers;
    const long long tw0 = clock64();
    while (ld_volatile_shared(&S.ready[kb]) != c) __nanosleep(32);
    wait_cycles += clock64() - tw0;
    __threadfence_block();
    const DpBuf<E2>& B = S.buf[kb];
    const int32_t cnt = B.cnt;
    const bool staged = B.n2 <= E2;
    for (int32_t tb = 0; tb < cnt; tb += 32) {
      const int32_t P = j0 + tb;
      const int32_t nb = min(32, cnt - tb);
      const int32_t c0 = 224 - P - lane;
      const int32_t kn_lim = -P - lane;  // Kn (candidate P + lane) loses c iff av + kn_lim >= 0
#pragma unroll 1
      for (int32_t u = 0; u < nb; ++u) {
        const int32_t t = tb + u;
        if (lane == u) Kn = (u == 0 ? bvr * 256 : 0) + 31 - u;
        if (staged) {
          // most steps have at most two in-window in-edges: apply two unconditionally
          // (masked to zero past the step's range), loop over the rest
          const int32_t eb = B.off2[t], ee = B.off2[t + 1];
          const int2 x0 = B.e2[eb], x1 = B.e2[eb + 1];
          const int32_t s0 = eb < ee ? x0.y : 0, s1 = eb + 1 < ee ? x1.y : 0;
          const int32_t r0 = (x0.x + c0) >> 5, r1 = (x1.x + c0) >> 5;
#pragma unroll
          for (int r = 0; r < NR; ++r) K[r] -= (r <= r0 ? s0 : 0) + (r <= r1 ? s1 : 0);
          Kn -= (x0.x + kn_lim >= 0 ? s0 : 0) + (x1.x + kn_lim >= 0 ? s1 : 0);
          for (int32_t e = eb + 2; e < ee; ++e) {
            const int2 x = B.e2[e];
            const int32_t rmax = (x.x + c0) >> 5;
#pragma unroll
            for (int r = 0; r < NR; ++r) K[r] -= r <= rmax ? x.y : 0;
            Kn -= x.x + kn_lim >= 0 ? x.y : 0;
          }
        } else {
          const int32_t eb = B.off[t], ee = B.off[t + 1];
          for (int32_t e = eb; e < ee; ++e) {
            const int32_t k = B.ioff[t] + (e - eb);
            const int32_t av = a.pos_of[a.in_src[k]];
            if (av < P - 224) continue;
            const int32_t sub = static_cast<int32_t>(a.in_cost[k]) << 8;
            const int32_t rmax = (av + c0) >> 5;
#pragma unroll
            for (int r = 0; r < NR; ++r) K[r] -= r <= rmax ? sub : 0;
            Kn -= av + kn_lim >= 0 ? sub : 0;
          }
        }
        off += B.out[t];
        // minimum over the old candidates i in [lo[p+1], P] (tree)
        const int32_t lo = B.lo[t];
        const int32_t rmin = (lo + c0 + 31) >> 5;
        int32_t mv[8];
#pragma unroll
        for (int r = 0; r < NR; ++r) mv[r] = r >= rmin ? K[r] : INT32_MAX;
        mv[7] = (lane == 0 && P >= lo) ? Kn : INT32_MAX;
        const int32_t m01 = min(mv[0], mv[1]), m23 = min(mv[2], mv[3]), m45 = min(mv[4], mv[5]),
                      m67 = min(mv[6], mv[7]);
        S.mt[u][lane] = min(min(m01, m23), min(m45, m67));
        if (lane >= 1 && lane <= u) S.ct[u][lane] = Kn;
      }
      __syncwarp();
      int32_t R = INT32_MAX, kmin = 0;
      if (lane < nb) {
        int32_t r4[4] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX};
#pragma unroll
        for (int q = 0; q < 32; ++q) r4[q & 3] = min(r4[q & 3], S.mt[lane][q]);
        R = min(min(r4[0], r4[1]), min(r4[2], r4[3]));
        kmin = B.lo[tb + lane] - P;
      }
      for (int k = 1; k < nb; ++k) {
        const int32_t b = __shfl_sync(FULL, R, k - 1) >> 8;
        const int32_t cc = S.ct[lane][k];
        if (lane >= k && k >= kmin) R = min(R, cc + b * 256);
      }
      if (lane < nb) a.prev_cut[P + lane + 1] = P + 31 - (R & 255);
      const int32_t bk = __shfl_up_sync(FULL, R, 1) >> 8;
      if (lane >= 1) Kn += bk * 256;
#pragma unroll
      for (int r = 0; r < NR - 1; ++r) K[r] = K[r + 1] + 32;
      K[NR - 1] = Kn + 32;
      bvr = __shfl_sync(FULL, R, nb - 1) >> 8;
      if (bvr > (1 << 20) || bvr < -(1 << 20)) {
#pragma unroll
        for (int r = 0; r < NR; ++r)
          if (K[r] < kUnfilled) K[r] -= bvr * 256;
        off += bvr;
        bvr = 0;
      }
      __syncwarp();
    }
    __syncwarp();
    if (lane == 0) *reinterpret_cast<volatile int*>(&S.consumed) = c + 1;
  }
  if (lane == 0 && a.debug) {
    a.debug[0] = clock64() - t_start;
    a.debug[1] = wait_cycles;
    a.debug[2] = 0;
  }
}

// ---------------------------------------------------------------- DP v5 records
// What the staging warps compute per chunk for v3 (dp_stage), computed once for every
// position in parallel when the order is complete: lo (window start under the memory
// limit, by binary search over the position-order memory prefix), the first-exceed check,
// and the in-window in-edges (source position >= block start - 224) — the first four in
// 16-byte records, the rest in an overflow list (order-free: they are summed).
__global__ void k_mem_by_pos(const int32_t* seq, const int64_t* mem, int32_t n, int64_t* out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p <= n; p += (int64_t)gridDim.x * blockDim.x)
    out[p] = p < n ? mem[seq[p]] : 0;
}

__global__ void __launch_bounds__(256) k_dp_records(DpArgs a, const int64_t* mp, int4* rec01, int4* rec23, int4* recz,
                                                    int32_t* bext, int2* ovf, int* ovf_count) {
  const int lane = threadIdx.x & 31;
  const int32_t n = a.n;
  for (int64_t p0 = blockIdx.x * (int64_t)blockDim.x; p0 < n; p0 += (int64_t)gridDim.x * blockDim.x) {
    const int32_t p = static_cast<int32_t>(p0) + threadIdx.x;
    int32_t cnt = 0;
    if (p < n) {
      const int32_t v = a.seq[p];
      if (a.mem[v] > a.limit) atomicMin(a.first_exceed, p);
      // lo: smallest i in [max(0, j - R), j - 1] with mp[j] - mp[i] <= limit, j = p + 1
      const int32_t j = p + 1;
      int32_t lo = max(0, j - a.range), hi = j - 1;
      const int64_t pj = mp[j];
      while (lo < hi) {
        const int32_t mid = (lo + hi) >> 1;
        if (pj - mp[mid] <= a.limit) hi = mid; else lo = mid + 1;
      }
      const int32_t P = p & ~31;
      const int32_t kb = a.in_off[v], ke = a.in_off[v + 1];
      int2 x[4] = {make_int2(0, 0), make_int2(0, 0), make_int2(0, 0), make_int2(0, 0)};
      for (int32_t k = kb; k < ke; ++k) {
        const int32_t av = a.pos_of[a.in_src[k]];
        if (av < P - 224) continue;
        const int2 e = make_int2(av, static_cast<int32_t>(a.in_cost[k]) << 8);
        if (cnt < 4) x[cnt] = e;
        ++cnt;
      }
      int32_t off = 0;
      if (cnt > 4) {
        off = atomicAdd(ovf_count, cnt - 4);
        int32_t q = 0;
        for (int32_t k = kb; k < ke; ++k) {
          const int32_t av = a.pos_of[a.in_src[k]];
          if (av < P - 224) continue;
          if (q >= 4) ovf[off + q - 4] = make_int2(av, static_cast<int32_t>(a.in_cost[k]) << 8);
          ++q;
        }
      }
      rec01[p] = make_int4(x[0].x, x[0].y, x[1].x, x[1].y);
      rec23[p] = make_int4(x[2].x, x[2].y, x[3].x, x[3].y);
      recz[p] = make_int4(lo, off, max(0, cnt - 4), 0);
    }
    const unsigned any = __ballot_sync(FULL, cnt > 4);
    if (lane == 0 && p < n + 31) bext[p >> 5] = any != 0;
  }
}

// ---------------------------------------------------------------- DP v5 (order known)
// The v3 recurrence for graphs whose order is complete before the DP starts (tree peel,
// fixpoint.cu), on kDp5Slots = 8 slot warps, one chain warp and the staging warps.
//  * Slots.  v3's eight candidate rows (seven old rows + the block's own candidates) live
//    in a ring, one slot per warp: in block b slot b & 7 holds the block's candidates and
//    slot s the old row r = (s - b - 1) & 7, so v3's register rotation becomes "+32 on
//    every key" in each warp (the tie byte of a fixed candidate grows by 32 per block).
//    Lane l of row r holds candidate i = P - 224 + 32 r + l (P = block start; the new slot:
//    i = P + l); an in-edge from position a lowers it iff a >= i, and it is eligible at a
//    step iff i >= lo.  Per step a slot warp applies the step's in-window in-edges (the
//    first four from staged records, broadcast loads) and stores its per-lane minimum; per
//    block it reduces its 32 x 32 minima (lane = step) and arrives at the block's barrier.
//  * Chain.  One warp runs v3's phase B for block b while the slot warps already work on
//    block b + 1: it takes the slot minima, then the 32-step chain over the block's own
//    candidates — candidate P included (k = 0, with the carried best[P]), so the new slot
//    never needs a chain result to start — and publishes the block's best values.  Only
//    the warp whose slot becomes row 6 at b + 1 waits for chain(b) (to add those values);
//    all slot warps stay at most one block ahead.
//  * Rebase.  Keys are 32-bit (value << 8 | tie byte) relative to a moving frame; when
//    chain(b) sees the carried value leave +-2^20 it publishes a shift that every warp
//    applies at the start of block b + 2, one block later than v3 (the slot warps are
//    already in block b + 1), and the chain adjusts its carry accordingly.
// Bit-identical to v3 (tests/test_gpu_paths.py, test_gpu_fixpoint.py).
constexpr int kDp5Slots = 8;
// A chunk's records (k_dp_records), copied by a staging warp.
struct Dp5Buf {
  int4 r01[kCh];
  int4 r23[kCh];
  int4 rz[kCh];
  int32_t bext[kCh / 32];
  int32_t cnt, n2;
};

template <int E2>
struct DpSmem5 {
  Dp5Buf buf[kDpProducers];
  int32_t mt[kDp5Slots][32][33];  // per slot warp, private: minimum per step and lane
  int32_t ct[2][32][33];          // new slot's keys per step (lanes <= step), by block parity
  int32_t rw[2][kDp5Slots][32];   // per slot warp: minimum per step, by block parity
  int32_t bk[2][32];              // chain: best values of the block's candidates
  int32_t rebase[2];              // chain(b): frame shift applied from block b + 2 on
  int chain_done;                 // chains completed
  int ready[kDpProducers];
  int consumed;
};
constexpr int kDp5Threads = (kDp5Slots + 1 + kDpProducers) * 32;

__device__ __forceinline__ void dp5_arrive(int p) {
  asm volatile("bar.arrive %0, %1;" ::"r"(3 + p), "r"((kDp5Slots + 1) * 32) : "memory");
}
__device__ __forceinline__ void dp5_wait(int p) {
  asm volatile("bar.sync %0, %1;" ::"r"(3 + p), "r"((kDp5Slots + 1) * 32) : "memory");
}

// One step of a slot warp (u: step in the block; q, q2, z: the position's staged records).
// NEW: the block's own candidates (enter at their step, keys to ct); else an old row
// (minimum to mt).
template <bool NEW, bool EXT, int E2>
__device__ __forceinline__ void dp5_step(const Dp5Buf& B, DpSmem5<E2>& S, int32_t (*__restrict__ mtw)[33],
                                         int p, int32_t u, const int4& q, const int4& q2, const int4& z, int32_t il,
                                         int lane, int32_t& K, const int2* ovf) {
  if (NEW && lane == u) K = 31 - u;  // enters with best = 0 (the chain adds it) + tie byte
  K -= (q.x >= il ? q.y : 0) + (q.z >= il ? q.w : 0) + (q2.x >= il ? q2.y : 0) + (q2.z >= il ? q2.w : 0);
  if (EXT && z.z) {
    for (int32_t e = z.y; e < z.y + z.z; ++e) {
      const int2 x = ovf[e];
      K -= x.x >= il ? x.y : 0;
    }
  }
  if (NEW) {
    if (lane <= u) S.ct[p][u][lane] = K;
  } else {
    mtw[u][lane] = il >= z.x ? K : INT32_MAX;
  }
}


template <bool NEW, int E2>
__device__ __forceinline__ void dp5_block(const DpArgs& a, const Dp5Buf& B, DpSmem5<E2>& S,
                                          int32_t (*mtw)[33], int p, int32_t tb, int32_t nb, bool staged, int32_t P,
                                          int32_t il, int lane, int32_t& K) {
  const int4* __restrict__ r01 = B.r01;
  const int4* __restrict__ r23 = B.r23;
  const int4* __restrict__ rz = B.rz;
  if (staged && nb == 32 && !B.bext[tb >> 5]) {  // no position beyond four in-window in-edges
    // records of step u + 4 load while step u computes
    int4 q0 = r01[tb], q02 = r23[tb], z0 = rz[tb];
    int4 q1 = r01[tb + 1], q12 = r23[tb + 1], z1 = rz[tb + 1];
    int4 q2 = r01[tb + 2], q22 = r23[tb + 2], z2 = rz[tb + 2];
    int4 q3 = r01[tb + 3], q32 = r23[tb + 3], z3 = rz[tb + 3];
#pragma unroll 8
    for (int32_t u = 0; u < 32; ++u) {
      const int32_t tn = tb + min(u + 4, 31);
      const int4 qn = r01[tn], qn2 = r23[tn], zn = rz[tn];
      dp5_step<NEW, false>(B, S, mtw, p, u, q0, q02, z0, il, lane, K, a.ovf);
      q0 = q1; q02 = q12; z0 = z1;
      q1 = q2; q12 = q22; z1 = z2;
      q2 = q3; q22 = q32; z2 = z3;
      q3 = qn; q32 = qn2; z3 = zn;
    }
    return;
  }
  for (int32_t u = 0; u < nb; ++u) {
    const int32_t t = tb + u;
    dp5_step<NEW, true>(B, S, mtw, p, u, r01[t], r23[t], rz[t], il, lane, K, a.ovf);
  }
}

// DP v5 staging: copy a chunk's records (12 KB) into its buffer; one warp per buffer.
template <int E2>
__device__ void dp_producer_v5(const DpArgs& a, DpSmem5<E2>& S, int k, int lane) {
  for (int32_t c = k;; c += kDpProducers) {
    const int32_t j0 = c * kCh;
    if (j0 >= a.n) break;
    const int32_t cnt = min(kCh, a.n - j0);
    while (ld_volatile_shared(&S.consumed) < c - kDpProducers + 1) __nanosleep(2000);  // a chunk lasts ~10 us
    Dp5Buf& B = S.buf[k];
    for (int32_t t = lane; t < cnt; t += 32) {
      B.r01[t] = a.rec01[j0 + t];
      B.r23[t] = a.rec23[j0 + t];
      B.rz[t] = a.recz[j0 + t];
    }
    if (lane < kCh / 32) B.bext[lane] = lane * 32 < cnt ? a.bext[(j0 >> 5) + lane] : 0;
    if (lane == 0) {
      B.cnt = cnt;
      B.n2 = 0;
    }
    __syncwarp();
    __threadfence_block();
    if (lane == 0) *reinterpret_cast<volatile int*>(&S.ready[k]) = c;
  }
}

template <int E2>
__device__ void dp_slot_v5(const DpArgs& a, DpSmem5<E2>& S, int w) {
  const int lane = threadIdx.x & 31;
  const int32_t n = a.n;
  constexpr int32_t kUnfilled = 0x3f000000;
  int32_t K = kUnfilled;
  long long cyc_wait = 0;
  int32_t blk = 0;
  int32_t(*mtw)[33] = S.mt[w];
  for (int32_t c = 0;; ++c) {
    const int32_t j0 = c * kCh;
    if (j0 >= n) break;
    const int kb = c % kDpProducers;
    while (ld_volatile_shared(&S.ready[kb]) != c) __nanosleep(32);
    __threadfence_block();
    const Dp5Buf& B = S.buf[kb];
    const int32_t cnt = B.cnt;
    const bool staged = B.n2 <= E2;
    for (int32_t tb = 0; tb < cnt; tb += 32, ++blk) {
      const int32_t P = j0 + tb;
      const int32_t nb = min(32, cnt - tb);
      const int p = blk & 1;
      const int32_t r = (w - blk - 1) & 7;  // 7: this block's own candidates
      if (blk >= 2) {  // at most one block ahead of the chain; then the frame shift of chain(blk - 2)
        const long long t0 = a.debug ? clock64() : 0;
        while (ld_volatile_shared(&S.chain_done) < blk - 1) __nanosleep(20);
        __threadfence_block();
        if (a.debug) cyc_wait += clock64() - t0;
        const int32_t d = S.rebase[p];
        if (d != 0 && K < kUnfilled) K -= d * 256;
      }
      const int32_t il = r == 7 ? P + lane : P - 224 + 32 * r + lane;  // this lane's candidate
      if (r == 7) dp5_block<true>(a, B, S, mtw, p, tb, nb, staged, P, il, lane, K);
      else dp5_block<false>(a, B, S, mtw, p, tb, nb, staged, P, il, lane, K);
      __syncwarp();
      // row 6 holds the previous block's candidates: their best values (chain(blk - 1)) are
      // added now — to the keys, and inside the reduction to the stored minima
      const bool fix = r == 6 && blk >= 1;
      if (fix) {
        const long long t0 = a.debug ? clock64() : 0;
        while (ld_volatile_shared(&S.chain_done) < blk) __nanosleep(20);
        __threadfence_block();
        if (a.debug) cyc_wait += clock64() - t0;
        K += S.bk[(blk - 1) & 1][lane] * 256;
      }
      int32_t m = INT32_MAX;
      if (r != 7 && lane < nb) {
        int32_t r4[4] = {INT32_MAX, INT32_MAX, INT32_MAX, INT32_MAX};
        if (fix) {
          const int32_t* bkp = S.bk[(blk - 1) & 1];
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const int32_t x = mtw[lane][q];
            r4[q & 3] = min(r4[q & 3], x == INT32_MAX ? INT32_MAX : x + bkp[q] * 256);
          }
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q) r4[q & 3] = min(r4[q & 3], mtw[lane][q]);
        }
        m = min(min(r4[0], r4[1]), min(r4[2], r4[3]));
      }
      S.rw[p][w][lane] = m;
      K += 32;
      __syncwarp();
      dp5_arrive(p);
    }
  }
  if (w == 0 && lane == 0 && a.debug) a.debug[5] = cyc_wait;
}

template <int E2>
__device__ void dp_chain_v5(const DpArgs& a, DpSmem5<E2>& S) {
  const int lane = threadIdx.x & 31;
  const int32_t n = a.n;
  const long long t_start = clock64();
  long long cyc_chain = 0, cyc_wait = 0, cyc_ld = 0, cyc_loop = 0;
  int32_t carry = 0;  // best[P] of the next block, in that block's frame
  int32_t pend = 0;   // shift published by the previous chain
  int32_t blk = 0;
  for (int32_t c = 0;; ++c) {
    const int32_t j0 = c * kCh;
    if (j0 >= n) break;
    const int kb = c % kDpProducers;
    while (ld_volatile_shared(&S.ready[kb]) != c) __nanosleep(32);
    __threadfence_block();
    const Dp5Buf& B = S.buf[kb];
    const int32_t cnt = B.cnt;
    for (int32_t tb = 0; tb < cnt; tb += 32, ++blk) {
      const int32_t P = j0 + tb;
      const int32_t nb = min(32, cnt - tb);
      const int p = blk & 1;
      const long long t0 = a.debug ? clock64() : 0;
      dp5_wait(p);
      const long long t1 = a.debug ? clock64() : 0;
      int32_t R = INT32_MAX, kmin = 0;
      if (lane < nb) {
#pragma unroll
        for (int q = 0; q < kDp5Slots; ++q) R = min(R, S.rw[p][q][lane]);
        kmin = B.rz[tb + lane].x - P;
      }
      int32_t cc[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) cc[k] = S.ct[p][lane][k];
      if (a.debug) {
        const long long tl = clock64();
        cyc_ld += tl - t1;
      }
      const long long t2 = a.debug ? clock64() : 0;
      if (0 >= kmin) R = min(R, cc[0] + carry * 256);
      if (nb == 32) {
        // two candidates per shuffle round: with R_{k-1} (final) and lane k's partial R_k
        // fetched together, every lane finishes R_k itself (candidate k is always eligible
        // at its own step), so b_{k+1} needs no second round trip
        int32_t ukk[32];
#pragma unroll
        for (int k = 1; k < 32; k += 2) ukk[k] = S.ct[p][k][k];
#pragma unroll
        for (int k = 1; k < 32; k += 2) {
          const int32_t x = __shfl_sync(FULL, R, k - 1), y = __shfl_sync(FULL, R, k);
          const int32_t bk = x & ~255;  // (R_{k-1} >> 8) * 256
          if (k + 1 < 32) {
            const int32_t bk1 = min(y, ukk[k] + bk) & ~255;
            if (lane >= k && k >= kmin) R = min(R, cc[k] + bk);
            if (lane >= k + 1 && k + 1 >= kmin) R = min(R, cc[k + 1] + bk1);
          } else {
            if (lane >= k && k >= kmin) R = min(R, cc[k] + bk);
          }
        }
      } else {
        for (int k = 1; k < nb; ++k) {
          const int32_t b = __shfl_sync(FULL, R, k - 1) & ~255;
          const int32_t ck = S.ct[p][lane][k];
          if (lane >= k && k >= kmin) R = min(R, ck + b);
        }
      }
      if (a.debug) cyc_loop += clock64() - t2;
      const int32_t up = __shfl_up_sync(FULL, R, 1) >> 8;
      S.bk[p][lane] = lane == 0 ? carry : up;
      const int32_t cout = __shfl_sync(FULL, R, nb - 1) >> 8;
      carry = cout - pend;  // into the next block's frame
      const int32_t d = (carry > (1 << 20) || carry < -(1 << 20)) ? carry : 0;
      if (lane == 0) S.rebase[p] = d;  // frame of block blk + 2 = frame of blk + 1 - d
      pend = d;
      __syncwarp();
      __threadfence_block();  // shared-memory results before the flag (the global store follows it)
      if (lane == 0) *reinterpret_cast<volatile int*>(&S.chain_done) = blk + 1;
      if (lane < nb) a.prev_cut[P + lane + 1] = P + 31 - (R & 255);
      if (a.debug) {
        cyc_wait += t1 - t0;
        cyc_chain += clock64() - t1;
      }
    }
    __syncwarp();
    if (lane == 0) *reinterpret_cast<volatile int*>(&S.consumed) = c + 1;
  }
  if (lane == 0 && a.debug) {
    a.debug[0] = clock64() - t_start;
    a.debug[1] = 0;
    a.debug[2] = 0;
    a.debug[4] = cyc_wait;
    a.debug[6] = cyc_chain;
    a.debug[2] = cyc_ld;
    a.debug[7] = cyc_loop;
  }
}

// Up to kPeelDpBatch independent graphs per launch.  Shared mode (k_peel_dp_shared): one
// CTA per graph — warp 0 peels, warp 1 runs the DP recurrence, warps 2, 3, 5 stage DP
// chunks (warp 4 exits at once so that the peel warp keeps its SM sub-partition: warps map
// to sub-partitions by index mod 4); shared memory holds the peel's region (8,192 buckets),
// then the DP's (1,024 staged in-edges per chunk).  The peel and DP talk through the
// progress counter only, so one SM per graph and no co-scheduling.  Pair mode (k_peel_dp,
// a single graph): the peel warp and the DP warps get an SM each, with the full-size tables
// (cooperative launch: the two CTAs must be co-resident).
constexpr int kPeelDpBatch = 8;
constexpr int kPeelDpWarps = 6;
constexpr int kDpPairWarps = 1 + kDpProducers;
struct PeelDpBatch {
  PeelArgs pa[kPeelDpBatch];
  DpArgs da[kPeelDpBatch];
};
constexpr size_t kPeelSmemV5 = sizeof(int4) * kStackCache + sizeof(int64_t) * kFreedCap + sizeof(int32_t) * 96;
constexpr size_t kPeelRegion = (std::max(kPeelSmemV5, sizeof(V6Smem<kV6BucketBits>)) + 127) / 128 * 128;
constexpr size_t kPeelRegionShared = (std::max(kPeelSmemV5, sizeof(V6Smem<kV6BucketBitsShared>)) + 127) / 128 * 128;
constexpr size_t kSmemPair =
    std::max(kPeelRegion, std::max(sizeof(DpSmem), sizeof(DpSmem3<kE2Cap>)));
constexpr size_t kSmemShared = kPeelRegionShared + std::max(sizeof(DpSmem), sizeof(DpSmem3<kE2CapShared>));
static_assert(kSmemPair <= 227 * 1024 && kSmemShared <= 227 * 1024, "peel / DP shared memory exceeds one SM");

__global__ void __launch_bounds__(kDpPairWarps * 32, 1) k_peel_dp(const __grid_constant__ PeelDpBatch b) {
  extern __shared__ int4 smem4[];
  const int warp = threadIdx.x >> 5;
  if (blockIdx.x == 0) {
    if (warp == 0) peel_dispatch<kV6BucketBits>(b.pa[0], smem4);
    return;
  }
  const DpArgs& da = b.da[0];
  if (da.v3) {
    DpSmem3<kE2Cap>& S = *reinterpret_cast<DpSmem3<kE2Cap>*>(smem4);
    if (threadIdx.x < kDpProducers) S.ready[threadIdx.x] = -1;
    if (threadIdx.x == 0) S.consumed = 0;
    __syncthreads();
    if (warp == 0) dp_compute_v3(da, S);
    else dp_producer(da, S, warp - 1, threadIdx.x & 31);
  } else if (warp == 0) {
    dp_warp(da, *reinterpret_cast<DpSmem*>(smem4));
  }
}

// Launched with kPeelDpWarps * 32 threads, or with kPeelDpExclusive threads whose extra
// warps exit at once: their registers keep other kernels' CTAs off the SM, so the peel warp
// does not share its issue slots and L1 (DP_PEEL_EXCLUSIVE=1).
constexpr int kPeelDpExclusive = 512;
__global__ void __launch_bounds__(kPeelDpExclusive, 1) k_peel_dp_shared(const __grid_constant__ PeelDpBatch b) {
  extern __shared__ int4 smem4[];
  const int warp = threadIdx.x >> 5;
  if (warp >= kPeelDpWarps) return;
  const PeelArgs& pa = b.pa[blockIdx.x];
  const DpArgs& da = b.da[blockIdx.x];
  int4* dsm = smem4 + kPeelRegionShared / sizeof(int4);
  DpSmem3<kE2CapShared>& S = *reinterpret_cast<DpSmem3<kE2CapShared>*>(dsm);
  if (da.v3) {
    if (threadIdx.x < kDpProducers) S.ready[threadIdx.x] = -1;
    if (threadIdx.x == 0) S.consumed = 0;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(kPeelDpWarps * 32) : "memory");  // the working warps only
  if (warp == 0) {
    peel_dispatch<kV6BucketBitsShared>(pa, smem4);
  } else if (warp == 1) {
    if (da.v3) dp_compute_v3(da, S);
    else dp_warp(da, *reinterpret_cast<DpSmem*>(dsm));
  } else if (da.v3 && warp != 4) {
    dp_producer(da, S, warp == 5 ? 2 : warp - 2, threadIdx.x & 31);
  }
}

// DP v5 alone on a finished order (tree peel): one CTA per graph — kDp5Slots slot warps,
// the chain warp, kDpProducers staging warps.
constexpr size_t kSmemDp5 = sizeof(DpSmem5<kE2Cap>);
static_assert(kSmemDp5 <= 227 * 1024, "DP v5 shared memory exceeds one SM");
__global__ void __launch_bounds__(kDp5Threads, 1) k_dp_only(const __grid_constant__ PeelDpBatch b) {
  extern __shared__ int4 smem4[];
  const DpArgs& da = b.da[blockIdx.x];
  DpSmem5<kE2Cap>& S = *reinterpret_cast<DpSmem5<kE2Cap>*>(smem4);
  if (threadIdx.x < kDpProducers) S.ready[threadIdx.x] = -1;
  if (threadIdx.x == 0) {
    S.consumed = 0;
    S.chain_done = 0;
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5;
  if (warp < kDp5Slots) dp_slot_v5(da, S, warp);
  else if (warp == kDp5Slots) dp_chain_v5(da, S);
  else dp_producer_v5(da, S, warp - kDp5Slots - 1, threadIdx.x & 31);
}

__global__ void k_slot16(const int32_t* out_off, const int32_t* out_dst, const int32_t* rank, int32_t m, int4* slot) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = out_dst[k];
    slot[k] = make_int4(c, rank[c], out_off[c], out_off[c + 1] - out_off[c]);
  }
}

__global__ void k_rank_keys2(const int64_t* cpath, const int32_t* by_id, int32_t n, uint64_t* keys, int32_t* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = by_id[i];
    keys[i] = ~(static_cast<uint64_t>(cpath[v]) ^ (1ull << 63));
    vals[i] = v;
  }
}

__global__ void k_rank_of2(const int32_t* by_rank, int32_t n, int32_t* rank) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    rank[by_rank[r]] = static_cast<int32_t>(r);
}

__global__ void k_src_flags2(const int32_t* by_rank, const int32_t* in_off, int32_t n, int32_t* flag) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = by_rank[r];
    flag[r] = (in_off[v + 1] - in_off[v]) == 0 ? 1 : 0;
  }
}

__global__ void k_src_place2(const int32_t* by_rank, const int32_t* flag, const int32_t* pos, const int32_t* out_off,
                             int32_t n, const int32_t* nsrc_p, bool stack, int4* buf) {
  const int32_t nsrc = *nsrc_p;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[r]) continue;
    const int32_t v = by_rank[r], p = pos[r];
    buf[stack ? nsrc - 1 - p : p] = make_int4(v, out_off[v], out_off[v + 1] - out_off[v], 0);
  }
}

__global__ void k_node_rec2(const int32_t* in_off, const int32_t* out_off, const int32_t* rank, int32_t n, int2* nr2) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t deg = min(out_off[v + 1] - out_off[v], 255);
    nr2[v] = make_int2(in_off[v + 1] - in_off[v], rank[v] | (deg << 24));
  }
}

__global__ void k_ell(const int32_t* out_off, const int32_t* out_dst, int32_t n, int ew, int32_t* ell) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (int64_t)n * ew; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = i / ew;
    const int32_t q = static_cast<int32_t>(i - v * ew);
    const int32_t b = out_off[v], d = out_off[v + 1] - b;
    ell[i] = (q < d && d <= ew) ? out_dst[b + q] : -1;
  }
}

__global__ void k_src_place_v5(const int32_t* by_rank, const int32_t* flag, const int32_t* pos, const int32_t* out_off,
                               int32_t n, const int32_t* nsrc_p, int2* buf) {
  const int32_t nsrc = *nsrc_p;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[r]) continue;
    const int32_t v = by_rank[r], p = pos[r];
    buf[nsrc - 1 - p] = make_int2(v, min(out_off[v + 1] - out_off[v], 255));
  }
}

// meta(c) = rank | min(indeg, 127) << 24 | (out-degree > 8) << 31
__device__ __forceinline__ int32_t v6_meta(const int32_t* in_off, const int32_t* out_off, const int32_t* rank,
                                           int32_t c) {
  const int32_t ind = min(in_off[c + 1] - in_off[c], 127);
  const bool lng = out_off[c + 1] - out_off[c] > 8;
  return static_cast<int32_t>(static_cast<uint32_t>(rank[c]) | (static_cast<uint32_t>(ind) << 24) |
                              (lng ? 0x80000000u : 0u));
}

// 8-slot rows sorted by child rank (ascending); -1 padded; long rows (> 8) left empty.
__global__ void k_ell6(const int32_t* in_off, const int32_t* out_off, const int32_t* out_dst, const int32_t* rank,
                       int32_t n, int2* ell) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = out_off[v], d = out_off[v + 1] - b;
    int2 r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = make_int2(-1, 0);
    if (d <= 8) {
      for (int q = 0; q < d; ++q) {
        const int32_t c = out_dst[b + q];
        int2 x = make_int2(c, v6_meta(in_off, out_off, rank, c));
        // insertion by rank (low 24 bits)
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (x.x >= 0 && (r[j].x < 0 || (x.y & 0xffffff) < (r[j].y & 0xffffff))) {
            const int2 t = r[j];
            r[j] = x;
            x = t;
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) ell[v * 8 + q] = r[q];
  }
}

__global__ void k_cmeta(const int32_t* in_off, const int32_t* out_off, const int32_t* out_dst, const int32_t* rank,
                        int32_t m, int2* cm) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = out_dst[k];
    cm[k] = make_int2(c, v6_meta(in_off, out_off, rank, c));
  }
}

__global__ void k_src_place_v6(const int32_t* by_rank, const int32_t* flag, const int32_t* pos, const int32_t* out_off,
                               int32_t n, const int32_t* nsrc_p, int32_t* buf) {
  const int32_t nsrc = *nsrc_p;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[r]) continue;
    const int32_t v = by_rank[r];
    buf[nsrc - 1 - pos[r]] = v | (out_off[v + 1] - out_off[v] > 8 ? kV6Long : 0);
  }
}

__global__ void k_scatter_pos_of(const int32_t* seq, int32_t n, int32_t* pos_of) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    pos_of[seq[p]] = static_cast<int32_t>(p);
}

__global__ void k_dense16(const int32_t* in_off, int32_t n, uint32_t* words, int* bad) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; 2 * j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = static_cast<int32_t>(2 * j);
    const int32_t d0 = in_off[v + 1] - in_off[v];
    const int32_t d1 = v + 1 < n ? in_off[v + 2] - in_off[v + 1] : 0;
    if (d0 >= 65535 || d1 >= 65535) atomicExch(bad, 1);
    words[j] = static_cast<uint32_t>(d0 & 0xffff) | (static_cast<uint32_t>(d1 & 0xffff) << 16);
  }
}

__global__ void k_indeg_init2(const int32_t* in_off, int32_t n, int32_t* indeg) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    indeg[v] = in_off[v + 1] - in_off[v];
}

__global__ void k_max_abs(const int64_t* x, int32_t n, unsigned long long* out) {
  unsigned long long m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = x[i] < 0 ? -x[i] : x[i];
    m = static_cast<unsigned long long>(v) > m ? static_cast<unsigned long long>(v) : m;
  }
  // one atomic per warp (one per thread serialised ~600K same-address atomics: 0.4 ms)
  for (int o = 16; o; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, m, o);
    m = y > m ? y : m;
  }
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

__global__ void k_out_sum(const int32_t* out_off, const int64_t* out_cost, int32_t n, int64_t* out_sum) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = 0;
    for (int32_t k = out_off[v]; k < out_off[v + 1]; ++k) s += out_cost[k];
    out_sum[v] = s;
  }
}

size_t peel_smem() { return kPeelRegion; }  // k_peel2 (topo_order)

}  // namespace

// Builds the peel inputs (ranks, 16-byte slot records, initial stack, in-degrees).
// Ranks, source flags and the peel counters; the tree peel's job when wanted (launched by
// the caller together with other graphs' jobs: tree_run).
void peel_prepare_begin(DevGraph& g, int policy, const int64_t* cpath, PeelState& st, int32_t* seq,
                        int32_t* pos_of, bool tree) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  const int32_t n = g.n;
  DevBuf<int32_t> by_id;
  node_order_by_id(g, by_id);
  st.by_rank.alloc(ctx, n);
  st.rank.alloc(ctx, n);
  if (policy == DP_TOPO_CPD) {
    DevBuf<uint64_t> keys(ctx, n), keys_out(ctx, n);
    DevBuf<int32_t> vals(ctx, n);
    DP_LAUNCH(ctx, k_rank_keys2, grid_for(n, B), B, 0, cpath, by_id.p, n, keys.p, vals.p);
    sort_pairs_u64(ctx, keys.p, keys_out.p, vals.p, st.by_rank.p, n, 0, 64);
  } else {
    DP_CUDA(cudaMemcpyAsync(st.by_rank.p, by_id.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  DP_LAUNCH(ctx, k_rank_of2, grid_for(n, B), B, 0, st.by_rank.p, n, st.rank.p);
  st.flag.alloc(ctx, (size_t)n + 1);
  st.fpos.alloc(ctx, (size_t)n + 1);
  st.flag.zero();
  DP_LAUNCH(ctx, k_src_flags2, grid_for(n, B), B, 0, st.by_rank.p, g.in_off.p, n, st.flag.p);
  exclusive_scan_i32(ctx, st.flag.p, st.fpos.p, (int64_t)n + 1);
  st.stack_mode = policy != DP_TOPO_M;
  st.counters.alloc(ctx, 3);
  st.counters.zero();
  // the number of sources (the scan's total) stays on the device
  DP_CUDA(cudaMemcpyAsync(st.counters.p + 2, st.fpos.p + n, sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
  st.tree.reset();
  st.tree_ok = false;
  if (st.stack_mode && seq != nullptr && tree && fixpoint_wanted(g)) {
    st.skip.alloc(ctx, 1);
    st.skip.zero();
    st.tree = fixpoint_prepare(g, st.by_rank.p, st.rank.p, st.flag.p, st.fpos.p, seq, pos_of, st.skip.p,
                               st.counters.p, st.counters.p + 1);
  }
}

// The one-warp peel's inputs (v6 / v5 / FIFO layouts).
void peel_prepare_end(DevGraph& g, PeelState& st, bool force_v5) {
  dp_ctx* ctx = g.ctx;
  const int B = 256;
  const int32_t n = g.n, m = g.m_ok;
  const int32_t* nsrc_p = st.fpos.p + n;
  const int32_t* by_rank = st.by_rank.p;
  const int32_t* rank = st.rank.p;
  // v6 for sparse graphs (m <= 6n), and in dense mode for graphs whose rows mostly exceed
  // v5's 32 on-chip slots (m > 32n: config #4 wide's coarse graph, 45 children per node:
  // 78 -> 50 ms; the deep one, 27 per node, stays on v5: 4.4 vs 7.1 ms).
  // DP_PEEL_V6_DENSE=0 / 1: never / always when dense mode applies.
  const bool dense_ok = n <= v6_dense_cap<kV6BucketBits>() && getenv("DP_PEEL_NO_DENSE") == nullptr;
  const char* v6d = getenv("DP_PEEL_V6_DENSE");
  const bool v6_dense =
      dense_ok && (v6d ? v6d[0] == '1' : static_cast<int64_t>(m) > 32 * static_cast<int64_t>(n));
  st.v6 = st.stack_mode && n < (1 << 24) && (static_cast<int64_t>(m) <= 6 * static_cast<int64_t>(n) || v6_dense) &&
          !force_v5 && getenv("DP_PEEL_V5") == nullptr;
  if (st.v6) {
    st.ell6.alloc(ctx, (size_t)n * 4);
    DP_LAUNCH(ctx, k_ell6, grid_for(n, B), B, 0, g.in_off.p, g.out_off.p, g.out_dst.p, rank, n,
              reinterpret_cast<int2*>(st.ell6.p));
    st.cmeta.alloc(ctx, m > 0 ? m : 1);
    DP_LAUNCH(ctx, k_cmeta, grid_for(m, B), B, 0, g.in_off.p, g.out_off.p, g.out_dst.p, rank, m, st.cmeta.p);
    st.gsid.alloc(ctx, (size_t)n + 1);
    DP_LAUNCH(ctx, k_src_place_v6, grid_for(n, B), B, 0, by_rank, st.flag.p, st.fpos.p, g.out_off.p, n, nsrc_p,
              st.gsid.p);
    st.indeg.alloc(ctx, n);
    DP_LAUNCH(ctx, k_indeg_init2, grid_for(n, B), B, 0, g.in_off.p, n, st.indeg.p);
    st.gover.alloc(ctx, n);
    st.gover.zero();
    st.spill.alloc(ctx, m > 0 ? m : 1);
    if (n <= v6_dense_cap<kV6BucketBits>() && getenv("DP_PEEL_NO_DENSE") == nullptr) {
      st.dense16.alloc(ctx, (n + 1) / 2);
      st.dense_bad.alloc(ctx, 1);
      st.dense_bad.zero();
      DP_LAUNCH(ctx, k_dense16, grid_for((n + 1) / 2, B), B, 0, g.in_off.p, n, st.dense16.p, st.dense_bad.p);
    }
    return;
  }
  st.gstack.alloc(ctx, (size_t)n + 1);
  if (st.stack_mode && n < (1 << 24)) {
    st.ellw = n > 262144 ? 8 : 32;
    st.nr2.alloc(ctx, n);
    DP_LAUNCH(ctx, k_node_rec2, grid_for(n, B), B, 0, g.in_off.p, g.out_off.p, rank, n, st.nr2.p);
    st.ell.alloc(ctx, (size_t)n * st.ellw);
    DP_LAUNCH(ctx, k_ell, grid_for((int64_t)n * st.ellw, B), B, 0, g.out_off.p, g.out_dst.p, n, st.ellw, st.ell.p);
    st.gstack2.alloc(ctx, (size_t)n + 1);
    DP_LAUNCH(ctx, k_src_place_v5, grid_for(n, B), B, 0, by_rank, st.flag.p, st.fpos.p, g.out_off.p, n, nsrc_p,
              st.gstack2.p);
  } else {
    if (st.stack_mode) fail(DP_E_UNSUPPORTED, "graphs with 2^24 or more nodes are not supported by the peel");
    DP_LAUNCH(ctx, k_src_place2, grid_for(n, B), B, 0, by_rank, st.flag.p, st.fpos.p, g.out_off.p, n, nsrc_p,
              st.stack_mode, st.gstack.p);
    st.indeg.alloc(ctx, n);
    DP_LAUNCH(ctx, k_indeg_init2, grid_for(n, B), B, 0, g.in_off.p, n, st.indeg.p);
    st.slot.alloc(ctx, m > 0 ? m : 1);
    DP_LAUNCH(ctx, k_slot16, grid_for(m, B), B, 0, g.out_off.p, g.out_dst.p, rank, m, st.slot.p);
  }
  st.spill.alloc(ctx, m > 0 ? m : 1);
}

void peel_prepare(DevGraph& g, int policy, const int64_t* cpath, PeelState& st, bool force_v5) {
  peel_prepare_begin(g, policy, cpath, st, nullptr, nullptr, false);
  peel_prepare_end(g, st, force_v5);
}

// Launches the tree peels of states that have one (one launch per kTreeBatch graphs), waits,
// and records which proofs held (PeelState::tree_ok); one host round trip.
void tree_run(dp_ctx* ctx, PeelState* const* sts, int count) {
  std::vector<TreeJob*> jobs;
  std::vector<int> idx;
  for (int i = 0; i < count; ++i)
    if (sts[i] && sts[i]->tree) {
      jobs.push_back(sts[i]->tree.get());
      idx.push_back(i);
    }
  if (jobs.empty()) return;
  fixpoint_launch_batch(ctx, jobs.data(), static_cast<int>(jobs.size()));
  std::vector<int> ok(jobs.size(), 0);
  for (size_t q = 0; q < jobs.size(); ++q) download_bytes(ctx, &ok[q], sts[idx[q]]->skip.p, sizeof(int));
  sync(ctx);
  for (size_t q = 0; q < jobs.size(); ++q) {
    sts[idx[q]]->tree_ok = ok[q] != 0;
    sts[idx[q]]->tree.reset();  // stream-ordered frees after the launch
  }
}

static PeelArgs peel_args(DevGraph& g, PeelState& st, int32_t* seq, int32_t* pos_of, bool progress) {
  PeelArgs a{};
  a.n = g.n;
  a.slot = st.slot.p;
  a.indeg = st.indeg.p;
  a.gstack = st.gstack.p;
  a.nsrc = st.counters.p + 2;
  a.stack_mode = st.stack_mode;
  a.seq = seq;
  a.pos_of = pos_of;
  a.progress = progress ? st.counters.p : nullptr;
  a.emitted = st.counters.p + 1;
  a.freed_spill = st.spill.p;
  a.nr2 = st.nr2.p;
  a.ell = st.ell.p;
  a.ellw = st.ellw;
  a.out_off = g.out_off.p;
  a.out_dst = g.out_dst.p;
  a.gstack2 = st.gstack2.p;
  a.v6 = st.v6;
  a.ell6 = st.ell6.p;
  a.cmeta = st.cmeta.p;
  a.rem_big = st.indeg.p;
  a.gsid = st.gsid.p;
  a.gover = st.gover.p;
  a.prefetch = getenv("DP_PEEL_NO_PREFETCH") == nullptr;
  a.skip = st.skip.p;
  a.dense16 = st.dense16.p;
  a.dense_bad = st.dense_bad.p;
  return a;
}

std::vector<int32_t> topo_order_batch(DevGraph* const* gs, int count, int policy, const int64_t* const* cpath,
                                      int32_t* const* seq, int32_t* const* pos_of, bool tree) {
  std::vector<int32_t> emitted(count, 0);
  if (count == 0) return emitted;
  dp_ctx* ctx = gs[0]->ctx;
  const size_t sm = peel_smem();
  static bool attr = false;
  if (!attr) {
    DP_CUDA(cudaFuncSetAttribute(k_peel2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
    attr = true;
  }
  std::vector<std::unique_ptr<PeelState>> st(count);
  std::vector<int> live;
  std::vector<PeelState*> sp;
  for (int i = 0; i < count; ++i) {
    if (gs[i]->n == 0) continue;
    st[i].reset(new PeelState);
    peel_prepare_begin(*gs[i], policy, cpath[i], *st[i], seq[i], pos_of[i], tree);
    live.push_back(i);
    sp.push_back(st[i].get());
  }
  tree_run(ctx, sp.data(), static_cast<int>(sp.size()));
  std::vector<int> run;  // graphs the one-warp peel orders
  double bytes = 0.0;
  for (int i : live)
    if (!st[i]->tree_ok) {
      peel_prepare_end(*gs[i], *st[i], false);
      run.push_back(i);
      bytes += 72.0 * gs[i]->n + 8.0 * gs[i]->m_ok;
    }
  if (!run.empty()) {
    StageScope s(ctx, policy == DP_TOPO_CPD ? "cpd_peel" : "peel", bytes);
    for (size_t b0 = 0; b0 < run.size(); b0 += kPeelBatch) {
      const int k = static_cast<int>(std::min<size_t>(kPeelBatch, run.size() - b0));
      PeelBatch batch{};
      for (int q = 0; q < k; ++q) {
        const int i = run[b0 + q];
        batch.a[q] = peel_args(*gs[i], *st[i], seq[i], pos_of[i], false);
      }
      DP_LAUNCH(ctx, k_peel2, k, 32, sm, batch);
    }
  }
  for (int i : live) download_bytes(ctx, &emitted[i], st[i]->counters.p + 1, sizeof(int32_t));
  sync(ctx);
  for (int i : run)
    if (st[i]->stack_mode && emitted[i] == gs[i]->n)
      DP_LAUNCH(ctx, k_scatter_pos_of, grid_for(gs[i]->n, 256), 256, 0, seq[i], gs[i]->n, pos_of[i]);
  return emitted;
}

int32_t topo_order(DevGraph& g, int policy, const int64_t* cpath, int32_t* seq, int32_t* pos_of) {
  DevGraph* gs[1] = {&g};
  const int64_t* cp[1] = {cpath};
  int32_t* sq[1] = {seq};
  int32_t* po[1] = {pos_of};
  return topo_order_batch(gs, 1, policy, cp, sq, po)[0];
}

struct PeelDpJob {
  dp_ctx* ctx = nullptr;
  DevGraph* g = nullptr;
  int32_t* seq = nullptr;
  int32_t* pos_of = nullptr;
  PeelState st;
  DevBuf<int64_t> out_sum;
  DevBuf<unsigned long long> mx;
  DevBuf<long long> dbg;
  PeelArgs pa{};
  DpArgs da{};
  double bytes = 0.0;  // algorithmic bytes (stage timing)
  // DP v5 records (k_dp_records)
  DevBuf<int64_t> mp;
  DevBuf<int4> rec01, rec23, recz;
  DevBuf<int32_t> bext;
  DevBuf<int2> ovf;
  DevBuf<int> ovfc;
  // peel_dp_prepare_begin -> _finish
  int32_t range = 0;
  int64_t limit = 0;
  int32_t* prev_cut = nullptr;
  int* first_exceed = nullptr;
  unsigned long long max_out = 0;
};

PeelDpJob* peel_dp_prepare_begin(DevGraph& g, const int64_t* cpath, int32_t range, int64_t limit, int32_t* seq,
                                 int32_t* pos_of, int32_t* prev_cut, int* first_exceed) {
  dp_ctx* ctx = g.ctx;
  const int32_t n = g.n;
  auto* j = new PeelDpJob;
  PeelDpHandle guard(j);
  j->ctx = ctx;
  j->range = range;
  j->limit = limit;
  j->prev_cut = prev_cut;
  j->first_exceed = first_exceed;
  j->out_sum.alloc(ctx, n);
  DP_LAUNCH(ctx, k_out_sum, grid_for(n, 256), 256, 0, g.out_off.p, g.out_cost.p, n, j->out_sum.p);
  // 32-bit keys need every window value within +-2^22 of the window minimum: bounded
  // by R x (largest out-cost sum of a position) + largest single cost.
  j->mx.alloc(ctx, 1);
  j->mx.zero();
  DP_LAUNCH(ctx, k_max_abs, grid_for(n, 256), 256, 0, j->out_sum.p, n, j->mx.p);
  DP_LAUNCH(ctx, k_max_abs, grid_for(g.m_ok, 256), 256, 0, g.out_cost.p, g.m_ok, j->mx.p);
  // the peel's preparation is enqueued before the one host round trip of this function;
  // with a tree peel the one-warp peel's inputs wait for its verdict (peel_dp_launch)
  peel_prepare_begin(g, DP_TOPO_CPD, cpath, j->st, seq, pos_of, true);
  if (!j->st.tree) peel_prepare_end(g, j->st, false);
  j->g = &g;
  j->seq = seq;
  j->pos_of = pos_of;
  download_bytes(ctx, &j->max_out, j->mx.p, sizeof(unsigned long long));  // read after the caller's sync
  guard.j = nullptr;
  return j;
}

void peel_dp_prepare_finish(PeelDpJob* j) {
  dp_ctx* ctx = j->ctx;
  DevGraph& g = *j->g;
  const int32_t n = g.n;
  const int32_t range = j->range;
  const unsigned long long max_out = j->max_out;
  DpArgs& da = j->da;
  da.keys32 = static_cast<double>(max_out) * (range + 2) < static_cast<double>(1 << 21);
  // the block recurrence lets relative values drift for up to 2 x 32 steps before a rebase
  da.block32 = static_cast<double>(max_out) * (range + 2 + 64) < static_cast<double>(1 << 21) &&
               getenv("DP_DP_PERSTEP") == nullptr;
  da.v3 = da.keys32 && da.block32 && range <= 225 && getenv("DP_DP_V2") == nullptr;
  da.n = n;
  da.range = range;
  da.seq = j->seq;
  da.pos_of = j->pos_of;
  da.mem = g.mem.p;
  da.out_sum = j->out_sum.p;
  da.in_off = g.in_off.p;
  da.in_src = g.in_src.p;
  da.in_cost = g.in_cost.p;
  da.limit = j->limit;
  da.prev_cut = j->prev_cut;
  da.first_exceed = j->first_exceed;
  j->dbg.alloc(ctx, 8);
  j->dbg.zero();
  da.debug = getenv("DP_DEBUG_DP") ? j->dbg.p : nullptr;
  da.progress = j->st.counters.p;
  // algorithmic bytes: peel 64 B row + 8 B seq/pos_of per node; DP 4+8+8+4 B per position
  // (node, memory, out-cost sum, cut) + 12 B per in-edge (source position, cost)
  j->bytes = 92.0 * n + 12.0 * g.m_ok;
}

PeelDpJob* peel_dp_prepare(DevGraph& g, const int64_t* cpath, int32_t range, int64_t limit, int32_t* seq,
                           int32_t* pos_of, int32_t* prev_cut, int* first_exceed) {
  PeelDpJob* j = peel_dp_prepare_begin(g, cpath, range, limit, seq, pos_of, prev_cut, first_exceed);
  PeelDpHandle guard(j);
  sync(g.ctx);
  peel_dp_prepare_finish(j);
  guard.j = nullptr;
  return j;
}

void peel_dp_launch(dp_ctx* ctx, PeelDpJob* const* jobs, int count) {
  static bool attr = false;
  if (!attr) {
    DP_CUDA(cudaFuncSetAttribute(k_peel_dp, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemPair)));
    DP_CUDA(cudaFuncSetAttribute(k_peel_dp_shared, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(kSmemShared)));
    DP_CUDA(cudaFuncSetAttribute(k_dp_only, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemDp5)));
    attr = true;
  }
  // tree peels of all graphs in one go; the one-warp peel's inputs where a proof failed
  {
    std::vector<PeelState*> sp;
    for (int q = 0; q < count; ++q) sp.push_back(&jobs[q]->st);
    std::vector<char> had(count);
    for (int q = 0; q < count; ++q) had[q] = jobs[q]->st.tree != nullptr;
    tree_run(ctx, sp.data(), count);
    for (int q = 0; q < count; ++q) {
      PeelDpJob* j = jobs[q];
      if (had[q] && !j->st.tree_ok) peel_prepare_end(*j->g, j->st, false);
      j->pa = peel_args(*j->g, j->st, j->seq, j->pos_of, true);
      j->pa.debug = j->da.debug ? j->dbg.p + 3 : nullptr;
    }
  }
  // finished orders: the multi-warp DP alone (DP v4), one CTA per graph
  std::vector<PeelDpJob*> dp4, rest;
  for (int q = 0; q < count; ++q) {
    if (jobs[q]->st.tree_ok && jobs[q]->da.v3 && getenv("DP_DP_V3") == nullptr) dp4.push_back(jobs[q]);
    else rest.push_back(jobs[q]);
  }
  if (!dp4.empty()) {  // the per-position records of every finished order
    StageScope s(ctx, "dp records", 0.0);
    for (PeelDpJob* j : dp4) {
      const int32_t n = j->da.n;
      const int32_t m = j->g->m_ok;
      DevBuf<int64_t> tmp(ctx, (size_t)n + 1);
      j->mp.alloc(ctx, (size_t)n + 1);
      DP_LAUNCH(ctx, k_mem_by_pos, grid_for((int64_t)n + 1, 256), 256, 0, j->da.seq, j->da.mem, n, tmp.p);
      exclusive_scan_i64(ctx, tmp.p, j->mp.p, (int64_t)n + 1);
      j->rec01.alloc(ctx, n);
      j->rec23.alloc(ctx, n);
      j->recz.alloc(ctx, n);
      j->bext.alloc(ctx, (size_t)n / 32 + 1);
      j->ovf.alloc(ctx, m > 0 ? m : 1);
      j->ovfc.alloc(ctx, 1);
      j->ovfc.zero();
      DP_LAUNCH(ctx, k_dp_records, grid_for(n, 256), 256, 0, j->da, j->mp.p, j->rec01.p, j->rec23.p, j->recz.p,
                j->bext.p, j->ovf.p, j->ovfc.p);
      j->da.rec01 = j->rec01.p;
      j->da.rec23 = j->rec23.p;
      j->da.recz = j->recz.p;
      j->da.bext = j->bext.p;
      j->da.ovf = j->ovf.p;
    }
  }
  for (size_t b0 = 0; b0 < dp4.size(); b0 += kPeelDpBatch) {
    const int k = static_cast<int>(std::min<size_t>(kPeelDpBatch, dp4.size() - b0));
    PeelDpBatch batch{};
    double bytes = 0.0;
    for (int q = 0; q < k; ++q) {
      batch.da[q] = dp4[b0 + q]->da;
      bytes += 32.0 * dp4[b0 + q]->da.n + 12.0 * dp4[b0 + q]->g->m_ok;
    }
    StageScope s(ctx, "dp", bytes);
    DP_LAUNCH(ctx, k_dp_only, k, kDp5Threads, kSmemDp5, batch);
  }
  // one graph: pair mode (an SM each for peel and DP); several: shared mode (an SM per graph)
  const bool pair = count == 1 && rest.size() == 1 && getenv("DP_PEEL_DP_SHARED") == nullptr;
  for (size_t b0 = 0; b0 < rest.size(); b0 += kPeelDpBatch) {
    const int k = static_cast<int>(std::min<size_t>(kPeelDpBatch, rest.size() - b0));
    PeelDpBatch batch{};
    double bytes = 0.0;
    for (int q = 0; q < k; ++q) {
      batch.pa[q] = rest[b0 + q]->pa;
      batch.da[q] = rest[b0 + q]->da;
      bytes += rest[b0 + q]->bytes;
    }
    StageScope s(ctx, "peel+dp (streamed)", bytes);
    if (pair) {
      void* args[] = {&batch};
      DP_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_peel_dp), 2, kDpPairWarps * 32, args,
                                          kSmemPair, ctx->stream));
      ++ctx->launches;
    } else {
      DP_LAUNCH(ctx, k_peel_dp_shared, k, getenv("DP_PEEL_EXCLUSIVE") ? kPeelDpExclusive : kPeelDpWarps * 32,
                kSmemShared, batch);
    }
  }
  for (int q = 0; q < count; ++q) {
    PeelDpJob* j = jobs[q];
    if (j->da.debug) {
      long long h[8];
      j->dbg.download(h, 8);
      sync(ctx);
      if (j->st.tree_ok && j->da.v3)
        fprintf(stderr,
                "[peel_dp] dp v5: chain warp waiting %.1f ms, chaining %.1f ms (loads %.1f, loop %.1f); slot warp 0 "
                "waiting %.1f ms\n",
                h[4] / 1.965e6, h[6] / 1.965e6, h[2] / 1.965e6, h[7] / 1.965e6, h[5] / 1.965e6);
      fprintf(stderr,
              "[peel_dp] dp %s: total %.1f ms, waiting %.1f ms, staging %.1f ms; peel warp %.1f ms (at 1.965 GHz)\n",
              j->st.tree_ok && j->da.v3 ? "v5 (8 slot warps + chain warp, tree-peeled order)" : "warp", h[0] / 1.965e6, h[1] / 1.965e6,
              h[2] / 1.965e6, h[3] / 1.965e6);
    }
  }
}

void peel_dp_release(PeelDpJob* j) { delete j; }

int32_t peel_dp_stream(DevGraph& g, const int64_t* cpath, int32_t range, int64_t limit, int32_t* seq, int32_t* pos_of,
                       int32_t* prev_cut, int* first_exceed) {
  if (g.n == 0) return 0;
  PeelDpHandle h(peel_dp_prepare(g, cpath, range, limit, seq, pos_of, prev_cut, first_exceed));
  peel_dp_launch(g.ctx, &h.j, 1);
  return scalar_to_host(g.ctx, h.j->st.counters.p + 1);
}

// Node indices sorted by id ascending (identity for dense ids): the rank of DFS / M-TOPO.
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
