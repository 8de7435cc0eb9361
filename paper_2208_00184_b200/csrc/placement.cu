// placement.cu — Order-Place and Adjusting placement (Optimal Operator Placement) on
// the GPU, bit-exact with placement.cpp (/root/reference/proj/src):
//   DeviceTimeline::find_slot / reserve   :13-32
//   order_place                           :128-159
//   est_on_device / adjusting_placement   :81-96, :161-218
//   expand_placement                      :239-268
//
// Both heuristics are sequential over the coarse order.  They run as one CTA each (the
// two CTAs of one launch run concurrently on two SMs).  Per node the adjusting CTA
//   1. reduces the in-edges into per-device maxima A[d] = max finish (same device) and
//      B[d] = max finish + cost, so pre_t(d) = max(0, A[d], max_{d' != d} B[d']);
//   2. lets warp d answer find_slot(pre_t(d), w) on device d's timeline;
//   3. applies the EST / back-cost rule in one thread and commits with one warp.
//
// find_slot is answered without the reference's linear scan.  Per device the busy
// intervals are kept sorted by start with PM[k] = max(E[0..k]) and
// GQ[k] = E[k] > PM[k-1] ? S[k] - PM[k-1] : -1, plus per-32 block maxima of GQ: the
// reference loop breaks at k0 (first PM[k] > earliest) when S[k0] - earliest >= dur,
// otherwise at the first k > k0 with GQ[k] >= dur, returning PM[k-1] — else PM[K-1].
#include <algorithm>
#include <cstdlib>

#include "placement.cuh"

namespace dpb {

namespace {

constexpr int kMaxD = 256;
constexpr unsigned FULL = 0xffffffffu;

// Blocked device timeline (DeviceTimeline, placement.cpp:13-32).  Intervals sorted by
// start (upper_bound insert) live in blocks of 32 (one lane per entry); blocks are kept
// in sequence by POSITION with per-position meta: physical id, count, max end, end
// prefix max over all blocks up to here (pmEnd), first entry, and an upper bound of the
// gaps inside the block (computed with the block-local end prefix max; the true prefix
// max can only be larger, so the true gaps only smaller: false positives are re-checked).
// An insert touches one block (split in halves when full) instead of shifting the whole
// timeline; pmEnd changes propagate forward only while they change (rarely past one).
// Semantics are the reference's exactly: with PM[k] = max(E[0..k]) the scan stops at the
// first interval with PM > earliest if its start leaves room, else at the first later
// interval k with E[k] > PM[k-1] and S[k] - PM[k-1] >= dur, returning PM[k-1]; else the
// overall max end (zero-length intervals included).
constexpr int kTB = 32;

// With the meta in global memory (large coarse graphs) the gap scan of find_slot reads
// G[p] = an upper bound of every gap of block p including its first one against the carry
// (max(gub[p], fS[p] - pmEnd[p-1] when fE[p] > pmEnd[p-1])) and SG[P] = max G over the
// 32 positions of super-block P, so a scan costs at most three dependent rounds; with the
// meta in shared memory the scan reads gub / fS / fE directly (G, SG null).
struct TLView {
  int64_t *S, *E;                                 // [maxb][kTB] by physical block id
  int32_t *id, *cnt;                              // [maxb] by position
  int64_t *maxE, *pmEnd, *fS, *fE, *gub;          // [maxb] by position
  int64_t *G, *SG;                                // [maxb], [maxb / 32 + 1] (global meta only)
  int32_t* nb;                                    // blocks in use (shared memory)
};

struct TLArrays {
  int64_t *S, *E, *maxE, *pmEnd, *fS, *fE, *gub, *G, *SG;
  int32_t *id, *cnt;
  int32_t maxb;
  int32_t* nb;  // shared memory, set by the kernel
  __device__ TLView view(int d) const {
    const int64_t eo = (int64_t)d * maxb * kTB, mo = (int64_t)d * maxb, so = (int64_t)d * (maxb / 32 + 1);
    return TLView{S + eo, E + eo, id + mo, cnt + mo, maxE + mo, pmEnd + mo, fS + mo, fE + mo, gub + mo,
                  G ? G + mo : nullptr, SG ? SG + so : nullptr, nb + d};
  }
};

// G of position p >= 1 from its meta and the carry pmEnd[p - 1] (position 0 has no carry)
__device__ __forceinline__ int64_t tl_gbound(int32_t p, int64_t gub, int64_t fs, int64_t fe, int64_t carry) {
  return (p > 0 && fe > carry && fs - carry > gub) ? fs - carry : gub;
}

// SG of the super-blocks P0..P1 from G (warp-collective)
__device__ void tl_sg(const TLView t, int32_t P0, int32_t P1, int32_t nb) {
  const int lane = threadIdx.x & 31;
  for (int32_t P = P0; P <= P1; ++P) {
    const int32_t p = P * 32 + lane;
    int64_t x = p < nb ? t.G[p] : -1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const int64_t y = __shfl_xor_sync(FULL, x, o);
      x = y > x ? y : x;
    }
    if (lane == 0) t.SG[P] = x;
  }
  __syncwarp();
}

// First index in [lo, hi] whose predicate holds (monotone false...true; pred(hi) true).
template <typename Pred>
__device__ __forceinline__ int32_t warp_first_true(int32_t lo, int32_t hi, Pred pred) {
  const int lane = threadIdx.x & 31;
  while (hi - lo >= 32) {
    const int32_t step = (hi - lo + 32) >> 5;
    const int32_t q = min(lo + lane * step, hi);
    const unsigned b = __ballot_sync(FULL, pred(q));
    if (b == 0) {
      lo = min(lo + 31 * step, hi) + 1;
    } else {
      const int f = __ffs(b) - 1;
      const int32_t qf = min(lo + f * step, hi);
      if (f > 0) lo = min(lo + (f - 1) * step, hi) + 1;
      hi = qf;
    }
  }
  const int32_t idx = lo + lane;
  const unsigned b = __ballot_sync(FULL, idx <= hi && pred(idx));
  return lo + __ffs(b) - 1;
}

__device__ __forceinline__ int64_t warp_incl_max(int64_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v = y > v ? y : v;
  }
  return v;
}

// Full-warp 64-bit max / min: redux.sync on the high and low words of order-preserving
// (sign-biased) values.  (Partial-mask redux is emulated in software on sm_100a.)
__device__ __forceinline__ long long warp_max_i64(long long x) {
  const uint64_t u = static_cast<uint64_t>(x) ^ 0x8000000000000000ull;
  const uint32_t hi = __reduce_max_sync(FULL, static_cast<uint32_t>(u >> 32));
  const uint32_t lo = __reduce_max_sync(FULL, static_cast<uint32_t>(u >> 32) == hi ? static_cast<uint32_t>(u) : 0u);
  return static_cast<long long>(((static_cast<uint64_t>(hi) << 32) | lo) ^ 0x8000000000000000ull);
}
__device__ __forceinline__ long long warp_min_i64(long long x) {
  const uint64_t u = static_cast<uint64_t>(x) ^ 0x8000000000000000ull;
  const uint32_t hi = __reduce_min_sync(FULL, static_cast<uint32_t>(u >> 32));
  const uint32_t lo =
      __reduce_min_sync(FULL, static_cast<uint32_t>(u >> 32) == hi ? static_cast<uint32_t>(u) : 0xffffffffu);
  return static_cast<long long>(((static_cast<uint64_t>(hi) << 32) | lo) ^ 0x8000000000000000ull);
}

struct BlockLoad {
  int64_t s, e, pm, pmprev;  // this lane's entry, PM at it, PM before it (with carry)
  int32_t c;
};

// Loads block at position pos (lane = entry) with the PM carried in from earlier blocks.
__device__ __forceinline__ BlockLoad tl_load(const TLView t, int32_t pos) {
  const int lane = threadIdx.x & 31;
  BlockLoad r;
  const int32_t b = t.id[pos];
  r.c = t.cnt[pos];
  const int64_t carry = pos > 0 ? t.pmEnd[pos - 1] : INT64_MIN;
  r.s = lane < r.c ? t.S[(int64_t)b * kTB + lane] : INT64_MAX;
  r.e = lane < r.c ? t.E[(int64_t)b * kTB + lane] : INT64_MIN;
  const int64_t inc = warp_incl_max(r.e);
  r.pm = inc > carry ? inc : carry;
  const int64_t up = __shfl_up_sync(FULL, r.pm, 1);
  r.pmprev = lane == 0 ? carry : up;
  return r;
}

// Block at position pos whose id, count and carried-in PM are already known: one load.
__device__ __forceinline__ BlockLoad tl_load_known(const TLView t, int32_t b, int32_t c, int64_t carry) {
  const int lane = threadIdx.x & 31;
  BlockLoad r;
  r.c = c;
  r.s = lane < c ? t.S[(int64_t)b * kTB + lane] : INT64_MAX;
  r.e = lane < c ? t.E[(int64_t)b * kTB + lane] : INT64_MIN;
  const int64_t inc = warp_incl_max(r.e);
  r.pm = inc > carry ? inc : carry;
  const int64_t up = __shfl_up_sync(FULL, r.pm, 1);
  r.pmprev = lane == 0 ? carry : up;
  return r;
}

// DeviceTimeline::find_slot(earliest, dur) (placement.cpp:13-21); warp-collective.
// Nodes arrive in topological order, so `earliest` is nearly always inside the last 32
// block positions: their meta comes in one round of independent loads (lane = position),
// the block holding the first PM > earliest in a second, and the gap candidates after it
// need only their entries.  Otherwise: a 32-ary search over all positions.
__device__ int64_t tl_query(const TLView t, int32_t K, int64_t gmax, int64_t last, int64_t earliest, int64_t dur,
                           int32_t* hint) {
  const int lane = threadIdx.x & 31;
  const int32_t nb = *t.nb;
  *hint = nb - 1;  // the block reserve() will insert into (a guess tl_insert checks)
  if (K == 0 || last <= earliest) return earliest;
  const int32_t lo = nb > 32 ? nb - 32 : 0;
  const int32_t p = lo + lane;
  const bool in = p < nb;
  int64_t wpm = INT64_MAX, wgu = -1, wfe = 0, wfs = 0;
  int32_t wid = 0, wc = 0;
  if (in) {
    wpm = t.pmEnd[p];
    wgu = t.gub[p];
    wfe = t.fE[p];
    wfs = t.fS[p];
    wid = t.id[p];
    wc = t.cnt[p];
  }
  const int64_t pm_lo = lo > 0 ? t.pmEnd[lo - 1] : INT64_MIN;
  if (pm_lo > earliest) {
    // first interval with PM > earliest: its block is the first position with pmEnd > earliest
    const int32_t j = warp_first_true(0, lo - 1, [&](int32_t q) { return t.pmEnd[q] > earliest; });
    BlockLoad L = tl_load(t, j);
    const int k0 = __ffs(__ballot_sync(FULL, lane < L.c && L.pm > earliest)) - 1;
    const int64_t s0 = __shfl_sync(FULL, L.s, k0);
    if (s0 >= earliest && s0 - earliest >= dur) {
      *hint = k0 > 0 || j == 0 ? j : j - 1;
      return earliest;
    }
    if (gmax < dur) return last;
    {
      const bool fit = lane > k0 && lane < L.c && L.e > L.pmprev && L.s - L.pmprev >= dur;
      const unsigned bal = __ballot_sync(FULL, fit);
      if (bal) {
        *hint = j;
        return __shfl_sync(FULL, L.pmprev, __ffs(bal) - 1);
      }
    }
    if (t.G) {  // candidates by G, super-blocks by SG
      int32_t P = j >> 5;
      const int32_t Pn = (nb - 1) >> 5;
      unsigned bal = __ballot_sync(FULL, P * 32 + lane > j && P * 32 + lane < nb && t.G[P * 32 + lane] >= dur);
      for (;;) {
        while (bal) {
          const int32_t pos = P * 32 + __ffs(bal) - 1;
          bal &= bal - 1;
          L = tl_load(t, pos);
          const bool fit = lane < L.c && L.e > L.pmprev && L.s - L.pmprev >= dur;
          const unsigned b2 = __ballot_sync(FULL, fit);
          if (b2) {
            *hint = b2 & 1u ? pos - 1 : pos;
            return __shfl_sync(FULL, L.pmprev, __ffs(b2) - 1);
          }
        }
        int32_t nP = -1;
        for (int32_t P0 = P + 1; P0 <= Pn && nP < 0; P0 += 32) {
          const unsigned sb = __ballot_sync(FULL, P0 + lane <= Pn && t.SG[P0 + lane] >= dur);
          if (sb) nP = P0 + __ffs(sb) - 1;
        }
        if (nP < 0) return last;
        P = nP;
        bal = __ballot_sync(FULL, P * 32 + lane < nb && t.G[P * 32 + lane] >= dur);
      }
    }
    for (int32_t p0 = j + 1; p0 < nb; p0 += 32) {
      const int32_t q = p0 + lane;
      bool cand = false;
      if (q < nb) {
        const int64_t pe = t.pmEnd[q - 1];
        cand = t.gub[q] >= dur || (t.fE[q] > pe && t.fS[q] - pe >= dur);
      }
      unsigned bal = __ballot_sync(FULL, cand);
      while (bal) {
        const int32_t pos = p0 + __ffs(bal) - 1;
        bal &= bal - 1;
        L = tl_load(t, pos);
        const bool fit = lane < L.c && L.e > L.pmprev && L.s - L.pmprev >= dur;
        const unsigned b2 = __ballot_sync(FULL, fit);
        if (b2) {
          *hint = b2 & 1u ? pos - 1 : pos;
          return __shfl_sync(FULL, L.pmprev, __ffs(b2) - 1);
        }
      }
    }
    return last;
  }
  // inside the window (pmEnd[nb - 1] = last > earliest)
  const int64_t wup = __shfl_up_sync(FULL, wpm, 1);  // (every lane shuffles)
  const int64_t wprev = lane == 0 ? pm_lo : wup;      // pmEnd[p - 1]
  const int jl = __ffs(__ballot_sync(FULL, in && wpm > earliest)) - 1;
  BlockLoad L = tl_load_known(t, __shfl_sync(FULL, wid, jl), __shfl_sync(FULL, wc, jl), __shfl_sync(FULL, wprev, jl));
  const int k0 = __ffs(__ballot_sync(FULL, lane < L.c && L.pm > earliest)) - 1;
  const int64_t s0 = __shfl_sync(FULL, L.s, k0);
  const int32_t jw = lo + jl;
  if (s0 >= earliest && s0 - earliest >= dur) {
    *hint = k0 > 0 || jw == 0 ? jw : jw - 1;
    return earliest;
  }
  if (gmax < dur) return last;
  {
    const bool fit = lane > k0 && lane < L.c && L.e > L.pmprev && L.s - L.pmprev >= dur;
    const unsigned bal = __ballot_sync(FULL, fit);
    if (bal) {
      *hint = jw;
      return __shfl_sync(FULL, L.pmprev, __ffs(bal) - 1);
    }
  }
  unsigned bal = __ballot_sync(FULL, in && lane > jl && (wgu >= dur || (wfe > wprev && wfs - wprev >= dur)));
  while (bal) {
    const int q = __ffs(bal) - 1;
    bal &= bal - 1;
    L = tl_load_known(t, __shfl_sync(FULL, wid, q), __shfl_sync(FULL, wc, q), __shfl_sync(FULL, wprev, q));
    const bool fit = lane < L.c && L.e > L.pmprev && L.s - L.pmprev >= dur;
    const unsigned b2 = __ballot_sync(FULL, fit);
    if (b2) {
      *hint = b2 & 1u ? lo + q - 1 : lo + q;
      return __shfl_sync(FULL, L.pmprev, __ffs(b2) - 1);
    }
  }
  return last;
}

// Recomputes the meta of the block at position pos from its entries (warp-collective)
// and propagates pmEnd forward while it changes.  Returns the block's gap upper bound.
// *ghi (optional): the last position whose G was rewritten.
__device__ int64_t tl_meta(const TLView t, int32_t pos, int32_t nb, bool propagate = true, int32_t* ghi = nullptr) {
  const int lane = threadIdx.x & 31;
  const int32_t b = t.id[pos], c = t.cnt[pos];
  const int64_t s = lane < c ? t.S[(int64_t)b * kTB + lane] : INT64_MAX;
  const int64_t e = lane < c ? t.E[(int64_t)b * kTB + lane] : INT64_MIN;
  const int64_t inc = warp_incl_max(e);
  const int64_t prev = __shfl_up_sync(FULL, inc, 1);
  int64_t g = (lane >= 1 && lane < c && e > prev) ? s - prev : -1;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t y = __shfl_xor_sync(FULL, g, o);
    g = y > g ? y : g;
  }
  const int64_t mx = __shfl_sync(FULL, inc, 31);
  const int64_t fs = __shfl_sync(FULL, s, 0), fe = __shfl_sync(FULL, e, 0);
  int32_t last_g = pos;
  if (lane == 0) {
    t.maxE[pos] = mx;
    t.fS[pos] = fs;
    t.fE[pos] = fe;
    t.gub[pos] = g;
    const int64_t carry = pos > 0 ? t.pmEnd[pos - 1] : INT64_MIN;
    int64_t pm = carry > mx ? carry : mx;
    t.pmEnd[pos] = pm;
    int32_t lc = pos;  // the last position whose pmEnd was rewritten
    for (int32_t q = pos + 1; propagate && q < nb; ++q) {  // forward while it changes
      const int64_t np = t.maxE[q] > pm ? t.maxE[q] : pm;
      if (np == t.pmEnd[q]) break;
      t.pmEnd[q] = np;
      pm = np;
      lc = q;
    }
    if (t.G) {  // G depends on the block and its carry: pos, and every q whose carry changed
      t.G[pos] = tl_gbound(pos, g, fs, fe, carry);
      if (propagate) {
        last_g = min(lc + 1, nb - 1);
        for (int32_t q = pos + 1; q <= last_g; ++q)
          t.G[q] = tl_gbound(q, t.gub[q], t.fS[q], t.fE[q], t.pmEnd[q - 1]);
      }
    }
  }
  last_g = __shfl_sync(FULL, last_g, 0);
  if (ghi) *ghi = last_g;
  __syncwarp();
  return g;
}

// DeviceTimeline::reserve(start, dur) (placement.cpp:23-32): upper_bound insert into the
// last block whose first start <= s.  Block splits (a full target block) take
// tl_insert_split; every other insert is done from registers: one round of meta loads at
// the target (guessed by the query: `hint`, checked here), one for the block's entries,
// then the stores (the block's meta rebuilt from the entries in registers, the prefix
// maxima propagated only when the block's own changed).
__device__ void tl_insert_split(const TLView t, int32_t* Kp, int64_t* gmaxp, int64_t* lastp, int64_t s, int64_t dur,
                                int32_t nb, int32_t j0) {
  const int lane = threadIdx.x & 31;
  const int64_t e = s + dur;
  const int64_t last = *lastp;
  int64_t gnew = -1;  // gaps this insert may create (upper bound bookkeeping)
  int32_t j = j0, sg_lo = j0, sg_hi = -1;
  if (t.cnt[j] == kTB) {  // split in halves: the upper half moves to a new block after j
    const int32_t nbid = nb;  // ids are allocated densely: the next free id is nb
    const int32_t b = t.id[j];
    if (lane >= kTB / 2) {
      t.S[(int64_t)nbid * kTB + lane - kTB / 2] = t.S[(int64_t)b * kTB + lane];
      t.E[(int64_t)nbid * kTB + lane - kTB / 2] = t.E[(int64_t)b * kTB + lane];
    }
    // shift positions j+1 .. nb-1 up by one (from the top, 32 at a time)
    for (int32_t top = nb; top > j + 1; top -= 32) {
      const int32_t lo = max(j + 1, top - 32);
      const int32_t q = lo + lane;
      int32_t vi = 0, vc = 0;
      int64_t m1 = 0, m2 = 0, m3 = 0, m4 = 0, m5 = 0, m6 = 0;
      const bool act = q < top;
      if (act) {
        vi = t.id[q]; vc = t.cnt[q]; m1 = t.maxE[q]; m2 = t.pmEnd[q]; m3 = t.fS[q]; m4 = t.fE[q]; m5 = t.gub[q];
        if (t.G) m6 = t.G[q];
      }
      __syncwarp();
      if (act) {
        t.id[q + 1] = vi; t.cnt[q + 1] = vc; t.maxE[q + 1] = m1; t.pmEnd[q + 1] = m2; t.fS[q + 1] = m3;
        t.fE[q + 1] = m4; t.gub[q + 1] = m5;
        if (t.G) t.G[q + 1] = m6;
      }
      __syncwarp();
    }
    if (lane == 0) {
      t.id[j + 1] = nbid;
      t.cnt[j + 1] = kTB / 2;
      t.cnt[j] = kTB / 2;
      t.pmEnd[j + 1] = t.pmEnd[j];  // placeholder until tl_meta below
      *t.nb = ++nb;
    }
    nb = __shfl_sync(FULL, nb, 0);  // every lane's bound (tl_sg loops over it)
    tl_meta(t, j, nb, false);  // position j + 1 is not valid yet: no propagation
    tl_meta(t, j + 1, nb);
    sg_hi = nb - 1;  // every later position moved
    if (t.fS[j + 1] <= s) ++j;
  }
  // insert into block j at the upper_bound position
  const int32_t b = t.id[j], c = t.cnt[j];
  const int64_t vs = lane < c ? t.S[(int64_t)b * kTB + lane] : INT64_MAX;
  const int64_t ve = lane < c ? t.E[(int64_t)b * kTB + lane] : 0;
  const int q = __popc(__ballot_sync(FULL, lane < c && vs <= s));
  __syncwarp();
  if (lane >= q && lane < c) {
    t.S[(int64_t)b * kTB + lane + 1] = vs;
    t.E[(int64_t)b * kTB + lane + 1] = ve;
  }
  if (lane == q) {
    t.S[(int64_t)b * kTB + lane] = s;
    t.E[(int64_t)b * kTB + lane] = e;
  }
  if (lane == 0) t.cnt[j] = c + 1;
  __syncwarp();
  int32_t ghi;
  gnew = tl_meta(t, j, nb, true, &ghi);
  if (t.G) tl_sg(t, sg_lo >> 5, max(sg_hi, ghi) >> 5, nb);
  // the next block's first gap may have changed (its carry in); count it in the bound
  if (j + 1 < nb) {
    const int64_t pe = t.pmEnd[j];
    const int64_t g1 = t.fE[j + 1] > pe ? t.fS[j + 1] - pe : -1;
    gnew = g1 > gnew ? g1 : gnew;
  }
  // the first gap of block j itself (against its carry)
  {
    const int64_t pe = j > 0 ? t.pmEnd[j - 1] : INT64_MIN;
    if (j > 0 && t.fE[j] > pe) {
      const int64_t g0 = t.fS[j] - pe;
      gnew = g0 > gnew ? g0 : gnew;
    }
  }
  if (lane == 0) {
    if (gnew > *gmaxp) *gmaxp = gnew;
    *lastp = last > e ? last : e;
    *Kp = *Kp + 1;
  }
  __syncwarp();
}


__device__ void tl_insert(const TLView t, int32_t* Kp, int64_t* gmaxp, int64_t* lastp, int64_t s, int64_t dur,
                          int32_t hint) {
  const int lane = threadIdx.x & 31;
  const int64_t e = s + dur;
  const int32_t nb = *t.nb;
  const int64_t last = *lastp;
  if (nb == 0) {
    if (lane == 0) {
      t.id[0] = 0;
      t.cnt[0] = 1;
      t.S[0] = s;
      t.E[0] = e;
      t.maxE[0] = e;
      t.pmEnd[0] = e;
      t.fS[0] = s;
      t.fE[0] = e;
      t.gub[0] = -1;
      if (t.G) {
        t.G[0] = -1;
        t.SG[0] = -1;
      }
      *t.nb = 1;
      *Kp = 1;
      *lastp = e;
    }
    __syncwarp();
    return;
  }
  // target j: the last position with fS <= s (position 0 when s precedes everything)
  int32_t j = hint >= 0 && hint < nb ? hint : nb - 1;
  struct Row {
    int64_t fs, fs1, fe1, carry, pm;
    int32_t id, c;
  };
  auto load = [&](int32_t q) {
    Row r;
    r.fs = t.fS[q];
    r.fs1 = q + 1 < nb ? t.fS[q + 1] : INT64_MAX;
    r.fe1 = q + 1 < nb ? t.fE[q + 1] : 0;
    r.carry = q > 0 ? t.pmEnd[q - 1] : INT64_MIN;
    r.pm = t.pmEnd[q];
    r.id = t.id[q];
    r.c = t.cnt[q];
    return r;
  };
  Row r = load(j);
  if (!((j == 0 || r.fs <= s) && r.fs1 > s)) {
    if (t.fS[nb - 1] <= s) {
      j = nb - 1;
    } else {
      j = warp_first_true(0, nb - 1, [&](int32_t q) { return t.fS[q] > s; }) - 1;
      if (j < 0) j = 0;
    }
    r = load(j);
  }
  if (r.c == kTB) {
    tl_insert_split(t, Kp, gmaxp, lastp, s, dur, nb, j);
    return;
  }
  const int32_t gp = (j & ~31) + lane;
  const int64_t gsb = t.G && gp < nb ? t.G[gp] : -1;  // G of j's super-block
  const int32_t b = r.id, c = r.c;
  const int64_t vs = lane < c ? t.S[(int64_t)b * kTB + lane] : INT64_MAX;
  const int64_t ve = lane < c ? t.E[(int64_t)b * kTB + lane] : INT64_MIN;
  const int q = __popc(__ballot_sync(FULL, lane < c && vs <= s));
  const int64_t us = __shfl_up_sync(FULL, vs, 1), ue = __shfl_up_sync(FULL, ve, 1);
  const int64_t ns = lane < q ? vs : lane == q ? s : us;  // lanes > c: unused
  const int64_t ne = lane < q ? ve : lane == q ? e : ue;
  if (lane >= q && lane <= c) {
    t.S[(int64_t)b * kTB + lane] = ns;
    t.E[(int64_t)b * kTB + lane] = ne;
  }
  const int32_t c1 = c + 1;
  const int64_t em = lane < c1 ? ne : INT64_MIN;
  const int64_t inc = warp_incl_max(em);
  const int64_t pv = __shfl_up_sync(FULL, inc, 1);
  int64_t g = (lane >= 1 && lane < c1 && em > pv) ? ns - pv : -1;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const int64_t y = __shfl_xor_sync(FULL, g, o);
    g = y > g ? y : g;
  }
  const int64_t mx = __shfl_sync(FULL, inc, 31);
  const int64_t fs = __shfl_sync(FULL, ns, 0), fe = __shfl_sync(FULL, ne, 0);
  const int64_t pmn = r.carry > mx ? r.carry : mx;
  const int64_t gj = tl_gbound(j, g, fs, fe, r.carry);  // the block's gaps + its first one
  // + the next block's first gap (its carry is this block's prefix max)
  int64_t gnew = gj;
  if (j + 1 < nb && r.fe1 > pmn && r.fs1 - pmn > gnew) gnew = r.fs1 - pmn;
  int32_t lc = j;  // the last position whose prefix max changed
  if (lane == 0) {
    t.cnt[j] = c1;
    t.maxE[j] = mx;
    t.fS[j] = fs;
    t.fE[j] = fe;
    t.gub[j] = g;  // block-local, as tl_meta
    t.pmEnd[j] = pmn;
    if (pmn != r.pm) {  // forward while it changes
      int64_t pm = pmn;
      for (int32_t x = j + 1; x < nb; ++x) {
        const int64_t np = t.maxE[x] > pm ? t.maxE[x] : pm;
        if (np == t.pmEnd[x]) break;
        t.pmEnd[x] = np;
        pm = np;
        lc = x;
      }
    }
    if (gnew > *gmaxp) *gmaxp = gnew;
    *lastp = last > e ? last : e;
    *Kp = *Kp + 1;
  }
  if (t.G) {
    lc = __shfl_sync(FULL, lc, 0);
    if (pmn == r.pm) {  // only G[j] changed: its super-block's max from the loaded values
      int64_t x = gp == j ? gj : gsb;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t y = __shfl_xor_sync(FULL, x, o);
        x = y > x ? y : x;
      }
      if (lane == 0) {
        t.G[j] = gj;
        t.SG[j >> 5] = x;
      }
    } else {  // the carries of j+1 .. lc+1 changed too
      const int32_t hi = min(lc + 1, nb - 1);
      if (lane == 0) {
        t.G[j] = gj;
        for (int32_t x = j + 1; x <= hi; ++x) t.G[x] = tl_gbound(x, t.gub[x], t.fS[x], t.fE[x], t.pmEnd[x - 1]);
      }
      __syncwarp();
      tl_sg(t, j >> 5, hi >> 5, nb);
    }
  }
  __syncwarp();
}

struct PlaceArgs {
  int32_t n, D;
  const int32_t* seq;
  const int64_t* w;
  const int64_t* mem;
  const int32_t* in_off;
  const int32_t* in_src;
  const int64_t* in_cost;
  const int64_t* back;  // max out-edge cost per node (>= 0)
  const int64_t* cap;   // [D] sorted by id
  TLArrays tl[2];
  bool meta_smem;  // timeline block meta in dynamic shared memory (small coarse graphs)
  long long* debug;  // optional: cycles of each CTA
  int64_t* finish;      // [n] (adjust)
  int32_t* dev[2];      // [n] device position by node index (order, adjust)
  int64_t* pdm[2];      // [D]
  int32_t* flags[2];    // [0] oom
  bool run[2];
  bool decisions;
  int32_t *dec_prev, *dec_chosen;
  int64_t *dec_back, *dec_est;
  uint8_t *dec_reloc, *dec_be;
};

__device__ int32_t most_free(const int64_t* avail, int32_t D) {  // placement.cpp:72-78
  int32_t best = 0;
  for (int32_t d = 1; d < D; ++d)
    if (avail[d] > avail[best]) best = d;
  return best;
}

// Up to kPlaceBatch independent (order, graph) jobs per launch: CTA 2j runs job j's
// order_place, CTA 2j + 1 its adjusting_placement.
constexpr int kPlaceBatch = 8;
struct PlaceBatch {
  PlaceArgs a[kPlaceBatch];
};

__global__ void __launch_bounds__(256) k_place(const __grid_constant__ PlaceBatch batch) {
  const PlaceArgs& a = batch.a[blockIdx.x >> 1];
  __shared__ int32_t sK[kMaxD], snb[kMaxD];
  __shared__ int64_t sg[kMaxD], sl[kMaxD], savail[kMaxD], spdm[kMaxD], savail2[kMaxD];
  __shared__ long long sA[kMaxD], sB[kMaxD], sA2[kMaxD], sB2[kMaxD];
  __shared__ int64_t sest[kMaxD], spre[kMaxD];
  __shared__ int32_t shint[kMaxD];
  const int which = blockIdx.x & 1;  // 0 order_place, 1 adjusting_placement
  const long long t0 = clock64();
  if (!a.run[which]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int32_t D = a.D;
  TLArrays tl = a.tl[which];
  tl.nb = snb;
  if (a.meta_smem) {  // same layout as the global meta, carved from dynamic shared memory
    extern __shared__ int64_t dyn[];
    const int64_t mc = static_cast<int64_t>(D) * tl.maxb;
    tl.maxE = dyn;
    tl.pmEnd = dyn + mc;
    tl.fS = dyn + 2 * mc;
    tl.fE = dyn + 3 * mc;
    tl.gub = dyn + 4 * mc;
    tl.id = reinterpret_cast<int32_t*>(dyn + 5 * mc);
    tl.cnt = tl.id + mc;
    tl.G = nullptr;  // the scan reads the on-chip meta directly
    tl.SG = nullptr;
  }
  for (int d = tid; d < D; d += blockDim.x) {
    sK[d] = 0;
    snb[d] = 0;
    sg[d] = -1;
    sl[d] = 0;
    savail[d] = a.cap[d];
    sA[d] = LLONG_MIN;
    sB[d] = LLONG_MIN;
    sA2[d] = LLONG_MIN;
    sB2[d] = LLONG_MIN;
    spdm[d] = 0;
  }
  __syncthreads();
  int32_t* dev = a.dev[which];
  if (which == 0) {
    // order_place (placement.cpp:138-157): warp 0 only
    if (warp != 0) return;
    int32_t cursor = 0;
    bool oom = false;
    for (int32_t k = 0; k < a.n; ++k) {
      const int32_t v = a.seq[k];
      const int64_t w = a.w[v], mv = a.mem[v];
      int32_t target = -1;
      for (int32_t d0 = cursor; d0 < D; d0 += 32) {
        const int32_t d = d0 + lane;
        const unsigned b = __ballot_sync(FULL, d < D && savail[d] >= mv);
        if (b) {
          target = d0 + __ffs(b) - 1;
          break;
        }
      }
      if (target >= 0) {
        cursor = target;
      } else {
        target = most_free(savail, D);
        oom = true;
      }
      const TLView t = tl.view(target);
      int32_t hint;
      const int64_t start = tl_query(t, sK[target], sg[target], sl[target], 0, w, &hint);
      tl_insert(t, &sK[target], &sg[target], &sl[target], start, w, hint);
      if (lane == 0) {
        dev[v] = target;
        savail[target] -= mv;
        spdm[target] += mv;
      }
      __syncwarp();
    }
    for (int d = lane; d < D; d += 32) a.pdm[0][d] = spdm[d];
    if (lane == 0) a.flags[0][0] = oom ? 1 : 0;
    if (lane == 0 && a.debug) a.debug[0] = clock64() - t0;
    return;
  }
  // adjusting_placement (placement.cpp:172-216)
  // The static inputs of a step are loaded in a software pipeline over the order, one
  // dependent stage per step, so no step waits on a chain of global loads: during step k
  // the CTA loads node k+4's id, node k+3's row bounds / compute / memory / back cost, this
  // thread's in-edge of node k+2 (source, cost) and the finish time / device of node
  // k+1's source.  Two block barriers per node: X (in-edge maxima ready; the previous
  // node's commit done) and Y (the per-device queries done).  Every warp takes the
  // decision itself, then the commit warp inserts the node into its device's timeline
  // while the other warps already reduce the next node's in-edges.  So a finish time /
  // device loaded for node k+1 may predate the commits of nodes k-1 and k: every thread
  // keeps those two (it took their decisions) and patches them in.  In-edges beyond
  // blockDim.x per node are read in the step itself (node k-1 committed by then).
  __shared__ int64_t s_be_start;
  int32_t prev = 0;
  bool oom = false;
  const int32_t n = a.n;
  const int T = blockDim.x;
  const int cw = nwarps - 1;  // the commit warp (warp 0 holds the in-edges of small rows)
  int32_t v1 = -1, dv1 = 0, v2 = -1, dv2 = 0;  // nodes k-1, k-2: index, device, finish
  int64_t f1 = 0, f2 = 0;
  // stage registers: s (seq id), b (row), c (edge), d (edge with finish/device)
  int32_t s_v = -1;
  int32_t b_v = -1, b_ib = 0, b_ie = 0;
  int64_t b_w = 0, b_mv = 0, b_bk = 0;
  int32_t c_v = -1, c_ib = 0, c_ie = 0, c_p = -1;
  int64_t c_w = 0, c_mv = 0, c_c = 0, c_bk = 0;
  int32_t d_v = -1, d_ib = 0, d_ie = 0, d_p = -1, d_dd = 0;
  int64_t d_w = 0, d_mv = 0, d_c = 0, d_f = 0, d_bk = 0;
  // next-stage registers: loaded at step k (issue), moved into the stages only after the
  // step's work (shift), so no register move waits on a load in flight
  int32_t nd_v = -1, nd_ib = 0, nd_ie = 0, nd_p = -1, nd_dd = 0;
  int64_t nd_w = 0, nd_mv = 0, nd_c = 0, nd_f = 0, nd_bk = 0;
  int32_t nc_v = -1, nc_ib = 0, nc_ie = 0, nc_p = -1;
  int64_t nc_w = 0, nc_mv = 0, nc_c = 0, nc_bk = 0;
  int32_t nb_v = -1, nb_ib = 0, nb_ie = 0;
  int64_t nb_w = 0, nb_mv = 0, nb_bk = 0;
  int32_t ns_v = -1;
  // 0, but opaque to the compiler's uniformity analysis: the pipelined node loads then
  // count as per-thread values and stay in vector registers.  With a provably uniform
  // address the loaded row / weight / memory go to uniform registers, and the R2UR that
  // moves them there waits for the load right where it is issued (~1.5 us per node).
  // (threadIdx.x < blockDim.x <= 1024 < n + 4096, which ptxas cannot fold: n is a parameter)
  const int32_t divz = static_cast<uint32_t>(tid) >= static_cast<uint32_t>(a.n) + 4096u ? 1 : 0;
  auto issue = [&](int32_t k) {  // loads issued at step k, consumed one step later
    // node k+1: finish / device of this thread's in-edge source (from stage c)
    nd_v = c_v; nd_ib = c_ib; nd_ie = c_ie; nd_p = c_p; nd_dd = 0;
    nd_w = c_w; nd_mv = c_mv; nd_c = c_c; nd_f = 0; nd_bk = c_bk;
    if (nd_p >= 0) {
      nd_f = a.finish[nd_p];
      nd_dd = dev[nd_p];
    }
    // node k+2: this thread's in-edge (from stage b)
    nc_v = b_v; nc_ib = b_ib; nc_ie = b_ie; nc_p = -1;
    nc_w = b_w; nc_mv = b_mv; nc_c = 0; nc_bk = b_bk;
    if (nc_v >= 0 && nc_ib + tid < nc_ie) {
      nc_p = a.in_src[nc_ib + tid];
      nc_c = a.in_cost[nc_ib + tid];
    }
    // node k+3: row bounds, compute, memory, back cost (from stage s)
    nb_v = s_v; nb_ib = 0; nb_ie = 0;
    nb_w = 0; nb_mv = 0; nb_bk = 0;
    if (nb_v >= 0) {
      nb_ib = a.in_off[nb_v];
      nb_ie = a.in_off[nb_v + 1];
      nb_w = a.w[nb_v];
      nb_mv = a.mem[nb_v];
      nb_bk = a.back[nb_v];
    }
    // node k+4: id
    ns_v = k + 4 < n ? a.seq[k + 4 + divz] : -1;
  };
  auto shift = [&] {
    d_v = nd_v; d_ib = nd_ib; d_ie = nd_ie; d_p = nd_p; d_dd = nd_dd; d_w = nd_w; d_mv = nd_mv; d_c = nd_c; d_f = nd_f;
    d_bk = nd_bk;
    c_v = nc_v; c_ib = nc_ib; c_ie = nc_ie; c_p = nc_p; c_w = nc_w; c_mv = nc_mv; c_c = nc_c; c_bk = nc_bk;
    b_v = nb_v; b_ib = nb_ib; b_ie = nb_ie; b_w = nb_w; b_mv = nb_mv; b_bk = nb_bk;
    s_v = ns_v;
  };
  for (int32_t k = -4; k < 0; ++k) {  // after this: d = node 0, c = 1, b = 2, s = 3
    issue(k);
    shift();
  }
  __syncthreads();
  long long ph[6] = {0, 0, 0, 0, 0, 0}, tp = 0;
  auto mark = [&](int i) {
    if (a.debug && tid == 0) {
      const long long t = clock64();
      ph[i] += t - tp;
      tp = t;
    }
  };
  if (a.debug && tid == 0) tp = clock64();
  for (int32_t k = 0; k < n; ++k) {
    const int32_t v = d_v;
    const int64_t w = d_w, mv = d_mv, back = d_bk;
    // this step's inputs, then the next steps' loads (consumed from step k+1 on)
    const int32_t my_p = d_p, my_dd0 = d_dd, ib = d_ib, ie = d_ie;
    const int64_t my_c = d_c, my_f0 = d_f;
    issue(k);
    // available memory and the in-edge maxima double-buffered by node parity: the commit of
    // node k-1 writes one copy while node k's decision reads the other, and node k's in-edge
    // reduction fills one pair of maxima while the other is reset after node k-1's queries
    int64_t* const avail = (k & 1) ? savail2 : savail;
    int64_t* const avail_next = (k & 1) ? savail : savail2;
    long long* const cA = (k & 1) ? sA2 : sA;
    long long* const cB = (k & 1) ? sB2 : sB;
    mark(0);
    {
      // per-device maxima of the node's in-edges, warp by warp: one device at a time (ballot
      // over the lanes still unassigned, full-warp 64-bit max by two redux.sync on
      // order-preserving words), then one shared-memory update per (warp, device) instead of
      // a contended CAS per edge (64-bit shared atomicMax is a CAS loop on sm_100a)
      const bool act = my_p >= 0;
      int64_t f = my_f0;
      int32_t dd = my_dd0;
      if (my_p == v1) {
        f = f1;
        dd = dv1;
      } else if (my_p == v2) {
        f = f2;
        dd = dv2;
      }
      unsigned todo = __ballot_sync(FULL, act);  // (rows over 32 in-edges: every warp with edges)
      while (todo) {
        const int leader = __ffs(todo) - 1;
        const int32_t d = __shfl_sync(FULL, dd, leader);
        const bool mine = act && dd == d;
        todo &= ~__ballot_sync(FULL, mine);
        const long long ga = warp_max_i64(mine ? f : LLONG_MIN), gb = warp_max_i64(mine ? f + my_c : LLONG_MIN);
        if (lane == leader) {
          atomicMax(&cA[d], ga);
          atomicMax(&cB[d], gb);
        }
      }
    }
    for (int32_t q = ib + T + tid; q < ie; q += T) {
      const int32_t p = a.in_src[q];
      int64_t f = a.finish[p];
      int32_t dd = dev[p];
      if (p == v1) {
        f = f1;
        dd = dv1;
      }
      atomicMax(&cA[dd], static_cast<long long>(f));
      atomicMax(&cB[dd], static_cast<long long>(f + a.in_cost[q]));
    }
    __syncthreads();  // X
    mark(1);
    for (int32_t d = warp; d < D; d += nwarps) {
      long long mb = LLONG_MIN;
      for (int32_t x = lane; x < D; x += 32)
        if (x != d) mb = max(mb, cB[x]);
#pragma unroll
      for (int o = 16; o; o >>= 1) mb = max(mb, __shfl_xor_sync(FULL, mb, o));
      int64_t pre = 0;
      if (cA[d] > pre) pre = cA[d];
      if (mb > pre) pre = mb;
      int64_t est = kNever;
      int32_t hint = -1;
      if (avail[d] >= mv) est = tl_query(tl.view(d), sK[d], sg[d], sl[d], pre, w, &hint);
      if (lane == 0) {
        sest[d] = est;
        spre[d] = pre;
        shint[d] = hint;
      }
    }
    __syncthreads();  // Y
    mark(2);
    // the decision (placement.cpp:185-210), by every warp (lanes = devices): best = the
    // lowest position among the feasible devices with the least est
    int32_t best = -1;
    int64_t bestv = kNever;
    for (int32_t d0 = 0; d0 < D; d0 += 32) {
      const int32_t d = d0 + lane;
      const bool ok = d < D && avail[d] >= mv;
      const int64_t e = ok ? sest[d] : kNever;
      const int64_t m = warp_min_i64(e);
      const unsigned hit = __ballot_sync(FULL, ok && e == m);
      if (hit && (best < 0 || m < bestv)) {
        best = d0 + __ffs(hit) - 1;
        bestv = m;
      }
    }
    const int64_t ep = sest[prev];
    int32_t chosen;
    int64_t start = 0;
    bool be = false, reloc = false;
    if (best >= 0 && (ep == kNever || ep - bestv > back)) {
      chosen = best;
      start = bestv;
      reloc = chosen != prev;
    } else if (ep != kNever) {
      chosen = prev;
      start = ep;
    } else {
      chosen = most_free(avail, D);
      be = true;
      oom = true;
    }
    if (a.decisions && tid == 0) {
      a.dec_prev[k] = prev;
      a.dec_back[k] = back;
      a.dec_chosen[k] = chosen;
      a.dec_reloc[k] = reloc;
      a.dec_be[k] = be;
    }
    for (int d = tid; d < D; d += blockDim.x) {  // the queries are done with this node's maxima
      cA[d] = LLONG_MIN;
      cB[d] = LLONG_MIN;
    }
    if (a.decisions)
      for (int d = tid; d < D; d += blockDim.x) a.dec_est[(int64_t)k * D + d] = sest[d];
    int32_t hint = shint[chosen];  // (read before the next node's queries rewrite it)
    if (be) {  // block-uniform: the start needs a query on the most free device
      if (warp == cw) {
        start = tl_query(tl.view(chosen), sK[chosen], sg[chosen], sl[chosen], spre[chosen], w, &hint);
        if (lane == 0) s_be_start = start;
      }
      __syncthreads();
      start = s_be_start;
    }
    if (warp == cw) {
      const TLView t = tl.view(chosen);
      tl_insert(t, &sK[chosen], &sg[chosen], &sl[chosen], start, w, hint);
      for (int d = lane; d < D; d += 32) avail_next[d] = avail[d] - (d == chosen ? mv : 0);
      if (lane == 0) {
        a.finish[v] = start + w;
        dev[v] = chosen;
        spdm[chosen] += mv;
      }
    }
    v2 = v1;
    dv2 = dv1;
    f2 = f1;
    v1 = v;
    dv1 = chosen;
    f1 = start + w;
    prev = chosen;
    shift();  // this step's loads have had the whole step to arrive
    mark(3);
  }
  __syncthreads();  // the last commit
  if (a.debug && tid == 0)
    for (int i = 0; i < 5; ++i) a.debug[2 + i] = ph[i];
  for (int d = tid; d < D; d += blockDim.x) a.pdm[1][d] = spdm[d];
  if (tid == 0) a.flags[1][0] = oom ? 1 : 0;
  if (tid == 0 && a.debug) a.debug[1] = clock64() - t0;
}

__global__ void k_back_cost(const int32_t* out_off, const int64_t* out_cost, int32_t n, int64_t* back) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = 0;
    if (out_cost)
      for (int32_t k = out_off[v]; k < out_off[v + 1]; ++k) b = out_cost[k] > b ? out_cost[k] : b;
    back[v] = b;
  }
}

__global__ void k_expand(const int32_t* cl, const int32_t* cdev, const int64_t* mem, int32_t n, int32_t D,
                         int32_t* dev_node, int64_t* pdm) {
  extern __shared__ unsigned long long sm[];
  for (int d = threadIdx.x; d < D; d += blockDim.x) sm[d] = 0;
  __syncthreads();
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = cdev[cl[v]];
    dev_node[v] = d;
    atomicAdd(&sm[d], static_cast<unsigned long long>(mem[v]));
  }
  __syncthreads();
  for (int d = threadIdx.x; d < D; d += blockDim.x)
    if (sm[d]) atomicAdd(reinterpret_cast<unsigned long long*>(&pdm[d]), sm[d]);
}

void alloc_tl(dp_ctx* ctx, int32_t D, int32_t n, DevBuf<int64_t>& store, DevBuf<int32_t>& store32, TLArrays& t) {
  // a device holding K intervals uses at most K/16 + 1 blocks (splits leave halves of 16)
  const int64_t maxb = n / (kTB / 2) + 2;
  const int64_t ent = (int64_t)D * maxb * kTB, meta = (int64_t)D * maxb, sg = (int64_t)D * (maxb / 32 + 1);
  store.alloc(ctx, static_cast<size_t>(2 * ent + 6 * meta + sg));
  store32.alloc(ctx, static_cast<size_t>(2 * meta));
  t.S = store.p;
  t.E = store.p + ent;
  t.maxE = store.p + 2 * ent;
  t.pmEnd = t.maxE + meta;
  t.fS = t.pmEnd + meta;
  t.fE = t.fS + meta;
  t.gub = t.fE + meta;
  t.G = t.gub + meta;
  t.SG = t.G + meta;
  t.id = store32.p;
  t.cnt = store32.p + meta;
  t.maxb = static_cast<int32_t>(maxb);
  t.nb = nullptr;
}

}  // namespace

Devices devices_sorted(const dp_devices_t* d) {
  if (d->count <= 0) fail(DP_E_INVALID_VALUE, "device list is empty");
  std::vector<std::pair<int32_t, int64_t>> v;
  for (int32_t i = 0; i < d->count; ++i) v.push_back({d->id[i], d->memory_bytes[i]});
  std::sort(v.begin(), v.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  Devices out;
  for (size_t i = 0; i < v.size(); ++i) {
    if (v[i].second <= 0) fail(DP_E_INVALID_VALUE, "device %d has non-positive memory capacity", v[i].first);
    if (i && v[i].first == v[i - 1].first) fail(DP_E_DUPLICATE_ID, "device id %d repeats", v[i].first);
    out.ids.push_back(v[i].first);
    out.cap.push_back(v[i].second);
  }
  out.D = static_cast<int32_t>(out.ids.size());
  return out;
}

struct PlaceJob {
  dp_ctx* ctx = nullptr;
  PlaceArgs a{};
  DevBuf<int64_t> back, cap, finish;
  DevBuf<int64_t> store[2];
  DevBuf<int32_t> store32[2];
  DevBuf<long long> dbg;
  size_t dyn = 0;
};

PlaceJob* place_prepare(DevGraph& g, const int32_t* seq, const Devices& devs, PlaceOut* order_out,
                        PlaceOut* adjust_out, bool want_decisions) {
  dp_ctx* ctx = g.ctx;
  const int32_t n = g.n, D = devs.D;
  if (D > kMaxD) fail(DP_E_UNSUPPORTED, "at most %d devices are supported", kMaxD);
  auto* j = new PlaceJob;
  PlaceHandle guard(j);
  j->ctx = ctx;
  PlaceArgs& a = j->a;
  a.n = n;
  a.D = D;
  a.seq = seq;
  a.w = g.w.p;
  a.mem = g.mem.p;
  a.in_off = g.in_off.p;
  a.in_src = g.in_src.p;
  a.in_cost = g.in_cost.p;
  j->back.alloc(ctx, n > 0 ? n : 1);
  j->cap.alloc(ctx, D);
  j->finish.alloc(ctx, n > 0 ? n : 1);
  j->cap.upload(devs.cap.data(), D);
  DP_LAUNCH(ctx, k_back_cost, grid_for(n, 256), 256, 0, g.out_off.p, g.has_cost ? g.out_cost.p : nullptr, n,
            j->back.p);
  a.back = j->back.p;
  a.cap = j->cap.p;
  a.finish = j->finish.p;
  PlaceOut* outs[2] = {order_out, adjust_out};
  for (int w = 0; w < 2; ++w) {
    a.run[w] = outs[w] != nullptr;
    if (!outs[w]) continue;
    alloc_tl(ctx, D, n > 0 ? n : 1, j->store[w], j->store32[w], a.tl[w]);
    outs[w]->dev.alloc(ctx, n > 0 ? n : 1);
    outs[w]->per_dev_mem.alloc(ctx, D);
    outs[w]->flags.alloc(ctx, 1);
    a.dev[w] = outs[w]->dev.p;
    a.pdm[w] = outs[w]->per_dev_mem.p;
    a.flags[w] = outs[w]->flags.p;
  }
  a.decisions = want_decisions && adjust_out;
  if (a.decisions) {
    adjust_out->dec_prev.alloc(ctx, n > 0 ? n : 1);
    adjust_out->dec_chosen.alloc(ctx, n > 0 ? n : 1);
    adjust_out->dec_back.alloc(ctx, n > 0 ? n : 1);
    adjust_out->dec_est.alloc(ctx, (size_t)(n > 0 ? n : 1) * D);
    adjust_out->dec_reloc.alloc(ctx, n > 0 ? n : 1);
    adjust_out->dec_be.alloc(ctx, n > 0 ? n : 1);
    a.dec_prev = adjust_out->dec_prev.p;
    a.dec_chosen = adjust_out->dec_chosen.p;
    a.dec_back = adjust_out->dec_back.p;
    a.dec_est = adjust_out->dec_est.p;
    a.dec_reloc = adjust_out->dec_reloc.p;
    a.dec_be = adjust_out->dec_be.p;
  }
  // block meta on chip when it fits: (5 x 8 + 2 x 4) bytes per block slot
  const size_t meta_bytes = static_cast<size_t>(48) * D * std::max(a.tl[0].maxb, a.tl[1].maxb);
  a.meta_smem = meta_bytes <= 186 * 1024 && getenv("DP_PLACE_GLOBAL_META") == nullptr;  // + ~38 KB static
  j->dyn = a.meta_smem ? meta_bytes : 0;
  j->dbg.alloc(ctx, 8);
  a.debug = getenv("DP_DEBUG_PLACE") ? j->dbg.p : nullptr;
  if (a.debug) j->dbg.zero();
  guard.j = nullptr;
  return j;
}

void place_launch(dp_ctx* ctx, PlaceJob* const* jobs, int count) {
  StageScope st(ctx, "placement", 0.0);
  for (int b0 = 0; b0 < count; b0 += kPlaceBatch) {
    const int k = std::min(kPlaceBatch, count - b0);
    PlaceBatch batch{};
    size_t dyn = 0;
    for (int q = 0; q < k; ++q) {
      batch.a[q] = jobs[b0 + q]->a;
      dyn = std::max(dyn, jobs[b0 + q]->dyn);
    }
    if (dyn) {
      static size_t attr = 0;
      if (dyn > attr) {
        DP_CUDA(cudaFuncSetAttribute(k_place, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn)));
        attr = dyn;
      }
    }
    DP_LAUNCH(ctx, k_place, 2 * k, 256, dyn, batch);
  }
  for (int q = 0; q < count; ++q) {
    PlaceJob* j = jobs[q];
    if (j->a.debug) {
      long long h[8];
      j->dbg.download(h, 8);
      sync(ctx);
      fprintf(stderr, "[place] order_place %.2f ms, adjusting %.2f ms (n=%d, D=%d, meta %s)\n", h[0] / 1.965e6,
              h[1] / 1.965e6, j->a.n, j->a.D, j->a.meta_smem ? "smem" : "global");
      fprintf(stderr, "[place] adjusting phases: loads %.2f, in-edges %.2f, find_slot %.2f, decide+commit %.2f ms\n",
              h[2] / 1.965e6, h[3] / 1.965e6, h[4] / 1.965e6, h[5] / 1.965e6);
    }
  }
}

void place_release(PlaceJob* j) { delete j; }

void place_dev(DevGraph& g, const int32_t* seq, const Devices& devs, PlaceOut* order_out, PlaceOut* adjust_out,
               bool want_decisions) {
  PlaceHandle h(place_prepare(g, seq, devs, order_out, adjust_out, want_decisions));
  place_launch(g.ctx, &h.j, 1);
}

void expand_dev(DevGraph& g, const int32_t* node_cluster, const int32_t* coarse_dev, int32_t D, int32_t* dev_node,
                int64_t* per_dev_mem) {
  dp_ctx* ctx = g.ctx;
  DP_CUDA(cudaMemsetAsync(per_dev_mem, 0, sizeof(int64_t) * D, ctx->stream));
  DP_LAUNCH(ctx, k_expand, grid_for(g.n, 256, 2 * ctx->num_sms), 256, sizeof(unsigned long long) * D, node_cluster,
            coarse_dev, g.mem.p, g.n, D, dev_node, per_dev_mem);
}

}  // namespace dpb
