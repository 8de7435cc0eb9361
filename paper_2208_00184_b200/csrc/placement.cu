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

#include "placement.cuh"

namespace dpb {

namespace {

constexpr int kMaxD = 256;
constexpr unsigned FULL = 0xffffffffu;

struct TLView {
  int64_t *S, *E, *PM, *GQ, *BG;
};

struct TLArrays {
  int64_t *S, *E, *PM, *GQ, *BG;
  int32_t cap, nb;
  __device__ TLView view(int d) const {
    return TLView{S + (int64_t)d * cap, E + (int64_t)d * cap, PM + (int64_t)d * cap, GQ + (int64_t)d * cap,
                  BG + (int64_t)d * nb};
  }
};

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

// DeviceTimeline::find_slot(earliest, dur) (placement.cpp:13-21); warp-collective.
__device__ int64_t tl_query(const TLView t, int32_t K, int64_t gmax, int64_t last, int64_t earliest, int64_t dur) {
  const int lane = threadIdx.x & 31;
  if (K == 0 || last <= earliest) return earliest;
  const int32_t k0 = warp_first_true(0, K - 1, [&](int32_t q) { return t.PM[q] > earliest; });
  const int64_t sk = t.S[k0];
  if (sk >= earliest && sk - earliest >= dur) return earliest;
  if (gmax < dur) return last;
  const int32_t k = k0 + 1;
  if (k >= K) return last;
  const int32_t blk = k >> 5;
  {
    const int32_t idx = (blk << 5) + lane;
    const unsigned b = __ballot_sync(FULL, idx >= k && idx < K && t.GQ[idx] >= dur);
    if (b) return t.PM[(blk << 5) + __ffs(b) - 2];
  }
  const int32_t nblk = (K + 31) >> 5;
  for (int32_t b0 = blk + 1; b0 < nblk; b0 += 32) {
    const int32_t bb = b0 + lane;
    const unsigned bal = __ballot_sync(FULL, bb < nblk && t.BG[bb] >= dur);
    if (bal) {
      const int32_t fb = b0 + __ffs(bal) - 1;
      const int32_t idx = (fb << 5) + lane;
      const unsigned b2 = __ballot_sync(FULL, idx < K && t.GQ[idx] >= dur);
      return t.PM[(fb << 5) + __ffs(b2) - 2];
    }
  }
  return last;
}

// DeviceTimeline::reserve(start, dur) (placement.cpp:23-32): upper_bound insert.
__device__ void tl_insert(const TLView t, int32_t* Kp, int64_t* gmaxp, int64_t* lastp, int64_t s, int64_t dur) {
  const int lane = threadIdx.x & 31;
  const int64_t e = s + dur;
  const int32_t K = *Kp;
  const int64_t last = *lastp;
  int32_t q;
  if (K == 0 || t.S[K - 1] <= s) {
    q = K;
  } else {
    q = warp_first_true(0, K - 1, [&](int32_t x) { return t.S[x] > s; });
  }
  if (q == K) {
    if (lane == 0) {
      t.S[q] = s;
      t.E[q] = e;
      const int64_t pm = K ? (last > e ? last : e) : e;
      t.PM[q] = pm;
      const int64_t gq = (K == 0) ? -1 : (e > last ? s - last : -1);
      t.GQ[q] = gq;
      const int32_t b = q >> 5;
      t.BG[b] = (q & 31) == 0 ? gq : (t.BG[b] > gq ? t.BG[b] : gq);
      if (gq > *gmaxp) *gmaxp = gq;
      *lastp = pm;
      *Kp = K + 1;
    }
    __syncwarp();
    return;
  }
  for (int32_t top = K; top > q; top -= 32) {
    const int32_t base = max(q, top - 32);
    const int32_t idx = base + lane;
    const bool act = idx < top;
    int64_t vs = 0, ve = 0, vp = 0, vg = 0;
    if (act) {
      vs = t.S[idx];
      ve = t.E[idx];
      vp = t.PM[idx];
      vg = t.GQ[idx];
    }
    __syncwarp();
    if (act) {
      t.S[idx + 1] = vs;
      t.E[idx + 1] = ve;
      t.PM[idx + 1] = vp;
      t.GQ[idx + 1] = vg;
    }
    __syncwarp();
  }
  const int32_t Kn = K + 1;
  if (lane == 0) {
    t.S[q] = s;
    t.E[q] = e;
    const int64_t prev = q ? t.PM[q - 1] : INT64_MIN;
    t.PM[q] = prev > e ? prev : e;
  }
  __syncwarp();
  for (int32_t idx = q + 1 + lane; idx < Kn; idx += 32) {
    const int64_t pm = t.PM[idx];
    if (pm < e) t.PM[idx] = e;
  }
  __syncwarp();
  for (int32_t idx = max(q, 1) + lane; idx < Kn; idx += 32) {
    const int64_t pp = t.PM[idx - 1];
    const int64_t ev = t.E[idx];
    t.GQ[idx] = ev > pp ? t.S[idx] - pp : -1;
  }
  if (q == 0 && lane == 0) t.GQ[0] = -1;
  __syncwarp();
  const int32_t lastb = (Kn - 1) >> 5;
  for (int32_t b = (q >> 5) + lane; b <= lastb; b += 32) {
    int64_t mx = INT64_MIN;
    const int32_t hi = min((b << 5) + 31, Kn - 1);
    for (int32_t i = b << 5; i <= hi; ++i) mx = max(mx, t.GQ[i]);
    t.BG[b] = mx;
  }
  __syncwarp();
  int64_t mx = -1;
  for (int32_t b = lane; b <= lastb; b += 32) mx = max(mx, t.BG[b]);
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
  if (lane == 0) {
    *gmaxp = mx;
    *lastp = last > e ? last : e;
    *Kp = Kn;
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

__global__ void __launch_bounds__(256) k_place(PlaceArgs a) {
  __shared__ int32_t sK[kMaxD];
  __shared__ int64_t sg[kMaxD], sl[kMaxD], savail[kMaxD], spdm[kMaxD];
  __shared__ long long sA[kMaxD], sB[kMaxD];
  __shared__ int64_t sest[kMaxD], spre[kMaxD];
  __shared__ int32_t s_chosen, s_be;
  __shared__ int64_t s_start;
  const int which = blockIdx.x;  // 0 order_place, 1 adjusting_placement
  if (!a.run[which]) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int32_t D = a.D;
  const TLArrays tl = a.tl[which];
  for (int d = tid; d < D; d += blockDim.x) {
    sK[d] = 0;
    sg[d] = -1;
    sl[d] = 0;
    savail[d] = a.cap[d];
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
      const int64_t start = tl_query(t, sK[target], sg[target], sl[target], 0, w);
      tl_insert(t, &sK[target], &sg[target], &sl[target], start, w);
      if (lane == 0) {
        dev[v] = target;
        savail[target] -= mv;
        spdm[target] += mv;
      }
      __syncwarp();
    }
    for (int d = lane; d < D; d += 32) a.pdm[0][d] = spdm[d];
    if (lane == 0) a.flags[0][0] = oom ? 1 : 0;
    return;
  }
  // adjusting_placement (placement.cpp:172-216)
  int32_t prev = 0;
  bool oom = false;
  for (int32_t k = 0; k < a.n; ++k) {
    const int32_t v = a.seq[k];
    const int64_t w = a.w[v], mv = a.mem[v];
    for (int d = tid; d < D; d += blockDim.x) {
      sA[d] = LLONG_MIN;
      sB[d] = LLONG_MIN;
    }
    __syncthreads();
    const int32_t ib = a.in_off[v], ie = a.in_off[v + 1];
    for (int32_t q = ib + tid; q < ie; q += blockDim.x) {
      const int32_t p = a.in_src[q];
      const int64_t f = a.finish[p];
      const int32_t dd = dev[p];
      atomicMax(&sA[dd], static_cast<long long>(f));
      atomicMax(&sB[dd], static_cast<long long>(f + a.in_cost[q]));
    }
    __syncthreads();
    for (int32_t d = warp; d < D; d += nwarps) {
      long long mb = LLONG_MIN;
      for (int32_t x = lane; x < D; x += 32)
        if (x != d) mb = max(mb, sB[x]);
#pragma unroll
      for (int o = 16; o; o >>= 1) mb = max(mb, __shfl_xor_sync(FULL, mb, o));
      int64_t pre = 0;
      if (sA[d] > pre) pre = sA[d];
      if (mb > pre) pre = mb;
      int64_t est = kNever;
      if (savail[d] >= mv) est = tl_query(tl.view(d), sK[d], sg[d], sl[d], pre, w);
      if (lane == 0) {
        sest[d] = est;
        spre[d] = pre;
      }
    }
    __syncthreads();
    if (tid == 0) {
      const int64_t back = a.back[v];
      int32_t best = -1;
      for (int32_t d = 0; d < D; ++d)
        if (savail[d] >= mv && (best < 0 || sest[d] < sest[best])) best = d;
      int32_t chosen;
      int64_t start = 0;
      bool reloc = false, be = false;
      if (best >= 0 && (sest[prev] == kNever || sest[prev] - sest[best] > back)) {
        chosen = best;
        start = sest[best];
        reloc = chosen != prev;
      } else if (sest[prev] != kNever) {
        chosen = prev;
        start = sest[prev];
      } else {
        chosen = most_free(savail, D);
        be = true;
        oom = true;
      }
      if (a.decisions) {
        a.dec_prev[k] = prev;
        a.dec_back[k] = back;
        a.dec_chosen[k] = chosen;
        a.dec_reloc[k] = reloc;
        a.dec_be[k] = be;
      }
      s_chosen = chosen;
      s_start = start;
      s_be = be;
    }
    __syncthreads();
    if (a.decisions)
      for (int d = tid; d < D; d += blockDim.x) a.dec_est[(int64_t)k * D + d] = sest[d];
    const int32_t chosen = s_chosen;
    if (warp == (chosen % nwarps)) {
      const TLView t = tl.view(chosen);
      int64_t start = s_start;
      if (s_be) start = tl_query(t, sK[chosen], sg[chosen], sl[chosen], spre[chosen], w);
      tl_insert(t, &sK[chosen], &sg[chosen], &sl[chosen], start, w);
      if (lane == 0) {
        a.finish[v] = start + w;
        dev[v] = chosen;
        savail[chosen] -= mv;
        spdm[chosen] += mv;
      }
    }
    prev = chosen;
    __syncthreads();
  }
  for (int d = tid; d < D; d += blockDim.x) a.pdm[1][d] = spdm[d];
  if (tid == 0) a.flags[1][0] = oom ? 1 : 0;
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

void alloc_tl(dp_ctx* ctx, int32_t D, int32_t cap, DevBuf<int64_t>& store, TLArrays& t) {
  const int64_t nb = cap / 32 + 2;
  const int64_t per = (int64_t)D * cap;
  store.alloc(ctx, static_cast<size_t>(4 * per + (int64_t)D * nb));
  t.S = store.p;
  t.E = store.p + per;
  t.PM = store.p + 2 * per;
  t.GQ = store.p + 3 * per;
  t.BG = store.p + 4 * per;
  t.cap = cap;
  t.nb = static_cast<int32_t>(nb);
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

void place_dev(DevGraph& g, const int32_t* seq, const Devices& devs, PlaceOut* order_out, PlaceOut* adjust_out,
               bool want_decisions) {
  dp_ctx* ctx = g.ctx;
  const int32_t n = g.n, D = devs.D;
  if (D > kMaxD) fail(DP_E_UNSUPPORTED, "at most %d devices are supported", kMaxD);
  PlaceArgs a{};
  a.n = n;
  a.D = D;
  a.seq = seq;
  a.w = g.w.p;
  a.mem = g.mem.p;
  a.in_off = g.in_off.p;
  a.in_src = g.in_src.p;
  a.in_cost = g.in_cost.p;
  DevBuf<int64_t> back(ctx, n > 0 ? n : 1), cap(ctx, D), finish(ctx, n > 0 ? n : 1);
  cap.upload(devs.cap.data(), D);
  DP_LAUNCH(ctx, k_back_cost, grid_for(n, 256), 256, 0, g.out_off.p, g.has_cost ? g.out_cost.p : nullptr, n, back.p);
  a.back = back.p;
  a.cap = cap.p;
  a.finish = finish.p;
  DevBuf<int64_t> store[2];
  PlaceOut* outs[2] = {order_out, adjust_out};
  for (int w = 0; w < 2; ++w) {
    a.run[w] = outs[w] != nullptr;
    if (!outs[w]) continue;
    alloc_tl(ctx, D, n > 0 ? n : 1, store[w], a.tl[w]);
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
  StageScope st(ctx, "placement", 0.0);
  DP_LAUNCH(ctx, k_place, 2, 256, 0, a);
}

void expand_dev(DevGraph& g, const int32_t* node_cluster, const int32_t* coarse_dev, int32_t D, int32_t* dev_node,
                int64_t* per_dev_mem) {
  dp_ctx* ctx = g.ctx;
  DP_CUDA(cudaMemsetAsync(per_dev_mem, 0, sizeof(int64_t) * D, ctx->stream));
  DP_LAUNCH(ctx, k_expand, grid_for(g.n, 256, 2 * ctx->num_sms), 256, sizeof(unsigned long long) * D, node_cluster,
            coarse_dev, g.mem.p, g.n, D, dev_node, per_dev_mem);
}

}  // namespace dpb
