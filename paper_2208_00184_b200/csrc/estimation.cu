// estimation.cu — the Standard Evaluation (estimation.cpp, /root/reference/proj/src) on the
// GPU, bit-exact in fp64:
//   fit_node_models   :67-88   per node, least squares over the batches (thread per node)
//   least_squares     :16-39   sums in batch order; __d*_rn so nothing contracts to FMA
//   estimate_graph    :90-119  node-parallel predict + llround; edge-parallel scaling
//   fit_comm_model    :121-140 one thread (the sums are order-sensitive)
//   deviation_report  :148-192 per-node deviations in parallel, the two means summed by
//                              one thread in node order (the reference's rounding)
// Inputs are joined by node id with device radix sorts (the reference's unordered_maps).
#include <algorithm>
#include <set>
#include <vector>

#include "abi_util.cuh"
#include "results.h"

namespace dpb {
namespace {

__device__ __forceinline__ uint64_t id_key(int64_t id) { return static_cast<uint64_t>(id) ^ (1ull << 63); }

struct Fit {
  double slope, intercept, residual;
};

// least_squares (estimation.cpp:16-39) over points (x[b], y[b]) in order.
__device__ Fit least_squares_dev(const double* x, const double* y, int32_t B, int64_t stride) {
  double sx = 0, sy = 0;
  for (int32_t b = 0; b < B; ++b) {
    sx = __dadd_rn(sx, x[b * stride]);
    sy = __dadd_rn(sy, y[b * stride]);
  }
  const double nB = static_cast<double>(static_cast<size_t>(B));
  const double mx = __ddiv_rn(sx, nB), my = __ddiv_rn(sy, nB);
  double sxx = 0, sxy = 0;
  for (int32_t b = 0; b < B; ++b) {
    const double dx = __dsub_rn(x[b * stride], mx), dy = __dsub_rn(y[b * stride], my);
    sxx = __dadd_rn(sxx, __dmul_rn(dx, dx));
    sxy = __dadd_rn(sxy, __dmul_rn(dx, dy));
  }
  Fit f;
  f.slope = sxx > 0 ? __ddiv_rn(sxy, sxx) : 0.0;
  f.intercept = __dsub_rn(my, __dmul_rn(f.slope, mx));
  double ss = 0;
  for (int32_t b = 0; b < B; ++b) {
    const double r = __dsub_rn(y[b * stride], __dadd_rn(__dmul_rn(f.slope, x[b * stride]), f.intercept));
    ss = __dadd_rn(ss, __dmul_rn(r, r));
  }
  f.residual = __dsqrt_rn(ss);
  return f;
}

__global__ void k_sample_keys(const int64_t* ids, int64_t m, uint64_t* keys, int32_t* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = id_key(ids[i]);
    vals[i] = static_cast<int32_t>(i);
  }
}

// Batch b's samples in id order vs batch 0's: flags [0] mismatch, [1] duplicate in b.
__global__ void k_universe_check(const uint64_t* keys, const int64_t* off, int32_t B, int64_t n, int* flags) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * B; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = static_cast<int32_t>(i / n);
    const int64_t k = i - (int64_t)b * n;
    const uint64_t v = keys[off[b] + k];
    if (k > 0 && keys[off[b] + k - 1] == v) atomicExch(&flags[1], 1);
    if (b > 0 && keys[off[0] + k] != v) atomicExch(&flags[0], 1);
  }
}

// Node-major matrices of x = batch size and y = sample values, node k = k-th smallest id.
__global__ void k_fit(const int32_t* perm, const int64_t* off, const int64_t* bsize, const int64_t* mem,
                      const int64_t* time, int32_t B, int64_t n, double* xs, double* ym, double* yt,
                      double* out /* [n][6] */) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double* x = xs + k * B;
    double* m = ym + k * B;
    double* t = yt + k * B;
    for (int32_t b = 0; b < B; ++b) {
      const int32_t s = perm[off[b] + k];
      x[b] = static_cast<double>(bsize[b]);
      m[b] = static_cast<double>(mem[s]);
      t[b] = static_cast<double>(time[s]);
    }
    const Fit fm = least_squares_dev(x, m, B, 1);
    const Fit ft = least_squares_dev(x, t, B, 1);
    double* o = out + k * 6;
    o[0] = fm.slope;
    o[1] = fm.intercept;
    o[2] = fm.residual;
    o[3] = ft.slope;
    o[4] = ft.intercept;
    o[5] = ft.residual;
  }
}

__device__ __forceinline__ int64_t find_sorted(const int64_t* ids, int64_t n, int64_t id) {
  int64_t lo = 0, hi = n - 1;
  while (lo <= hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ids[mid] < id) lo = mid + 1; else if (ids[mid] > id) hi = mid - 1; else return mid;
  }
  return -1;
}

// estimate_graph nodes (estimation.cpp:101-112): predict(target) = slope * x + intercept.
__global__ void k_est_nodes(const int64_t* node_id, int64_t n, const int64_t* mid, int64_t nm, const double* model,
                            double target, int64_t* mem_out, int64_t* w_out, unsigned long long* first_missing) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = find_sorted(mid, nm, node_id[v]);
    if (k < 0) {
      atomicMin(first_missing, static_cast<unsigned long long>(v));
      continue;
    }
    const double* f = model + k * 6;
    const double pm = __dadd_rn(__dmul_rn(f[0], target), f[1]);
    const double pt = __dadd_rn(__dmul_rn(f[3], target), f[4]);
    const int64_t a = static_cast<int64_t>(llround(pm)), b = static_cast<int64_t>(llround(pt));
    mem_out[v] = a > 0 ? a : 0;
    w_out[v] = b > 0 ? b : 0;
  }
}

// estimate_graph edges (:114-119): bytes * (override or target / reference).
__global__ void k_est_edges(const int64_t* src, const int64_t* dst, const int64_t* bytes, int64_t m,
                            const int64_t* ov_src, const int64_t* ov_dst, const double* ov_f, int64_t nov,
                            double ratio, int64_t* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    double f = ratio;
    int64_t lo = 0, hi = nov - 1;  // overrides sorted by (src, dst), unique
    while (lo <= hi) {
      const int64_t mid = (lo + hi) >> 1;
      const bool less = ov_src[mid] < src[e] || (ov_src[mid] == src[e] && ov_dst[mid] < dst[e]);
      const bool more = ov_src[mid] > src[e] || (ov_src[mid] == src[e] && ov_dst[mid] > dst[e]);
      if (less) lo = mid + 1; else if (more) hi = mid - 1; else { f = ov_f[mid]; break; }
    }
    const int64_t b = static_cast<int64_t>(llround(__dmul_rn(static_cast<double>(bytes[e]), f)));
    out[e] = b > 0 ? b : 0;
  }
}

// fit_comm_model (:121-140): one thread, sums in sample order.
__global__ void k_comm_fit(const int64_t* bytes, const double* us, int64_t n, double* out) {
  if (blockIdx.x || threadIdx.x) return;
  double sx = 0, sy = 0;
  for (int64_t i = 0; i < n; ++i) {
    sx = __dadd_rn(sx, static_cast<double>(bytes[i]));
    sy = __dadd_rn(sy, us[i]);
  }
  const double nn = static_cast<double>(static_cast<size_t>(n));
  const double mx = __ddiv_rn(sx, nn), my = __ddiv_rn(sy, nn);
  double sxx = 0, sxy = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double dx = __dsub_rn(static_cast<double>(bytes[i]), mx), dy = __dsub_rn(us[i], my);
    sxx = __dadd_rn(sxx, __dmul_rn(dx, dx));
    sxy = __dadd_rn(sxy, __dmul_rn(dx, dy));
  }
  const double slope = sxx > 0 ? __ddiv_rn(sxy, sxx) : 0.0;
  const double intercept = __dsub_rn(my, __dmul_rn(slope, mx));
  out[0] = slope > 0.0 ? slope : 0.0;  // std::max(0.0, .)
  out[1] = intercept > 0.0 ? intercept : 0.0;
}

// deviation_report per node (:166-181): relative deviations, zero flags.
__global__ void k_dev_nodes(const int64_t* est_id, const int64_t* est_mem, const int64_t* est_w, int64_t n,
                            const int64_t* mids, const int32_t* midx, int64_t nm, const int64_t* meas_mem,
                            const int64_t* meas_w, double* dm, double* dt, uint8_t* zm, uint8_t* zt,
                            unsigned long long* first_missing) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = find_sorted(mids, nm, est_id[v]);
    if (k < 0) {
      atomicMin(first_missing, static_cast<unsigned long long>(v));
      continue;
    }
    const int32_t s = midx[k];
    const int64_t mm = meas_mem[s], mw = meas_w[s];
    zm[v] = mm == 0;
    zt[v] = mw == 0;
    dm[v] = mm == 0 ? 0.0 : __ddiv_rn(fabs(static_cast<double>(est_mem[v] - mm)), static_cast<double>(mm));
    dt[v] = mw == 0 ? 0.0 : __ddiv_rn(fabs(static_cast<double>(est_w[v] - mw)), static_cast<double>(mw));
  }
}

// The two means: one thread, node order (:174-190).
__global__ void k_dev_means(const double* dm, const double* dt, const uint8_t* zm, const uint8_t* zt, int64_t n,
                            double* out) {
  if (blockIdx.x || threadIdx.x) return;
  double ms = 0, ts = 0;
  int64_t mc = 0, tc = 0;
  for (int64_t v = 0; v < n; ++v) {
    if (!zm[v]) {
      ms = __dadd_rn(ms, dm[v]);
      ++mc;
    }
    if (!zt[v]) {
      ts = __dadd_rn(ts, dt[v]);
      ++tc;
    }
  }
  out[0] = mc ? __ddiv_rn(ms, static_cast<double>(mc)) : 0.0;
  out[1] = tc ? __ddiv_rn(ts, static_cast<double>(tc)) : 0.0;
}

struct SortedIds {
  DevBuf<uint64_t> keys;   // ascending, sign-flipped ids
  DevBuf<int32_t> idx;     // original index (stable: later occurrences after earlier)
};

void sort_ids(dp_ctx* ctx, const int64_t* ids_dev, int64_t m, SortedIds& out) {
  DevBuf<uint64_t> k(ctx, m > 0 ? m : 1);
  DevBuf<int32_t> v(ctx, m > 0 ? m : 1);
  out.keys.alloc(ctx, m > 0 ? m : 1);
  out.idx.alloc(ctx, m > 0 ? m : 1);
  DP_LAUNCH(ctx, k_sample_keys, grid_for(m, 256), 256, 0, ids_dev, m, k.p, v.p);
  sort_pairs_u64(ctx, k.p, out.keys.p, v.p, out.idx.p, m, 0, 64);
}

}  // namespace
}  // namespace dpb

using namespace dpb;

extern "C" {

int dp_fit_node_models(dp_ctx_t* ctx, const dp_profiles_t* p, dp_node_models_t** out) {
  DP_API_BEGIN(ctx)
  if (!p || !out || p->n_batches < 0) fail(DP_E_ARGUMENT, "null profiles / output");
  const int32_t B = p->n_batches;
  // check_profiles (estimation.cpp:42-64)
  std::set<int64_t> sizes(p->batch_size, p->batch_size + B);
  if (sizes.size() < 2)
    fail(DP_E_INSUFFICIENT_SAMPLES, "need at least 2 distinct batch sizes, got %zu", sizes.size());
  const int64_t n = p->node_off[1] - p->node_off[0];
  for (int32_t b = 0; b < B; ++b)
    if (p->node_off[b + 1] - p->node_off[b] != n)
      fail(DP_E_NODE_UNIVERSE_MISMATCH, "batch %lld profiles a different node set", (long long)p->batch_size[b]);
  const int64_t m = p->node_off[B] - p->node_off[0];
  DevBuf<int64_t> ids(ctx, m > 0 ? m : 1), mem(ctx, m > 0 ? m : 1), tim(ctx, m > 0 ? m : 1), off(ctx, B + 1),
      bsz(ctx, B);
  ids.upload(p->node_id + p->node_off[0], m);
  mem.upload(p->memory_bytes + p->node_off[0], m);
  tim.upload(p->compute_us + p->node_off[0], m);
  std::vector<int64_t> hoff(B + 1);
  for (int32_t b = 0; b <= B; ++b) hoff[b] = p->node_off[b] - p->node_off[0];
  off.upload(hoff.data(), B + 1);
  bsz.upload(p->batch_size, B);
  // sort every batch's samples by id: one key sort over (batch, id) is a per-batch sort
  DevBuf<uint64_t> k(ctx, m > 0 ? m : 1), ko(ctx, m > 0 ? m : 1);
  DevBuf<int32_t> v(ctx, m > 0 ? m : 1), perm(ctx, m > 0 ? m : 1);
  DP_LAUNCH(ctx, k_sample_keys, grid_for(m, 256), 256, 0, ids.p, m, k.p, v.p);
  for (int32_t b = 0; b < B; ++b)
    if (hoff[b + 1] > hoff[b])
      sort_pairs_u64(ctx, k.p + hoff[b], ko.p + hoff[b], v.p + hoff[b], perm.p + hoff[b], hoff[b + 1] - hoff[b], 0,
                     64);
  DevBuf<int> flags(ctx, 2);
  flags.zero();
  DP_LAUNCH(ctx, k_universe_check, grid_for(n * B, 256), 256, 0, ko.p, off.p, B, n, flags.p);
  int hf[2];
  flags.download(hf, 2);
  sync(ctx);
  if (hf[0] || hf[1]) {
    // error path: name the first batch (in order) whose set differs and the smallest
    // universe id it misses (the reference names the first in hash order)
    std::vector<uint64_t> keys = to_host(ctx, ko.p, m);
    for (int32_t b = 0; b < B; ++b) {
      for (int64_t i = 1; i < n; ++i)
        if (keys[hoff[b] + i] == keys[hoff[b] + i - 1])
          fail(DP_E_INVALID_VALUE, "batch %lld lists node %lld twice", (long long)p->batch_size[b],
               (long long)(keys[hoff[b] + i] ^ (1ull << 63)));
    }
    for (int32_t b = 1; b < B; ++b) {
      int64_t j = 0;
      for (int64_t i = 0; i < n; ++i) {
        const uint64_t u = keys[i];
        while (j < n && keys[hoff[b] + j] < u) ++j;
        if (j >= n || keys[hoff[b] + j] != u)
          fail(DP_E_NODE_UNIVERSE_MISMATCH, "node %lld missing from batch %lld", (long long)(u ^ (1ull << 63)),
               (long long)p->batch_size[b]);
      }
    }
  }
  DevBuf<double> xs(ctx, (size_t)(n > 0 ? n : 1) * B), ym(ctx, (size_t)(n > 0 ? n : 1) * B),
      yt(ctx, (size_t)(n > 0 ? n : 1) * B), fit(ctx, (size_t)(n > 0 ? n : 1) * 6);
  DP_LAUNCH(ctx, k_fit, grid_for(n, 128), 128, 0, perm.p, off.p, bsz.p, mem.p, tim.p, B, n, xs.p, ym.p, yt.p, fit.p);
  auto* r = halloc<dp_node_models_t>(1);
  r->n = n;
  r->node_id = halloc<int64_t>(n);
  r->fit = halloc<double>(n * 6);
  std::vector<uint64_t> k0 = to_host(ctx, ko.p, n);
  for (int64_t i = 0; i < n; ++i) r->node_id[i] = static_cast<int64_t>(k0[i] ^ (1ull << 63));
  fit.download(r->fit, n * 6);
  sync(ctx);
  *out = r;
  DP_API_END
}

void dp_node_models_free(dp_node_models_t* m) {
  if (!m) return;
  std::free(m->node_id);
  std::free(m->fit);
  std::free(m);
}

int dp_estimate_graph(dp_ctx_t* ctx, const dp_graph_t* base, const dp_node_models_t* models, int64_t target_batch,
                      int64_t reference_batch, int64_t n_override, const int64_t* ov_src, const int64_t* ov_dst,
                      const double* ov_factor, dp_graph_out_t** out) {
  DP_API_BEGIN(ctx)
  if (!base || !models || !out) fail(DP_E_ARGUMENT, "null argument");
  if (target_batch <= 0) fail(DP_E_INVALID_VALUE, "target batch must be > 0");
  if (reference_batch <= 0) fail(DP_E_INVALID_VALUE, "reference batch must be > 0");
  const int64_t n = base->n_nodes, m = base->n_edges, nm = models->n;
  DevBuf<int64_t> id(ctx, n > 0 ? n : 1), mid(ctx, nm > 0 ? nm : 1), mo(ctx, n > 0 ? n : 1), wo(ctx, n > 0 ? n : 1);
  DevBuf<double> fit(ctx, (size_t)(nm > 0 ? nm : 1) * 6);
  id.upload(base->node_id, n);
  mid.upload(models->node_id, nm);  // ascending (dp_fit_node_models output)
  fit.upload(models->fit, nm * 6);
  DevBuf<unsigned long long> miss(ctx, 1);
  unsigned long long none = ~0ull;
  miss.upload(&none, 1);
  DP_LAUNCH(ctx, k_est_nodes, grid_for(n, 256), 256, 0, id.p, n, mid.p, nm, fit.p, static_cast<double>(target_batch),
            mo.p, wo.p, miss.p);
  // overrides: sorted by (src, dst), the last duplicate wins
  std::vector<int64_t> os, od;
  std::vector<double> of;
  {
    std::vector<int64_t> order(static_cast<size_t>(n_override));
    for (int64_t i = 0; i < n_override; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) {
      return ov_src[a] < ov_src[b] || (ov_src[a] == ov_src[b] && ov_dst[a] < ov_dst[b]);
    });
    for (size_t i = 0; i < order.size(); ++i) {
      const int64_t a = order[i];
      if (!os.empty() && os.back() == ov_src[a] && od.back() == ov_dst[a]) {
        of.back() = ov_factor[a];
        continue;
      }
      os.push_back(ov_src[a]);
      od.push_back(ov_dst[a]);
      of.push_back(ov_factor[a]);
    }
  }
  const int64_t nov = static_cast<int64_t>(os.size());
  DevBuf<int64_t> es(ctx, m > 0 ? m : 1), ed(ctx, m > 0 ? m : 1), eb(ctx, m > 0 ? m : 1), eo(ctx, m > 0 ? m : 1),
      vs(ctx, nov > 0 ? nov : 1), vd(ctx, nov > 0 ? nov : 1);
  DevBuf<double> vf(ctx, nov > 0 ? nov : 1);
  es.upload(base->edge_src, m);
  ed.upload(base->edge_dst, m);
  eb.upload(base->edge_bytes, m);
  vs.upload(os.data(), nov);
  vd.upload(od.data(), nov);
  vf.upload(of.data(), nov);
  const double ratio = static_cast<double>(target_batch) / static_cast<double>(reference_batch);
  DP_LAUNCH(ctx, k_est_edges, grid_for(m, 256), 256, 0, es.p, ed.p, eb.p, m, vs.p, vd.p, vf.p, nov, ratio, eo.p);
  const unsigned long long first = scalar_to_host(ctx, miss.p);
  if (first != ~0ull)
    fail(DP_E_UNKNOWN_NODE, "no fitted model for node %lld", (long long)base->node_id[first]);
  dp_graph_out_t* g = new_graph_out(n, m);
  std::memcpy(g->node_id, base->node_id, sizeof(int64_t) * n);
  mo.download(g->memory_bytes, n);
  wo.download(g->compute_us, n);
  for (int64_t i = 0; i < n; ++i) g->group[i] = base->group ? base->group[i] : -1;
  std::memcpy(g->edge_src, base->edge_src, sizeof(int64_t) * m);
  std::memcpy(g->edge_dst, base->edge_dst, sizeof(int64_t) * m);
  eo.download(g->edge_bytes, m);
  sync(ctx);
  *out = g;
  DP_API_END
}

int dp_fit_comm_model(dp_ctx_t* ctx, int64_t n, const int64_t* bytes, const double* us, dp_comm_t* out) {
  DP_API_BEGIN(ctx)
  if (!out || (n > 0 && (!bytes || !us))) fail(DP_E_ARGUMENT, "null argument");
  if (n < 2) fail(DP_E_INSUFFICIENT_SAMPLES, "need at least 2 transfer samples");
  std::set<int64_t> distinct(bytes, bytes + n);
  if (distinct.size() < 2) fail(DP_E_INSUFFICIENT_SAMPLES, "transfer samples need 2 distinct byte counts");
  DevBuf<int64_t> b(ctx, n);
  DevBuf<double> u(ctx, n), r(ctx, 2);
  b.upload(bytes, n);
  u.upload(us, n);
  DP_LAUNCH(ctx, k_comm_fit, 1, 32, 0, b.p, u.p, n, r.p);
  double h[2];
  r.download(h, 2);
  sync(ctx);
  out->k_us_per_byte = h[0];
  out->b_us = h[1];
  DP_API_END
}

int dp_deviation_report(dp_ctx_t* ctx, const dp_graph_t* est, const dp_graph_t* meas, dp_deviation_t** out) {
  DP_API_BEGIN(ctx)
  if (!est || !meas || !out) fail(DP_E_ARGUMENT, "null argument");
  const int64_t n = est->n_nodes, mm = meas->n_nodes;
  DevBuf<int64_t> mid(ctx, mm > 0 ? mm : 1), mmem(ctx, mm > 0 ? mm : 1), mw(ctx, mm > 0 ? mm : 1);
  mid.upload(meas->node_id, mm);
  mmem.upload(meas->memory_bytes, mm);
  mw.upload(meas->compute_us, mm);
  SortedIds s;
  sort_ids(ctx, mid.p, mm, s);
  // actual[id] = &node keeps the last occurrence of an id; count the distinct ids
  std::vector<uint64_t> keys = to_host(ctx, s.keys.p, mm);
  std::vector<int32_t> idx = to_host(ctx, s.idx.p, mm);
  std::vector<int64_t> uid;
  std::vector<int32_t> uix;
  for (int64_t i = 0; i < mm; ++i) {
    if (i + 1 < mm && keys[i + 1] == keys[i]) continue;  // stable sort: the last index comes last
    uid.push_back(static_cast<int64_t>(keys[i] ^ (1ull << 63)));
    uix.push_back(idx[i]);
  }
  if (static_cast<int64_t>(uid.size()) != n)
    fail(DP_E_NODE_UNIVERSE_MISMATCH, "estimated and measured graphs have different node counts");
  const int64_t nu = static_cast<int64_t>(uid.size());
  DevBuf<int64_t> ud(ctx, nu > 0 ? nu : 1), eid(ctx, n > 0 ? n : 1), emem(ctx, n > 0 ? n : 1), ew(ctx, n > 0 ? n : 1);
  DevBuf<int32_t> ux(ctx, nu > 0 ? nu : 1);
  ud.upload(uid.data(), nu);
  ux.upload(uix.data(), nu);
  eid.upload(est->node_id, n);
  emem.upload(est->memory_bytes, n);
  ew.upload(est->compute_us, n);
  DevBuf<double> dm(ctx, n > 0 ? n : 1), dt(ctx, n > 0 ? n : 1), means(ctx, 2);
  DevBuf<uint8_t> zm(ctx, n > 0 ? n : 1), zt(ctx, n > 0 ? n : 1);
  DevBuf<unsigned long long> miss(ctx, 1);
  unsigned long long none = ~0ull;
  miss.upload(&none, 1);
  DP_LAUNCH(ctx, k_dev_nodes, grid_for(n, 256), 256, 0, eid.p, emem.p, ew.p, n, ud.p, ux.p, nu, mmem.p, mw.p, dm.p,
            dt.p, zm.p, zt.p, miss.p);
  const unsigned long long first = scalar_to_host(ctx, miss.p);
  if (first != ~0ull)
    fail(DP_E_NODE_UNIVERSE_MISMATCH, "node %lld missing from measured graph", (long long)est->node_id[first]);
  DP_LAUNCH(ctx, k_dev_means, 1, 32, 0, dm.p, dt.p, zm.p, zt.p, n, means.p);
  std::vector<double> hm = to_host(ctx, dm.p, n), ht = to_host(ctx, dt.p, n), mean = to_host(ctx, means.p, 2);
  std::vector<uint8_t> hzm = to_host(ctx, zm.p, n), hzt = to_host(ctx, zt.p, n);
  // std::map outputs (ascending id; a repeated estimated id keeps its last value)
  std::vector<int64_t> order(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return est->node_id[a] < est->node_id[b]; });
  auto* r = halloc<dp_deviation_t>(1);
  r->memory_id = halloc<int64_t>(n);
  r->memory_dev = halloc<double>(n);
  r->time_id = halloc<int64_t>(n);
  r->time_dev = halloc<double>(n);
  r->zero_memory = halloc<int64_t>(n);
  r->zero_time = halloc<int64_t>(n);
  for (int32_t which = 0; which < 2; ++which) {
    const std::vector<double>& d = which ? ht : hm;
    const std::vector<uint8_t>& z = which ? hzt : hzm;
    int64_t* ids = which ? r->time_id : r->memory_id;
    double* vals = which ? r->time_dev : r->memory_dev;
    int64_t cnt = 0;
    for (size_t q = 0; q < order.size(); ++q) {
      const int64_t v = order[q];
      if (z[v]) continue;
      if (cnt > 0 && ids[cnt - 1] == est->node_id[v]) {
        vals[cnt - 1] = d[v];  // later write to the same key
        continue;
      }
      ids[cnt] = est->node_id[v];
      vals[cnt] = d[v];
      ++cnt;
    }
    (which ? r->n_time : r->n_memory) = cnt;
    int64_t* zl = which ? r->zero_time : r->zero_memory;
    int64_t zc = 0;
    for (size_t q = 0; q < order.size(); ++q)
      if (z[order[q]]) zl[zc++] = est->node_id[order[q]];
    (which ? r->n_zero_time : r->n_zero_memory) = zc;
  }
  r->mean_memory = mean[0];
  r->mean_time = mean[1];
  *out = r;
  DP_API_END
}

void dp_deviation_free(dp_deviation_t* d) {
  if (!d) return;
  std::free(d->memory_id);
  std::free(d->memory_dev);
  std::free(d->time_id);
  std::free(d->time_dev);
  std::free(d->zero_memory);
  std::free(d->zero_time);
  std::free(d);
}

}  // extern "C"
