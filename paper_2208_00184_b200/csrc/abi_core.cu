// abi_core.cu — C-ABI entry points of the graph core and orderings
// (include/dagplace_b200.h).  Each call: host SoA -> HBM, GPU kernels, results -> host.
#include <algorithm>
#include <new>

#include "abi_util.cuh"
#include "graph.cuh"
#include "peel.cuh"
#include "results.h"

namespace dpb {
namespace {

__global__ void k_ccr_sums(const int64_t* w, int32_t n, const int64_t* bytes, int32_t m, double ck, double cb,
                           unsigned long long* out /* [0] compute, [1] comm, [2] negative bytes flag */) {
  unsigned long long sc = 0, sm = 0;
  int neg = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    sc += static_cast<unsigned long long>(w[i]);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = bytes[e];
    if (b < 0) neg = 1;
    else sm += static_cast<unsigned long long>(comm_cost_dev(b, ck, cb));
  }
  for (int o = 16; o; o >>= 1) {
    sc += __shfl_down_sync(0xffffffffu, sc, o);
    sm += __shfl_down_sync(0xffffffffu, sm, o);
    neg |= __shfl_down_sync(0xffffffffu, neg, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], sc);
    atomicAdd(&out[1], sm);
    if (neg) atomicOr(&out[2], 1ull);
  }
}

__global__ void k_gather_ids(const int64_t* id, const int32_t* idx, int32_t n, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = id ? id[idx[i]] : idx[i];
}

__global__ void k_cpath(const int64_t* t, const int64_t* b, int32_t n, int64_t* c) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c[i] = t[i] + b[i];
}

// is_valid_topo_order on ids (ordering.cpp:116-132): seq ids sorted with positions.
__global__ void k_seq_keys(const int64_t* seq, int64_t len, uint64_t* keys, int32_t* vals) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = static_cast<uint64_t>(seq[i]) ^ (1ull << 63);
    vals[i] = static_cast<int32_t>(i);
  }
}
__device__ int32_t seq_pos(const uint64_t* keys, const int32_t* vals, int64_t len, int64_t id) {
  uint64_t k = static_cast<uint64_t>(id) ^ (1ull << 63);
  int64_t lo = 0, hi = len;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  return (lo < len && keys[lo] == k) ? vals[lo] : -1;
}
__global__ void k_order_check(const uint64_t* keys, const int32_t* vals, int64_t len, const int64_t* node_id,
                              int32_t n, const int64_t* src, const int64_t* dst, int32_t m, int* ok) {
  int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < len; i += nth)
    if (i > 0 && keys[i] == keys[i - 1]) atomicExch(ok, 0);
  for (int64_t i = tid; i < n; i += nth)
    if (seq_pos(keys, vals, len, node_id[i]) < 0) atomicExch(ok, 0);
  for (int64_t e = tid; e < m; e += nth) {
    int32_t u = seq_pos(keys, vals, len, src[e]), v = seq_pos(keys, vals, len, dst[e]);
    if (u < 0 || v < 0 || u >= v) atomicExch(ok, 0);
  }
}

}  // namespace

void require_valid_dev(DevGraph& g, const dp_graph_t* h, bool cycle_check) {
  Validation v = graph_validate(g, h, false, cycle_check);
  if (v.code) fail(v.code, "%s", v.message.c_str());
}

void prepare_graph(DevGraph& g, dp_ctx* ctx, const dp_graph_t* h) {
  graph_upload(g, ctx, h);
  graph_resolve(g);
  graph_adjacency(g);
}

// compute_levels (graph.cpp:217-269) on a validated device graph; cycle -> error.
void levels_dev(DevGraph& g, dp_comm_t comm, DevBuf<int64_t>& t, DevBuf<int64_t>& b, DevBuf<int64_t>& c,
                bool chainlike) {
  dp_ctx* ctx = g.ctx;
  graph_costs(g, comm);
  t.alloc(ctx, g.n > 0 ? g.n : 1);
  b.alloc(ctx, g.n > 0 ? g.n : 1);
  c.alloc(ctx, g.n > 0 ? g.n : 1);
  {
    StageScope st(ctx, "levels", 40.0 * g.m_ok + 48.0 * g.n);
    if (!graph_levels_indexorder(g, t.p, b.p, chainlike)) graph_kahn(g, t.p, b.p, nullptr);
  }
  if (g.processed != g.n) {
    std::vector<int64_t> wit = graph_cycle_witness(g);
    fail(DP_E_CYCLE_DETECTED, "cycle: [%s]", join_ids(wit).c_str());
  }
  DP_LAUNCH(ctx, k_cpath, grid_for(g.n, 256), 256, 0, t.p, b.p, g.n, c.p);
}

// levels_dev(g, comm, t, b, c, chainlike = false) of several graphs: one index-order check
// and shared sweep / dataflow launches (graphs_levels_indexorder), Kahn for the others.
void levels_dev_batch(DevGraph* const* gs, int count, dp_comm_t comm, DevBuf<int64_t>* const* t,
                      DevBuf<int64_t>* const* b, DevBuf<int64_t>* const* c) {
  if (count == 0) return;
  dp_ctx* ctx = gs[0]->ctx;
  double bytes = 0.0;
  std::vector<int64_t*> tp(count), bp(count);
  for (int i = 0; i < count; ++i) {
    DevGraph& g = *gs[i];
    graph_costs(g, comm);
    t[i]->alloc(ctx, g.n > 0 ? g.n : 1);
    b[i]->alloc(ctx, g.n > 0 ? g.n : 1);
    c[i]->alloc(ctx, g.n > 0 ? g.n : 1);
    tp[i] = t[i]->p;
    bp[i] = b[i]->p;
    bytes += 40.0 * g.m_ok + 48.0 * g.n;
  }
  {
    StageScope st(ctx, "levels", bytes);
    std::vector<char> ok = graphs_levels_indexorder(gs, count, tp.data(), bp.data());
    for (int i = 0; i < count; ++i)
      if (!ok[i]) graph_kahn(*gs[i], tp[i], bp[i], nullptr);
  }
  for (int i = 0; i < count; ++i) {
    DevGraph& g = *gs[i];
    if (g.processed != g.n) {
      std::vector<int64_t> wit = graph_cycle_witness(g);
      fail(DP_E_CYCLE_DETECTED, "cycle: [%s]", join_ids(wit).c_str());
    }
    DP_LAUNCH(ctx, k_cpath, grid_for(g.n, 256), 256, 0, t[i]->p, b[i]->p, g.n, c[i]->p);
  }
}

// levels_dev(g, comm, t, b, c, chainlike = true) of several graphs: one index-order check
// (one host sync) and one sweep launch per direction for all of them.
void levels_dev_chainlike_batch(DevGraph* const* gs, int count, dp_comm_t comm, DevBuf<int64_t>* const* t,
                                DevBuf<int64_t>* const* b, DevBuf<int64_t>* const* c) {
  if (count == 0) return;
  dp_ctx* ctx = gs[0]->ctx;
  double bytes = 0.0;
  for (int i = 0; i < count; ++i) {
    DevGraph& g = *gs[i];
    graph_costs(g, comm);
    t[i]->alloc(ctx, g.n > 0 ? g.n : 1);
    b[i]->alloc(ctx, g.n > 0 ? g.n : 1);
    c[i]->alloc(ctx, g.n > 0 ? g.n : 1);
    bytes += 40.0 * g.m_ok + 48.0 * g.n;
  }
  {
    StageScope st(ctx, "levels", bytes);
    std::vector<char> ok(count, 0);
    bool flow = getenv("DP_LEVELS_FLOW") != nullptr;
    for (int i = 0; i < count; ++i) flow = flow || coarse_flow_wanted(gs[i]->n);
    std::vector<DevGraph*> sg;
    std::vector<int64_t*> st_, sb;
    if (flow) {  // the small ones still take the sweep (graphs_levels_indexorder decides)
      std::vector<int64_t*> tp(count), bp(count);
      for (int i = 0; i < count; ++i) {
        tp[i] = t[i]->p;
        bp[i] = b[i]->p;
      }
      ok = graphs_levels_indexorder(gs, count, tp.data(), bp.data());
    } else if (!getenv("DP_LEVELS_KAHN")) {
      ok = graphs_index_topological(gs, count);
    }
    for (int i = 0; i < count && !flow; ++i) {
      if (!ok[i]) continue;
      sg.push_back(gs[i]);
      st_.push_back(t[i]->p);
      sb.push_back(b[i]->p);
      gs[i]->processed = gs[i]->n;
    }
    if (!sg.empty()) levels_sweep_launch(sg.data(), st_.data(), sb.data(), static_cast<int>(sg.size()));
    for (int i = 0; i < count; ++i)
      if (!ok[i]) graph_kahn(*gs[i], t[i]->p, b[i]->p, nullptr);
  }
  for (int i = 0; i < count; ++i) {
    DevGraph& g = *gs[i];
    if (g.processed != g.n) {
      std::vector<int64_t> wit = graph_cycle_witness(g);
      fail(DP_E_CYCLE_DETECTED, "cycle: [%s]", join_ids(wit).c_str());
    }
    DP_LAUNCH(ctx, k_cpath, grid_for(g.n, 256), 256, 0, t[i]->p, b[i]->p, g.n, c[i]->p);
  }
}

// is_valid_topo_order (ordering.cpp:116-132) for a host sequence of ids.
bool order_valid_dev(DevGraph& g, const int64_t* seq, int64_t len) {
  dp_ctx* ctx = g.ctx;
  if (len != g.n) return false;
  DevBuf<int64_t> s(ctx, len > 0 ? len : 1);
  s.upload(seq, len);
  DevBuf<uint64_t> k(ctx, len > 0 ? len : 1), ko(ctx, len > 0 ? len : 1);
  DevBuf<int32_t> v(ctx, len > 0 ? len : 1), vo(ctx, len > 0 ? len : 1);
  DP_LAUNCH(ctx, k_seq_keys, grid_for(len, 256), 256, 0, s.p, len, k.p, v.p);
  sort_pairs_u64(ctx, k.p, ko.p, v.p, vo.p, len, 0, 64);
  DevBuf<int> ok(ctx, 1);
  int one = 1;
  ok.upload(&one, 1);
  DP_LAUNCH(ctx, k_order_check, grid_for(std::max<int64_t>(len, g.m), 256), 256, 0, ko.p, vo.p, len, g.id.p,
            g.n, g.src_id.p, g.dst_id.p, g.m, ok.p);
  return scalar_to_host(ctx, ok.p) == 1;
}

void seq_ids(DevGraph& g, const int32_t* seq, int32_t n, int64_t* out_dev) {
  DP_LAUNCH(g.ctx, k_gather_ids, grid_for(n, 256), 256, 0, g.dense_ids ? nullptr : g.id.p, seq, n, out_dev);
}

}  // namespace dpb

using namespace dpb;

extern "C" {

int dp_comm_time(int64_t bytes, dp_comm_t comm, int64_t* out) {
  // graph.cpp:200-204; host-side scalar evaluation of the same formula the kernels use.
  if (bytes < 0) {
    set_last_error(DP_E_INVALID_VALUE, "negative byte count");
    return DP_E_INVALID_VALUE;
  }
  volatile double t = comm.k_us_per_byte * static_cast<double>(bytes);
  volatile double u = t + comm.b_us;
  *out = static_cast<int64_t>(llround(u));
  return DP_OK;
}

int dp_ccr(dp_ctx_t* ctx, const dp_graph_t* h, dp_comm_t comm, double* out) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  graph_upload(g, ctx, h);
  DevBuf<unsigned long long> sums(ctx, 3);
  sums.zero();
  DP_LAUNCH(ctx, k_ccr_sums, grid_for(std::max(g.n, g.m), 256, 4 * ctx->num_sms), 256, 0, g.w.p, g.n,
            g.bytes.p, g.m, comm.k_us_per_byte, comm.b_us, sums.p);
  unsigned long long s[3];
  sums.download(s, 3);
  sync(ctx);
  int64_t total_compute = static_cast<int64_t>(s[0]), total_comm = static_cast<int64_t>(s[1]);
  if (total_compute <= 0) fail(DP_E_ZERO_COMPUTE_TIME, "total compute time is zero");
  if (s[2]) fail(DP_E_INVALID_VALUE, "negative byte count");
  *out = static_cast<double>(total_comm) / static_cast<double>(total_compute);
  DP_API_END
}

int dp_validate(dp_ctx_t* ctx, const dp_graph_t* h, dp_violation_list_t** out) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  Validation v = graph_validate(g, h, true);
  auto* r = halloc<dp_violation_list_t>(1);
  int64_t k = static_cast<int64_t>(v.kinds.size());
  r->count = k;
  r->kind = halloc<int32_t>(k);
  r->node_off = halloc<int64_t>(k + 1);
  r->msg_off = halloc<int64_t>(k + 1);
  int64_t nn = 0, nm = 0;
  for (int64_t i = 0; i < k; ++i) {
    nn += static_cast<int64_t>(v.witnesses[i].size());
    nm += static_cast<int64_t>(v.messages[i].size());
  }
  r->nodes = halloc<int64_t>(nn);
  r->msg = halloc<char>(nm + 1);
  nn = nm = 0;
  for (int64_t i = 0; i < k; ++i) {
    r->kind[i] = v.kinds[i];
    r->node_off[i] = nn;
    r->msg_off[i] = nm;
    for (int64_t id : v.witnesses[i]) r->nodes[nn++] = id;
    std::memcpy(r->msg + nm, v.messages[i].data(), v.messages[i].size());
    nm += static_cast<int64_t>(v.messages[i].size());
  }
  r->node_off[k] = nn;
  r->msg_off[k] = nm;
  *out = r;
  DP_API_END
}

void dp_violation_list_free(dp_violation_list_t* v) {
  if (!v) return;
  std::free(v->kind); std::free(v->node_off); std::free(v->nodes); std::free(v->msg_off);
  std::free(v->msg); std::free(v);
}

int dp_require_valid(dp_ctx_t* ctx, const dp_graph_t* h) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  DP_API_END
}

int dp_graph_index(dp_ctx_t* ctx, const dp_graph_t* h, int32_t* es, int32_t* ed, int32_t* os, int32_t* ol,
                   int32_t* is, int32_t* il) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  graph_upload(g, ctx, h);
  graph_resolve(g);
  graph_index_checks(g, h);
  std::vector<int32_t> hs = to_host(ctx, g.esrc.p, g.m), hd = to_host(ctx, g.edst.p, g.m);
  graph_adjacency(g);
  std::memcpy(es, hs.data(), sizeof(int32_t) * g.m);
  std::memcpy(ed, hd.data(), sizeof(int32_t) * g.m);
  g.out_off.download(os, (size_t)g.n + 1);
  g.in_off.download(is, (size_t)g.n + 1);
  g.out_eid.download(ol, g.m);
  g.in_eid.download(il, g.m);
  sync(ctx);
  DP_API_END
}

int dp_compute_levels(dp_ctx_t* ctx, const dp_graph_t* h, dp_comm_t comm, int64_t* tl, int64_t* bl, int64_t* cp) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, false);
  DevBuf<int64_t> t, b, c;
  levels_dev(g, comm, t, b, c);
  t.download(tl, g.n);
  b.download(bl, g.n);
  c.download(cp, g.n);
  sync(ctx);
  DP_API_END
}

int dp_topo_order(dp_ctx_t* ctx, const dp_graph_t* h, int32_t policy, const int64_t* cpath, int64_t* seq_out) {
  DP_API_BEGIN(ctx)
  if (policy < DP_TOPO_M || policy > DP_TOPO_CPD) fail(DP_E_INVALID_VALUE, "unknown topo policy");
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  int32_t n = g.n;
  DevBuf<int64_t> cp;
  if (policy == DP_TOPO_CPD) {
    if (!cpath && n) fail(DP_E_ARGUMENT, "cpd_topo needs cpath");
    cp.alloc(ctx, n > 0 ? n : 1);
    cp.upload(cpath, n);
  }
  DevBuf<int32_t> seq(ctx, n > 0 ? n : 1), pos(ctx, n > 0 ? n : 1);
  int32_t emitted = topo_order(g, policy, cp.p, seq.p, pos.p);
  if (emitted != n) fail(DP_E_CYCLE_DETECTED, "graph has a cycle; topological order impossible");
  DevBuf<int64_t> ids(ctx, n > 0 ? n : 1);
  seq_ids(g, seq.p, n, ids.p);
  ids.download(seq_out, n);
  sync(ctx);
  DP_API_END
}

int dp_is_valid_topo_order(dp_ctx_t* ctx, const dp_graph_t* h, const int64_t* seq, int64_t len, int32_t* out) {
  DP_API_BEGIN(ctx)
  *out = 0;
  if (len != h->n_nodes) return DP_OK;
  DevGraph g;
  graph_upload(g, ctx, h);
  *out = order_valid_dev(g, seq, len) ? 1 : 0;
  DP_API_END
}

}  // extern "C"
