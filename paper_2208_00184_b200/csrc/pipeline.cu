#include <chrono>
#include <cstdlib>
// pipeline.cu — evaluate_pipeline (pipeline.cpp:27-111, /root/reference/proj/src) with
// every intermediate resident in HBM.  The generation window of pipeline.cpp:67-79
// (fuse -> coarse levels + cpd_topo -> order_place + adjusting_placement -> 2x expand)
// runs as one stream of kernels; only the results cross PCIe.
#include <algorithm>
#include <array>
#include <memory>

#include "abi_util.cuh"
#include "fusion.cuh"
#include "peel.cuh"
#include "placement.cuh"
#include "results.h"
#include "simulate.cuh"

namespace dpb {

dp_graph_out_t* graph_to_host_async(DevGraph& g, bool dense_ids_out, Finalizers& fin);
dp_placement_result_t* placement_to_host_async(dp_ctx* ctx, const Devices& devs, PlaceOut& p, int32_t n,
                                               std::shared_ptr<const std::vector<int64_t>> seq_ids, bool decisions,
                                               Finalizers& fin);
dp_sim_report_t* sim_report(DevGraph& g, const Devices& devs, const int32_t* dev_pos_dev, bool trace);

namespace {

__global__ void k_ccr(const int64_t* w, int32_t n, const int64_t* cost, int32_t m, unsigned long long* out) {
  unsigned long long sc = 0, sm = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    sc += static_cast<unsigned long long>(w[i]);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
    sm += static_cast<unsigned long long>(cost[e]);
  for (int o = 16; o; o >>= 1) {
    sc += __shfl_down_sync(0xffffffffu, sc, o);
    sm += __shfl_down_sync(0xffffffffu, sm, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&out[0], sc);
    atomicAdd(&out[1], sm);
  }
}

}  // namespace

struct Resident {
  dp_ctx* ctx = nullptr;
  const dp_graph_t* host = nullptr;  // only for error messages during generate
  dp_graph_t host_copy{};
  std::vector<int64_t> h_id, h_src, h_dst;  // what host_copy points at (dp_resident_create)
  DevGraph g;
  dp_devices_t dev_in{};                      // the caller's list, checked at placement
  std::vector<int32_t> dev_in_id;
  std::vector<int64_t> dev_in_mem;
  Devices devs;
  dp_comm_t comm{};
  dp_pipeline_config_t cfg{};
  int64_t limit = 1;
  bool decisions = true;
  // window outputs
  FuseOut f;
  DevBuf<int64_t> ct, cb, cc;
  DevBuf<int32_t> cseq, cpos;
  PlaceOut po, pa;
  DevBuf<int32_t> dev_order, dev_adjust;
  DevBuf<int64_t> pdm_order, pdm_adjust;
  double original_ccr = 0.0;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
};

double ccr_dev(DevGraph& g) {
  dp_ctx* ctx = g.ctx;
  DevBuf<unsigned long long> s(ctx, 2);
  s.zero();
  DP_LAUNCH(ctx, k_ccr, grid_for(std::max(g.n, g.m), 256, 4 * ctx->num_sms), 256, 0, g.w.p, g.n, g.cost.p, g.m, s.p);
  unsigned long long h[2];
  s.download(h, 2);
  sync(ctx);
  const int64_t tc = static_cast<int64_t>(h[0]);
  if (tc <= 0) fail(DP_E_ZERO_COMPUTE_TIME, "total compute time is zero");
  return static_cast<double>(static_cast<int64_t>(h[1])) / static_cast<double>(tc);
}

// Index + validation of an uploaded graph (pipeline.cpp:33).
void resident_validate(Resident& r, bool cycle_check) {
  DevGraph& g = r.g;
  StageScope st(r.ctx, "index+validate", 16.0 * g.m + 8.0 * g.n);
  graph_resolve(g);
  graph_adjacency(g);
  Validation v = graph_validate(g, r.host, false, cycle_check);
  if (v.code) fail(v.code, "%s", v.message.c_str());
}

// resident_validate(r, false) of several graphs with three host round trips in all (id
// density; adjacency facts; first violations) instead of three per graph.  Violations are
// reported graph by graph in order.
void resident_validate_batch(Resident* const* rs, int count, std::vector<Validation>* found = nullptr) {
  if (count == 1 && !found) {
    resident_validate(*rs[0], false);
    return;
  }
  dp_ctx* ctx = rs[0]->ctx;
  double bytes = 0.0;
  for (int i = 0; i < count; ++i) bytes += 16.0 * rs[i]->g.m + 8.0 * rs[i]->g.n;
  StageScope st(ctx, "index+validate", bytes);
  std::vector<ResolveState> R(count);
  std::vector<AdjState> A(count);
  std::vector<ValState> V(count);
  for (int i = 0; i < count; ++i) graph_resolve_begin(rs[i]->g, R[i]);
  sync(ctx);
  for (int i = 0; i < count; ++i) {
    graph_resolve_end(rs[i]->g, R[i]);
    graph_adjacency_begin(rs[i]->g, A[i]);
  }
  sync(ctx);
  for (int i = 0; i < count; ++i) {
    graph_adjacency_end(rs[i]->g, A[i]);
    graph_validate_begin(rs[i]->g, V[i]);
  }
  sync(ctx);
  for (int i = 0; i < count; ++i) {
    Validation v = graph_validate_end(rs[i]->g, rs[i]->host, V[i], false, false);
    if (found) found->push_back(std::move(v));
    else if (v.code) fail(v.code, "%s", v.message.c_str());
  }
}

// The end of the generation window (pipeline.cpp:67-79): 2x expand.
void generate_tail(Resident& r) {
  dp_ctx* ctx = r.ctx;
  DevGraph& g = r.g;
  const int32_t D = r.devs.D;
  r.dev_order.alloc(ctx, g.n > 0 ? g.n : 1);
  r.dev_adjust.alloc(ctx, g.n > 0 ? g.n : 1);
  r.pdm_order.alloc(ctx, D);
  r.pdm_adjust.alloc(ctx, D);
  StageScope st(ctx, "expand", 2.0 * (12.0 * g.n));
  expand_dev(g, r.f.node_cluster.p, r.po.dev.p, D, r.dev_order.p, r.pdm_order.p);
  expand_dev(g, r.f.node_cluster.p, r.pa.dev.p, D, r.dev_adjust.p, r.pdm_adjust.p);
}

// Generation windows of independent graphs on one stream (graphs already validated, with
// costs): each graph's fuse_begin, ONE launch of all the streamed peel + DP cores, each
// graph's traceback and coarse graph, ONE launch (per direction) of all the coarse-level
// sweeps, ONE launch of all the coarse CPD peels, ONE launch of all the placements, expand.
void generate_windows(Resident* const* rs, int count) {
  dp_ctx* ctx = rs[0]->ctx;
  std::vector<std::unique_ptr<FuseStage>> fs;
  std::vector<PeelDpJob*> jobs;
  // graphs sharing the comm model and a streamed range: their levels in shared launches
  // (fuse_order cannot fail then, so errors keep the graph-by-graph order)
  bool same = rs[0]->cfg.fusion_range >= 1 && rs[0]->cfg.fusion_range <= 256;
  for (int i = 1; i < count; ++i)
    same = same && rs[i]->comm.k_us_per_byte == rs[0]->comm.k_us_per_byte && rs[i]->comm.b_us == rs[0]->comm.b_us &&
           rs[i]->cfg.fusion_range == rs[0]->cfg.fusion_range;
  for (int i = 0; i < count; ++i) fs.emplace_back(new FuseStage);
  if (same && count > 1) {
    std::vector<DevGraph*> gs(count);
    std::vector<int64_t> lim(count);
    std::vector<FuseOut*> fo(count);
    std::vector<FuseStage*> fp(count);
    for (int i = 0; i < count; ++i) {
      gs[i] = &rs[i]->g;
      lim[i] = rs[i]->limit;
      fo[i] = &rs[i]->f;
      fp[i] = fs[i].get();
    }
    fuse_begin_batch(gs.data(), count, rs[0]->comm, rs[0]->cfg.fusion_range, lim.data(), fo.data(), fp.data());
  } else {
    for (int i = 0; i < count; ++i)
      fuse_begin(rs[i]->g, rs[i]->comm, rs[i]->cfg.fusion_range, rs[i]->limit, rs[i]->f, *fs[i]);
  }
  for (int i = 0; i < count; ++i)
    if (fs[i]->streamed) jobs.push_back(fs[i]->job.j);
  if (!jobs.empty()) peel_dp_launch(ctx, jobs.data(), static_cast<int>(jobs.size()));
  {
    std::vector<DevGraph*> gs(count);
    std::vector<FuseOut*> fo(count);
    std::vector<FuseStage*> fp(count);
    for (int i = 0; i < count; ++i) {
      gs[i] = &rs[i]->g;
      fo[i] = &rs[i]->f;
      fp[i] = fs[i].get();
    }
    fuse_end_batch(gs.data(), count, fo.data(), fp.data());
  }
  // coarse levels + cpd_topo of all graphs: one sweep launch per direction, one peel launch
  std::vector<DevGraph*> cg(count);
  std::vector<DevBuf<int64_t>*> ct(count), cb(count), cc(count);
  for (int i = 0; i < count; ++i) {
    cg[i] = &rs[i]->f.coarse;
    ct[i] = &rs[i]->ct;
    cb[i] = &rs[i]->cb;
    cc[i] = &rs[i]->cc;
  }
  levels_dev_chainlike_batch(cg.data(), count, rs[0]->comm, ct.data(), cb.data(), cc.data());
  std::vector<const int64_t*> cpath(count);
  std::vector<int32_t*> cseq(count), cpos(count);
  for (int i = 0; i < count; ++i) {
    Resident& r = *rs[i];
    const int32_t k = r.f.coarse.n;
    r.cseq.alloc(ctx, k > 0 ? k : 1);
    r.cpos.alloc(ctx, k > 0 ? k : 1);
    cpath[i] = r.cc.p;
    cseq[i] = r.cseq.p;
    cpos[i] = r.cpos.p;
  }
  topo_order_batch(cg.data(), count, DP_TOPO_CPD, cpath.data(), cseq.data(), cpos.data(), false);
  std::vector<std::unique_ptr<PlaceHandle>> ph;
  std::vector<PlaceJob*> pj;
  for (int i = 0; i < count; ++i) {
    Resident& r = *rs[i];
    // SchedulerState::for_devices runs inside order_place (placement.cpp:132,34-53), after
    // the graph, ccr and fuse errors: the device list is checked here, not at init
    r.devs = devices_sorted(&r.dev_in);
    ph.emplace_back(new PlaceHandle(place_prepare(r.f.coarse, r.cseq.p, r.devs, &r.po, &r.pa, r.decisions)));
    pj.push_back(ph.back()->j);
  }
  place_launch(ctx, pj.data(), count);
  for (int i = 0; i < count; ++i) generate_tail(*rs[i]);
}

// Everything after the H2D upload: index, validation (pipeline.cpp:33), ccr (:58),
// cluster limit (:60-65) and the generation window (:67-79).
void resident_generate(Resident* const* rs, int count, bool with_ccr) {
  dp_ctx* ctx = rs[0]->ctx;
  StageScope whole(ctx, "generate", 0.0);
  const bool dbg = getenv("DP_DEBUG_SYNC") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t s0 = ctx->sync_count;
  if (!with_ccr && count == 1) {
    resident_validate_batch(rs, count);
    graph_costs(rs[0]->g, rs[0]->comm);
  } else if (!with_ccr) {
    std::vector<Validation> found;
    resident_validate_batch(rs, count, &found);
    for (int i = 0; i < count; ++i) {
      if (found[i].code) {  // the earlier graphs' windows come first
        if (i > 0) generate_windows(rs, i);
        fail(found[i].code, "%s", found[i].message.c_str());
      }
      graph_costs(rs[i]->g, rs[i]->comm);
    }
  } else {  // validation (pipeline.cpp:33) and ccr (:58), one round trip each for all the graphs
    std::vector<Validation> found;
    resident_validate_batch(rs, count, &found);
    for (int i = 0; i < count; ++i)
      if (!found[i].code) graph_costs(rs[i]->g, rs[i]->comm);
    std::vector<DevBuf<unsigned long long>> sums(count);
    std::vector<unsigned long long> h(2 * (size_t)count, 0ull);
    for (int i = 0; i < count; ++i) {
      if (found[i].code) continue;
      DevGraph& g = rs[i]->g;
      sums[i].alloc(ctx, 2);
      sums[i].zero();
      DP_LAUNCH(ctx, k_ccr, grid_for(std::max(g.n, g.m), 256, 4 * ctx->num_sms), 256, 0, g.w.p, g.n, g.cost.p, g.m,
                sums[i].p);
      sums[i].download(h.data() + 2 * i, 2);
    }
    sync(ctx);
    for (int i = 0; i < count; ++i) {  // errors graph by graph: its violation, then its ccr
      const int64_t tc = static_cast<int64_t>(h[2 * i]);
      if (found[i].code || tc <= 0) {
        // the earlier graphs' windows come first (as in a loop of single calls)
        if (i > 0) generate_windows(rs, i);
        if (found[i].code) fail(found[i].code, "%s", found[i].message.c_str());
        fail(DP_E_ZERO_COMPUTE_TIME, "total compute time is zero");
      }
      rs[i]->original_ccr = static_cast<double>(static_cast<int64_t>(h[2 * i + 1])) / static_cast<double>(tc);
    }
  }
  const auto t1 = std::chrono::steady_clock::now();
  const int64_t s1 = ctx->sync_count;
  generate_windows(rs, count);
  if (dbg) {
    sync(ctx);
    const auto t2 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "[sync] %d graphs: validate %.1f ms (%lld syncs), windows %.1f ms (%lld syncs)\n", count, ms(t0, t1),
            (long long)(s1 - s0), ms(t1, t2), (long long)(ctx->sync_count - s1));
  }
}

void resident_init(Resident& r, dp_ctx* ctx, const dp_graph_t* h, const dp_devices_t* devices, dp_comm_t comm,
                   const dp_pipeline_config_t* cfg, cudaStream_t copy = nullptr, cudaEvent_t done = nullptr) {
  if (devices->count <= 0) fail(DP_E_INVALID_VALUE, "device list is empty");
  r.ctx = ctx;
  r.host = h;
  r.comm = comm;
  r.cfg = *cfg;  // fusion_range < 1 fails in fuse like fusion.cpp:96
  r.dev_in_id.assign(devices->id, devices->id + devices->count);
  r.dev_in_mem.assign(devices->memory_bytes, devices->memory_bytes + devices->count);
  r.dev_in = dp_devices_t{devices->count, r.dev_in_id.data(), r.dev_in_mem.data()};
  int64_t min_cap = devices->memory_bytes[0];
  for (int32_t i = 0; i < devices->count; ++i) min_cap = std::min(min_cap, devices->memory_bytes[i]);
  r.limit = std::max<int64_t>(1, static_cast<int64_t>(static_cast<double>(min_cap) * r.cfg.cluster_mem_fraction));
  graph_upload(r.g, ctx, h, copy, done);
}

// Expanded placement with every device listed (present where it received nodes).
dp_placement_result_t* expanded_to_host_async(dp_ctx* ctx, const Devices& devs, const int32_t* dev,
                                              const int64_t* pdm, int32_t n, Finalizers& fin) {
  const int32_t D = devs.D;
  dp_placement_result_t* p = new_placement(n, D, 0);
  auto d = std::make_shared<std::vector<int32_t>>(n);
  auto m = std::make_shared<std::vector<int64_t>>(D);
  if (n) download_bytes(ctx, d->data(), dev, sizeof(int32_t) * n);
  download_bytes(ctx, m->data(), pdm, sizeof(int64_t) * D);
  std::vector<int32_t> ids = devs.ids;
  fin.push_back([p, d, m, ids, n, D] {
    std::vector<uint8_t> present(D, 0);
    for (int32_t v = 0; v < n; ++v) {
      p->device[v] = ids[(*d)[v]];
      present[(*d)[v]] = 1;
    }
    for (int32_t i = 0; i < D; ++i) {
      p->device_ids[i] = ids[i];
      p->per_device_memory[i] = present[i] ? (*m)[i] : 0;
      p->device_present[i] = present[i];
    }
  });
  return p;
}

// ccr (graph.cpp:206-215) of a device graph into *out after sync(ctx) and `fin`.
void ccr_async(DevGraph& g, double* out, Finalizers& fin) {
  dp_ctx* ctx = g.ctx;
  DevBuf<unsigned long long> s(ctx, 2);
  s.zero();
  DP_LAUNCH(ctx, k_ccr, grid_for(std::max(g.n, g.m), 256, 4 * ctx->num_sms), 256, 0, g.w.p, g.n, g.cost.p, g.m, s.p);
  auto h = std::make_shared<std::array<unsigned long long, 2>>();
  download_bytes(ctx, h->data(), s.p, sizeof(unsigned long long) * 2);
  fin.push_back([h, out] {
    const int64_t tc = static_cast<int64_t>((*h)[0]);
    if (tc <= 0) fail(DP_E_ZERO_COMPUTE_TIME, "total compute time is zero");
    *out = static_cast<double>(static_cast<int64_t>((*h)[1])) / static_cast<double>(tc);
  });
}

}  // namespace dpb

struct dp_resident : dpb::Resident {};

using namespace dpb;

extern "C" {

int dp_pipeline(dp_ctx_t* ctx, const dp_graph_t* h, const dp_devices_t* devices, dp_comm_t comm,
                const dp_pipeline_config_t* cfg, dp_pipeline_result_t** out) {
  const dp_graph_t* hs[1] = {h};
  return dp_pipeline_batch(ctx, 1, hs, devices, comm, cfg, out);
}

int dp_pipeline_batch(dp_ctx_t* ctx, int32_t count, const dp_graph_t* const* graphs, const dp_devices_t* devices,
                      dp_comm_t comm, const dp_pipeline_config_t* cfg, dp_pipeline_result_t** out) {
  DP_API_BEGIN(ctx)
  if (count < 0) fail(DP_E_INVALID_VALUE, "graph count must be >= 0");
  const bool dbg = getenv("DP_DEBUG_PIPE") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto span_ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto h0 = now();
  std::vector<std::unique_ptr<Resident>> rs;
  std::vector<Resident*> rp;
  // several graphs: uploads on the context's copy stream, graph i's validation waits only
  // for its own copies (the later graphs' uploads overlap it)
  std::vector<cudaEvent_t> up;
  struct UpGuard {  // before the graphs are freed (stream-ordered on ctx->stream): order the
    dp_ctx* c;       // frees after every copy, also when a graph fails before its wait
    std::vector<cudaEvent_t>& v;
    ~UpGuard() {
      for (auto e : v) {
        cudaStreamWaitEvent(c->stream, e, 0);
        cudaEventDestroy(e);
      }
    }
  } up_guard{ctx, up};
  if (count > 1 && !ctx->copy_stream)
    DP_CUDA(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  for (int32_t i = 0; i < count; ++i) {
    rs.emplace_back(new Resident);
    rp.push_back(rs.back().get());
    cudaEvent_t e = nullptr;
    if (count > 1) {
      DP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      up.push_back(e);
    }
    resident_init(*rs.back(), ctx, graphs[i], devices, comm, cfg, count > 1 ? ctx->copy_stream : nullptr, e);
  }
  if (dbg) sync(ctx);
  const auto h1 = now();
  cudaEvent_t e0, e1;
  DP_CUDA(cudaEventCreate(&e0));
  DP_CUDA(cudaEventCreate(&e1));
  struct EvGuard {
    cudaEvent_t a, b;
    ~EvGuard() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  } guard{e0, e1};
  // require_valid + ccr precede the window (pipeline.cpp:33, :58)
  for (int32_t i = 0; i < count; ++i) {
    Resident* r = rp[i];
    if (!up.empty()) DP_CUDA(cudaStreamWaitEvent(ctx->stream, up[i], 0));
    try {
      resident_validate(*r, true);
      graph_costs(r->g, comm);
      r->original_ccr = ccr_dev(r->g);
    } catch (const DpFail&) {
      // a loop of single calls would have run the earlier graphs' windows first: their
      // errors take precedence over this graph's
      if (i > 0) generate_windows(rp.data(), i);
      throw;
    }
  }
  if (dbg) sync(ctx);
  const auto h2 = now();
  DP_CUDA(cudaEventRecord(e0, ctx->stream));
  if (count > 0) generate_windows(rp.data(), count);
  DP_CUDA(cudaEventRecord(e1, ctx->stream));
  if (dbg) sync(ctx);
  const auto h3 = now();
  std::vector<dp_pipeline_result_t*> res(static_cast<size_t>(count), nullptr);
  struct ResGuard {
    std::vector<dp_pipeline_result_t*>& v;
    ~ResGuard() {
      for (auto* x : v)
        if (x) dp_pipeline_result_free(x);
    }
  } res_guard{res};
  float ms = 0;
  DP_CUDA(cudaEventSynchronize(e1));
  DP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  // every graph's downloads first, one sync, then the host-side assembly
  Finalizers fin;
  for (int32_t i = 0; i < count; ++i) {
    Resident& r = *rp[i];
    DevGraph& coarse = r.f.coarse;
    const int32_t k = coarse.n, n = r.g.n;
    auto* x = res[i] = halloc<dp_pipeline_result_t>(1);
    x->original_nodes = n;
    x->original_edges = r.g.m;
    x->original_ccr = r.original_ccr;
    x->coarse_nodes = k;
    x->coarse_edges = coarse.m;
    x->fusion = halloc<dp_fusion_result_t>(1);
    x->fusion->coarse = graph_to_host_async(coarse, true, fin);
    x->fusion->map = fuse_map_to_host_async(r.g, r.f, fin);
    auto cs = std::make_shared<std::vector<int32_t>>(k);
    if (k) download_bytes(ctx, cs->data(), r.cseq.p, sizeof(int32_t) * k);
    x->coarse_sequence = halloc<int64_t>(k);
    auto cids = std::make_shared<std::vector<int64_t>>(static_cast<size_t>(k));
    fin.push_back([x, cs, cids, k] {
      for (int32_t q = 0; q < k; ++q) (*cids)[q] = x->coarse_sequence[q] = (*cs)[q];
    });
    x->coarse_order = placement_to_host_async(ctx, r.devs, r.po, k, cids, false, fin);
    x->coarse_adjust = placement_to_host_async(ctx, r.devs, r.pa, k, cids, true, fin);
    x->order_expanded = expanded_to_host_async(ctx, r.devs, r.dev_order.p, r.pdm_order.p, n, fin);
    x->adjust_expanded = expanded_to_host_async(ctx, r.devs, r.dev_adjust.p, r.pdm_adjust.p, n, fin);
    x->generation_ms = ms;  // the window of the whole call (all graphs of a batch)
    x->coarse_ccr = 0.0;
    if (coarse.m > 0) ccr_async(coarse, &x->coarse_ccr, fin);  // pipeline.cpp:83
    x->order_makespan = x->adjust_makespan = -1;
  }
  sync(ctx);
  for (auto& f : fin) f();
  if (cfg->simulate) {  // pipeline.cpp:89-90 (full reports kept for simulate == 2)
    const bool full = cfg->simulate == 2;
    for (int32_t i = 0; i < count; ++i) {
      Resident& r = *rp[i];
      dp_sim_report_t* so = sim_report(r.g, r.devs, r.dev_order.p, full);
      res[i]->order_makespan = so->makespan;
      if (full) res[i]->order_sim = so; else free_sim(so);
      dp_sim_report_t* sa = sim_report(r.g, r.devs, r.dev_adjust.p, full);
      res[i]->adjust_makespan = sa->makespan;
      if (full) res[i]->adjust_sim = sa; else free_sim(sa);
    }
  }
  if (dbg) {
    const auto h4 = now();
    fprintf(stderr, "[dp_pipeline] upload %.1f ms, validate+ccr %.1f ms, window %.1f ms, results %.1f ms\n",
            span_ms(h0, h1), span_ms(h1, h2), span_ms(h2, h3), span_ms(h3, h4));
  }
  for (int32_t i = 0; i < count; ++i) {
    out[i] = res[i];
    res[i] = nullptr;
  }
  DP_API_END
}

int dp_resident_create(dp_ctx_t* ctx, const dp_graph_t* h, const dp_devices_t* devices, dp_comm_t comm,
                       const dp_pipeline_config_t* cfg, dp_resident_t** out) {
  DP_API_BEGIN(ctx)
  auto* r = new dp_resident;
  try {
    resident_init(*r, ctx, h, devices, comm, cfg);
    // a private copy of the ids / edge endpoints for error messages raised by later
    // generate calls (the caller may free its arrays once the graph is on the device)
    r->h_id.assign(h->node_id, h->node_id + h->n_nodes);
    r->h_src.assign(h->edge_src, h->edge_src + h->n_edges);
    r->h_dst.assign(h->edge_dst, h->edge_dst + h->n_edges);
    r->host_copy = *h;
    r->host_copy.node_id = r->h_id.data();
    r->host_copy.edge_src = r->h_src.data();
    r->host_copy.edge_dst = r->h_dst.data();
    r->host_copy.compute_us = nullptr;
    r->host_copy.memory_bytes = nullptr;
    r->host_copy.edge_bytes = nullptr;
    r->host_copy.group = nullptr;
    r->host = &r->host_copy;
    sync(ctx);
  } catch (...) {
    delete r;
    throw;
  }
  *out = r;
  DP_API_END
}

int dp_resident_generate(dp_resident_t* r) {
  DP_API_BEGIN(r ? r->ctx : nullptr)
  Resident* rs[1] = {r};
  resident_generate(rs, 1, false);
  DP_API_END
}

int dp_resident_generate_batch(dp_resident_t* const* rs, int32_t count) {
  if (count == 0) return 0;
  DP_API_BEGIN(count > 0 && rs && rs[0] ? rs[0]->ctx : nullptr)
  for (int32_t i = 0; i < count; ++i)
    if (!rs[i] || rs[i]->ctx != rs[0]->ctx) fail(DP_E_INVALID_VALUE, "batched residents must share one context");
  std::vector<Resident*> v(rs, rs + count);
  resident_generate(v.data(), count, false);
  DP_API_END
}

int dp_resident_fetch(dp_resident_t* r, int32_t* order_device, int32_t* adjust_device, int64_t* coarse_nodes,
                      int64_t* coarse_edges) {
  DP_API_BEGIN(r ? r->ctx : nullptr)
  dp_ctx* ctx = r->ctx;
  const int32_t n = r->g.n;
  // device positions -> ids on the host side of the copy
  std::vector<int32_t> a = to_host(ctx, r->dev_order.p, n), b = to_host(ctx, r->dev_adjust.p, n);
  for (int32_t v = 0; v < n; ++v) {
    order_device[v] = r->devs.ids[a[v]];
    adjust_device[v] = r->devs.ids[b[v]];
  }
  if (coarse_nodes) *coarse_nodes = r->f.coarse.n;
  if (coarse_edges) *coarse_edges = r->f.coarse.m;
  DP_API_END
}

void dp_resident_destroy(dp_resident_t* r) {
  if (!r) return;
  cudaSetDevice(r->ctx->device);
  cudaStreamSynchronize(r->ctx->stream);
  r->ctx->pending.clear();
  delete r;
}

}  // extern "C"
