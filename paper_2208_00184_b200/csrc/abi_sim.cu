// abi_sim.cu — C-ABI entry points of the simulator (simulator.cpp:56-310).
#include <algorithm>

#include "abi_util.cuh"
#include "placement.cuh"
#include "results.h"
#include "simulate.cuh"

namespace dpb {
namespace {

__global__ void k_sim_stats(const int32_t* esrc, const int32_t* edst, const int64_t* bytes, int32_t m,
                            const int32_t* dev, const int64_t* mem, int32_t n, int32_t D,
                            unsigned long long* out /* [0] count [1] bytes [2..2+D) peak */) {
  extern __shared__ unsigned long long sm[];
  for (int d = threadIdx.x; d < D + 2; d += blockDim.x) sm[d] = 0;
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    if (dev[esrc[e]] != dev[edst[e]]) {
      atomicAdd(&sm[0], 1ull);
      atomicAdd(&sm[1], static_cast<unsigned long long>(bytes[e]));
    }
  }
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&sm[2 + dev[v]], static_cast<unsigned long long>(mem[v]));
  __syncthreads();
  for (int d = threadIdx.x; d < D + 2; d += blockDim.x)
    if (sm[d]) atomicAdd(&out[d], sm[d]);
}

}  // namespace

// Placement -> device positions with the checks of simulator.cpp:61-92.
std::vector<int32_t> sim_positions(const dp_graph_t* h, const int32_t* device_of_node, const Devices& devs) {
  std::vector<int32_t> pos(static_cast<size_t>(h->n_nodes));
  for (int64_t v = 0; v < h->n_nodes; ++v) {
    const int32_t d = device_of_node[v];
    if (d == INT32_MIN) fail(DP_E_UNPLACED_NODE, "node %lld has no device", (long long)h->node_id[v]);
    auto it = std::lower_bound(devs.ids.begin(), devs.ids.end(), d);
    if (it == devs.ids.end() || *it != d)
      fail(DP_E_INVALID_VALUE, "node %lld placed on unknown device %d", (long long)h->node_id[v], d);
    pos[v] = static_cast<int32_t>(it - devs.ids.begin());
  }
  return pos;
}

// SimulationReport (simulator.cpp:210-250) for one placement already on the device.
dp_sim_report_t* sim_report(DevGraph& g, const Devices& devs, const int32_t* dev_pos_dev, bool trace) {
  dp_ctx* ctx = g.ctx;
  const int32_t D = devs.D;
  SimInput in;
  in.node_dev = dev_pos_dev;
  in.D = D;
  in.trace = trace;
  SimOutput out;
  int32_t Q = sim_queue_cap();
  simulate_dev(g, in, out, Q);
  int64_t ms = scalar_to_host(ctx, out.makespan.p);
  while (ms < 0 && g.n) {  // a ring overflowed: re-run with larger rings
    Q = sim_queue_grow(g, Q);
    simulate_dev(g, in, out, Q);
    ms = scalar_to_host(ctx, out.makespan.p);
  }
  DevBuf<unsigned long long> st(ctx, (size_t)D + 2);
  st.zero();
  DP_LAUNCH(ctx, k_sim_stats, grid_for(std::max(g.n, g.m), 256, 4 * ctx->num_sms), 256,
            sizeof(unsigned long long) * (D + 2), g.esrc.p, g.edst.p, g.bytes.p, g.m, dev_pos_dev, g.mem.p, g.n, D,
            st.p);
  std::vector<unsigned long long> hs = to_host(ctx, st.p, (size_t)D + 2);
  const int64_t cross = static_cast<int64_t>(hs[0]);
  dp_sim_report_t* r = new_sim(D, trace ? g.n + 2 * cross : 0);
  r->makespan = g.n ? ms : 0;
  r->cross_transfer_count = cross;
  r->cross_transfer_bytes = static_cast<int64_t>(hs[1]);
  for (int32_t d = 0; d < D; ++d) {
    r->device_ids[d] = devs.ids[d];
    r->capacity[d] = devs.cap[d];
    r->peak_memory[d] = static_cast<int64_t>(hs[2 + d]);
    if (r->peak_memory[d] > r->capacity[d]) r->oom_flag = 1;
  }
  if (trace && g.n) {
    // trace records sorted by (start, compute-before-transfer, id) (simulator.cpp:223-250)
    const int32_t n = g.n, m = g.m;
    std::vector<int64_t> ts = to_host(ctx, out.tstart.p, (size_t)n + m), te = to_host(ctx, out.tend.p, (size_t)n + m);
    std::vector<int32_t> dv = to_host(ctx, dev_pos_dev, n);
    std::vector<int32_t> es = to_host(ctx, g.esrc.p, m), ed = to_host(ctx, g.edst.p, m);
    std::vector<int64_t> ids = to_host(ctx, g.id.p, n), sid = to_host(ctx, g.src_id.p, m), did = to_host(ctx, g.dst_id.p, m);
    std::vector<int32_t> tasks;
    tasks.reserve(static_cast<size_t>(n + cross));
    for (int32_t v = 0; v < n; ++v) tasks.push_back(v);
    for (int32_t e = 0; e < m; ++e)
      if (dv[es[e]] != dv[ed[e]]) tasks.push_back(n + e);
    std::sort(tasks.begin(), tasks.end(), [&](int32_t a, int32_t b) {
      if (ts[a] != ts[b]) return ts[a] < ts[b];
      const bool xa = a >= n, xb = b >= n;
      if (xa != xb) return !xa;
      if (xa) return a < b;
      return ids[a] < ids[b];
    });
    int64_t w = 0;
    for (int32_t t : tasks) {
      if (t >= n) {
        const int32_t e = t - n;
        for (int k = 0; k < 2; ++k) {
          r->tr_kind[w] = k ? DP_TASK_RECEIVE : DP_TASK_SEND;
          r->tr_node[w] = -1;
          r->tr_src[w] = sid[e];
          r->tr_dst[w] = did[e];
          r->tr_device[w] = devs.ids[dv[k ? ed[e] : es[e]]];
          r->tr_start[w] = ts[t];
          r->tr_end[w] = te[t];
          ++w;
        }
      } else {
        r->tr_kind[w] = DP_TASK_COMPUTE;
        r->tr_node[w] = ids[t];
        r->tr_src[w] = -1;
        r->tr_dst[w] = -1;
        r->tr_device[w] = devs.ids[dv[t]];
        r->tr_start[w] = ts[t];
        r->tr_end[w] = te[t];
        ++w;
      }
    }
  }
  return r;
}

}  // namespace dpb

using namespace dpb;

extern "C" {

int dp_simulate(dp_ctx_t* ctx, const dp_graph_t* h, const int32_t* device_of_node, const dp_devices_t* devices,
                dp_comm_t comm, int32_t want_trace, dp_sim_report_t** out) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  Devices devs = devices_sorted(devices);
  std::vector<int32_t> pos = sim_positions(h, device_of_node, devs);
  graph_costs(g, comm);
  DevBuf<int32_t> dpos(ctx, g.n > 0 ? g.n : 1);
  dpos.upload(pos.data(), g.n);
  *out = sim_report(g, devs, dpos.p, want_trace != 0);
  DP_API_END
}

int dp_simulate_candidates(dp_ctx_t* ctx, const dp_graph_t* h, const int32_t* node_cluster, int64_t n_clusters,
                           const uint8_t* cand, int64_t B, const dp_devices_t* devices, dp_comm_t comm,
                           int64_t* makespans, int64_t* argmin) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  Devices devs = devices_sorted(devices);
  for (int64_t i = 0; i < B * n_clusters; ++i)
    if (cand[i] >= devs.D) fail(DP_E_INVALID_VALUE, "candidate device position %d out of range", cand[i]);
  for (int64_t v = 0; v < h->n_nodes; ++v)
    if (node_cluster[v] < 0 || node_cluster[v] >= n_clusters)
      fail(DP_E_INVALID_CLUSTER_MAP, "node %lld has no cluster", (long long)h->node_id[v]);
  graph_costs(g, comm);
  DevBuf<uint8_t> dc(ctx, B * n_clusters > 0 ? B * n_clusters : 1);
  DevBuf<int32_t> dcl(ctx, g.n > 0 ? g.n : 1);
  dc.upload(cand, B * n_clusters);
  dcl.upload(node_cluster, g.n);
  SimInput in;
  in.cand = dc.p;
  in.node_cluster = dcl.p;
  in.n_clusters = static_cast<int32_t>(n_clusters);
  in.n_candidates = B;
  in.D = devs.D;
  SimOutput o;
  simulate_batch_dev(g, in, o);
  o.makespan.download(makespans, B);
  sync(ctx);
  int64_t best = -1;
  for (int64_t b = 0; b < B; ++b)
    if (best < 0 || makespans[b] < makespans[best]) best = b;  // first strict minimum
  *argmin = best;
  DP_API_END
}

int dp_brute_force_optimal(dp_ctx_t* ctx, const dp_graph_t* h, const dp_devices_t* devices, dp_comm_t comm,
                           int32_t* best_dev, int64_t* best_ms) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  const int64_t n = h->n_nodes;
  if (n > 12 || devices->count > 3)
    fail(DP_E_INSTANCE_TOO_LARGE, "exhaustive search limited to 12 nodes and 3 devices");
  if (devices->count <= 0) fail(DP_E_INVALID_VALUE, "device list is empty");
  // sorted devices (no validity checks yet: simulate() performs them, simulator.cpp:61-75)
  std::vector<std::pair<int32_t, int64_t>> ds;
  for (int32_t i = 0; i < devices->count; ++i) ds.push_back({devices->id[i], devices->memory_bytes[i]});
  std::sort(ds.begin(), ds.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  const int32_t Dn = static_cast<int32_t>(ds.size());
  // nodes by ascending id; odometer over them, last varies fastest (simulator.cpp:268-303)
  std::vector<int32_t> by_id(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) by_id[i] = static_cast<int32_t>(i);
  std::sort(by_id.begin(), by_id.end(), [&](int32_t a, int32_t b) { return h->node_id[a] < h->node_id[b]; });
  int64_t total = 1;
  for (int64_t i = 0; i < n; ++i) total *= Dn;
  std::vector<uint8_t> cands;
  std::vector<int64_t> order_idx;
  std::vector<int32_t> choice(static_cast<size_t>(n), 0);
  for (int64_t c = 0; c < total; ++c) {
    int64_t x = c;
    for (int64_t p = n - 1; p >= 0; --p) {
      choice[p] = static_cast<int32_t>(x % Dn);
      x /= Dn;
    }
    std::vector<int64_t> used(Dn, 0);
    bool feasible = true;
    for (int64_t p = 0; p < n && feasible; ++p) {
      used[choice[p]] += h->memory_bytes[by_id[p]];
      feasible = used[choice[p]] <= ds[choice[p]].second;
    }
    if (!feasible) continue;
    order_idx.push_back(c);
    for (int64_t v = 0; v < n; ++v) cands.push_back(0);
    uint8_t* row = cands.data() + cands.size() - n;
    for (int64_t p = 0; p < n; ++p) row[by_id[p]] = static_cast<uint8_t>(choice[p]);
  }
  if (order_idx.empty()) fail(DP_E_INSTANCE_INFEASIBLE, "no memory-feasible assignment exists");
  Devices devs = devices_sorted(devices);
  graph_costs(g, comm);
  const int64_t B = static_cast<int64_t>(order_idx.size());
  DevBuf<uint8_t> dc(ctx, cands.size());
  dc.upload(cands.data(), cands.size());
  std::vector<int32_t> ident(static_cast<size_t>(n));
  for (int64_t v = 0; v < n; ++v) ident[v] = static_cast<int32_t>(v);
  DevBuf<int32_t> dcl(ctx, n > 0 ? n : 1);
  dcl.upload(ident.data(), n);
  SimInput in;
  in.cand = dc.p;
  in.node_cluster = dcl.p;
  in.n_clusters = static_cast<int32_t>(n);
  in.n_candidates = B;
  in.D = devs.D;
  SimOutput o;
  simulate_batch_dev(g, in, o);
  std::vector<int64_t> ms = to_host(ctx, o.makespan.p, B);
  int64_t best = 0;
  for (int64_t b = 1; b < B; ++b)
    if (ms[b] < ms[best]) best = b;
  for (int64_t v = 0; v < n; ++v) best_dev[v] = devs.ids[cands[best * n + v]];
  *best_ms = ms[best];
  DP_API_END
}

}  // extern "C"
