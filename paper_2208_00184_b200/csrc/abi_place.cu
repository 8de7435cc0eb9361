// abi_place.cu — C-ABI entry points of the placement stage (placement.cpp:128-268).
#include <algorithm>
#include <unordered_map>

#include "abi_util.cuh"
#include "placement.cuh"
#include "results.h"

namespace dpb {

// GraphIndex ctor errors (graph_index.cpp:12-18, 44-50) on an uploaded, resolved graph.
void graph_index_checks(DevGraph& g, const dp_graph_t* h) {
  dp_ctx* ctx = g.ctx;
  if (!g.dense_ids && g.n > 1) {
    std::vector<uint64_t> keys = to_host(ctx, g.sorted_key.p, g.n);
    std::vector<int32_t> idx = to_host(ctx, g.sorted_idx.p, g.n);
    int32_t bad = INT32_MAX;
    int64_t bad_id = 0;
    for (int32_t s = 1; s < g.n; ++s) {
      if (keys[s] == keys[s - 1] && idx[s] < bad) {
        bad = idx[s];
        bad_id = static_cast<int64_t>(keys[s] ^ (1ull << 63));
      }
    }
    if (bad != INT32_MAX) fail(DP_E_DUPLICATE_ID, "node id %lld is not unique", (long long)bad_id);
  }
  std::vector<int32_t> hs = to_host(ctx, g.esrc.p, g.m), hd = to_host(ctx, g.edst.p, g.m);
  for (int32_t e = 0; e < g.m; ++e) {
    if (hs[e] < 0) fail(DP_E_UNKNOWN_NODE, "node %lld not in graph", (long long)h->edge_src[e]);
    if (hd[e] < 0) fail(DP_E_UNKNOWN_NODE, "node %lld not in graph", (long long)h->edge_dst[e]);
  }
}

// Host view of a device placement (device positions -> ids).
dp_placement_result_t* placement_to_host_async(dp_ctx* ctx, const Devices& devs, PlaceOut& p, int32_t n,
                                               std::shared_ptr<const std::vector<int64_t>> seq_ids, bool decisions,
                                               Finalizers& fin) {
  const int32_t D = devs.D;
  dp_placement_result_t* r = new_placement(n, D, decisions ? n : 0);
  auto dev = std::make_shared<std::vector<int32_t>>(n);
  auto pdm = std::make_shared<std::vector<int64_t>>(D);
  auto oom = std::make_shared<int32_t>(0);
  if (n) download_bytes(ctx, dev->data(), p.dev.p, sizeof(int32_t) * n);
  download_bytes(ctx, pdm->data(), p.per_dev_mem.p, sizeof(int64_t) * D);
  download_bytes(ctx, oom.get(), p.flags.p, sizeof(int32_t));
  auto prev = std::make_shared<std::vector<int32_t>>(), ch = std::make_shared<std::vector<int32_t>>();
  const bool dec = decisions && n;
  if (dec) {
    prev->resize(n);
    ch->resize(n);
    download_bytes(ctx, prev->data(), p.dec_prev.p, sizeof(int32_t) * n);
    download_bytes(ctx, ch->data(), p.dec_chosen.p, sizeof(int32_t) * n);
    p.dec_est.download(r->dec_est, (size_t)n * D);
    p.dec_back.download(r->dec_back_cost, n);
    p.dec_reloc.download(r->dec_relocated, n);
    p.dec_be.download(r->dec_best_effort, n);
  }
  std::vector<int32_t> ids = devs.ids;
  fin.push_back([r, dev, pdm, oom, prev, ch, dec, ids, seq_ids, n, D] {
    for (int32_t v = 0; v < n; ++v) r->device[v] = ids[(*dev)[v]];
    for (int32_t d = 0; d < D; ++d) {
      r->device_ids[d] = ids[d];
      r->per_device_memory[d] = (*pdm)[d];
      r->device_present[d] = 1;
    }
    r->oom_risk = *oom;
    if (dec) {
      for (int32_t k = 0; k < n; ++k) {
        r->dec_node[k] = (*seq_ids)[k];
        r->dec_prev[k] = ids[(*prev)[k]];
        r->dec_chosen[k] = ids[(*ch)[k]];
      }
    }
  });
  return r;
}

dp_placement_result_t* placement_to_host(dp_ctx* ctx, const Devices& devs, PlaceOut& p, int32_t n,
                                         const std::vector<int64_t>* seq_ids, bool decisions) {
  Finalizers fin;
  auto seq = std::make_shared<const std::vector<int64_t>>(seq_ids ? *seq_ids : std::vector<int64_t>());
  dp_placement_result_t* r = placement_to_host_async(ctx, devs, p, n, seq, decisions, fin);
  sync(ctx);
  for (auto& x : fin) x();
  return r;
}

namespace {

int place_api(dp_ctx* ctx, const dp_graph_t* h, const int64_t* seq, int64_t len, const dp_devices_t* devices,
              const dp_comm_t* comm, dp_placement_result_t** out) {
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  if (!order_valid_dev(g, seq, len)) fail(DP_E_INVALID_VALUE, "order is not a topological order of this graph");
  Devices devs = devices_sorted(devices);
  if (comm) graph_costs(g, *comm);
  const int32_t n = g.n;
  DevBuf<int64_t> sid(ctx, n > 0 ? n : 1);
  sid.upload(seq, n);
  DevBuf<int32_t> sidx(ctx, n > 0 ? n : 1);
  graph_ids_to_index(g, sid.p, sidx.p, n);
  PlaceOut p;
  place_dev(g, sidx.p, devs, comm ? nullptr : &p, comm ? &p : nullptr, comm != nullptr);
  std::vector<int64_t> ids(seq, seq + n);
  *out = placement_to_host(ctx, devs, p, n, &ids, comm != nullptr);
  return DP_OK;
}

}  // namespace
}  // namespace dpb

using namespace dpb;

extern "C" {

int dp_order_place(dp_ctx_t* ctx, const dp_graph_t* coarse, const int64_t* seq, int64_t len,
                   const dp_devices_t* devices, dp_placement_result_t** out) {
  DP_API_BEGIN(ctx)
  place_api(ctx, coarse, seq, len, devices, nullptr, out);
  DP_API_END
}

int dp_adjusting_placement(dp_ctx_t* ctx, const dp_graph_t* coarse, const int64_t* seq, int64_t len,
                           const dp_devices_t* devices, dp_comm_t comm, dp_placement_result_t** out) {
  DP_API_BEGIN(ctx)
  place_api(ctx, coarse, seq, len, devices, &comm, out);
  DP_API_END
}

int dp_expand_placement(dp_ctx_t* ctx, const dp_graph_t* h, const int32_t* node_cluster, int64_t n_clusters,
                        const int64_t* member_off, const int64_t* members, const int32_t* coarse_device,
                        const uint8_t* coarse_placed, dp_placement_result_t** out) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  graph_upload(g, ctx, h);
  graph_resolve(g);
  graph_index_checks(g, h);
  const int64_t n = h->n_nodes;
  // ClusterMap / coarse placement checks in the reference's iteration order
  // (placement.cpp:242-266) — validation of caller input.
  int64_t mapped = 0;
  for (int64_t i = 0; i < n; ++i) mapped += node_cluster[i] >= 0;
  if (mapped != n)
    fail(DP_E_INVALID_CLUSTER_MAP, "cluster map covers %lld nodes, graph has %lld", (long long)mapped, (long long)n);
  std::unordered_map<int64_t, int32_t> index;
  index.reserve(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) index.emplace(h->node_id[i], static_cast<int32_t>(i));
  std::vector<uint8_t> seen(static_cast<size_t>(n), 0);
  int64_t covered = 0;
  std::vector<int32_t> dev_ids;
  for (int64_t c = 0; c < n_clusters; ++c) {
    if (coarse_placed && !coarse_placed[c]) fail(DP_E_UNPLACED_NODE, "cluster %lld has no device", (long long)c);
    dev_ids.push_back(coarse_device[c]);
    for (int64_t q = member_off[c]; q < member_off[c + 1]; ++q) {
      auto it = index.find(members[q]);
      if (it == index.end()) fail(DP_E_UNKNOWN_NODE, "node %lld not in graph", (long long)members[q]);
      if (seen[it->second]) fail(DP_E_INVALID_CLUSTER_MAP, "node %lld appears in two clusters", (long long)members[q]);
      seen[it->second] = 1;
      ++covered;
    }
  }
  if (covered != n) fail(DP_E_INVALID_CLUSTER_MAP, "expanded placement does not cover the graph");
  // devices that receive nodes, ascending id -> positions
  std::vector<int32_t> used;
  for (int64_t c = 0; c < n_clusters; ++c)
    if (member_off[c + 1] > member_off[c]) used.push_back(coarse_device[c]);
  std::sort(used.begin(), used.end());
  used.erase(std::unique(used.begin(), used.end()), used.end());
  const int32_t D = static_cast<int32_t>(used.size());
  // the map the expansion follows is the clusters' member lists (not node_cluster)
  std::vector<int32_t> cl(static_cast<size_t>(n), 0), cpos(static_cast<size_t>(n_clusters > 0 ? n_clusters : 1), 0);
  for (int64_t c = 0; c < n_clusters; ++c) {
    cpos[c] = static_cast<int32_t>(std::lower_bound(used.begin(), used.end(), coarse_device[c]) - used.begin());
    for (int64_t q = member_off[c]; q < member_off[c + 1]; ++q) cl[index[members[q]]] = static_cast<int32_t>(c);
  }
  DevBuf<int32_t> dcl(ctx, n > 0 ? n : 1), dcp(ctx, n_clusters > 0 ? n_clusters : 1), dev(ctx, n > 0 ? n : 1);
  DevBuf<int64_t> pdm(ctx, D > 0 ? D : 1);
  dcl.upload(cl.data(), n);
  dcp.upload(cpos.data(), n_clusters);
  expand_dev(g, dcl.p, dcp.p, D, dev.p, pdm.p);
  dp_placement_result_t* r = new_placement(n, D, 0);
  std::vector<int32_t> hd = to_host(ctx, dev.p, n);
  pdm.download(r->per_device_memory, D);
  sync(ctx);
  for (int64_t v = 0; v < n; ++v) r->device[v] = used[hd[v]];
  for (int32_t d = 0; d < D; ++d) {
    r->device_ids[d] = used[d];
    r->device_present[d] = 1;
  }
  *out = r;
  DP_API_END
}

}  // extern "C"
