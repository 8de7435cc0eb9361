// abi_fusion.cu — C-ABI entry points of the fusion stage (fusion.cpp:16-335).
#include <algorithm>
#include <unordered_map>
#include <unordered_set>

#include "abi_util.cuh"
#include "fusion.cuh"
#include "peel.cuh"
#include "results.h"

namespace dpb {
namespace {

__global__ void k_scatter_pos(const int32_t* seq, int32_t n, int32_t* pos_of) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    pos_of[seq[p]] = static_cast<int32_t>(p);
}

__global__ void k_cl_by_node(const int32_t* cl_of_pos, const int32_t* pos_of, int32_t n, int32_t* out) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[v] = cl_of_pos[pos_of[v]];
}

__global__ void k_tot_from_map(const int32_t* cl, const int64_t* w, const int64_t* mem, int32_t n, int64_t* tw,
                               int64_t* tm) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    atomic_add_i64(&tw[cl[v]], w[v]);
    atomic_add_i64(&tm[cl[v]], mem[v]);
  }
}

// Reachability u ->* v avoiding the direct edge (merge_is_safe, fusion.cpp:33-50):
// persistent level-synchronous BFS.
struct BfsArgs {
  const int32_t* out_off;
  const int32_t* out_dst;
  const int32_t* out_eid;
  int32_t ui, vi, direct;
  int32_t* visited;
  int32_t* queue;
  int* counters;  // [0] tail, [1] found
  unsigned* bar;
};
__global__ void __launch_bounds__(256) k_bfs(BfsArgs a) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  int32_t lb = 0;
  int32_t le = a.counters[0];
  grid_barrier(a.bar, gridDim.x);
  for (;;) {
    if (le == lb) break;  // run to completion: an early exit on `found` could split the barrier
    for (int64_t i = lb + tid; i < le; i += nth) {
      int32_t u = a.queue[i];
      for (int32_t k = a.out_off[u]; k < a.out_off[u + 1]; ++k) {
        if (u == a.ui && a.out_eid[k] == a.direct) continue;
        int32_t x = a.out_dst[k];
        if (x == a.vi) {
          atomicExch(&a.counters[1], 1);
          continue;
        }
        bool fresh = atomicExch(&a.visited[x], 1) == 0;
        int slot = warp_append(&a.counters[0], fresh);
        if (fresh) a.queue[slot] = x;
      }
    }
    grid_barrier(a.bar, gridDim.x, &a.counters[0], &a.counters[2]);
    lb = le;
    le = *((volatile int*)&a.counters[2]);
  }
}

__global__ void k_find_direct(const int32_t* out_off, const int32_t* out_dst, const int32_t* out_eid, int32_t ui,
                              int32_t vi, int* direct) {
  for (int32_t k = out_off[ui] + threadIdx.x; k < out_off[ui + 1]; k += blockDim.x)
    if (out_dst[k] == vi) atomicMin(direct, out_eid[k]);
}

}  // namespace

dp_graph_out_t* graph_to_host_async(DevGraph& g, bool dense_ids_out, Finalizers& fin) {
  dp_ctx* ctx = g.ctx;
  dp_graph_out_t* o = new_graph_out(g.n, g.m);
  if (dense_ids_out) {
    for (int32_t i = 0; i < g.n; ++i) o->node_id[i] = i;
  } else {
    g.id.download(o->node_id, g.n);
  }
  g.w.download(o->compute_us, g.n);
  g.mem.download(o->memory_bytes, g.n);
  if (g.has_group) g.group.download(o->group, g.n);
  auto s = std::make_shared<std::vector<int32_t>>(g.m), d = std::make_shared<std::vector<int32_t>>(g.m);
  if (g.m) {
    download_bytes(ctx, s->data(), g.esrc.p, sizeof(int32_t) * g.m);
    download_bytes(ctx, d->data(), g.edst.p, sizeof(int32_t) * g.m);
  }
  g.bytes.download(o->edge_bytes, g.m);
  const bool has_group = g.has_group;
  const int32_t n = g.n, m = g.m;
  fin.push_back([o, s, d, dense_ids_out, has_group, n, m] {
    if (!has_group)
      for (int32_t i = 0; i < n; ++i) o->group[i] = -1;
    for (int32_t e = 0; e < m; ++e) {
      o->edge_src[e] = dense_ids_out ? (*s)[e] : o->node_id[(*s)[e]];
      o->edge_dst[e] = dense_ids_out ? (*d)[e] : o->node_id[(*d)[e]];
    }
  });
  return o;
}

dp_graph_out_t* graph_to_host(DevGraph& g, bool dense_ids_out) {
  Finalizers fin;
  dp_graph_out_t* o = graph_to_host_async(g, dense_ids_out, fin);
  sync(g.ctx);
  for (auto& x : fin) x();
  return o;
}

}  // namespace dpb

using namespace dpb;

extern "C" {

int dp_merge_is_safe(dp_ctx_t* ctx, const dp_graph_t* h, int64_t u, int64_t v, int32_t* out) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  int32_t ui = graph_index_of(g, u);
  if (ui < 0) fail(DP_E_UNKNOWN_NODE, "node %lld not in graph", (long long)u);
  int32_t vi = graph_index_of(g, v);
  if (vi < 0) fail(DP_E_UNKNOWN_NODE, "node %lld not in graph", (long long)v);
  DevBuf<int> direct(ctx, 1);
  int big = INT32_MAX;
  direct.upload(&big, 1);
  DP_LAUNCH(ctx, k_find_direct, 1, 256, 0, g.out_off.p, g.out_dst.p, g.out_eid.p, ui, vi, direct.p);
  int de = scalar_to_host(ctx, direct.p);
  if (de == INT32_MAX) fail(DP_E_NO_SUCH_EDGE, "no edge (%lld,%lld)", (long long)u, (long long)v);
  DevBuf<int32_t> visited(ctx, g.n), queue(ctx, (size_t)g.n + 1);
  visited.zero();
  int one = 1;
  DP_CUDA(cudaMemcpyAsync(visited.p + ui, &one, sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
  DP_CUDA(cudaMemcpyAsync(queue.p, &ui, sizeof(int32_t), cudaMemcpyHostToDevice, ctx->stream));
  DevBuf<int> counters(ctx, 3);
  int c0[3] = {1, 0, 0};
  counters.upload(c0, 3);
  DevBuf<unsigned> bar(ctx, 2);
  bar.zero();
  BfsArgs a{g.out_off.p, g.out_dst.p, g.out_eid.p, ui, vi, de, visited.p, queue.p, counters.p, bar.p};
  int per_sm = 0;
  DP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfs, 256, 0));
  int grid = std::max(1, std::min(per_sm * ctx->num_sms, std::max(1, g.n / 256)));
  grid = std::min(grid, 2 * ctx->num_sms);
  void* args[] = {&a};
  DP_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k_bfs), grid, 256, args, 0, ctx->stream));
  ++ctx->launches;
  int res[2];
  counters.download(res, 2);
  sync(ctx);
  *out = res[1] ? 0 : 1;
  DP_API_END
}

int dp_optimal_breakpoints(dp_ctx_t* ctx, const dp_graph_t* h, const int64_t* seq, int64_t len, dp_comm_t comm,
                           int32_t range, int64_t limit, dp_cluster_map_t** out) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  if (!order_valid_dev(g, seq, len)) fail(DP_E_INVALID_VALUE, "order is not a topological order of this graph");
  if (range < 1) fail(DP_E_INVALID_VALUE, "exploration range must be >= 1");
  if (limit <= 0) fail(DP_E_INVALID_VALUE, "cluster memory limit must be > 0");
  const int32_t n = g.n;
  if (n == 0) {
    *out = new_cluster_map(0, 0, 0);
    return DP_OK;
  }
  graph_costs(g, comm);
  DevBuf<int64_t> sid(ctx, n);
  sid.upload(seq, n);
  DevBuf<int32_t> sidx(ctx, n), pos(ctx, n);
  graph_ids_to_index(g, sid.p, sidx.p, n);
  DP_LAUNCH(ctx, k_scatter_pos, grid_for(n, 256), 256, 0, sidx.p, n, pos.p);
  Clusters cl;
  breakpoints_dev(g, sidx.p, pos.p, range, limit, cl);
  dp_cluster_map_t* m = new_cluster_map(n, cl.k, cl.k > 0 ? cl.k - 1 : 0);
  DevBuf<int32_t> byn(ctx, n);
  DP_LAUNCH(ctx, k_cl_by_node, grid_for(n, 256), 256, 0, cl.cl_of_pos.p, pos.p, n, byn.p);
  byn.download(m->node_cluster, n);
  cl.tot_w.download(m->total_compute, cl.k);
  cl.tot_mem.download(m->total_memory, cl.k);
  std::vector<int32_t> cuts = to_host(ctx, cl.cut_pos.p, (size_t)cl.k + 1);
  std::memcpy(m->members, seq, sizeof(int64_t) * n);  // clusters_from_cuts: members in sequence order
  for (int32_t c = 0; c <= cl.k; ++c) m->member_off[c] = cuts[c];
  for (int32_t c = 1; c < cl.k; ++c) m->breakpoints[c - 1] = cuts[c];
  *out = m;
  DP_API_END
}

int dp_build_coarse_graph(dp_ctx_t* ctx, const dp_graph_t* h, const int64_t* seq, int64_t len,
                          const int64_t* map_ids, const int32_t* map_cluster, int64_t map_count, int64_t n_clusters,
                          const int32_t* cluster_ids, const int64_t* member_off, const int64_t* members,
                          dp_graph_out_t** out) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  if (!order_valid_dev(g, seq, len)) fail(DP_E_INVALID_VALUE, "order is not a topological order of this graph");
  // ClusterMap consistency (fusion.cpp:178-203): input validation of the caller's map.
  std::unordered_map<int64_t, int32_t> map;
  map.reserve(static_cast<size_t>(map_count));
  for (int64_t i = 0; i < map_count; ++i) map[map_ids[i]] = map_cluster[i];
  if (static_cast<int64_t>(map.size()) != h->n_nodes)
    fail(DP_E_INVALID_CLUSTER_MAP, "cluster map does not cover the node set");
  std::unordered_set<int64_t> accounted;
  accounted.reserve(static_cast<size_t>(h->n_nodes));
  for (int64_t c = 0; c < n_clusters; ++c) {
    if (cluster_ids[c] != static_cast<int32_t>(c) || member_off[c + 1] == member_off[c])
      fail(DP_E_INVALID_CLUSTER_MAP, "cluster %lld is empty or misnumbered", (long long)c);
    for (int64_t q = member_off[c]; q < member_off[c + 1]; ++q) {
      auto it = map.find(members[q]);
      if (it == map.end() || it->second != cluster_ids[c] || !accounted.insert(members[q]).second)
        fail(DP_E_INVALID_CLUSTER_MAP, "node %lld is not mapped consistently", (long long)members[q]);
    }
  }
  for (int64_t i = 0; i < h->n_nodes; ++i)
    if (!accounted.count(h->node_id[i]))
      fail(DP_E_INVALID_CLUSTER_MAP, "node %lld missing from cluster map", (long long)h->node_id[i]);
  const int32_t n = g.n, k = static_cast<int32_t>(n_clusters);
  std::vector<int32_t> cl(n);
  for (int32_t i = 0; i < n; ++i) cl[i] = map[h->node_id[i]];
  DevBuf<int32_t> dcl(ctx, n > 0 ? n : 1);
  dcl.upload(cl.data(), n);
  DevBuf<int64_t> tw(ctx, k > 0 ? k : 1), tm(ctx, k > 0 ? k : 1);
  tw.zero();
  tm.zero();
  DP_LAUNCH(ctx, k_tot_from_map, grid_for(n, 256), 256, 0, dcl.p, g.w.p, g.mem.p, n, tw.p, tm.p);
  DevGraph coarse;
  coarse_graph_dev(g, dcl.p, k, tw.p, tm.p, coarse);
  *out = graph_to_host(coarse, true);
  DP_API_END
}

int dp_contract_colocation_groups(dp_ctx_t* ctx, const dp_graph_t* h, dp_contraction_t** out) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  Contraction c;
  contract_dev(g, c, true);
  graph_kahn(c.work, nullptr, nullptr, nullptr);
  if (c.work.processed != c.work.n) {
    std::vector<int64_t> wit = graph_cycle_witness(c.work);
    fail(DP_E_CYCLE_DETECTED, "co-location groups are inconsistent with a DAG: cycle: [%s]", join_ids(wit).c_str());
  }
  auto* r = halloc<dp_contraction_t>(1);
  r->contracted = graph_to_host(c.work, false);
  int32_t nc = c.work.n;
  r->member_off = halloc<int64_t>((int64_t)nc + 1);
  r->members = halloc<int64_t>(g.n);
  c.mem_off.download(r->member_off, (size_t)nc + 1);
  c.mem_ids.download(r->members, g.n);
  sync(ctx);
  *out = r;
  DP_API_END
}

int dp_fuse(dp_ctx_t* ctx, const dp_graph_t* h, dp_comm_t comm, int32_t range, int64_t limit,
            dp_fusion_result_t** out) {
  DP_API_BEGIN(ctx)
  DevGraph g;
  prepare_graph(g, ctx, h);
  require_valid_dev(g, h, true);
  FuseOut f;
  fuse_dev(g, comm, range, limit, f);
  auto* r = halloc<dp_fusion_result_t>(1);
  r->coarse = graph_to_host(f.coarse, true);
  r->map = fuse_map_to_host(g, f);
  *out = r;
  DP_API_END
}

}  // extern "C"
