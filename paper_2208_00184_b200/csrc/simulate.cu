// simulate.cu — makespan simulation of placements on the GPU, bit-exact with
// simulate() (simulator.cpp:56-252, /root/reference/proj/src).
//
// One warp simulates one placement; lane e owns engine e (3 per device: compute, send,
// receive; simulator.cpp:26-28).  Because every engine runs at most one task, the event
// heap of the reference collapses into the lanes' end times: the next event time is a
// warp min-reduction.  Engine queues are rings in HBM keyed like the reference's
// std::set<(ready, kind, id)> (simulator.cpp:32,51): ready times are enqueued in
// non-decreasing order, so an insert is an append plus a short backward shift inside
// the run of equal ready times.  try_start (simulator.cpp:148-179): an idle compute
// engine starts its head; a transfer starts when it heads both its send and receive
// queues and both engines are idle — one pass suffices because a start only makes its
// own engines busy.  Completions at one time are applied before the next try_start, so
// zero-duration tasks replay at the same `now` exactly like the reference.
//
// A batch of candidate placements is spread over persistent warps (one candidate per
// warp at a time).  A candidate whose ring would overflow is marked and re-run with
// 16x larger rings (up to the exact bound, every task queued once per engine).
#include <algorithm>

#include "simulate.cuh"

namespace dpb {
namespace {

struct QE {
  int64_t ready;
  int64_t sk;    // node id (compute) or edge index (transfer)
  int64_t meta;  // task (bits 0-31) | other engine (bits 32-47) | kind (bit 48)
};

__device__ __forceinline__ bool qe_less(const QE& a, const QE& b) {
  if (a.ready != b.ready) return a.ready < b.ready;
  const int64_t ka = (a.meta >> 48) & 1, kb = (b.meta >> 48) & 1;
  if (ka != kb) return ka < kb;
  if (a.sk != b.sk) return a.sk < b.sk;
  return static_cast<int32_t>(a.meta) < static_cast<int32_t>(b.meta);
}

constexpr int kWarpsPerBlock = 4;
constexpr int kStage = 128;

struct SimArgs {
  int32_t n, m, D, E, Q;
  const int32_t* out_off;
  const int32_t* out_dst;
  const int32_t* out_eid;
  const int32_t* edst;
  const int64_t* cost;
  const int64_t* w;
  const int64_t* id;  // null: dense ids
  const int32_t* indeg;
  const int32_t* node_dev;
  const uint8_t* cand;
  const int32_t* ncl;
  int32_t ncls;
  int64_t B;
  const int64_t* cand_list;  // optional subset of candidate indices (re-runs)
  int32_t* deps;
  uint8_t* devv;
  QE* queues;
  int64_t* tstart;
  int64_t* tend;
  int64_t* makespan;
  unsigned long long* next;
};

__global__ void __launch_bounds__(kWarpsPerBlock * 32) k_sim(SimArgs a) {
  __shared__ int32_t s_task[kWarpsPerBlock][kStage];
  __shared__ int16_t s_ea[kWarpsPerBlock][kStage];
  __shared__ int16_t s_eb[kWarpsPerBlock][kStage];
  __shared__ int64_t s_sk[kWarpsPerBlock][kStage];
  __shared__ int32_t s_head[kWarpsPerBlock][32];
  __shared__ int32_t s_go[kWarpsPerBlock][32];
  __shared__ uint8_t s_busy[kWarpsPerBlock][32];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wl;
  const int32_t n = a.n, E = a.E, Q = a.Q;
  int32_t* deps = a.deps + gw * n;
  uint8_t* devv = a.devv + gw * n;
  QE* myq = a.queues + (gw * E + (lane < E ? lane : 0)) * (int64_t)Q;
  const int type = lane % 3;
  int32_t* st_task = s_task[wl];
  int16_t* st_ea = s_ea[wl];
  int16_t* st_eb = s_eb[wl];
  int64_t* st_sk = s_sk[wl];

  for (;;) {
    unsigned long long bi = 0;
    if (lane == 0) bi = atomicAdd(a.next, 1ull);
    bi = __shfl_sync(0xffffffffu, bi, 0);
    if (static_cast<int64_t>(bi) >= a.B) break;
    const int64_t b = a.cand_list ? a.cand_list[bi] : static_cast<int64_t>(bi);
    for (int32_t v = lane; v < n; v += 32) {
      devv[v] = a.node_dev ? static_cast<uint8_t>(a.node_dev[v])
                           : a.cand[b * a.ncls + a.ncl[v]];
      deps[v] = a.indeg[v];
    }
    __syncwarp();
    bool busy = false, overflow = false;
    int32_t cur = -1, head = 0, tail = 0;
    int64_t endt = 0, now = 0;
    int ns = 0;

    auto flush = [&]() {
      __syncwarp();
      if (lane < E) {
        for (int i = 0; i < ns; ++i) {
          if (st_ea[i] != lane && st_eb[i] != lane) continue;
          const int32_t t = st_task[i];
          const bool xfer = t >= n;
          const int other = xfer ? (st_ea[i] == lane ? st_eb[i] : st_ea[i]) : 0;
          QE q{now, st_sk[i],
               static_cast<int64_t>(static_cast<uint32_t>(t)) | (static_cast<int64_t>(other) << 32) |
                   (static_cast<int64_t>(xfer ? 1 : 0) << 48)};
          if (tail - head >= Q) {
            overflow = true;
            continue;
          }
          int32_t pos = tail;
          while (pos > head) {
            const QE& pv = myq[(pos - 1) & (Q - 1)];
            if (pv.ready != now || !qe_less(q, pv)) break;
            myq[pos & (Q - 1)] = pv;
            --pos;
          }
          myq[pos & (Q - 1)] = q;
          ++tail;
        }
      }
      __syncwarp();
      ns = 0;
    };
    auto stage = [&](bool want, int32_t t, int ea, int eb, int64_t sk) {
      const unsigned bm = __ballot_sync(0xffffffffu, want);
      if (want) {
        const int at = ns + __popc(bm & ((1u << lane) - 1));
        st_task[at] = t;
        st_ea[at] = static_cast<int16_t>(ea);
        st_eb[at] = static_cast<int16_t>(eb);
        st_sk[at] = sk;
      }
      ns += __popc(bm);
      if (ns > kStage - 32) flush();
    };

    // sources are ready at t = 0 (simulator.cpp:181-183)
    for (int32_t v0 = 0; v0 < n; v0 += 32) {
      const int32_t v = v0 + lane;
      const bool src = v < n && a.indeg[v] == 0;
      stage(src, v, src ? 3 * devv[v] : 0, -1, src ? (a.id ? a.id[v] : v) : 0);
    }
    flush();

    for (;;) {
      // ---- try_start(now)
      const bool idle = lane < E && !busy && head != tail;
      QE h{0, 0, 0};
      if (idle) h = myq[head & (Q - 1)];
      const int32_t ht = idle ? static_cast<int32_t>(h.meta) : -1;
      s_head[wl][lane] = ht;
      s_busy[wl][lane] = busy ? 1 : 0;
      s_go[wl][lane] = -1;
      __syncwarp();
      if (idle && type == 0) {
        busy = true;
        cur = ht;
        endt = now + a.w[ht];
        ++head;
      } else if (idle && type == 1) {
        const int r = static_cast<int>((h.meta >> 32) & 0xffff);
        if (!s_busy[wl][r] && s_head[wl][r] == ht) {
          busy = true;
          cur = ht;
          endt = now + a.cost[ht - n];
          ++head;
          s_go[wl][r] = ht;
        }
      }
      __syncwarp();
      if (idle && type == 2 && s_go[wl][lane] == ht) {
        busy = true;
        cur = ht;
        endt = now + a.cost[ht - n];
        ++head;
      }
      if (a.tstart && busy && (idle) && cur == ht) {
        if (type != 2) {
          a.tstart[cur] = now;
          a.tend[cur] = endt;
        }
      }
      // ---- next completion time
      int64_t nx = busy ? endt : INT64_MAX;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t y = __shfl_xor_sync(0xffffffffu, nx, o);
        nx = y < nx ? y : nx;
      }
      if (nx == INT64_MAX) break;
      now = nx;
      // ---- completions at `now` (simulator.cpp:189-203)
      unsigned cm = __ballot_sync(0xffffffffu, busy && endt == now);
      const int32_t my_cur = cur;
      if (busy && endt == now) busy = false;
      while (cm) {
        const int c = __ffs(cm) - 1;
        cm &= cm - 1;
        if (c % 3 == 2) continue;  // receive side of a transfer: the send lane handles it
        const int32_t t = __shfl_sync(0xffffffffu, my_cur, c);
        if (t < n) {
          const int dv = devv[t];
          const int32_t kb = a.out_off[t], ke = a.out_off[t + 1];
          for (int32_t k0 = kb; k0 < ke; k0 += 32) {
            const int32_t k = k0 + lane;
            bool want = false;
            int32_t task = 0;
            int ea = 0, eb = -1;
            int64_t sk = 0;
            if (k < ke) {
              const int32_t x = a.out_dst[k];
              const int dx = devv[x];
              if (dx != dv) {
                const int32_t eid = a.out_eid[k];
                want = true;
                task = n + eid;
                ea = 3 * dv + 1;
                eb = 3 * dx + 2;
                sk = eid;
              } else {
                const int32_t d = deps[x] - 1;
                deps[x] = d;
                if (d == 0) {
                  want = true;
                  task = x;
                  ea = 3 * dx;
                  sk = a.id ? a.id[x] : x;
                }
              }
            }
            stage(want, task, ea, eb, sk);
          }
        } else {
          bool want = false;
          int32_t x = 0;
          if (lane == 0) {
            x = a.edst[t - n];
            const int32_t d = deps[x] - 1;
            deps[x] = d;
            want = d == 0;
          }
          x = __shfl_sync(0xffffffffu, x, 0);
          stage(want, x, 3 * devv[x], -1, a.id ? a.id[x] : x);
        }
        __syncwarp();
      }
      flush();
    }
    const unsigned ov = __ballot_sync(0xffffffffu, overflow);
    if (lane == 0) a.makespan[b] = ov ? -1 : now;
    __syncwarp();
  }
}

// Placements on more than 10 devices (E = 3D > 32 engines): the same event loop with the
// engines strided over the lanes (lane l owns engines l, l + 32, ...) and their state
// (busy, running task, end time, ring head/tail) in shared memory, one warp per CTA.
// Semantics are those of k_sim: engines are independent within a try_start pass except
// for the send -> receive handshake, which is resolved in the same two phases.
__global__ void __launch_bounds__(32) k_sim_wide(SimArgs a) {
  extern __shared__ __align__(16) unsigned char s_raw[];
  const int32_t n = a.n, E = a.E, Q = a.Q;
  int64_t* e_end = reinterpret_cast<int64_t*>(s_raw);
  int64_t* st_sk = e_end + E;
  int32_t* e_cur = reinterpret_cast<int32_t*>(st_sk + kStage);
  int32_t* e_head = e_cur + E;
  int32_t* e_tail = e_head + E;
  int32_t* e_ht = e_tail + E;  // head task of an idle engine with work, else -1
  int32_t* e_go = e_ht + E;
  int32_t* st_task = e_go + E;
  int32_t* st_ea = st_task + kStage;
  int32_t* st_eb = st_ea + kStage;
  uint8_t* e_busy = reinterpret_cast<uint8_t*>(st_eb + kStage);
  const int lane = threadIdx.x & 31;
  const int64_t gw = blockIdx.x;
  int32_t* deps = a.deps + gw * n;
  uint8_t* devv = a.devv + gw * n;
  QE* qbase = a.queues + gw * E * (int64_t)Q;

  for (;;) {
    unsigned long long bi = 0;
    if (lane == 0) bi = atomicAdd(a.next, 1ull);
    bi = __shfl_sync(0xffffffffu, bi, 0);
    if (static_cast<int64_t>(bi) >= a.B) break;
    const int64_t b = a.cand_list ? a.cand_list[bi] : static_cast<int64_t>(bi);
    for (int32_t v = lane; v < n; v += 32) {
      devv[v] = a.node_dev ? static_cast<uint8_t>(a.node_dev[v]) : a.cand[b * a.ncls + a.ncl[v]];
      deps[v] = a.indeg[v];
    }
    for (int e = lane; e < E; e += 32) {
      e_busy[e] = 0;
      e_cur[e] = -1;
      e_end[e] = 0;
      e_head[e] = 0;
      e_tail[e] = 0;
    }
    __syncwarp();
    bool overflow = false;
    int64_t now = 0;
    int ns = 0;

    auto push = [&](int e, int i) {
      QE* q_ = qbase + static_cast<int64_t>(e) * Q;
      const int32_t t = st_task[i];
      const bool xfer = t >= n;
      const int other = xfer ? (st_ea[i] == e ? st_eb[i] : st_ea[i]) : 0;
      QE q{now, st_sk[i],
           static_cast<int64_t>(static_cast<uint32_t>(t)) | (static_cast<int64_t>(other) << 32) |
               (static_cast<int64_t>(xfer ? 1 : 0) << 48)};
      const int32_t head = e_head[e];
      int32_t tail = e_tail[e];
      if (tail - head >= Q) {
        overflow = true;
        return;
      }
      int32_t pos = tail;
      while (pos > head) {
        const QE& pv = q_[(pos - 1) & (Q - 1)];
        if (pv.ready != now || !qe_less(q, pv)) break;
        q_[pos & (Q - 1)] = pv;
        --pos;
      }
      q_[pos & (Q - 1)] = q;
      e_tail[e] = tail + 1;
    };
    auto flush = [&]() {
      __syncwarp();
      for (int i = 0; i < ns; ++i) {  // engine e is owned by lane e % 32: no two lanes touch one ring
        if ((st_ea[i] & 31) == lane) push(st_ea[i], i);
        if (st_eb[i] >= 0 && (st_eb[i] & 31) == lane) push(st_eb[i], i);
      }
      __syncwarp();
      ns = 0;
    };
    auto stage = [&](bool want, int32_t t, int ea, int eb, int64_t sk) {
      const unsigned bm = __ballot_sync(0xffffffffu, want);
      if (want) {
        const int at = ns + __popc(bm & ((1u << lane) - 1));
        st_task[at] = t;
        st_ea[at] = ea;
        st_eb[at] = eb;
        st_sk[at] = sk;
      }
      ns += __popc(bm);
      if (ns > kStage - 32) flush();
    };

    for (int32_t v0 = 0; v0 < n; v0 += 32) {
      const int32_t v = v0 + lane;
      const bool src = v < n && a.indeg[v] == 0;
      stage(src, v, src ? 3 * devv[v] : 0, -1, src ? (a.id ? a.id[v] : v) : 0);
    }
    flush();

    for (;;) {
      // ---- try_start(now): phase 1 publishes every idle engine's head task
      for (int e = lane; e < E; e += 32) {
        const bool idle = !e_busy[e] && e_head[e] != e_tail[e];
        e_ht[e] = idle ? static_cast<int32_t>(qbase[static_cast<int64_t>(e) * Q + (e_head[e] & (Q - 1))].meta) : -1;
        e_go[e] = -1;
      }
      __syncwarp();
      // phase 2: compute engines start; send engines start iff their task heads an idle
      // receive engine (receive engines are only modified in phase 3)
      for (int e = lane; e < E; e += 32) {
        const int32_t ht = e_ht[e];
        if (ht < 0) continue;
        const int type = e % 3;
        if (type == 0) {
          e_busy[e] = 1;
          e_cur[e] = ht;
          e_end[e] = now + a.w[ht];
          e_head[e] += 1;
        } else if (type == 1) {
          const QE h = qbase[static_cast<int64_t>(e) * Q + (e_head[e] & (Q - 1))];
          const int r = static_cast<int>((h.meta >> 32) & 0xffff);
          if (!e_busy[r] && e_ht[r] == ht) {
            e_busy[e] = 1;
            e_cur[e] = ht;
            e_end[e] = now + a.cost[ht - n];
            e_head[e] += 1;
            e_go[r] = ht;
          }
        } else {
          continue;
        }
        if (a.tstart && e_busy[e] && e_cur[e] == ht) {
          a.tstart[ht] = now;
          a.tend[ht] = e_end[e];
        }
      }
      __syncwarp();
      for (int e = lane; e < E; e += 32) {
        const int32_t ht = e_ht[e];
        if (e % 3 == 2 && ht >= 0 && e_go[e] == ht) {
          e_busy[e] = 1;
          e_cur[e] = ht;
          e_end[e] = now + a.cost[ht - n];
          e_head[e] += 1;
        }
      }
      // ---- next completion time
      int64_t nx = INT64_MAX;
      for (int e = lane; e < E; e += 32)
        if (e_busy[e] && e_end[e] < nx) nx = e_end[e];
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const int64_t y = __shfl_xor_sync(0xffffffffu, nx, o);
        nx = y < nx ? y : nx;
      }
      if (nx == INT64_MAX) break;
      now = nx;
      // ---- completions at `now` (simulator.cpp:189-203), engines in index order
      for (int e0 = 0; e0 < E; e0 += 32) {
        const int e = e0 + lane;
        const bool fin = e < E && e_busy[e] && e_end[e] == now;
        unsigned cm = __ballot_sync(0xffffffffu, fin);
        const int32_t my_cur = e < E ? e_cur[e] : -1;
        __syncwarp();
        if (fin) e_busy[e] = 0;
        while (cm) {
          const int c = __ffs(cm) - 1;
          cm &= cm - 1;
          if ((e0 + c) % 3 == 2) continue;  // receive side of a transfer: the send engine handles it
          const int32_t t = __shfl_sync(0xffffffffu, my_cur, c);
          if (t < n) {
            const int dv = devv[t];
            const int32_t kb = a.out_off[t], ke = a.out_off[t + 1];
            for (int32_t k0 = kb; k0 < ke; k0 += 32) {
              const int32_t k = k0 + lane;
              bool want = false;
              int32_t task = 0;
              int ea = 0, eb = -1;
              int64_t sk = 0;
              if (k < ke) {
                const int32_t x = a.out_dst[k];
                const int dx = devv[x];
                if (dx != dv) {
                  const int32_t eid = a.out_eid[k];
                  want = true;
                  task = n + eid;
                  ea = 3 * dv + 1;
                  eb = 3 * dx + 2;
                  sk = eid;
                } else {
                  const int32_t d = deps[x] - 1;
                  deps[x] = d;
                  if (d == 0) {
                    want = true;
                    task = x;
                    ea = 3 * dx;
                    sk = a.id ? a.id[x] : x;
                  }
                }
              }
              stage(want, task, ea, eb, sk);
            }
          } else {
            bool want = false;
            int32_t x = 0;
            if (lane == 0) {
              x = a.edst[t - n];
              const int32_t d = deps[x] - 1;
              deps[x] = d;
              want = d == 0;
            }
            x = __shfl_sync(0xffffffffu, x, 0);
            stage(want, x, 3 * devv[x], -1, a.id ? a.id[x] : x);
          }
          __syncwarp();
        }
      }
      flush();
    }
    const unsigned ov = __ballot_sync(0xffffffffu, overflow);
    if (lane == 0) a.makespan[b] = ov ? -1 : now;
    __syncwarp();
  }
}

size_t wide_smem(int32_t E) {
  return static_cast<size_t>(E) * (8 + 5 * 4 + 1) + kStage * (8 + 3 * 4) + 16;
}

void run_sim(DevGraph& g, const SimInput& in, SimOutput& out, int32_t Q, int64_t count, const int64_t* cand_list) {
  dp_ctx* ctx = g.ctx;
  const int32_t n = g.n, m = g.m, D = in.D, E = 3 * D;
  // device positions are bytes (candidate rows, the per-warp device array)
  if (D > 256) fail(DP_E_UNSUPPORTED, "simulate supports at most 256 devices per placement (got %d)", D);
  if (n == 0 || count == 0) return;
  const bool wide = E > 32;
  const int wpb = wide ? 1 : kWarpsPerBlock;
  // Each warp's event loop is latency-bound (dependent HBM/L2 accesses per event), so
  // throughput comes from concurrency: up to 32 resident warps per SM.
  int64_t warps = std::min<int64_t>(count, static_cast<int64_t>(ctx->num_sms) * 32);
  // bound the per-warp workspace (rings + dependency counters) to ~16 GiB of HBM
  const int64_t per_warp = static_cast<int64_t>(E) * Q * sizeof(QE) + 5ll * n;
  while (warps > 1 && warps * per_warp > (16ll << 30)) warps /= 2;
  const int64_t blocks = (warps + wpb - 1) / wpb;
  warps = blocks * wpb;
  DevBuf<int32_t> indeg(ctx, n), deps(ctx, (size_t)warps * n);
  DevBuf<uint8_t> devv(ctx, (size_t)warps * n);
  DevBuf<QE> queues(ctx, (size_t)warps * E * Q);
  DevBuf<unsigned long long> next(ctx, 1);
  next.zero();
  std::vector<int32_t> hoff = to_host(ctx, g.in_off.p, (size_t)n + 1);
  std::vector<int32_t> hdeg(n);
  for (int32_t v = 0; v < n; ++v) hdeg[v] = hoff[v + 1] - hoff[v];
  indeg.upload(hdeg.data(), n);
  SimArgs a{};
  a.n = n;
  a.m = m;
  a.D = D;
  a.E = E;
  a.Q = Q;
  a.out_off = g.out_off.p;
  a.out_dst = g.out_dst.p;
  a.out_eid = g.out_eid.p;
  a.edst = g.edst.p;
  a.cost = g.cost.p;
  a.w = g.w.p;
  a.id = g.dense_ids ? nullptr : g.id.p;
  a.indeg = indeg.p;
  a.node_dev = in.node_dev;
  a.cand = in.cand;
  a.ncl = in.node_cluster;
  a.ncls = in.n_clusters;
  a.B = count;
  a.cand_list = cand_list;
  a.deps = deps.p;
  a.devv = devv.p;
  a.queues = queues.p;
  a.tstart = in.trace ? out.tstart.p : nullptr;
  a.tend = in.trace ? out.tend.p : nullptr;
  a.makespan = out.makespan.p;
  a.next = next.p;
  StageScope st(ctx, "simulate", 0.0);
  if (wide) {
    const size_t sm = wide_smem(E);
    if (sm > 48 * 1024) DP_CUDA(cudaFuncSetAttribute(k_sim_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    DP_LAUNCH(ctx, k_sim_wide, static_cast<int>(blocks), 32, sm, a);
  } else {
    DP_LAUNCH(ctx, k_sim, static_cast<int>(blocks), kWarpsPerBlock * 32, 0, a);
  }
}

}  // namespace

void simulate_dev(DevGraph& g, const SimInput& in, SimOutput& out, int32_t queue_cap) {
  dp_ctx* ctx = g.ctx;
  out.makespan.alloc(ctx, in.n_candidates > 0 ? in.n_candidates : 1);
  if (in.trace) {
    out.tstart.alloc(ctx, (size_t)g.n + g.m);
    out.tend.alloc(ctx, (size_t)g.n + g.m);
  }
  if (g.n == 0) {
    out.makespan.zero();
    return;
  }
  run_sim(g, in, out, queue_cap, in.n_candidates, nullptr);
}

int32_t sim_queue_cap() {
  // DP_SIM_QUEUE (diagnostic, power of two >= 1) shrinks the first-pass rings so tests can
  // force the overflow -> exact-capacity re-run path
  if (const char* e = getenv("DP_SIM_QUEUE")) {
    const int q = atoi(e);
    if (q >= 1 && (q & (q - 1)) == 0) return q;
  }
  return 1024;
}

void simulate_batch_dev(DevGraph& g, const SimInput& in, SimOutput& out) {
  dp_ctx* ctx = g.ctx;
  int32_t Q = sim_queue_cap();
  simulate_dev(g, in, out, Q);
  if (g.n == 0) return;
  for (;;) {  // re-run overflowed candidates with 16x larger rings, up to the exact bound
    std::vector<int64_t> ms = to_host(ctx, out.makespan.p, in.n_candidates);
    std::vector<int64_t> redo;
    for (int64_t b = 0; b < in.n_candidates; ++b)
      if (ms[b] < 0) redo.push_back(b);
    if (redo.empty()) return;
    Q = sim_queue_grow(g, Q);
    DevBuf<int64_t> list(ctx, redo.size());
    list.upload(redo.data(), redo.size());
    run_sim(g, in, out, Q, static_cast<int64_t>(redo.size()), list.p);
  }
}

int32_t sim_queue_grow(const DevGraph& g, int32_t Q) {
  int32_t exact = 1;
  while (exact < g.n + g.m + 1) exact <<= 1;  // every task is queued at most once per engine
  if (Q >= exact) fail(DP_E_CUDA, "simulate: engine queue overflow at the exact capacity");
  return static_cast<int32_t>(std::min<int64_t>(exact, static_cast<int64_t>(Q) * 16));
}

}  // namespace dpb
