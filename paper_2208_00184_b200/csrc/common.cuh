// common.cuh — context, stream-ordered buffers, errors, launch accounting, grid barrier.
#pragma once
#include <functional>
#include <memory>

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "../../include/dagplace_b200.h"

namespace dpb {

// ------------------------------------------------------------------ errors
// Internal failures travel as DpFail and are converted to a status code at the C-ABI
// boundary (abi.cu); no exception ever crosses extern "C".
struct DpFail {
  int code;
  std::string msg;  // message body without the "<Kind>: " prefix
};

const char* kind_name(int code);
[[noreturn]] void fail(int code, const char* fmt, ...);
void set_last_error(int code, const std::string& body);

#define DP_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess) ::dpb::fail(DP_E_CUDA, "%s (%s:%d)", cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                             \
  } while (0)

// ------------------------------------------------------------------ context
struct Stage {
  const char* name;
  cudaEvent_t a, b;
  double bytes;
};

}  // namespace dpb

struct dp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int64_t launches = 0;
  int64_t tree_stats[5] = {0, 0, 0, 0, 0};  // tree-peel outcomes (DP_DEBUG_FIXPOINT)
  int64_t sync_count = 0;                    // host round trips (diagnostics)
  bool timing = false;
  std::vector<dpb::Stage> stages;      // events of the last timed call
  std::vector<dpb::Stage> event_pool;  // recycled events
  size_t event_next = 0;
  std::vector<double> stage_ms;        // resolved durations
  // Device->host results are staged through a pinned arena and copied to their
  // destination at the next dpb::sync: a D2H copy into pageable memory would block the
  // calling thread until the stream drains (and serialise concurrent contexts).
  struct PendingCopy {
    void* dst;
    size_t off, bytes;
  };
  char* pin = nullptr;
  size_t pin_cap = 0, pin_off = 0;
  std::vector<PendingCopy> pending;
  // Host waits block on this event (cudaEventBlockingSync) instead of spinning: many
  // contexts driven by more host threads than cores must not burn the cores they share.
  cudaEvent_t sync_ev = nullptr;
  // A private stream-ordered pool per context: with the device's shared default pool, a
  // block freed on one context's stream could be handed to another context's stream
  // with an inserted cross-stream dependency, coupling independent replicas.
  cudaMemPool_t pool = nullptr;
  // Host->device copies of batched calls run here (created on first use), so the first
  // graphs' validation overlaps the later graphs' uploads.
  cudaStream_t copy_stream = nullptr;
};

namespace dpb {

void ctx_activate(dp_ctx* ctx);

// Stage timing: CUDA events recorded on the context stream around each stage.
void stage_reset(dp_ctx* ctx);
size_t stage_begin(dp_ctx* ctx, const char* name, double bytes);
void stage_end(dp_ctx* ctx, size_t idx);
void stage_resolve(dp_ctx* ctx);

struct StageScope {
  dp_ctx* ctx;
  size_t idx = 0;
  bool on;
  StageScope(dp_ctx* c, const char* name, double bytes = 0.0) : ctx(c), on(c->timing) {
    if (on) idx = stage_begin(ctx, name, bytes);
  }
  ~StageScope() {
    if (on) stage_end(ctx, idx);
  }
};

#define DP_LAUNCH(ctx, kernel, grid, block, smem, ...)                         \
  do {                                                                         \
    if ((grid) > 0) {                                                          \
      kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);         \
      ++(ctx)->launches;                                                       \
      DP_CUDA(cudaGetLastError());                                             \
    }                                                                          \
  } while (0)

inline int grid_for(int64_t n, int block, int max_blocks = 148 * 16) {
  int64_t g = (n + block - 1) / block;
  if (g > max_blocks) g = max_blocks;
  return static_cast<int>(g);
}

// ------------------------------------------------------------------ device buffers
// Stream-ordered allocations (cudaMallocAsync on the context stream); the pool keeps
// freed blocks cached so repeated pipeline calls do not hit the driver.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  dp_ctx* ctx = nullptr;
  DevBuf() = default;
  DevBuf(dp_ctx* c, size_t count) { alloc(c, count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), ctx(o.ctx) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; ctx = o.ctx;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(dp_ctx* c, size_t count) {
    release();
    ctx = c;
    n = count;
    if (count) {
      cudaError_t e = c->pool ? cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), count * sizeof(T), c->pool,
                                                        c->stream)
                              : cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), c->stream);
      if (e != cudaSuccess) {
        p = nullptr;
        fail(DP_E_OUT_OF_MEMORY, "device allocation of %zu bytes failed: %s", count * sizeof(T),
             cudaGetErrorString(e));
      }
    }
  }
  void ensure(dp_ctx* c, size_t count) {
    if (count > n || !p) alloc(c, count < 1 ? 1 : count);
  }
  void release() {
    if (p) cudaFreeAsync(p, ctx->stream);
    p = nullptr;
    n = 0;
  }
  void zero() {
    if (p && n) DP_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), ctx->stream));
  }
  void fill_bytes(int v) {
    if (p && n) DP_CUDA(cudaMemsetAsync(p, v, n * sizeof(T), ctx->stream));
  }
  void upload(const T* host, size_t count) {
    if (count) DP_CUDA(cudaMemcpyAsync(p, host, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
  }
  void download(T* host, size_t count) const;
  T* get() const { return p; }
};

// Stream-ordered D2H copy of `bytes` into `host` through the pinned arena; `host` is
// valid after the next sync(ctx).
void download_bytes(dp_ctx* ctx, void* host, const void* dev, size_t bytes);
// Waits for the context stream and completes the pending D2H copies.
void sync(dp_ctx* ctx);
// Host-side steps to run after the next sync(ctx), in order (results assembled from
// downloads that several graphs enqueue before one sync).
using Finalizers = std::vector<std::function<void()>>;
// Drops pending copies (error paths: their destinations may be gone).
void discard_pending(dp_ctx* ctx);

template <typename T>
void DevBuf<T>::download(T* host, size_t count) const {
  if (count) download_bytes(ctx, host, p, count * sizeof(T));
}

template <typename T>
inline std::vector<T> to_host(dp_ctx* ctx, const T* dev, size_t count) {
  std::vector<T> h(count);
  if (count) {
    download_bytes(ctx, h.data(), dev, count * sizeof(T));
    sync(ctx);
  }
  return h;
}
template <typename T>
inline T scalar_to_host(dp_ctx* ctx, const T* dev) {
  T v{};
  download_bytes(ctx, &v, dev, sizeof(T));
  sync(ctx);
  return v;
}

// ------------------------------------------------------------------ device helpers
constexpr int64_t kNever = INT64_MAX;

// comm_time (graph.cpp:200-204): fp64 k*bytes then + b, each correctly rounded (no
// FMA contraction), then llround (half away from zero).
__device__ __forceinline__ int64_t comm_cost_dev(int64_t bytes, double k, double b) {
  double t = __dmul_rn(k, static_cast<double>(bytes));
  t = __dadd_rn(t, b);
  return static_cast<int64_t>(llround(t));
}

__device__ __forceinline__ unsigned long long as_ull(int64_t v) {
  return static_cast<unsigned long long>(v);
}

__device__ __forceinline__ void atomic_max_i64(int64_t* p, int64_t v) {
  atomicMax(reinterpret_cast<long long*>(p), static_cast<long long>(v));
}
__device__ __forceinline__ void atomic_min_i64(int64_t* p, int64_t v) {
  atomicMin(reinterpret_cast<long long*>(p), static_cast<long long>(v));
}
__device__ __forceinline__ void atomic_add_i64(int64_t* p, int64_t v) {
  atomicAdd(reinterpret_cast<unsigned long long*>(p), static_cast<unsigned long long>(v));
}

// Warp-aggregated append: returns the slot for this lane (all `active` lanes call).
__device__ __forceinline__ int warp_append(int* counter, bool want) {
  unsigned mask = __ballot_sync(__activemask(), want);
  if (!want) return -1;
  int leader = __ffs(mask) - 1;
  int lane = threadIdx.x & 31;
  int base = 0;
  if (lane == leader) base = atomicAdd(counter, __popc(mask));
  base = __shfl_sync(mask, base, leader);
  return base + __popc(mask & ((1u << lane) - 1));
}

// Sense-reversing grid barrier for persistent kernels launched cooperatively (every CTA
// resident).  `bar[0]` = arrival count, `bar[1]` = generation.  When `snap_src` is set,
// the last CTA to arrive copies *snap_src into *snap_dst before releasing the others, so
// every CTA reads one consistent value produced before the barrier (e.g. the end of the
// next frontier) even though fast CTAs start appending right after it.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks, const int* snap_src = nullptr,
                                             int* snap_dst = nullptr) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      if (snap_src) *((volatile int*)snap_dst) = *((volatile const int*)snap_src);
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
        __nanosleep(32);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// ------------------------------------------------------------------ CUB wrappers (sort.cu)
// Stable LSD radix sorts (keys ascending over [begin_bit, end_bit)).
void sort_pairs_u32(dp_ctx* ctx, const uint32_t* keys_in, uint32_t* keys_out, const int32_t* vals_in,
                    int32_t* vals_out, int64_t count, int end_bit);
void sort_pairs_u64(dp_ctx* ctx, const uint64_t* keys_in, uint64_t* keys_out, const int32_t* vals_in,
                    int32_t* vals_out, int64_t count, int begin_bit, int end_bit);
void sort_pairs_u64_i64(dp_ctx* ctx, const uint64_t* keys_in, uint64_t* keys_out,
                        const int64_t* vals_in, int64_t* vals_out, int64_t count, int end_bit);
void exclusive_scan_i32(dp_ctx* ctx, const int32_t* in, int32_t* out, int64_t count);
void exclusive_scan_i64(dp_ctx* ctx, const int64_t* in, int64_t* out, int64_t count);
void inclusive_scan_i64(dp_ctx* ctx, const int64_t* in, int64_t* out, int64_t count);
// Sum runs of equal keys (sorted input); *num_runs written on device.
void reduce_by_key_u64(dp_ctx* ctx, const uint64_t* keys, uint64_t* unique_out, const int64_t* vals,
                       int64_t* sums_out, int64_t* num_runs, int64_t count);

int bits_for(uint64_t max_value);

}  // namespace dpb
