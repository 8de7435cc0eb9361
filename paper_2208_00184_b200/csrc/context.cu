#include <cstdlib>
// context.cu — dp_ctx lifecycle, thread-local last error, stage timing.
#include <cstring>

#include "common.cuh"

namespace dpb {

namespace {
thread_local std::string g_err_msg;
thread_local int g_err_code = 0;
}  // namespace

const char* kind_name(int code) {
  static const char* names[] = {"OK",
                                "CycleDetected",
                                "DanglingEdge",
                                "DuplicateId",
                                "DuplicateEdge",
                                "InvalidValue",
                                "ZeroComputeTime",
                                "NoSuchEdge",
                                "NodeExceedsClusterLimit",
                                "GroupExceedsClusterLimit",
                                "InfeasiblePartition",
                                "InvalidClusterMap",
                                "InsufficientSamples",
                                "UnknownNode",
                                "NodeUniverseMismatch",
                                "UnplacedNode",
                                "InstanceTooLarge",
                                "InstanceInfeasible",
                                "UnreachableTargetCcr",
                                "ParseError"};
  if (code >= 0 && code <= 19) return names[code];
  switch (code) {
    case DP_E_CUDA: return "CudaError";
    case DP_E_ARGUMENT: return "InvalidArgument";
    case DP_E_OUT_OF_MEMORY: return "OutOfMemory";
    case DP_E_UNSUPPORTED: return "Unsupported";
    default: return "UnknownError";
  }
}

void fail(int code, const char* fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw DpFail{code, buf};
}

// DagError::what() == "<Kind>: <message>" (error.hpp:37-41).
void set_last_error(int code, const std::string& body) {
  g_err_code = code;
  g_err_msg = std::string(kind_name(code)) + ": " + body;
}

void ctx_activate(dp_ctx* ctx) { DP_CUDA(cudaSetDevice(ctx->device)); }

void stage_reset(dp_ctx* ctx) {
  for (auto& s : ctx->stages) ctx->event_pool.push_back(s);
  ctx->stages.clear();
  ctx->stage_ms.clear();
}

size_t stage_begin(dp_ctx* ctx, const char* name, double bytes) {
  Stage s;
  if (!ctx->event_pool.empty()) {
    s = ctx->event_pool.back();
    ctx->event_pool.pop_back();
  } else {
    DP_CUDA(cudaEventCreate(&s.a));
    DP_CUDA(cudaEventCreate(&s.b));
  }
  s.name = name;
  s.bytes = bytes;
  DP_CUDA(cudaEventRecord(s.a, ctx->stream));
  ctx->stages.push_back(s);
  return ctx->stages.size() - 1;
}

void stage_end(dp_ctx* ctx, size_t idx) {
  if (idx >= ctx->stages.size()) return;
  DP_CUDA(cudaEventRecord(ctx->stages[idx].b, ctx->stream));
}

void download_bytes(dp_ctx* ctx, void* host, const void* dev, size_t bytes) {
  if (!bytes) return;
  const size_t need = (bytes + 255) & ~static_cast<size_t>(255);
  if (ctx->pin_off + need > ctx->pin_cap) {
    sync(ctx);  // completes (and empties) the pending copies
    // grow only for a single copy larger than the arena: growing to everything pending
    // (hundreds of MB per context) costs cudaFreeHost / cudaHostAlloc, which stall every
    // stream, for no measured gain
    if (need > ctx->pin_cap) {
      if (ctx->pin) cudaFreeHost(ctx->pin);
      ctx->pin = nullptr;
      ctx->pin_cap = 0;
      const size_t cap = std::max<size_t>(need, 1 << 20);
      DP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&ctx->pin), cap, cudaHostAllocDefault));
      ctx->pin_cap = cap;
    }
  }
  DP_CUDA(cudaMemcpyAsync(ctx->pin + ctx->pin_off, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream));
  ctx->pending.push_back({host, ctx->pin_off, bytes});
  ctx->pin_off += need;
}

void sync(dp_ctx* ctx) {
  ++ctx->sync_count;
  if (ctx->sync_ev) {
    DP_CUDA(cudaEventRecord(ctx->sync_ev, ctx->stream));
    DP_CUDA(cudaEventSynchronize(ctx->sync_ev));
  } else {
    DP_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  for (const auto& c : ctx->pending) std::memcpy(c.dst, ctx->pin + c.off, c.bytes);
  ctx->pending.clear();
  ctx->pin_off = 0;
}

void discard_pending(dp_ctx* ctx) {
  ctx->pending.clear();
}

void stage_resolve(dp_ctx* ctx) {
  ctx->stage_ms.clear();
  sync(ctx);
  for (auto& s : ctx->stages) {
    float ms = 0;
    DP_CUDA(cudaEventElapsedTime(&ms, s.a, s.b));
    ctx->stage_ms.push_back(ms);
  }
}

}  // namespace dpb

using namespace dpb;

extern "C" {

const char* dp_last_error_message(void) { return g_err_msg.c_str(); }
int32_t dp_last_error_code(void) { return g_err_code; }

int dp_ctx_create(int device, void* stream, dp_ctx_t** out) {
  try {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count <= device || device < 0) {
      fail(DP_E_CUDA, "no CUDA device %d available (%s); libdagplace_b200 has no CPU fallback", device,
           e == cudaSuccess ? "device count" : cudaGetErrorString(e));
    }
    cudaDeviceProp prop;
    DP_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) {
      fail(DP_E_CUDA, "device %d is sm_%d%d; this build targets sm_100a (B200)", device, prop.major, prop.minor);
    }
    DP_CUDA(cudaSetDevice(device));
    dp_ctx* ctx = new dp_ctx;
    ctx->device = device;
    ctx->stream = static_cast<cudaStream_t>(stream);
    ctx->num_sms = prop.multiProcessorCount;
    if (getenv("DP_SPIN_SYNC") == nullptr)
      DP_CUDA(cudaEventCreateWithFlags(&ctx->sync_ev, cudaEventBlockingSync | cudaEventDisableTiming));
    {
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      if (cudaMemPoolCreate(&ctx->pool, &props) == cudaSuccess) {
        uint64_t threshold = UINT64_MAX;  // keep freed blocks cached for the next call
        cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &threshold);
      } else {
        ctx->pool = nullptr;
        cudaGetLastError();
      }
    }
    *out = ctx;
    return DP_OK;
  } catch (const DpFail& f) {
    set_last_error(f.code, f.msg);
    return f.code;
  }
}

void dp_ctx_destroy(dp_ctx_t* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  ctx->pending.clear();
  if (ctx->pin) cudaFreeHost(ctx->pin);
  if (ctx->sync_ev) cudaEventDestroy(ctx->sync_ev);
  if (ctx->copy_stream) {
    cudaStreamSynchronize(ctx->copy_stream);
    cudaStreamDestroy(ctx->copy_stream);
  }
  if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
  for (auto& s : ctx->stages) ctx->event_pool.push_back(s);
  for (auto& s : ctx->event_pool) {
    cudaEventDestroy(s.a);
    cudaEventDestroy(s.b);
  }
  delete ctx;
}

int dp_ctx_set_stream(dp_ctx_t* ctx, void* stream) {
  ctx->stream = static_cast<cudaStream_t>(stream);
  return DP_OK;
}

int dp_ctx_synchronize(dp_ctx_t* ctx) {
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e == cudaSuccess) {
    for (const auto& c : ctx->pending) std::memcpy(c.dst, ctx->pin + c.off, c.bytes);
    ctx->pending.clear();
    ctx->pin_off = 0;
  }
  if (e != cudaSuccess) {
    set_last_error(DP_E_CUDA, cudaGetErrorString(e));
    return DP_E_CUDA;
  }
  return DP_OK;
}

int64_t dp_ctx_launch_count(const dp_ctx_t* ctx) { return ctx->launches; }

int dp_ctx_peel_stats(const dp_ctx_t* ctx, int64_t* out5) {
  for (int i = 0; i < 5; ++i) out5[i] = ctx->tree_stats[i];
  return DP_OK;
}

int dp_ctx_enable_stage_timing(dp_ctx_t* ctx, int32_t on) {
  ctx->timing = on != 0;
  return DP_OK;
}
int32_t dp_ctx_stage_count(const dp_ctx_t* ctx) { return static_cast<int32_t>(ctx->stage_ms.size()); }
const char* dp_ctx_stage_name(const dp_ctx_t* ctx, int32_t i) {
  return (i >= 0 && i < (int32_t)ctx->stages.size()) ? ctx->stages[i].name : "";
}
double dp_ctx_stage_ms(const dp_ctx_t* ctx, int32_t i) {
  return (i >= 0 && i < (int32_t)ctx->stage_ms.size()) ? ctx->stage_ms[i] : 0.0;
}
double dp_ctx_stage_bytes(const dp_ctx_t* ctx, int32_t i) {
  return (i >= 0 && i < (int32_t)ctx->stages.size()) ? ctx->stages[i].bytes : 0.0;
}

}  // extern "C"
