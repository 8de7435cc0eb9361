// abi_util.cuh — exception-to-status wrapping shared by the extern "C" entry points.
#pragma once

#include <new>

#include "common.cuh"

namespace dpb {
// Resolves the stage events of a timed call when the entry point returns normally.
struct StageResolver {
  dp_ctx* ctx;
  bool ok = false;
  explicit StageResolver(dp_ctx* c) : ctx(c) {}
  ~StageResolver() {
    if (ok && ctx && ctx->timing) {
      try {
        stage_resolve(ctx);
      } catch (...) {
      }
    }
  }
};
}  // namespace dpb

#define DP_API_BEGIN(ctx)                                                    \
  ::dpb::StageResolver dp_stage_resolver_(ctx);                              \
  try {                                                                      \
    if (!(ctx)) ::dpb::fail(DP_E_ARGUMENT, "null dp_ctx_t");                 \
    ::dpb::ctx_activate(ctx);                                                \
    if ((ctx)->timing) ::dpb::stage_reset(ctx);

#define DP_API_END                                                           \
    if (!dp_stage_resolver_.ctx->pending.empty()) ::dpb::sync(dp_stage_resolver_.ctx); \
    dp_stage_resolver_.ok = true;                                            \
  }                                                                          \
  catch (const ::dpb::DpFail& f_) {                                          \
    if (dp_stage_resolver_.ctx) ::dpb::discard_pending(dp_stage_resolver_.ctx); \
    ::dpb::set_last_error(f_.code, f_.msg);                                  \
    return f_.code;                                                          \
  }                                                                          \
  catch (const std::bad_alloc&) {                                            \
    if (dp_stage_resolver_.ctx) ::dpb::discard_pending(dp_stage_resolver_.ctx); \
    ::dpb::set_last_error(DP_E_OUT_OF_MEMORY, "host allocation failed");     \
    return DP_E_OUT_OF_MEMORY;                                               \
  }                                                                          \
  return DP_OK;

namespace dpb {
struct DevGraph;
void require_valid_dev(DevGraph& g, const dp_graph_t* h, bool cycle_check);
void prepare_graph(DevGraph& g, dp_ctx* ctx, const dp_graph_t* h);
template <typename T>
struct DevBuf;
void levels_dev(DevGraph& g, dp_comm_t comm, DevBuf<int64_t>& t, DevBuf<int64_t>& b, DevBuf<int64_t>& c,
                bool chainlike = false);
void levels_dev_batch(DevGraph* const* gs, int count, dp_comm_t comm, DevBuf<int64_t>* const* t,
                      DevBuf<int64_t>* const* b, DevBuf<int64_t>* const* c);
void levels_dev_chainlike_batch(DevGraph* const* gs, int count, dp_comm_t comm, DevBuf<int64_t>* const* t,
                                DevBuf<int64_t>* const* b, DevBuf<int64_t>* const* c);
void seq_ids(DevGraph& g, const int32_t* seq, int32_t n, int64_t* out_dev);
bool order_valid_dev(DevGraph& g, const int64_t* seq, int64_t len);
void graph_index_checks(DevGraph& g, const dp_graph_t* h);
}  // namespace dpb
