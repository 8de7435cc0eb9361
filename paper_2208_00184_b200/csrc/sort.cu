// sort.cu — device radix sort / scan / reduce-by-key primitives (CUB onesweep, compiled
// into this library for sm_100a) with stream-ordered temporary storage.
#include <cub/cub.cuh>

#include "common.cuh"

namespace dpb {

namespace {
struct Temp {
  DevBuf<unsigned char> buf;
};
}  // namespace

int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

void sort_pairs_u32(dp_ctx* ctx, const uint32_t* ki, uint32_t* ko, const int32_t* vi, int32_t* vo,
                    int64_t count, int end_bit) {
  if (count <= 0) return;
  size_t bytes = 0;
  DP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ki, ko, vi, vo, count, 0, end_bit, ctx->stream));
  Temp t;
  t.buf.alloc(ctx, bytes);
  DP_CUDA(cub::DeviceRadixSort::SortPairs(t.buf.p, bytes, ki, ko, vi, vo, count, 0, end_bit, ctx->stream));
  ctx->launches += (end_bit + 7) / 8 + 1;
}

void sort_pairs_u64(dp_ctx* ctx, const uint64_t* ki, uint64_t* ko, const int32_t* vi, int32_t* vo,
                    int64_t count, int begin_bit, int end_bit) {
  if (count <= 0) return;
  size_t bytes = 0;
  DP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ki, ko, vi, vo, count, begin_bit, end_bit,
                                          ctx->stream));
  Temp t;
  t.buf.alloc(ctx, bytes);
  DP_CUDA(cub::DeviceRadixSort::SortPairs(t.buf.p, bytes, ki, ko, vi, vo, count, begin_bit, end_bit,
                                          ctx->stream));
  ctx->launches += (end_bit - begin_bit + 7) / 8 + 1;
}

void sort_pairs_u64_i64(dp_ctx* ctx, const uint64_t* ki, uint64_t* ko, const int64_t* vi,
                        int64_t* vo, int64_t count, int end_bit) {
  if (count <= 0) return;
  size_t bytes = 0;
  DP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, ki, ko, vi, vo, count, 0, end_bit, ctx->stream));
  Temp t;
  t.buf.alloc(ctx, bytes);
  DP_CUDA(cub::DeviceRadixSort::SortPairs(t.buf.p, bytes, ki, ko, vi, vo, count, 0, end_bit, ctx->stream));
  ctx->launches += (end_bit + 7) / 8 + 1;
}

void exclusive_scan_i32(dp_ctx* ctx, const int32_t* in, int32_t* out, int64_t count) {
  if (count <= 0) return;
  size_t bytes = 0;
  DP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, count, ctx->stream));
  Temp t;
  t.buf.alloc(ctx, bytes);
  DP_CUDA(cub::DeviceScan::ExclusiveSum(t.buf.p, bytes, in, out, count, ctx->stream));
  ctx->launches += 2;
}

void exclusive_scan_i64(dp_ctx* ctx, const int64_t* in, int64_t* out, int64_t count) {
  if (count <= 0) return;
  size_t bytes = 0;
  DP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, count, ctx->stream));
  Temp t;
  t.buf.alloc(ctx, bytes);
  DP_CUDA(cub::DeviceScan::ExclusiveSum(t.buf.p, bytes, in, out, count, ctx->stream));
  ctx->launches += 2;
}

void inclusive_scan_i64(dp_ctx* ctx, const int64_t* in, int64_t* out, int64_t count) {
  if (count <= 0) return;
  size_t bytes = 0;
  DP_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, count, ctx->stream));
  Temp t;
  t.buf.alloc(ctx, bytes);
  DP_CUDA(cub::DeviceScan::InclusiveSum(t.buf.p, bytes, in, out, count, ctx->stream));
  ctx->launches += 2;
}

void reduce_by_key_u64(dp_ctx* ctx, const uint64_t* keys, uint64_t* uniq, const int64_t* vals,
                       int64_t* sums, int64_t* num_runs, int64_t count) {
  if (count <= 0) {
    DP_CUDA(cudaMemsetAsync(num_runs, 0, sizeof(int64_t), ctx->stream));
    return;
  }
  size_t bytes = 0;
  DP_CUDA(cub::DeviceReduce::ReduceByKey(nullptr, bytes, keys, uniq, vals, sums, num_runs,
                                         cuda::std::plus<int64_t>{}, count, ctx->stream));
  Temp t;
  t.buf.alloc(ctx, bytes);
  DP_CUDA(cub::DeviceReduce::ReduceByKey(t.buf.p, bytes, keys, uniq, vals, sums, num_runs,
                                         cuda::std::plus<int64_t>{}, count, ctx->stream));
  ctx->launches += 2;
}

}  // namespace dpb
