// sort.cu — device radix sort, scans and reduce-by-key for the graph build (CSR/CSC,
// id index, coarse-edge aggregation), hand-written for sm_100a with stream-ordered
// temporary storage.
//
// Radix sort: stable LSD over 8-bit digits, three launches per digit:
//   k_rs_hist     one 4,096-item tile per CTA (8 warps x 16 rounds of 32 consecutive
//                 items): per-tile digit histogram in shared memory -> hist[digit][tile]
//   scan          exclusive scan of the digit-major histogram = every (digit, tile)'s
//                 first output slot (the same scan as exclusive_scan_i32 below)
//   k_rs_scatter  re-reads the tile; a key's rank among its digit inside the tile is
//                 (same-digit keys in earlier warps) + (in earlier rounds of its warp) +
//                 (lower lanes of its round, __match_any_sync); the tile is reordered by
//                 digit in shared memory and written out in tile order, so each digit's
//                 run goes to consecutive global slots (coalesced stores).
// Items are read in order and ranked in order, so equal digits keep their input order
// (stability, which CSR/CSC construction relies on: graph_index.cpp:36-41).
// Scans: per-tile reduce -> scan of the tile sums (recursively) -> per-tile scan + offset.
#include "common.cuh"

namespace dpb {

int bits_for(uint64_t max_value) {
  int b = 0;
  while (b < 64 && (max_value >> b) != 0) ++b;
  return b < 1 ? 1 : b;
}

namespace {

constexpr int kRsWarps = 8;
constexpr int kRsRounds = 16;
constexpr int kRsTile = kRsWarps * kRsRounds * 32;  // 4,096 items per CTA
constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4,096 items per CTA

template <typename K>
__device__ __forceinline__ uint32_t digit_of(K k, int shift) {
  return static_cast<uint32_t>(k >> shift) & 0xffu;
}

template <typename K>
__global__ void __launch_bounds__(kRsWarps * 32) k_rs_hist(const K* keys, int64_t count, int shift, int32_t ntiles,
                                                           int32_t* hist) {
  __shared__ int32_t h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kRsTile;
  for (int i = threadIdx.x; i < kRsTile; i += blockDim.x) {
    const int64_t k = t0 + i;
    if (k < count) atomicAdd(&h[digit_of(keys[k], shift)], 1);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += blockDim.x) hist[static_cast<int64_t>(d) * ntiles + blockIdx.x] = h[d];
}

template <typename K, typename V>
__global__ void __launch_bounds__(kRsWarps * 32) k_rs_scatter(const K* kin, const V* vin, K* kout, V* vout,
                                                              int64_t count, int shift, int32_t ntiles,
                                                              const int32_t* offs) {
  __shared__ int32_t wcnt[kRsWarps][256];  // per-warp digit counts; then offsets inside the tile
  __shared__ int32_t base[256];            // global slot of the tile's first key of each digit
  __shared__ int32_t tstart[256];          // tile position of the tile's first key of each digit
  extern __shared__ unsigned char rs_stage[];  // the tile's keys and values in digit order
  K* sk = reinterpret_cast<K*>(rs_stage);
  V* sv = reinterpret_cast<V*>(sk + kRsTile);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < kRsWarps * 256; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  for (int d = threadIdx.x; d < 256; d += blockDim.x) base[d] = offs[static_cast<int64_t>(d) * ntiles + blockIdx.x];
  __syncthreads();
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kRsTile;
  const int64_t w0 = t0 + static_cast<int64_t>(warp) * kRsRounds * 32;
  K key[kRsRounds];
  V val[kRsRounds];
  int32_t rank[kRsRounds];
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    const int64_t k = w0 + r * 32 + lane;
    const bool ok = k < count;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    rank[r] = -1;
    if (ok) {
      key[r] = kin[k];
      val[r] = vin[k];
      const uint32_t d = digit_of(key[r], shift);
      const unsigned peers = __match_any_sync(act, d);
      const int32_t before = wcnt[warp][d];
      rank[r] = before + __popc(peers & ((1u << lane) - 1u));
      __syncwarp(act);
      if (lane == __ffs(peers) - 1) wcnt[warp][d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();
  // digit d's keys occupy tile positions [tstart[d], tstart[d] + total(d)); warp w's part of
  // them starts at tstart[d] + (digit-d keys of warps before w)
  if (threadIdx.x < 256) {
    const int d = threadIdx.x;
    int32_t s = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const int32_t c = wcnt[w][d];
      wcnt[w][d] = s;
      s += c;
    }
    tstart[d] = s;  // total for now; scanned below
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the 256 digit totals (8 per lane)
    int32_t v[8], sum = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      v[q] = tstart[lane * 8 + q];
      sum += v[q];
    }
    int32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    int32_t run = inc - sum;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      tstart[lane * 8 + q] = run;
      run += v[q];
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRsRounds; ++r) {
    if (rank[r] >= 0) {
      const uint32_t d = digit_of(key[r], shift);
      const int32_t at = tstart[d] + wcnt[warp][d] + rank[r];
      sk[at] = key[r];
      sv[at] = val[r];
    }
  }
  __syncthreads();
  // write out in tile order: consecutive positions of one digit go to consecutive slots
  const int32_t nt = static_cast<int32_t>(count - t0 < kRsTile ? count - t0 : kRsTile);
  for (int32_t i = threadIdx.x; i < nt; i += blockDim.x) {
    const K kk = sk[i];
    const uint32_t d = digit_of(kk, shift);
    const int64_t at = static_cast<int64_t>(base[d]) + (i - tstart[d]);
    kout[at] = kk;
    vout[at] = sv[i];
  }
}

// ---- scans (T = int32_t / int64_t); a CTA scans kScanTile items
template <typename T>
__device__ __forceinline__ T block_exclusive(T x, T* sw, T* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sw[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    T s = lane < nw ? sw[lane] : T(0);
    T si = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = __shfl_up_sync(0xffffffffu, si, o);
      if (lane >= o) si += y;
    }
    if (lane < nw) sw[lane] = si - s;
    if (lane == nw - 1) *total = si;
  }
  __syncthreads();
  const T r = sw[warp] + inc - x;
  __syncthreads();
  return r;
}

template <typename T>
__global__ void __launch_bounds__(kScanThreads) k_tile_sums(const T* in, int64_t count, T* sums) {
  __shared__ T sw[32];
  __shared__ T total;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanItems;
  T s = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q)
    if (t0 + q < count) s += in[t0 + q];
  block_exclusive(s, sw, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// out = exclusive (or inclusive) scan of the tile + offs[tile] (offs may be null)
template <typename T, bool INCLUSIVE>
__global__ void __launch_bounds__(kScanThreads) k_tile_scan(const T* in, int64_t count, const T* offs, T* out) {
  __shared__ T sw[32];
  __shared__ T total;
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * kScanTile + static_cast<int64_t>(threadIdx.x) * kScanItems;
  T v[kScanItems];
  T s = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    v[q] = t0 + q < count ? in[t0 + q] : T(0);
    s += v[q];
  }
  T run = block_exclusive(s, sw, &total) + (offs ? offs[blockIdx.x] : T(0));
#pragma unroll
  for (int q = 0; q < kScanItems; ++q) {
    if (INCLUSIVE) run += v[q];
    if (t0 + q < count) out[t0 + q] = run;
    if (!INCLUSIVE) run += v[q];
  }
}

template <typename T, bool INCLUSIVE>
void scan_impl(dp_ctx* ctx, const T* in, T* out, int64_t count) {
  if (count <= 0) return;
  const int64_t tiles = (count + kScanTile - 1) / kScanTile;
  if (tiles == 1) {
    k_tile_scan<T, INCLUSIVE><<<1, kScanThreads, 0, ctx->stream>>>(in, count, nullptr, out);
    ++ctx->launches;
    DP_CUDA(cudaGetLastError());
    return;
  }
  DevBuf<T> sums(ctx, tiles), offs(ctx, tiles);
  k_tile_sums<T><<<static_cast<unsigned>(tiles), kScanThreads, 0, ctx->stream>>>(in, count, sums.p);
  ++ctx->launches;
  DP_CUDA(cudaGetLastError());
  scan_impl<T, false>(ctx, sums.p, offs.p, tiles);
  k_tile_scan<T, INCLUSIVE><<<static_cast<unsigned>(tiles), kScanThreads, 0, ctx->stream>>>(in, count, offs.p, out);
  ++ctx->launches;
  DP_CUDA(cudaGetLastError());
}

template <typename K, typename V>
void radix_sort(dp_ctx* ctx, const K* ki, K* ko, const V* vi, V* vo, int64_t count, int begin_bit, int end_bit) {
  if (count <= 0) return;
  if (count > (int64_t(1) << 31) - kRsTile)
    fail(DP_E_UNSUPPORTED, "radix sort of %lld items exceeds the 2^31 limit", static_cast<long long>(count));
  const int passes = end_bit > begin_bit ? (end_bit - begin_bit + 7) / 8 : 0;
  if (passes == 0) {
    DP_CUDA(cudaMemcpyAsync(ko, ki, sizeof(K) * count, cudaMemcpyDeviceToDevice, ctx->stream));
    DP_CUDA(cudaMemcpyAsync(vo, vi, sizeof(V) * count, cudaMemcpyDeviceToDevice, ctx->stream));
    return;
  }
  const int32_t tiles = static_cast<int32_t>((count + kRsTile - 1) / kRsTile);
  DevBuf<int32_t> hist(ctx, static_cast<size_t>(256) * tiles), offs(ctx, static_cast<size_t>(256) * tiles);
  DevBuf<K> tk;
  DevBuf<V> tv;
  if (passes > 1) {
    tk.alloc(ctx, count);
    tv.alloc(ctx, count);
  }
  const size_t stage = static_cast<size_t>(kRsTile) * (sizeof(K) + sizeof(V));
  static bool attr = false;  // per (K, V) instantiation
  if (!attr) {
    DP_CUDA(cudaFuncSetAttribute(k_rs_scatter<K, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(stage)));
    attr = true;
  }
  // ping-pong so that the last pass writes ko / vo and the inputs are never written
  const K* sk = ki;
  const V* sv = vi;
  for (int p = 0; p < passes; ++p) {
    const bool to_out = ((passes - 1 - p) & 1) == 0;
    K* dk = to_out ? ko : tk.p;
    V* dv = to_out ? vo : tv.p;
    const int shift = begin_bit + 8 * p;
    k_rs_hist<K><<<tiles, kRsWarps * 32, 0, ctx->stream>>>(sk, count, shift, tiles, hist.p);
    ++ctx->launches;
    DP_CUDA(cudaGetLastError());
    scan_impl<int32_t, false>(ctx, hist.p, offs.p, static_cast<int64_t>(256) * tiles);
    k_rs_scatter<K, V><<<tiles, kRsWarps * 32, stage, ctx->stream>>>(sk, sv, dk, dv, count, shift, tiles, offs.p);
    ++ctx->launches;
    DP_CUDA(cudaGetLastError());
    sk = dk;
    sv = dv;
  }
}

// ---- reduce by key over sorted keys (runs of equal keys are contiguous)
__global__ void k_run_flags(const uint64_t* keys, int64_t count, int64_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// run r = runid[i] - 1 at its first item i: key and start; at its last item: the sum from
// the inclusive prefix of the values
__global__ void k_run_emit(const uint64_t* keys, const int64_t* runid, const int64_t* pre, int64_t count,
                           uint64_t* uniq, int64_t* start, int64_t* sums, int64_t* num_runs) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = runid[i] - 1;
    if (i == 0 || keys[i] != keys[i - 1]) {
      uniq[r] = keys[i];
      start[r] = i;
    }
    if (i == count - 1) *num_runs = r + 1;
  }
}
__global__ void k_run_sums(const int64_t* runid, const int64_t* pre, const int64_t* start, int64_t count,
                           int64_t* sums) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = runid[i] - 1;
    if (i == count - 1 || runid[i + 1] != runid[i]) {
      const int64_t s = start[r];
      sums[r] = pre[i] - (s > 0 ? pre[s - 1] : 0);
    }
  }
}

}  // namespace

void sort_pairs_u32(dp_ctx* ctx, const uint32_t* ki, uint32_t* ko, const int32_t* vi, int32_t* vo,
                    int64_t count, int end_bit) {
  radix_sort<uint32_t, int32_t>(ctx, ki, ko, vi, vo, count, 0, end_bit);
}

void sort_pairs_u64(dp_ctx* ctx, const uint64_t* ki, uint64_t* ko, const int32_t* vi, int32_t* vo,
                    int64_t count, int begin_bit, int end_bit) {
  radix_sort<uint64_t, int32_t>(ctx, ki, ko, vi, vo, count, begin_bit, end_bit);
}

void sort_pairs_u64_i64(dp_ctx* ctx, const uint64_t* ki, uint64_t* ko, const int64_t* vi,
                        int64_t* vo, int64_t count, int end_bit) {
  radix_sort<uint64_t, int64_t>(ctx, ki, ko, vi, vo, count, 0, end_bit);
}

void exclusive_scan_i32(dp_ctx* ctx, const int32_t* in, int32_t* out, int64_t count) {
  scan_impl<int32_t, false>(ctx, in, out, count);
}

void exclusive_scan_i64(dp_ctx* ctx, const int64_t* in, int64_t* out, int64_t count) {
  scan_impl<int64_t, false>(ctx, in, out, count);
}

void inclusive_scan_i64(dp_ctx* ctx, const int64_t* in, int64_t* out, int64_t count) {
  scan_impl<int64_t, true>(ctx, in, out, count);
}

void reduce_by_key_u64(dp_ctx* ctx, const uint64_t* keys, uint64_t* uniq, const int64_t* vals,
                       int64_t* sums, int64_t* num_runs, int64_t count) {
  if (count <= 0) {
    DP_CUDA(cudaMemsetAsync(num_runs, 0, sizeof(int64_t), ctx->stream));
    return;
  }
  DevBuf<int64_t> flag(ctx, count), runid(ctx, count), pre(ctx, count), start(ctx, count);
  DP_LAUNCH(ctx, k_run_flags, grid_for(count, 256), 256, 0, keys, count, flag.p);
  scan_impl<int64_t, true>(ctx, flag.p, runid.p, count);
  scan_impl<int64_t, true>(ctx, vals, pre.p, count);
  DP_LAUNCH(ctx, k_run_emit, grid_for(count, 256), 256, 0, keys, runid.p, pre.p, count, uniq, start.p, sums,
            num_runs);
  DP_LAUNCH(ctx, k_run_sums, grid_for(count, 256), 256, 0, runid.p, pre.p, start.p, count, sums);
}

}  // namespace dpb
