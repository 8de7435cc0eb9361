// gen.cu — deterministic synthetic inputs (host code; input synthesis, not the measured
// path).  The layered recipe is SURVEY §8(d)'s "common recipe", which uses the
// reference generator's range mapping (generator.cpp:32-46): u(lo,hi) = lo + rng() %
// (hi-lo+1) over std::mt19937_64.
#include <algorithm>
#include <numeric>
#include <random>
#include <vector>

#include "abi_util.cuh"

extern "C" {

int dp_gen_layered(int64_t n, int64_t width, int64_t fan_lo, int64_t fan_hi, uint64_t seed, int64_t* node_id,
                   int64_t* compute_us, int64_t* memory_bytes, int64_t* edge_src, int64_t* edge_dst,
                   int64_t* edge_bytes, int64_t* n_edges) {
  if (n < 0 || width < 1 || fan_lo < 0 || fan_hi < fan_lo) {
    dpb::set_last_error(DP_E_ARGUMENT, "invalid generator parameters");
    return DP_E_ARGUMENT;
  }
  std::mt19937_64 rng(seed);
  auto u = [&rng](int64_t lo, int64_t hi) -> int64_t {
    if (hi <= lo) return lo;
    const uint64_t span = static_cast<uint64_t>(hi - lo) + 1;
    return lo + static_cast<int64_t>(rng() % span);
  };
  for (int64_t i = 0; i < n; ++i) {
    node_id[i] = i;
    compute_us[i] = u(100, 900);
    memory_bytes[i] = u(1 << 19, 3 << 19);
  }
  struct E {
    int64_t s, d, b;
  };
  std::vector<E> edges;
  edges.reserve(static_cast<size_t>(n * (fan_lo + fan_hi) / 2 + 16));
  std::vector<int64_t> pool;
  for (int64_t v = width; v < n; ++v) {
    const int64_t layer = v / width;
    const int64_t lo = (layer - 1) * width, hi = std::min(lo + width, n);
    const int64_t k = std::min<int64_t>(hi - lo, u(fan_lo, fan_hi));
    pool.resize(static_cast<size_t>(hi - lo));
    std::iota(pool.begin(), pool.end(), lo);
    for (int64_t t = 0; t < k; ++t) {
      const int64_t pick = u(0, static_cast<int64_t>(pool.size()) - 1);
      const int64_t src = pool[static_cast<size_t>(pick)];
      pool.erase(pool.begin() + pick);
      edges.push_back({src, v, u(1 << 15, 3 << 15)});
    }
  }
  std::sort(edges.begin(), edges.end(), [](const E& a, const E& b) { return a.s != b.s ? a.s < b.s : a.d < b.d; });
  for (size_t e = 0; e < edges.size(); ++e) {
    edge_src[e] = edges[e].s;
    edge_dst[e] = edges[e].d;
    edge_bytes[e] = edges[e].b;
  }
  *n_edges = static_cast<int64_t>(edges.size());
  return DP_OK;
}

}  // extern "C"
