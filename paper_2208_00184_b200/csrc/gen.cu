// gen.cu — deterministic synthetic inputs (host code; input synthesis, not the measured
// path).  The layered recipe is SURVEY §8(d)'s "common recipe", which uses the
// reference generator's range mapping (generator.cpp:32-46): u(lo,hi) = lo + rng() %
// (hi-lo+1) over std::mt19937_64.
#include <algorithm>
#include <numeric>
#include <random>
#include <vector>

#include "abi_util.cuh"

namespace {

// k picks without replacement from the pool lo..hi-1, each u(0, |pool|-1) and erased
// from the pool (the recipe's std::vector::erase), without materialising the pool: the
// pick-th remaining entry is found by skipping the offsets already taken (k <= 6).
template <typename U, typename F>
void pick_distinct(U& u, int64_t lo, int64_t hi, int64_t k, std::vector<int64_t>& taken, F emit) {
  taken.clear();
  for (int64_t t = 0; t < k; ++t) {
    int64_t x = u(0, hi - lo - t - 1);
    size_t j = 0;
    for (; j < taken.size() && taken[j] <= x; ++j) ++x;
    taken.insert(taken.begin() + static_cast<std::ptrdiff_t>(j), x);
    emit(lo + x);
  }
}

}  // namespace

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
  std::vector<int64_t> taken;
  for (int64_t v = width; v < n; ++v) {
    const int64_t layer = v / width;
    const int64_t lo = (layer - 1) * width, hi = std::min(lo + width, n);
    const int64_t k = std::min<int64_t>(hi - lo, u(fan_lo, fan_hi));
    pick_distinct(u, lo, hi, k, taken, [&](int64_t src) { edges.push_back({src, v, u(1 << 15, 3 << 15)}); });
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

extern "C" {

// Config #5 candidate family: candidate 0 = base (cluster -> device
// position); candidate k > 0 = base with max(1, n_c/100) moves, each cluster rk() % n_c
// -> device rk() % D, rk = std::mt19937_64(k).  out: [count x n_c], candidates first..first+count-1.
int dp_gen_candidates(const uint8_t* base, int64_t n_clusters, int32_t D, int64_t first, int64_t count, uint8_t* out) {
  if (n_clusters < 1 || D < 1 || D > 255 || first < 0 || count < 0) {
    dpb::set_last_error(DP_E_ARGUMENT, "invalid candidate parameters");
    return DP_E_ARGUMENT;
  }
  const int64_t moves = std::max<int64_t>(1, n_clusters / 100);
  for (int64_t i = 0; i < count; ++i) {
    const int64_t k = first + i;
    uint8_t* row = out + i * n_clusters;
    std::copy(base, base + n_clusters, row);
    if (k == 0) continue;
    std::mt19937_64 rk(static_cast<uint64_t>(k));
    for (int64_t t = 0; t < moves; ++t) {
      const uint64_t c = rk() % static_cast<uint64_t>(n_clusters);
      const uint64_t d = rk() % static_cast<uint64_t>(D);
      row[c] = static_cast<uint8_t>(d);
    }
  }
  return DP_OK;
}

}  // extern "C"

extern "C" {

// Config #2: GNMT-like, 8 chains x T steps, node id = l*T + t.  Node costs
// by the common recipe in id order; then, l outer / t inner: chain edge (l,t)->(l,t+1),
// layer edge (l,t)->(l+1,t), and for l == 7, t % 16 == 0, t+1 < T the attention edge
// (7,t)->(0,t+1); bytes u(2^15, 3*2^15) in that emission order; edges sorted (src,dst).
int dp_gen_gnmt(int64_t chains, int64_t T, uint64_t seed, int64_t* node_id, int64_t* compute_us,
                int64_t* memory_bytes, int64_t* edge_src, int64_t* edge_dst, int64_t* edge_bytes, int64_t* n_edges) {
  std::mt19937_64 rng(seed);
  auto u = [&rng](int64_t lo, int64_t hi) -> int64_t {
    if (hi <= lo) return lo;
    return lo + static_cast<int64_t>(rng() % (static_cast<uint64_t>(hi - lo) + 1));
  };
  const int64_t n = chains * T;
  for (int64_t i = 0; i < n; ++i) {
    node_id[i] = i;
    compute_us[i] = u(100, 900);
    memory_bytes[i] = u(1 << 19, 3 << 19);
  }
  struct E {
    int64_t s, d, b;
  };
  std::vector<E> edges;
  for (int64_t l = 0; l < chains; ++l) {
    for (int64_t t = 0; t < T; ++t) {
      const int64_t id = l * T + t;
      if (t + 1 < T) edges.push_back({id, id + 1, u(1 << 15, 3 << 15)});
      if (l + 1 < chains) edges.push_back({id, id + T, u(1 << 15, 3 << 15)});
      if (l == chains - 1 && t % 16 == 0 && t + 1 < T) edges.push_back({id, t + 1, u(1 << 15, 3 << 15)});
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

// Config #3: BERT-like — the common layered recipe plus a skip edge
// (v - skip*W -> v) for every v >= skip*W with (v / W) % skip == 0, its bytes drawn
// right after v's fan-in picks; edges sorted (src,dst).
int dp_gen_bert(int64_t n, int64_t width, int64_t skip, uint64_t seed, int64_t* node_id, int64_t* compute_us,
                int64_t* memory_bytes, int64_t* edge_src, int64_t* edge_dst, int64_t* edge_bytes, int64_t* n_edges) {
  std::mt19937_64 rng(seed);
  auto u = [&rng](int64_t lo, int64_t hi) -> int64_t {
    if (hi <= lo) return lo;
    return lo + static_cast<int64_t>(rng() % (static_cast<uint64_t>(hi - lo) + 1));
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
  std::vector<int64_t> taken;
  for (int64_t v = width; v < n; ++v) {
    const int64_t layer = v / width;
    const int64_t lo = (layer - 1) * width, hi = std::min(lo + width, n);
    const int64_t k = std::min<int64_t>(hi - lo, u(2, 6));
    pick_distinct(u, lo, hi, k, taken, [&](int64_t src) { edges.push_back({src, v, u(1 << 15, 3 << 15)}); });
    if (v >= skip * width && (v / width) % skip == 0) edges.push_back({v - skip * width, v, u(1 << 15, 3 << 15)});
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
