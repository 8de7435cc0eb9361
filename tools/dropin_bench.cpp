// dropin_bench.cpp — times dagplace::evaluate_pipeline (pipeline.cpp:27-111) on config #4
// (SURVEY §8(d) layered recipe, 1M ops, 8 devices) through the C++ API, compiled against
// the UNCHANGED reference headers.  The same source links either to the B200 drop-in
// (libdagplace_core_b200.so -> build/dropin_bench_b200) or to the reference's own objects
// (oracle/_ref -> build/dropin_bench_ref), so the two print comparable lines:
//
//   build/dropin_bench_b200 [n] [width] [reps]
//
// Per call: wall time of evaluate_pipeline (AoS graph in, PipelineReport out, both
// simulations), the report's generation_wall_us (the reference's own window timer),
// the two makespans and a checksum of the chosen placement.
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <optional>
#include <random>
#include <string>
#include <vector>

#include "dagplace/pipeline.hpp"

using namespace dagplace;

static ComputationGraph layered(int64_t n, int64_t width, uint64_t seed) {
  std::mt19937_64 rng(seed);
  auto u = [&rng](int64_t lo, int64_t hi) -> int64_t {
    return hi <= lo ? lo : lo + static_cast<int64_t>(rng() % (static_cast<uint64_t>(hi - lo) + 1));
  };
  ComputationGraph g;
  g.nodes.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    g.nodes[i].id = i;
    g.nodes[i].name = "op" + std::to_string(i);
    g.nodes[i].compute_us = u(100, 900);
    g.nodes[i].memory_bytes = u(1 << 19, 3 << 19);
  }
  std::vector<int64_t> taken;
  for (int64_t v = width; v < n; ++v) {
    const int64_t lo = (v / width - 1) * width, hi = std::min(lo + width, n);
    const int64_t k = std::min<int64_t>(hi - lo, u(2, 6));
    taken.clear();
    for (int64_t t = 0; t < k; ++t) {
      int64_t x = u(0, hi - lo - t - 1);
      size_t j = 0;
      for (; j < taken.size() && taken[j] <= x; ++j) ++x;
      taken.insert(taken.begin() + static_cast<std::ptrdiff_t>(j), x);
      g.edges.push_back(TensorEdge{lo + x, v, u(1 << 15, 3 << 15)});
    }
  }
  std::sort(g.edges.begin(), g.edges.end(), [](const TensorEdge& a, const TensorEdge& b) {
    return a.src != b.src ? a.src < b.src : a.dst < b.dst;
  });
  return g;
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 1000000;
  const int64_t w = argc > 2 ? std::atoll(argv[2]) : 1024;
  const int reps = argc > 3 ? std::atoi(argv[3]) : 3;
  ComputationGraph g = layered(n, w, 12345);
  Bytes total = 0;
  for (const auto& nd : g.nodes) total += nd.memory_bytes;
  std::vector<DeviceSpec> devs;
  for (int d = 0; d < 8; ++d) devs.push_back(DeviceSpec{d, total / 8 + total / 32});
  const CommModel comm{0.001, 10.0};
  PipelineConfig cfg;
  for (int r = 0; r < reps; ++r) {
    const auto t0 = std::chrono::steady_clock::now();
    PipelineReport rep = evaluate_pipeline(g, std::nullopt, devs, comm, cfg);
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    uint64_t h = 1469598103934665603ull;
    for (const auto& nd : g.nodes) h = (h ^ static_cast<uint64_t>(rep.chosen_placement.assignment.at(nd.id))) * 1099511628211ull;
    std::printf("{\"call\": %d, \"n\": %lld, \"m\": %zu, \"evaluate_pipeline_s\": %.3f, \"generation_wall_us\": %lld, "
                "\"coarse_nodes\": %lld, \"order_makespan\": %lld, \"adjust_makespan\": %lld, "
                "\"chosen_trace\": %zu, \"chosen_hash\": \"%016llx\"}\n",
                r, static_cast<long long>(n), g.edges.size(), s, static_cast<long long>(rep.generation_wall_us),
                static_cast<long long>(rep.coarse_nodes), static_cast<long long>(rep.order_place.makespan_us),
                static_cast<long long>(rep.adjusting.makespan_us), rep.chosen_simulation.trace.size(),
                static_cast<unsigned long long>(h));
    std::fflush(stdout);
  }
  return 0;
}
