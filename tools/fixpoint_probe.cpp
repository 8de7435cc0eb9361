// Prototype (host, diagnostic only): how many rounds does the parallel characterisation
// of the CPD peel need at config #4?  sigma is the peel order iff sigma is topological and
// sigma = preorder(T(sigma)), T(sigma) = forest whose parent(v) is v's last-emitted
// predecessor, children (and roots) visited by rank (cpath desc, id asc)
// (ordering.cpp:40-77, 98-114).  Prints rounds and per-round convergence.
//
//   g++ -O2 -std=c++17 tools/fixpoint_probe.cpp -o /tmp/fp && /tmp/fp 1000000 1024
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

using i64 = int64_t;

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1000000;
  const int W = argc > 2 ? atoi(argv[2]) : 1024;
  const int start = argc > 3 ? atoi(argv[3]) : 0;  // 0: index order, 1: m_topo-like BFS by id
  std::mt19937_64 rng(12345);
  auto u = [&](i64 lo, i64 hi) { return lo + (i64)(rng() % (uint64_t)(hi - lo + 1)); };
  std::vector<i64> w(n), mem(n);
  for (int i = 0; i < n; ++i) { w[i] = u(100, 900); mem[i] = u(1 << 19, 3 << 19); }
  std::vector<std::pair<int, int>> E;
  std::vector<i64> eb;
  std::vector<int> pool;
  for (int v = W; v < n; ++v) {
    int l = v / W, lo = (l - 1) * W, hi = std::min(lo + W, n);
    pool.clear();
    for (int x = lo; x < hi; ++x) pool.push_back(x);
    int k = (int)u(2, 6);
    for (int t = 0; t < k && !pool.empty(); ++t) {
      int pick = (int)u(0, (i64)pool.size() - 1);
      E.push_back({pool[pick], v});
      pool.erase(pool.begin() + pick);
      eb.push_back(u(1 << 15, 3 << 15));
    }
  }
  std::vector<int> ord(E.size());
  for (size_t i = 0; i < ord.size(); ++i) ord[i] = (int)i;
  std::sort(ord.begin(), ord.end(), [&](int a, int b) { return E[a] < E[b]; });
  const int m = (int)E.size();
  std::vector<int> es(m), ed(m);
  std::vector<i64> ec(m);
  for (int i = 0; i < m; ++i) {
    es[i] = E[ord[i]].first; ed[i] = E[ord[i]].second;
    ec[i] = std::llround(0.001 * (double)eb[ord[i]] + 10.0);
  }
  std::vector<int> ooff(n + 1, 0), ioff(n + 1, 0);
  for (int i = 0; i < m; ++i) { ooff[es[i] + 1]++; ioff[ed[i] + 1]++; }
  for (int i = 0; i < n; ++i) { ooff[i + 1] += ooff[i]; ioff[i + 1] += ioff[i]; }
  std::vector<int> oe(m), ie(m), oc(ooff.begin(), ooff.end() - 1), ic(ioff.begin(), ioff.end() - 1);
  for (int i = 0; i < m; ++i) { oe[oc[es[i]]++] = i; ie[ic[ed[i]]++] = i; }
  // levels (index order is topological)
  std::vector<i64> tl(n, 0), bl(n, 0), cp(n);
  for (int v = 0; v < n; ++v)
    for (int k = ioff[v]; k < ioff[v + 1]; ++k) { int e = ie[k]; tl[v] = std::max(tl[v], tl[es[e]] + w[es[e]] + ec[e]); }
  for (int v = n - 1; v >= 0; --v) {
    i64 b = 0;
    for (int k = ooff[v]; k < ooff[v + 1]; ++k) { int e = oe[k]; b = std::max(b, bl[ed[e]] + ec[e]); }
    bl[v] = b + w[v];
  }
  for (int v = 0; v < n; ++v) cp[v] = tl[v] + bl[v];
  auto better = [&](int a, int b) { return cp[a] != cp[b] ? cp[a] > cp[b] : a < b; };
  // reference peel
  std::vector<int> indeg(n), seq;
  seq.reserve(n);
  std::vector<int> stack, src;
  for (int v = 0; v < n; ++v) { indeg[v] = ioff[v + 1] - ioff[v]; if (!indeg[v]) src.push_back(v); }
  std::sort(src.begin(), src.end(), better);
  for (int i = (int)src.size() - 1; i >= 0; --i) stack.push_back(src[i]);
  std::vector<int> fr;
  while (!stack.empty()) {
    int v = stack.back(); stack.pop_back(); seq.push_back(v);
    fr.clear();
    for (int k = ooff[v]; k < ooff[v + 1]; ++k) { int c = ed[oe[k]]; if (--indeg[c] == 0) fr.push_back(c); }
    std::sort(fr.begin(), fr.end(), better);
    for (int i = (int)fr.size() - 1; i >= 0; --i) stack.push_back(fr[i]);
  }
  // out rows sorted by child rank
  std::vector<int> rowc(m);
  for (int v = 0; v < n; ++v) {
    for (int k = ooff[v]; k < ooff[v + 1]; ++k) rowc[k] = ed[oe[k]];
    std::sort(rowc.begin() + ooff[v], rowc.begin() + ooff[v + 1], better);
  }
  // fixed point
  std::vector<int> sig(n), pos(n), par(n), nsig(n);
  if (start == 0) for (int i = 0; i < n; ++i) sig[i] = i;
  for (int i = 0; i < n; ++i) pos[sig[i]] = i;
  int depth = 0;
  { std::vector<int> lv(n, 0); for (int v = 0; v < n; ++v) for (int k = ioff[v]; k < ioff[v + 1]; ++k) lv[v] = std::max(lv[v], lv[es[ie[k]]] + 1); for (int v = 0; v < n; ++v) depth = std::max(depth, lv[v]); }
  printf("n=%d m=%d W=%d depth=%d\n", n, m, W, depth + 1);
  std::vector<int> st;
  for (int round = 1; round < 5000; ++round) {
    for (int v = 0; v < n; ++v) {
      int best = -1, bp = -1;
      for (int k = ioff[v]; k < ioff[v + 1]; ++k) { int p = es[ie[k]]; if (pos[p] > bp) { bp = pos[p]; best = p; } }
      par[v] = best;
    }
    // preorder via explicit stack over rank-sorted rows
    st.clear();
    for (int i = (int)src.size() - 1; i >= 0; --i) st.push_back(src[i]);
    int q = 0;
    while (!st.empty()) {
      int v = st.back(); st.pop_back(); nsig[q++] = v;
      for (int k = ooff[v + 1] - 1; k >= ooff[v]; --k) { int c = rowc[k]; if (par[c] == v) st.push_back(c); }
    }
    int changed = 0, prefix = 0, prefix_final = 0;
    while (prefix < n && nsig[prefix] == sig[prefix]) ++prefix;
    while (prefix_final < n && nsig[prefix_final] == seq[prefix_final]) ++prefix_final;
    int parchg = 0;
    for (int i = 0; i < n; ++i) changed += nsig[i] != sig[i];
    sig.swap(nsig);
    std::vector<int> opos = pos;
    for (int i = 0; i < n; ++i) pos[sig[i]] = i;
    for (int v = 0; v < n; ++v) { int best = -1, bp = -1; for (int k = ioff[v]; k < ioff[v + 1]; ++k) { int p = es[ie[k]]; if (pos[p] > bp) { bp = pos[p]; best = p; } } parchg += best != par[v]; }
    if (round <= 10 || round % 20 == 0 || changed == 0)
      printf("round %d: changed %d, stable prefix %d, prefix==peel %d, parents changing next %d\n", round, changed, prefix, prefix_final, parchg);
    if (changed == 0) {
      printf("converged after %d rounds; equals peel: %s\n", round, sig == seq ? "yes" : "NO");
      break;
    }
  }
  return 0;
}
