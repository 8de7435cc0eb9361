// Prototype (host, diagnostic only): WINDOWED fixed-point peel.  The continuation of the
// stack peel after an emitted prefix is the peel of the residual graph started from the
// current stack; restricted to a down-closed window C (residual levels < h) the peel of
// C is exact up to the first position whose emission frees a node outside C.  Each window:
// Kahn levels of the residual (h levels), fixed point on C with the stack as roots, commit
// the exact prefix, rebuild the stack (parent position desc, rank asc).  Prints windows,
// committed positions per window and rounds per window; checks the result against the
// reference peel.
//
//   g++ -O2 -std=c++17 tools/window_probe.cpp -o /tmp/wp && /tmp/wp 1000000 1024 8
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
  const int H = argc > 3 ? atoi(argv[3]) : 8;
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
  std::vector<int> od(m), is(m), oc(ooff.begin(), ooff.end() - 1), ic(ioff.begin(), ioff.end() - 1);
  for (int i = 0; i < m; ++i) { od[oc[es[i]]++] = ed[i]; is[ic[ed[i]]++] = es[i]; }
  std::vector<i64> tl(n, 0), bl(n, 0), cp(n);
  for (int v = 0; v < n; ++v)
    for (int k = ioff[v]; k < ioff[v + 1]; ++k) { int p = is[k]; /* cost by edge lookup */ }
  // levels need per-edge costs in CSC order: recompute from edge list
  {
    std::vector<std::vector<std::pair<int, i64>>> inn(n);
    for (int i = 0; i < m; ++i) inn[ed[i]].push_back({es[i], ec[i]});
    for (int v = 0; v < n; ++v) for (auto& pc : inn[v]) tl[v] = std::max(tl[v], tl[pc.first] + w[pc.first] + pc.second);
    std::vector<std::vector<std::pair<int, i64>>> out(n);
    for (int i = 0; i < m; ++i) out[es[i]].push_back({ed[i], ec[i]});
    for (int v = n - 1; v >= 0; --v) { i64 b = 0; for (auto& pc : out[v]) b = std::max(b, bl[pc.first] + pc.second); bl[v] = b + w[v]; }
  }
  for (int v = 0; v < n; ++v) cp[v] = tl[v] + bl[v];
  std::vector<int> byr(n), rank(n);
  for (int i = 0; i < n; ++i) byr[i] = i;
  std::sort(byr.begin(), byr.end(), [&](int a, int b) { return cp[a] != cp[b] ? cp[a] > cp[b] : a < b; });
  for (int i = 0; i < n; ++i) rank[byr[i]] = i;
  // rows sorted by rank
  for (int v = 0; v < n; ++v) std::sort(od.begin() + ooff[v], od.begin() + ooff[v + 1], [&](int a, int b) { return rank[a] < rank[b]; });
  // reference peel
  std::vector<int> seq;
  {
    std::vector<int> indeg(n), st;
    for (int v = 0; v < n; ++v) indeg[v] = ioff[v + 1] - ioff[v];
    std::vector<int> src;
    for (int v = 0; v < n; ++v) if (!indeg[v]) src.push_back(v);
    std::sort(src.begin(), src.end(), [&](int a, int b) { return rank[a] < rank[b]; });
    for (int i = (int)src.size() - 1; i >= 0; --i) st.push_back(src[i]);
    while (!st.empty()) {
      int v = st.back(); st.pop_back(); seq.push_back(v);
      std::vector<int> fr;
      for (int k = ooff[v]; k < ooff[v + 1]; ++k) if (--indeg[od[k]] == 0) fr.push_back(od[k]);
      for (int i = (int)fr.size() - 1; i >= 0; --i) st.push_back(fr[i]);  // rows are rank-sorted
    }
  }
  // windowed fixed point
  std::vector<int> rem(n), emitted_pos(n, -1), stackv;
  for (int v = 0; v < n; ++v) rem[v] = ioff[v + 1] - ioff[v];
  for (int v = 0; v < n; ++v) if (!rem[v]) stackv.push_back(v);
  std::sort(stackv.begin(), stackv.end(), [&](int a, int b) { return rank[a] < rank[b]; });  // top first
  std::vector<int> out_seq;
  out_seq.reserve(n);
  std::vector<int> lvl(n, -1), rem2(n), inC(n, 0), posC(n, -1), par(n), sz(n), pre(n);
  long windows = 0, total_rounds = 0, total_C = 0, max_rounds = 0;
  std::vector<int> C, levoff;
  while ((int)out_seq.size() < n) {
    ++windows;
    // Kahn over the residual from the stack, H levels
    C.clear();
    levoff.clear();
    for (int v : stackv) { C.push_back(v); inC[v] = 1; lvl[v] = 0; }
    levoff.push_back(0);
    std::vector<int> touched;
    size_t lb = 0;
    for (int L = 0; L < H && lb < C.size(); ++L) {
      size_t le = C.size();
      levoff.push_back((int)le);
      if (L == H - 1) break;
      for (size_t i = lb; i < le; ++i) {
        int v = C[i];
        for (int k = ooff[v]; k < ooff[v + 1]; ++k) {
          int c = od[k];
          if (emitted_pos[c] >= 0) continue;
          if (rem2[c] == 0 && !inC[c]) { rem2[c] = rem[c]; touched.push_back(c); }
          if (--rem2[c] == 0) { C.push_back(c); inC[c] = 1; lvl[c] = L + 1; }
        }
      }
      lb = le;
    }
    if (levoff.back() != (int)C.size()) levoff.push_back((int)C.size());
    const int nl = (int)levoff.size() - 1;
    total_C += C.size();
    // fixed point on C; roots = stack order; initial order = Kahn order
    for (size_t i = 0; i < C.size(); ++i) posC[C[i]] = (int)i;
    int rounds = 0;
    for (;;) {
      ++rounds;
      for (int v : C) {
        int best = -1, bp = -1;
        for (int k = ioff[v]; k < ioff[v + 1]; ++k) {
          int p = is[k];
          if (!inC[p]) continue;  // emitted prefix (all R-preds of v are in C)
          if (posC[p] > bp) { bp = posC[p]; best = p; }
        }
        par[v] = best;
      }
      for (int L = nl - 1; L >= 0; --L)
        for (int i = levoff[L]; i < levoff[L + 1]; ++i) {
          int v = C[i], s = 1;
          for (int k = ooff[v]; k < ooff[v + 1]; ++k) { int c = od[k]; if (inC[c] && par[c] == v) s += sz[c]; }
          sz[v] = s;
        }
      int acc = 0;
      for (int v : stackv) { pre[v] = acc; acc += sz[v]; }
      for (int L = 0; L < nl; ++L)
        for (int i = levoff[L]; i < levoff[L + 1]; ++i) {
          int v = C[i], a = pre[v] + 1;
          for (int k = ooff[v]; k < ooff[v + 1]; ++k) { int c = od[k]; if (inC[c] && par[c] == v) { pre[c] = a; a += sz[c]; } }
        }
      bool chg = false;
      for (int v : C) { if (pre[v] != posC[v]) chg = true; }
      for (int v : C) posC[v] = pre[v];
      if (!chg) break;
    }
    total_rounds += rounds;
    max_rounds = std::max<long>(max_rounds, rounds);
    // t = first restricted position whose emission frees a node outside C
    int t = (int)C.size() - 1;
    std::vector<int> outside;
    for (int v : C)
      for (int k = ooff[v]; k < ooff[v + 1]; ++k) {
        int c = od[k];
        if (!inC[c] && emitted_pos[c] < 0) outside.push_back(c);
      }
    std::sort(outside.begin(), outside.end());
    outside.erase(std::unique(outside.begin(), outside.end()), outside.end());
    for (int c : outside) {
      // c outside C: freed during sigma_C iff all residual preds in C
      bool all = true;
      int mx = -1;
      for (int k = ioff[c]; k < ioff[c + 1]; ++k) {
        int p = is[k];
        if (emitted_pos[p] >= 0) continue;
        if (!inC[p]) { all = false; break; }
        mx = std::max(mx, posC[p]);
      }
      if (all) t = std::min(t, mx);
    }
    // commit positions [0, t]
    std::vector<int> sc(C.size());
    for (int v : C) sc[posC[v]] = v;
    for (int q = 0; q <= t; ++q) {
      int v = sc[q];
      emitted_pos[v] = (int)out_seq.size();
      out_seq.push_back(v);
      for (int k = ooff[v]; k < ooff[v + 1]; ++k) --rem[od[k]];
    }
    // reset window marks
    for (int v : C) { inC[v] = 0; }
    for (int c : touched) rem2[c] = 0;
    // new stack: freed, unemitted; order (parent position desc, rank asc)
    std::vector<std::pair<int, int>> st;  // (parent pos, rank)
    std::vector<int> cand;
    for (int v : C) if (emitted_pos[v] < 0) cand.push_back(v);
    for (int c : outside) if (emitted_pos[c] < 0 && rem[c] == 0) cand.push_back(c);
    std::sort(cand.begin(), cand.end());
    cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
    stackv.clear();
    std::vector<std::pair<std::pair<int, int>, int>> keyed;
    for (int v : cand) {
      if (rem[v] != 0) continue;
      int pp = -1;
      for (int k = ioff[v]; k < ioff[v + 1]; ++k) pp = std::max(pp, emitted_pos[is[k]]);
      keyed.push_back({{-pp, rank[v]}, v});
    }
    std::sort(keyed.begin(), keyed.end());
    for (auto& x : keyed) stackv.push_back(x.second);
    if (windows <= 5 || windows % 200 == 0)
      printf("window %ld: |C|=%zu levels=%d rounds=%d commit=%d emitted=%zu stack=%zu\n", windows, C.size(), nl, rounds,
             t + 1, out_seq.size(), stackv.size());
  }
  printf("H=%d windows=%ld mean commit=%.1f mean |C|=%.1f mean rounds=%.2f max rounds=%ld equal=%s\n", H, windows,
         (double)n / windows, (double)total_C / windows, (double)total_rounds / windows, max_rounds,
         out_seq == seq ? "yes" : "NO");
  return 0;
}
