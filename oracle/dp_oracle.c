/*
 * dp_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C, flat-array restatement of the
 * reference's graph-analysis / placement-evaluation path (dagplace, /root/reference/proj).
 *
 * Parity pinning: every dpo_* function is checked against the unmodified reference
 * (oracle/_ref/libdagplace_ref.so, dpr_*) on the reference's golden vectors and on
 * seeded random graphs by tests/test_oracle_pinning.py.  The product (CUDA) path never
 * links or calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline may.
 *
 * Built with -ffp-contract=off: comm_time's k*bytes + b must not become an FMA
 * (graph.cpp:200-204).
 */
#include <limits.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "dp_results.h"

#define NEVER INT64_MAX

static _Thread_local char g_err[1024];
static _Thread_local int g_code;

static const char* kind_name(int code) {
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
  return (code >= 0 && code <= 19) ? names[code] : "UnknownError";
}

/* DagError(kind, msg).what() == "<Kind>: <msg>" (error.hpp:37-41). */
static int fail(int code, const char* fmt, ...) {
  char msg[900];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(msg, sizeof msg, fmt, ap);
  va_end(ap);
  snprintf(g_err, sizeof g_err, "%s: %s", kind_name(code), msg);
  g_code = code;
  return code;
}
const char* dpo_last_error_message(void) { return g_err; }

DPR_DEFINE_FREES(dpo_)

/* ------------------------------------------------------------------ small utils */
typedef struct {
  int64_t id;
  int32_t idx;
} IdIdx;

static int cmp_ididx(const void* a, const void* b) {
  const IdIdx* x = (const IdIdx*)a;
  const IdIdx* y = (const IdIdx*)b;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* Sorted (id, idx) table replacing GraphIndex::index_ (graph_index.cpp:12-18). */
typedef struct {
  IdIdx* t;
  int32_t n;
} IdMap;

static IdMap idmap_build(const int64_t* ids, int64_t n) {
  IdMap m;
  m.n = (int32_t)n;
  m.t = (IdIdx*)malloc(sizeof(IdIdx) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    m.t[i].id = ids[i];
    m.t[i].idx = (int32_t)i;
  }
  qsort(m.t, (size_t)n, sizeof(IdIdx), cmp_ididx);
  return m;
}
static int32_t idmap_find(const IdMap* m, int64_t id) { /* first idx with id, or -1 */
  int32_t lo = 0, hi = m->n;
  while (lo < hi) {
    int32_t mid = lo + (hi - lo) / 2;
    if (m->t[mid].id < id) lo = mid + 1; else hi = mid;
  }
  return (lo < m->n && m->t[lo].id == id) ? m->t[lo].idx : -1;
}
static void idmap_free(IdMap* m) { free(m->t); }

/* comm_time, graph.cpp:200-204. */
static int64_t comm_cost(int64_t bytes, dp_comm_t c) {
  double t = c.k_us_per_byte * (double)bytes;
  t = t + c.b_us;
  return (int64_t)llround(t);
}

int dpo_comm_time(int64_t bytes, dp_comm_t comm, int64_t* out) {
  if (bytes < 0) return fail(DP_E_INVALID_VALUE, "negative byte count");
  *out = comm_cost(bytes, comm);
  return 0;
}

/* ------------------------------------------------------------------ GraphIndex */
/* graph_index.cpp:8-42: endpoints as indices, CSR (out) / CSC (in) lists of edge
 * indices, stable in input edge order (counting sort). */
typedef struct {
  int32_t n, m;
  int32_t *esrc, *edst;
  int32_t *out_start, *out_list, *in_start, *in_list;
  IdMap ids;
} Index;

static void index_free(Index* ix) {
  free(ix->esrc); free(ix->edst); free(ix->out_start); free(ix->out_list);
  free(ix->in_start); free(ix->in_list); idmap_free(&ix->ids);
}

static int index_build(const dp_graph_t* g, Index* ix) {
  memset(ix, 0, sizeof *ix);
  int32_t n = (int32_t)g->n_nodes, m = (int32_t)g->n_edges;
  ix->n = n;
  ix->m = m;
  ix->ids = idmap_build(g->node_id, n);
  for (int32_t i = 1; i < n; ++i) {
    if (ix->ids.t[i].id == ix->ids.t[i - 1].id) {
      /* graph_index.cpp:13-17 reports the first index whose emplace fails. */
      int64_t dup_id = ix->ids.t[i].id;
      int32_t second = ix->ids.t[i].idx; /* sorted by (id, idx): i is a later index */
      for (int32_t j = i; j < n && ix->ids.t[j].id == dup_id; ++j) {
        if (ix->ids.t[j].idx < second) second = ix->ids.t[j].idx;
      }
      (void)second;
      index_free(ix);
      return fail(DP_E_DUPLICATE_ID, "node id %lld is not unique", (long long)dup_id);
    }
  }
  ix->esrc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  ix->edst = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  ix->out_start = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  ix->in_start = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
  ix->out_list = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  ix->in_list = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  for (int32_t e = 0; e < m; ++e) {
    int32_t s = idmap_find(&ix->ids, g->edge_src[e]);
    if (s < 0) {
      index_free(ix);
      return fail(DP_E_UNKNOWN_NODE, "node %lld not in graph", (long long)g->edge_src[e]);
    }
    int32_t d = idmap_find(&ix->ids, g->edge_dst[e]);
    if (d < 0) {
      index_free(ix);
      return fail(DP_E_UNKNOWN_NODE, "node %lld not in graph", (long long)g->edge_dst[e]);
    }
    ix->esrc[e] = s;
    ix->edst[e] = d;
    ix->out_start[s + 1]++;
    ix->in_start[d + 1]++;
  }
  for (int32_t v = 0; v < n; ++v) {
    ix->out_start[v + 1] += ix->out_start[v];
    ix->in_start[v + 1] += ix->in_start[v];
  }
  int32_t* of = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  int32_t* inf = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  memcpy(of, ix->out_start, sizeof(int32_t) * ((size_t)n + 1));
  memcpy(inf, ix->in_start, sizeof(int32_t) * ((size_t)n + 1));
  for (int32_t e = 0; e < m; ++e) {
    ix->out_list[of[ix->esrc[e]]++] = e;
    ix->in_list[inf[ix->edst[e]]++] = e;
  }
  free(of);
  free(inf);
  return 0;
}

int dpo_graph_index(const dp_graph_t* g, int32_t* esrc, int32_t* edst, int32_t* out_start,
                    int32_t* out_list, int32_t* in_start, int32_t* in_list) {
  Index ix;
  int rc = index_build(g, &ix);
  if (rc) return rc;
  memcpy(esrc, ix.esrc, sizeof(int32_t) * (size_t)ix.m);
  memcpy(edst, ix.edst, sizeof(int32_t) * (size_t)ix.m);
  memcpy(out_start, ix.out_start, sizeof(int32_t) * ((size_t)ix.n + 1));
  memcpy(in_start, ix.in_start, sizeof(int32_t) * ((size_t)ix.n + 1));
  memcpy(out_list, ix.out_list, sizeof(int32_t) * (size_t)ix.m);
  memcpy(in_list, ix.in_list, sizeof(int32_t) * (size_t)ix.m);
  index_free(&ix);
  return 0;
}

/* ------------------------------------------------------------------ validate */
typedef struct {
  int64_t count, cap;
  int32_t* kind;
  int64_t *node_off, *nodes, *msg_off;
  char* msg;
  int64_t nodes_len, nodes_cap, msg_len, msg_cap;
} VList;

static void vl_add(VList* v, int code, const int64_t* ids, int nids, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  int len = vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (v->count + 1 >= v->cap) {
    v->cap = v->cap ? v->cap * 2 : 16;
    v->kind = (int32_t*)realloc(v->kind, sizeof(int32_t) * (size_t)v->cap);
    v->node_off = (int64_t*)realloc(v->node_off, sizeof(int64_t) * (size_t)(v->cap + 1));
    v->msg_off = (int64_t*)realloc(v->msg_off, sizeof(int64_t) * (size_t)(v->cap + 1));
  }
  while (v->nodes_len + nids > v->nodes_cap) {
    v->nodes_cap = v->nodes_cap ? v->nodes_cap * 2 : 64;
    v->nodes = (int64_t*)realloc(v->nodes, sizeof(int64_t) * (size_t)v->nodes_cap);
  }
  while (v->msg_len + len + 1 > v->msg_cap) {
    v->msg_cap = v->msg_cap ? v->msg_cap * 2 : 1024;
    v->msg = (char*)realloc(v->msg, (size_t)v->msg_cap);
  }
  v->kind[v->count] = code;
  v->node_off[v->count] = v->nodes_len;
  v->msg_off[v->count] = v->msg_len;
  for (int i = 0; i < nids; ++i) v->nodes[v->nodes_len++] = ids[i];
  memcpy(v->msg + v->msg_len, buf, (size_t)len);
  v->msg_len += len;
  v->count++;
  v->node_off[v->count] = v->nodes_len;
  v->msg_off[v->count] = v->msg_len;
}

typedef struct {
  int64_t s, d;
  int32_t e;
} Pair;
static int cmp_pair(const void* a, const void* b) {
  const Pair* x = (const Pair*)a;
  const Pair* y = (const Pair*)b;
  if (x->s != y->s) return x->s < y->s ? -1 : 1;
  if (x->d != y->d) return x->d < y->d ? -1 : 1;
  return x->e < y->e ? -1 : (x->e > y->e);
}

/* find_cycle_witness, graph.cpp:71-94: start at the smallest remaining id, follow the
 * smallest successor inside `remaining` until an id repeats. */
static int64_t* cycle_witness(const dp_graph_t* g, const IdMap* ids, const uint8_t* remaining_idx,
                              int* out_len) {
  int32_t n = (int32_t)g->n_nodes;
  int64_t start = 0;
  int have = 0;
  for (int32_t v = 0; v < n; ++v) {
    if (remaining_idx[v] && (!have || g->node_id[v] < start)) {
      start = g->node_id[v];
      have = 1;
    }
  }
  int64_t* path = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  int32_t* pos_in_path = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int32_t v = 0; v < n; ++v) pos_in_path[v] = -1;
  int len = 0;
  int64_t cur = start;
  for (;;) {
    int32_t ci = idmap_find(ids, cur);
    if (pos_in_path[ci] >= 0) {
      int from = pos_in_path[ci];
      memmove(path, path + from, sizeof(int64_t) * (size_t)(len - from));
      *out_len = len - from;
      free(pos_in_path);
      return path;
    }
    pos_in_path[ci] = len;
    path[len++] = cur;
    int64_t best = 0;
    int found = 0;
    for (int64_t e = 0; e < g->n_edges; ++e) {
      if (g->edge_src[e] != cur) continue;
      int32_t di = idmap_find(ids, g->edge_dst[e]);
      if (!remaining_idx[di]) continue;
      if (!found || g->edge_dst[e] < best) {
        best = g->edge_dst[e];
        found = 1;
      }
    }
    if (!found) {
      *out_len = len;
      free(pos_in_path);
      return path;
    }
    cur = best;
  }
}

static void append_ids(char* buf, size_t cap, const int64_t* ids, int n) {
  size_t off = strlen(buf);
  for (int i = 0; i < n && off < cap; ++i) {
    off += (size_t)snprintf(buf + off, cap - off, i ? ",%lld" : "%lld", (long long)ids[i]);
  }
}

/* validate, graph.cpp:98-191: every violation in detection order. */
static void validate_into(const dp_graph_t* g, VList* v) {
  int32_t n = (int32_t)g->n_nodes;
  int64_t m = g->n_edges;
  IdMap ids = idmap_build(g->node_id, n);
  /* id_count via the sorted table (graph.cpp:105-106) */
  int32_t* count_of_idx = (int32_t*)calloc((size_t)(n ? n : 1), sizeof(int32_t));
  uint8_t* first_of_id = (uint8_t*)calloc((size_t)(n ? n : 1), 1);
  int any_dup = 0;
  for (int32_t i = 0; i < n;) {
    int32_t j = i;
    while (j < n && ids.t[j].id == ids.t[i].id) ++j;
    for (int32_t k = i; k < j; ++k) count_of_idx[ids.t[k].idx] = j - i;
    first_of_id[ids.t[i].idx] = 1; /* smallest index of that id (sorted by idx within id) */
    if (j - i > 1) any_dup = 1;
    i = j;
  }
  for (int32_t i = 0; i < n; ++i) { /* graph.cpp:108-120 */
    int64_t id = g->node_id[i];
    if (count_of_idx[i] > 1 && first_of_id[i]) {
      vl_add(v, DP_E_DUPLICATE_ID, &id, 1, "node id %lld appears %d times", (long long)id,
             count_of_idx[i]);
    }
    if (g->compute_us[i] < 0)
      vl_add(v, DP_E_INVALID_VALUE, &id, 1, "node %lld has negative compute_us", (long long)id);
    if (g->memory_bytes[i] < 0)
      vl_add(v, DP_E_INVALID_VALUE, &id, 1, "node %lld has negative memory_bytes", (long long)id);
  }
  /* duplicate edges among edges with ok endpoints (graph.cpp:122,149-154) */
  uint8_t* ok_ep = (uint8_t*)calloc((size_t)(m ? m : 1), 1);
  uint8_t* is_dup = (uint8_t*)calloc((size_t)(m ? m : 1), 1);
  Pair* pairs = (Pair*)malloc(sizeof(Pair) * (size_t)(m ? m : 1));
  int64_t np = 0;
  for (int64_t e = 0; e < m; ++e) {
    int ok = idmap_find(&ids, g->edge_src[e]) >= 0 && idmap_find(&ids, g->edge_dst[e]) >= 0 &&
             g->edge_src[e] != g->edge_dst[e];
    ok_ep[e] = (uint8_t)ok;
    if (ok) {
      pairs[np].s = g->edge_src[e];
      pairs[np].d = g->edge_dst[e];
      pairs[np].e = (int32_t)e;
      ++np;
    }
  }
  qsort(pairs, (size_t)np, sizeof(Pair), cmp_pair);
  for (int64_t k = 1; k < np; ++k) {
    if (pairs[k].s == pairs[k - 1].s && pairs[k].d == pairs[k - 1].d) is_dup[pairs[k].e] = 1;
  }
  free(pairs);
  int edges_resolvable = 1;
  for (int64_t e = 0; e < m; ++e) { /* graph.cpp:124-156 */
    int64_t s = g->edge_src[e], d = g->edge_dst[e];
    int64_t sd[2] = {s, d};
    int ok = 1;
    if (idmap_find(&ids, s) < 0) {
      vl_add(v, DP_E_DANGLING_EDGE, sd, 2, "edge (%lld,%lld) references missing node %lld",
             (long long)s, (long long)d, (long long)s);
      ok = 0;
    }
    if (idmap_find(&ids, d) < 0) {
      vl_add(v, DP_E_DANGLING_EDGE, sd, 2, "edge (%lld,%lld) references missing node %lld",
             (long long)s, (long long)d, (long long)d);
      ok = 0;
    }
    if (s == d) {
      vl_add(v, DP_E_CYCLE_DETECTED, &s, 1, "self-loop on node %lld", (long long)s);
      ok = 0;
    }
    if (g->edge_bytes[e] < 0)
      vl_add(v, DP_E_INVALID_VALUE, sd, 2, "edge (%lld,%lld) has negative tensor_bytes",
             (long long)s, (long long)d);
    if (ok && is_dup[e])
      vl_add(v, DP_E_DUPLICATE_EDGE, sd, 2,
             "parallel edge (%lld,%lld); aggregate tensor bytes upstream", (long long)s,
             (long long)d);
    edges_resolvable = edges_resolvable && ok;
  }
  /* Kahn acyclicity (graph.cpp:159-188); the id-keyed maps of the reference are
   * equivalent to index arrays once ids are unique. */
  if (edges_resolvable && !any_dup && n > 0) {
    int32_t* indeg = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    int32_t* ostart = (int32_t*)calloc((size_t)n + 1, sizeof(int32_t));
    int32_t* olist = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
    int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
    int32_t* queue = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
    for (int64_t e = 0; e < m; ++e) {
      ostart[idmap_find(&ids, g->edge_src[e]) + 1]++;
      indeg[idmap_find(&ids, g->edge_dst[e])]++;
    }
    for (int32_t i = 0; i < n; ++i) ostart[i + 1] += ostart[i];
    memcpy(fill, ostart, sizeof(int32_t) * ((size_t)n + 1));
    for (int64_t e = 0; e < m; ++e) {
      olist[fill[idmap_find(&ids, g->edge_src[e])]++] = idmap_find(&ids, g->edge_dst[e]);
    }
    int32_t head = 0, tail = 0;
    for (int32_t i = 0; i < n; ++i)
      if (indeg[i] == 0) queue[tail++] = i;
    int64_t emitted = 0;
    while (head < tail) {
      int32_t u = queue[head++];
      ++emitted;
      for (int32_t k = ostart[u]; k < ostart[u + 1]; ++k) {
        if (--indeg[olist[k]] == 0) queue[tail++] = olist[k];
      }
    }
    if (emitted != n) {
      uint8_t* rem = (uint8_t*)calloc((size_t)n, 1);
      for (int32_t i = 0; i < n; ++i) rem[i] = indeg[i] > 0;
      int wl = 0;
      int64_t* w = cycle_witness(g, &ids, rem, &wl);
      char buf[1000] = "cycle: [";
      append_ids(buf, sizeof buf - 2, w, wl);
      strcat(buf, "]");
      vl_add(v, DP_E_CYCLE_DETECTED, w, wl, "%s", buf);
      free(w);
      free(rem);
    }
    free(indeg); free(ostart); free(olist); free(fill); free(queue);
  }
  free(ok_ep); free(is_dup); free(count_of_idx); free(first_of_id);
  idmap_free(&ids);
}

int dpo_validate(const dp_graph_t* g, dp_violation_list_t** out) {
  VList v;
  memset(&v, 0, sizeof v);
  validate_into(g, &v);
  dp_violation_list_t* r = DPR_NEW(dp_violation_list_t, 1);
  r->count = v.count;
  r->kind = v.kind ? v.kind : DPR_NEW(int32_t, 1);
  r->node_off = v.node_off ? v.node_off : DPR_NEW(int64_t, 1);
  r->msg_off = v.msg_off ? v.msg_off : DPR_NEW(int64_t, 1);
  r->nodes = v.nodes ? v.nodes : DPR_NEW(int64_t, 1);
  r->msg = v.msg ? v.msg : DPR_NEW(char, 1);
  *out = r;
  return 0;
}

/* require_valid, graph.cpp:193-198. */
int dpo_require_valid(const dp_graph_t* g) {
  VList v;
  memset(&v, 0, sizeof v);
  validate_into(g, &v);
  int rc = 0;
  if (v.count) {
    char msg[900];
    int64_t len = v.msg_off[1] - v.msg_off[0];
    if (len > 899) len = 899;
    memcpy(msg, v.msg, (size_t)len);
    msg[len] = 0;
    rc = fail(v.kind[0], "%s", msg);
  }
  free(v.kind); free(v.node_off); free(v.nodes); free(v.msg_off); free(v.msg);
  return rc;
}

/* ccr, graph.cpp:206-215. */
int dpo_ccr(const dp_graph_t* g, dp_comm_t comm, double* out) {
  int64_t total_compute = 0, total_comm = 0;
  for (int64_t i = 0; i < g->n_nodes; ++i) total_compute += g->compute_us[i];
  if (total_compute <= 0) return fail(DP_E_ZERO_COMPUTE_TIME, "total compute time is zero");
  for (int64_t e = 0; e < g->n_edges; ++e) {
    if (g->edge_bytes[e] < 0) return fail(DP_E_INVALID_VALUE, "negative byte count");
    total_comm += comm_cost(g->edge_bytes[e], comm);
  }
  *out = (double)total_comm / (double)total_compute;
  return 0;
}

/* ------------------------------------------------------------------ levels */
static int64_t* edge_costs(const dp_graph_t* g, dp_comm_t comm) {
  int64_t* c = (int64_t*)malloc(sizeof(int64_t) * (size_t)(g->n_edges ? g->n_edges : 1));
  for (int64_t e = 0; e < g->n_edges; ++e) c[e] = comm_cost(g->edge_bytes[e], comm);
  return c;
}

/* compute_levels core, graph.cpp:222-261, on a built index. */
static void levels_core(const dp_graph_t* g, const Index* ix, const int64_t* cost, int64_t* tl,
                        int64_t* bl) {
  int32_t n = ix->n;
  int32_t* topo = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t* indeg = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t head = 0, tail = 0;
  for (int32_t v = 0; v < n; ++v) {
    indeg[v] = ix->in_start[v + 1] - ix->in_start[v];
    if (!indeg[v]) topo[tail++] = v;
  }
  while (head < tail) { /* Kahn FIFO, graph.cpp:236-244 */
    int32_t v = topo[head++];
    for (int32_t k = ix->out_start[v]; k < ix->out_start[v + 1]; ++k) {
      int32_t w = ix->edst[ix->out_list[k]];
      if (--indeg[w] == 0) topo[tail++] = w;
    }
  }
  for (int32_t v = 0; v < n; ++v) tl[v] = bl[v] = 0;
  for (int32_t i = 0; i < n; ++i) { /* graph.cpp:247-252 */
    int32_t v = topo[i];
    for (int32_t k = ix->in_start[v]; k < ix->in_start[v + 1]; ++k) {
      int32_t e = ix->in_list[k], p = ix->esrc[e];
      int64_t cand = tl[p] + g->compute_us[p] + cost[e];
      if (cand > tl[v]) tl[v] = cand;
    }
  }
  for (int32_t i = n - 1; i >= 0; --i) { /* graph.cpp:253-261 */
    int32_t v = topo[i];
    int64_t best = 0;
    for (int32_t k = ix->out_start[v]; k < ix->out_start[v + 1]; ++k) {
      int32_t e = ix->out_list[k];
      int64_t cand = bl[ix->edst[e]] + cost[e];
      if (cand > best) best = cand;
    }
    bl[v] = best + g->compute_us[v];
  }
  free(topo);
  free(indeg);
}

int dpo_compute_levels(const dp_graph_t* g, dp_comm_t comm, int64_t* tl, int64_t* bl,
                       int64_t* cp) {
  int rc = dpo_require_valid(g); /* graph.cpp:218 */
  if (rc) return rc;
  Index ix;
  if ((rc = index_build(g, &ix))) return rc;
  int64_t* cost = edge_costs(g, comm);
  levels_core(g, &ix, cost, tl, bl);
  for (int32_t v = 0; v < ix.n; ++v) cp[v] = tl[v] + bl[v];
  free(cost);
  index_free(&ix);
  return 0;
}

/* ------------------------------------------------------------------ peel */
/* Sort context for the policy comparators of ordering.cpp:81-114. */
static const int64_t* s_key_cpath;
static const int64_t* s_key_id;
static int s_desc_cpath; /* 1: cpath descending (initial), 0: ascending (children) */
static int s_desc_id;
static int cmp_policy(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  if (s_key_cpath && s_key_cpath[x] != s_key_cpath[y]) {
    int lt = s_key_cpath[x] < s_key_cpath[y];
    return s_desc_cpath ? (lt ? 1 : -1) : (lt ? -1 : 1);
  }
  if (s_key_id[x] == s_key_id[y]) return 0;
  int lt = s_key_id[x] < s_key_id[y];
  return s_desc_id ? (lt ? 1 : -1) : (lt ? -1 : 1);
}

/* peel, ordering.cpp:40-77.  The deque is a ring buffer of capacity n. */
static int peel_core(const dp_graph_t* g, const Index* ix, int policy, const int64_t* cpath,
                     int64_t* seq_out) {
  int32_t n = ix->n;
  int32_t cap = n + 1;
  int32_t* ring = (int32_t*)malloc(sizeof(int32_t) * (size_t)cap);
  int32_t* indeg = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t* srcs = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t* freed = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t ns = 0;
  for (int32_t v = 0; v < n; ++v) {
    indeg[v] = ix->in_start[v + 1] - ix->in_start[v];
    if (!indeg[v]) srcs[ns++] = v;
  }
  s_key_id = g->node_id;
  s_key_cpath = policy == DP_TOPO_CPD ? cpath : NULL;
  s_desc_cpath = 1; /* initial: cpath desc, id asc (ordering.cpp:435-438 / 81-96) */
  s_desc_id = 0;
  qsort(srcs, (size_t)ns, sizeof(int32_t), cmp_policy);
  int32_t head = 0, size = 0;
  for (int32_t i = 0; i < ns; ++i) ring[(head + size++) % cap] = srcs[i];
  int64_t emitted = 0;
  while (size) {
    int32_t v = ring[head];
    head = (head + 1) % cap;
    --size;
    seq_out[emitted++] = g->node_id[v];
    int32_t nf = 0;
    for (int32_t k = ix->out_start[v]; k < ix->out_start[v + 1]; ++k) {
      int32_t c = ix->edst[ix->out_list[k]];
      if (--indeg[c] == 0) freed[nf++] = c;
    }
    /* child order: M: id asc; DFS: id desc; CPD: cpath asc, id desc */
    s_desc_cpath = 0;
    s_desc_id = policy == DP_TOPO_M ? 0 : 1;
    qsort(freed, (size_t)nf, sizeof(int32_t), cmp_policy);
    for (int32_t i = 0; i < nf; ++i) {
      if (policy == DP_TOPO_M) {
        ring[(head + size) % cap] = freed[i];
      } else {
        head = (head - 1 + cap) % cap;
        ring[head] = freed[i];
      }
      ++size;
    }
  }
  free(ring); free(indeg); free(srcs); free(freed);
  if (emitted != n) return fail(DP_E_CYCLE_DETECTED, "graph has a cycle; topological order impossible");
  return 0;
}

int dpo_topo_order(const dp_graph_t* g, int32_t policy, const int64_t* cpath, int64_t* seq) {
  int rc = dpo_require_valid(g);
  if (rc) return rc;
  Index ix;
  if ((rc = index_build(g, &ix))) return rc;
  rc = peel_core(g, &ix, policy, cpath, seq);
  index_free(&ix);
  return rc;
}

/* is_valid_topo_order, ordering.cpp:116-132. */
static int valid_order(const dp_graph_t* g, const int64_t* seq, int64_t len) {
  if (len != g->n_nodes) return 0;
  IdMap pos = idmap_build(seq, len); /* idx = position */
  for (int64_t i = 1; i < len; ++i)
    if (pos.t[i].id == pos.t[i - 1].id) { idmap_free(&pos); return 0; }
  for (int64_t i = 0; i < g->n_nodes; ++i)
    if (idmap_find(&pos, g->node_id[i]) < 0) { idmap_free(&pos); return 0; }
  for (int64_t e = 0; e < g->n_edges; ++e) {
    int32_t u = idmap_find(&pos, g->edge_src[e]), v = idmap_find(&pos, g->edge_dst[e]);
    if (u < 0 || v < 0 || u >= v) { idmap_free(&pos); return 0; }
  }
  idmap_free(&pos);
  return 1;
}
int dpo_is_valid_topo_order(const dp_graph_t* g, const int64_t* seq, int64_t len, int32_t* out) {
  *out = valid_order(g, seq, len);
  return 0;
}

/* ------------------------------------------------------------------ fusion */
/* merge_is_safe, fusion.cpp:16-51. */
int dpo_merge_is_safe(const dp_graph_t* g, int64_t u, int64_t v, int32_t* out) {
  int rc = dpo_require_valid(g);
  if (rc) return rc;
  Index ix;
  if ((rc = index_build(g, &ix))) return rc;
  int32_t ui = idmap_find(&ix.ids, u);
  if (ui < 0) { index_free(&ix); return fail(DP_E_UNKNOWN_NODE, "node %lld not in graph", (long long)u); }
  int32_t vi = idmap_find(&ix.ids, v);
  if (vi < 0) { index_free(&ix); return fail(DP_E_UNKNOWN_NODE, "node %lld not in graph", (long long)v); }
  int32_t direct = -1;
  for (int32_t k = ix.out_start[ui]; k < ix.out_start[ui + 1]; ++k)
    if (ix.edst[ix.out_list[k]] == vi) { direct = ix.out_list[k]; break; }
  if (direct < 0) {
    index_free(&ix);
    return fail(DP_E_NO_SUCH_EDGE, "no edge (%lld,%lld)", (long long)u, (long long)v);
  }
  uint8_t* seen = (uint8_t*)calloc((size_t)ix.n, 1);
  int32_t* stack = (int32_t*)malloc(sizeof(int32_t) * ((size_t)ix.n + 1));
  int32_t sp = 0;
  stack[sp++] = ui;
  seen[ui] = 1;
  int safe = 1;
  while (sp && safe) {
    int32_t cur = stack[--sp];
    for (int32_t k = ix.out_start[cur]; k < ix.out_start[cur + 1]; ++k) {
      int32_t e = ix.out_list[k];
      if (e == direct && cur == ui) continue;
      int32_t nx = ix.edst[e];
      if (nx == vi) { safe = 0; break; }
      if (!seen[nx]) { seen[nx] = 1; stack[sp++] = nx; }
    }
  }
  *out = safe;
  free(seen); free(stack); index_free(&ix);
  return 0;
}

/* clusters_from_cuts, fusion.cpp:61-81. */
static dp_cluster_map_t* clusters_from_cuts(const dp_graph_t* g, const IdMap* ids,
                                            const int64_t* seq, const int32_t* cuts,
                                            int32_t ncuts) {
  int32_t k = ncuts - 1;
  dp_cluster_map_t* m = dpr_cluster_map_new(g->n_nodes, k, k > 0 ? k - 1 : 0);
  for (int64_t i = 0; i < g->n_nodes; ++i) m->node_cluster[i] = -1;
  int64_t off = 0;
  for (int32_t c = 0; c < k; ++c) {
    m->member_off[c] = off;
    for (int32_t p = cuts[c]; p < cuts[c + 1]; ++p) {
      int32_t idx = idmap_find(ids, seq[p]);
      m->members[off++] = seq[p];
      m->total_compute[c] += g->compute_us[idx];
      m->total_memory[c] += g->memory_bytes[idx];
      m->node_cluster[idx] = c;
    }
  }
  m->member_off[k] = off;
  for (int32_t c = 1; c + 1 < ncuts; ++c) m->breakpoints[c - 1] = cuts[c];
  return m;
}

/* optimal_breakpoints, fusion.cpp:85-171. */
int dpo_optimal_breakpoints(const dp_graph_t* g, const int64_t* seq, int64_t len, dp_comm_t comm,
                            int32_t range, int64_t limit, dp_cluster_map_t** out) {
  int rc = dpo_require_valid(g);
  if (rc) return rc;
  if (!valid_order(g, seq, len))
    return fail(DP_E_INVALID_VALUE, "order is not a topological order of this graph");
  if (range < 1) return fail(DP_E_INVALID_VALUE, "exploration range must be >= 1");
  if (limit <= 0) return fail(DP_E_INVALID_VALUE, "cluster memory limit must be > 0");
  Index ix;
  if ((rc = index_build(g, &ix))) return rc;
  int32_t n = (int32_t)len;
  if (n == 0) {
    int32_t zero = 0;
    *out = clusters_from_cuts(g, &ix.ids, seq, &zero, 1);
    index_free(&ix);
    return 0;
  }
  int32_t* pos_of_idx = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  int32_t* idx_at_pos = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  for (int32_t p = 0; p < n; ++p) {
    int32_t idx = idmap_find(&ix.ids, seq[p]);
    pos_of_idx[idx] = p;
    idx_at_pos[p] = idx;
  }
  int64_t* mem_prefix = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int32_t p = 0; p < n; ++p) {
    int32_t idx = idx_at_pos[p];
    if (g->memory_bytes[idx] > limit) {
      free(pos_of_idx); free(idx_at_pos); free(mem_prefix); index_free(&ix);
      return fail(DP_E_NODE_EXCEEDS_CLUSTER_LIMIT, "node %lld needs %lld bytes, cluster limit is %lld",
                  (long long)g->node_id[idx], (long long)g->memory_bytes[idx], (long long)limit);
    }
    mem_prefix[p + 1] = mem_prefix[p] + g->memory_bytes[idx];
  }
  int64_t* cost = edge_costs(g, comm);
  int64_t* forward = (int64_t*)calloc((size_t)n, sizeof(int64_t));
  int64_t* best = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n + 1));
  int32_t* prev_cut = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 1));
  for (int32_t j = 0; j <= n; ++j) { best[j] = NEVER; prev_cut[j] = -1; }
  best[0] = 0;
  for (int32_t j = 1; j <= n; ++j) {
    int32_t fp = j - 1, v = idx_at_pos[fp];
    int64_t out_sum = 0;
    for (int32_t k = ix.out_start[v]; k < ix.out_start[v + 1]; ++k) out_sum += cost[ix.out_list[k]];
    forward[fp] = out_sum;
    for (int32_t k = ix.in_start[v]; k < ix.in_start[v + 1]; ++k) {
      int32_t e = ix.in_list[k];
      forward[pos_of_idx[ix.esrc[e]]] -= cost[e];
    }
    int64_t wc = 0;
    int32_t lo = j - range > 0 ? j - range : 0;
    for (int32_t i = j - 1; i >= lo; --i) {
      wc += forward[i];
      if (mem_prefix[j] - mem_prefix[i] > limit) break;
      if (best[i] == NEVER) continue;
      int64_t cand = best[i] + wc;
      if (cand < best[j]) { best[j] = cand; prev_cut[j] = i; }
    }
    if (best[j] == NEVER) {
      free(pos_of_idx); free(idx_at_pos); free(mem_prefix); free(cost); free(forward);
      free(best); free(prev_cut); index_free(&ix);
      return fail(DP_E_INFEASIBLE_PARTITION, "no admissible cluster ends at position %d", j);
    }
  }
  int32_t* cuts = (int32_t*)malloc(sizeof(int32_t) * ((size_t)n + 2));
  int32_t nc = 0;
  for (int32_t c = n; c >= 0; c = prev_cut[c]) {
    cuts[nc++] = c;
    if (c == 0) break;
  }
  for (int32_t a = 0, b = nc - 1; a < b; ++a, --b) { int32_t t = cuts[a]; cuts[a] = cuts[b]; cuts[b] = t; }
  *out = clusters_from_cuts(g, &ix.ids, seq, cuts, nc);
  free(cuts); free(pos_of_idx); free(idx_at_pos); free(mem_prefix); free(cost); free(forward);
  free(best); free(prev_cut); index_free(&ix);
  return 0;
}

typedef struct {
  int64_t u, v, bytes;
} Edge3;
static int cmp_edge3(const void* a, const void* b) {
  const Edge3* x = (const Edge3*)a;
  const Edge3* y = (const Edge3*)b;
  if (x->u != y->u) return x->u < y->u ? -1 : 1;
  if (x->v != y->v) return x->v < y->v ? -1 : 1;
  return 0;
}
/* std::map<pair,Bytes> aggregation: sort by (u,v), sum runs (fusion.cpp:216-225). */
static int64_t aggregate_edges(Edge3* es, int64_t k) {
  qsort(es, (size_t)k, sizeof(Edge3), cmp_edge3);
  int64_t w = 0;
  for (int64_t r = 0; r < k; ++r) {
    if (w && es[w - 1].u == es[r].u && es[w - 1].v == es[r].v) es[w - 1].bytes += es[r].bytes;
    else es[w++] = es[r];
  }
  return w;
}

/* build_coarse_graph, fusion.cpp:173-229. */
int dpo_build_coarse_graph(const dp_graph_t* g, const int64_t* seq, int64_t len,
                           const int64_t* map_ids, const int32_t* map_cluster, int64_t map_count,
                           int64_t n_clusters, const int32_t* cluster_ids,
                           const int64_t* member_off, const int64_t* members,
                           dp_graph_out_t** out) {
  int rc = dpo_require_valid(g);
  if (rc) return rc;
  if (!valid_order(g, seq, len))
    return fail(DP_E_INVALID_VALUE, "order is not a topological order of this graph");
  /* node_to_cluster as an id-keyed map: later entries overwrite earlier (operator[]). */
  IdMap mids = idmap_build(map_ids, map_count);
  int64_t distinct = 0;
  for (int64_t i = 0; i < map_count; ++i)
    if (i == 0 || mids.t[i].id != mids.t[i - 1].id) ++distinct;
  /* value for an id = the last map entry with that id */
  #define MAP_LOOKUP(KEY_, outc)                                                  \
    do {                                                                        \
      int32_t lo_ = 0, hi_ = mids.n;                                            \
      while (lo_ < hi_) { int32_t md_ = lo_ + (hi_ - lo_) / 2;                  \
        if (mids.t[md_].id <= (KEY_)) lo_ = md_ + 1; else hi_ = md_; }            \
      outc = (lo_ > 0 && mids.t[lo_ - 1].id == (KEY_)) ? map_cluster[mids.t[lo_ - 1].idx] : INT32_MIN; \
    } while (0)
  if (distinct != g->n_nodes) {
    idmap_free(&mids);
    return fail(DP_E_INVALID_CLUSTER_MAP, "cluster map does not cover the node set");
  }
  IdMap ids = idmap_build(g->node_id, g->n_nodes);
  uint8_t* accounted = (uint8_t*)calloc((size_t)(g->n_nodes ? g->n_nodes : 1), 1);
  /* `accounted` is an unordered_set of ids; members not in the graph are tracked in a
   * side list so that repeats of them are detected too. */
  int64_t total_members = member_off[n_clusters];
  int64_t* foreign = (int64_t*)malloc(sizeof(int64_t) * (size_t)(total_members ? total_members : 1));
  int64_t nforeign = 0;
  for (int64_t c = 0; c < n_clusters; ++c) {
    if (cluster_ids[c] != (int32_t)c || member_off[c + 1] == member_off[c]) {
      free(accounted); free(foreign); idmap_free(&ids); idmap_free(&mids);
      return fail(DP_E_INVALID_CLUSTER_MAP, "cluster %lld is empty or misnumbered", (long long)c);
    }
    for (int64_t k = member_off[c]; k < member_off[c + 1]; ++k) {
      int64_t mid = members[k];
      int32_t mc;
      MAP_LOOKUP(mid, mc);
      int dup;
      int32_t gi = idmap_find(&ids, mid);
      if (gi >= 0) {
        dup = accounted[gi];
        accounted[gi] = 1;
      } else {
        dup = 0;
        for (int64_t f = 0; f < nforeign; ++f) if (foreign[f] == mid) dup = 1;
        if (!dup) foreign[nforeign++] = mid;
      }
      if (mc == INT32_MIN || mc != cluster_ids[c] || dup) {
        free(accounted); free(foreign); idmap_free(&ids); idmap_free(&mids);
        return fail(DP_E_INVALID_CLUSTER_MAP, "node %lld is not mapped consistently", (long long)mid);
      }
    }
  }
  for (int64_t i = 0; i < g->n_nodes; ++i) {
    if (!accounted[i]) {
      int64_t id = g->node_id[i];
      free(accounted); free(foreign); idmap_free(&ids); idmap_free(&mids);
      return fail(DP_E_INVALID_CLUSTER_MAP, "node %lld missing from cluster map", (long long)id);
    }
  }
  Edge3* es = (Edge3*)malloc(sizeof(Edge3) * (size_t)(g->n_edges ? g->n_edges : 1));
  int64_t k = 0;
  for (int64_t e = 0; e < g->n_edges; ++e) {
    int32_t cu, cv;
    MAP_LOOKUP(g->edge_src[e], cu);
    MAP_LOOKUP(g->edge_dst[e], cv);
    if (cu != cv) { es[k].u = cu; es[k].v = cv; es[k].bytes = g->edge_bytes[e]; ++k; }
  }
  #undef MAP_LOOKUP
  k = aggregate_edges(es, k);
  dp_graph_out_t* o = dpr_graph_out_new(n_clusters, k);
  for (int64_t c = 0; c < n_clusters; ++c) {
    o->node_id[c] = c;
    o->group[c] = -1;
    for (int64_t q = member_off[c]; q < member_off[c + 1]; ++q) {
      int32_t gi = idmap_find(&ids, members[q]);
      o->compute_us[c] += g->compute_us[gi];
      o->memory_bytes[c] += g->memory_bytes[gi];
    }
  }
  for (int64_t e = 0; e < k; ++e) {
    o->edge_src[e] = es[e].u;
    o->edge_dst[e] = es[e].v;
    o->edge_bytes[e] = es[e].bytes;
  }
  free(es); free(accounted); free(foreign); idmap_free(&ids); idmap_free(&mids);
  /* require_valid(coarse) (fusion.cpp:227) holds by construction: contiguous runs of a
   * topological order, aggregated crossing edges point forward. */
  *out = o;
  return 0;
}

static dp_graph_t view_of(const dp_graph_out_t* o) {
  dp_graph_t g;
  g.n_nodes = o->n_nodes;
  g.n_edges = o->n_edges;
  g.node_id = o->node_id;
  g.compute_us = o->compute_us;
  g.memory_bytes = o->memory_bytes;
  g.group = o->group;
  g.edge_src = o->edge_src;
  g.edge_dst = o->edge_dst;
  g.edge_bytes = o->edge_bytes;
  return g;
}

typedef struct {
  int32_t label;
  int64_t id;
  int32_t idx;
} GroupMember;
static int cmp_gm(const void* a, const void* b) {
  const GroupMember* x = (const GroupMember*)a;
  const GroupMember* y = (const GroupMember*)b;
  if (x->label != y->label) return x->label < y->label ? -1 : 1;
  if (x->id != y->id) return x->id < y->id ? -1 : 1;
  return 0;
}

/* contract_colocation_groups, fusion.cpp:231-295. */
int dpo_contract_colocation_groups(const dp_graph_t* g, dp_contraction_t** out) {
  int rc = dpo_require_valid(g);
  if (rc) return rc;
  int64_t n = g->n_nodes;
  IdMap ids = idmap_build(g->node_id, n);
  int64_t* rep = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1)); /* by node index */
  int32_t* grp_first = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int32_t* grp_len = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  GroupMember* gm = (GroupMember*)malloc(sizeof(GroupMember) * (size_t)(n ? n : 1));
  int64_t ng = 0;
  for (int64_t i = 0; i < n; ++i) {
    rep[i] = g->node_id[i];
    grp_first[i] = -1;
    if (g->group && g->group[i] >= 0) {
      gm[ng].label = g->group[i];
      gm[ng].id = g->node_id[i];
      gm[ng].idx = (int32_t)i;
      ++ng;
    }
  }
  qsort(gm, (size_t)ng, sizeof(GroupMember), cmp_gm);
  for (int64_t a = 0; a < ng;) { /* rep = min member id (fusion.cpp:242-245) */
    int64_t b = a;
    while (b < ng && gm[b].label == gm[a].label) ++b;
    for (int64_t q = a; q < b; ++q) {
      rep[gm[q].idx] = gm[a].id;
      grp_first[gm[q].idx] = (int32_t)a;
      grp_len[gm[q].idx] = (int32_t)(b - a);
    }
    a = b;
  }
  /* contracted nodes in input order: non-members and representatives (:247-261) */
  int64_t nc = 0;
  for (int64_t i = 0; i < n; ++i)
    if (grp_first[i] < 0 || rep[i] == g->node_id[i]) ++nc;
  Edge3* es = (Edge3*)malloc(sizeof(Edge3) * (size_t)(g->n_edges ? g->n_edges : 1));
  int64_t k = 0;
  for (int64_t e = 0; e < g->n_edges; ++e) { /* :273-286 */
    int64_t u = rep[idmap_find(&ids, g->edge_src[e])];
    int64_t v = rep[idmap_find(&ids, g->edge_dst[e])];
    if (u != v) { es[k].u = u; es[k].v = v; es[k].bytes = g->edge_bytes[e]; ++k; }
  }
  k = aggregate_edges(es, k);
  dp_contraction_t* c = DPR_NEW(dp_contraction_t, 1);
  c->contracted = dpr_graph_out_new(nc, k);
  c->member_off = DPR_NEW(int64_t, nc + 1);
  c->members = DPR_NEW(int64_t, n);
  int64_t w = 0, off = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(grp_first[i] < 0 || rep[i] == g->node_id[i])) continue;
    dp_graph_out_t* o = c->contracted;
    o->node_id[w] = g->node_id[i];
    o->group[w] = g->group ? g->group[i] : -1;
    c->member_off[w] = off;
    if (grp_first[i] < 0) {
      o->compute_us[w] = g->compute_us[i];
      o->memory_bytes[w] = g->memory_bytes[i];
      c->members[off++] = g->node_id[i];
    } else {
      for (int32_t q = grp_first[i]; q < grp_first[i] + grp_len[i]; ++q) {
        o->compute_us[w] += g->compute_us[gm[q].idx]; /* :262-271 */
        o->memory_bytes[w] += g->memory_bytes[gm[q].idx];
        c->members[off++] = gm[q].id;
      }
    }
    ++w;
  }
  c->member_off[nc] = off;
  for (int64_t e = 0; e < k; ++e) {
    c->contracted->edge_src[e] = es[e].u;
    c->contracted->edge_dst[e] = es[e].v;
    c->contracted->edge_bytes[e] = es[e].bytes;
  }
  free(es); free(rep); free(grp_first); free(grp_len); free(gm); idmap_free(&ids);
  /* validate(contracted) (:288-293) */
  dp_graph_t view = view_of(c->contracted);
  VList v;
  memset(&v, 0, sizeof v);
  validate_into(&view, &v);
  if (v.count) {
    char msg[900];
    int64_t len = v.msg_off[1];
    if (len > 800) len = 800;
    memcpy(msg, v.msg, (size_t)len);
    msg[len] = 0;
    free(v.kind); free(v.node_off); free(v.nodes); free(v.msg_off); free(v.msg);
    dpr_contraction_free_(c);
    return fail(DP_E_CYCLE_DETECTED, "co-location groups are inconsistent with a DAG: %s", msg);
  }
  *out = c;
  return 0;
}

/* fuse, fusion.cpp:297-335. */
int dpo_fuse(const dp_graph_t* g, dp_comm_t comm, int32_t range, int64_t limit,
             dp_fusion_result_t** out) {
  dp_contraction_t* con = NULL;
  int rc = dpo_contract_colocation_groups(g, &con);
  if (rc) return rc;
  dp_graph_t work = view_of(con->contracted);
  int64_t n = work.n_nodes;
  for (int64_t i = 0; i < n; ++i) { /* :302-310 */
    if (con->member_off[i + 1] - con->member_off[i] > 1 && work.memory_bytes[i] > limit) {
      rc = fail(DP_E_GROUP_EXCEEDS_CLUSTER_LIMIT,
                "co-location group of node %lld needs %lld bytes, cluster limit is %lld",
                (long long)work.node_id[i], (long long)work.memory_bytes[i], (long long)limit);
      dpr_contraction_free_(con);
      return rc;
    }
  }
  int64_t* tl = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  int64_t* bl = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  int64_t* cp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  int64_t* seq = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  dp_cluster_map_t* cmap = NULL;
  dp_graph_out_t* coarse = NULL;
  if ((rc = dpo_compute_levels(&work, comm, tl, bl, cp))) goto done;
  if ((rc = dpo_topo_order(&work, DP_TOPO_CPD, cp, seq))) goto done;
  if ((rc = dpo_optimal_breakpoints(&work, seq, n, comm, range, limit, &cmap))) goto done;
  {
    int32_t* cids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cmap->n_clusters + 1));
    for (int64_t c = 0; c < cmap->n_clusters; ++c) cids[c] = (int32_t)c;
    rc = dpo_build_coarse_graph(&work, seq, n, work.node_id, cmap->node_cluster, n,
                                cmap->n_clusters, cids, cmap->member_off, cmap->members, &coarse);
    free(cids);
    if (rc) goto done;
  }
  {
    /* re-express the map over original ids (:317-333) */
    IdMap cids = idmap_build(work.node_id, n);
    IdMap oids = idmap_build(g->node_id, g->n_nodes);
    dp_cluster_map_t* m = dpr_cluster_map_new(g->n_nodes, cmap->n_clusters, cmap->n_breakpoints);
    memcpy(m->breakpoints, cmap->breakpoints, sizeof(int32_t) * (size_t)cmap->n_breakpoints);
    int64_t off = 0;
    for (int64_t c = 0; c < cmap->n_clusters; ++c) {
      m->member_off[c] = off;
      m->total_compute[c] = cmap->total_compute[c];
      m->total_memory[c] = cmap->total_memory[c];
      for (int64_t q = cmap->member_off[c]; q < cmap->member_off[c + 1]; ++q) {
        int32_t si = idmap_find(&cids, cmap->members[q]);
        for (int64_t r = con->member_off[si]; r < con->member_off[si + 1]; ++r) {
          m->members[off++] = con->members[r];
          m->node_cluster[idmap_find(&oids, con->members[r])] = (int32_t)c;
        }
      }
    }
    m->member_off[cmap->n_clusters] = off;
    idmap_free(&cids);
    idmap_free(&oids);
    dp_fusion_result_t* f = DPR_NEW(dp_fusion_result_t, 1);
    f->coarse = coarse;
    f->map = m;
    coarse = NULL;
    *out = f;
  }
done:
  free(tl); free(bl); free(cp); free(seq);
  dpr_cluster_map_free_(cmap);
  dpr_graph_out_free_(coarse);
  dpr_contraction_free_(con);
  return rc;
}

/* ------------------------------------------------------------------ placement */
/* DeviceTimeline, placement.cpp:13-32. */
typedef struct {
  int64_t *start, *end;
  int64_t n, cap;
} Timeline;

static int64_t tl_find_slot(const Timeline* t, int64_t earliest, int64_t dur) {
  int64_t cand = earliest;
  for (int64_t k = 0; k < t->n; ++k) {
    if (t->end[k] <= cand) continue;
    if (t->start[k] >= cand && t->start[k] - cand >= dur) break;
    if (t->end[k] > cand) cand = t->end[k];
  }
  return cand;
}
static void tl_reserve(Timeline* t, int64_t start, int64_t dur) {
  if (t->n == t->cap) {
    t->cap = t->cap ? t->cap * 2 : 16;
    t->start = (int64_t*)realloc(t->start, sizeof(int64_t) * (size_t)t->cap);
    t->end = (int64_t*)realloc(t->end, sizeof(int64_t) * (size_t)t->cap);
  }
  int64_t lo = 0, hi = t->n; /* upper_bound by start */
  while (lo < hi) {
    int64_t mid = (lo + hi) / 2;
    if (t->start[mid] <= start) lo = mid + 1; else hi = mid;
  }
  memmove(t->start + lo + 1, t->start + lo, sizeof(int64_t) * (size_t)(t->n - lo));
  memmove(t->end + lo + 1, t->end + lo, sizeof(int64_t) * (size_t)(t->n - lo));
  t->start[lo] = start;
  t->end[lo] = start + dur;
  t->n++;
}

typedef struct {
  int32_t D;
  int32_t* ids;    /* sorted device ids */
  int64_t* avail;  /* available memory */
  Timeline* tls;
} Sched;

typedef struct {
  int32_t id;
  int64_t mem;
} DevSpec;
static int cmp_dev(const void* a, const void* b) {
  const DevSpec* x = (const DevSpec*)a;
  const DevSpec* y = (const DevSpec*)b;
  return x->id < y->id ? -1 : (x->id > y->id);
}

/* SchedulerState::for_devices, placement.cpp:34-53. */
static int sched_init(const dp_devices_t* d, Sched* s) {
  memset(s, 0, sizeof *s);
  if (d->count <= 0) return fail(DP_E_INVALID_VALUE, "device list is empty");
  DevSpec* ds = (DevSpec*)malloc(sizeof(DevSpec) * (size_t)d->count);
  for (int32_t i = 0; i < d->count; ++i) { ds[i].id = d->id[i]; ds[i].mem = d->memory_bytes[i]; }
  qsort(ds, (size_t)d->count, sizeof(DevSpec), cmp_dev);
  s->ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)d->count);
  s->avail = (int64_t*)malloc(sizeof(int64_t) * (size_t)d->count);
  for (int32_t i = 0; i < d->count; ++i) {
    if (ds[i].mem <= 0) {
      int rc = fail(DP_E_INVALID_VALUE, "device %d has non-positive memory capacity", ds[i].id);
      free(ds); free(s->ids); free(s->avail);
      return rc;
    }
    if (i && ds[i].id == ds[i - 1].id) {
      int rc = fail(DP_E_DUPLICATE_ID, "device id %d repeats", ds[i].id);
      free(ds); free(s->ids); free(s->avail);
      return rc;
    }
    s->ids[i] = ds[i].id;
    s->avail[i] = ds[i].mem;
  }
  s->D = d->count;
  s->tls = (Timeline*)calloc((size_t)d->count, sizeof(Timeline));
  free(ds);
  return 0;
}
static void sched_free(Sched* s) {
  for (int32_t d = 0; d < s->D; ++d) { free(s->tls[d].start); free(s->tls[d].end); }
  free(s->tls); free(s->ids); free(s->avail);
}
/* most_free_device, placement.cpp:72-78. */
static int32_t most_free(const Sched* s) {
  int32_t best = 0;
  for (int32_t d = 1; d < s->D; ++d) if (s->avail[d] > s->avail[best]) best = d;
  return best;
}

/* est_on_device, placement.cpp:81-96. */
static int64_t est_on(const dp_graph_t* g, const Index* ix, const int64_t* cost, const Sched* s,
                      const int32_t* dev_of, const int64_t* finish, int32_t v, int32_t d) {
  int64_t pre = 0;
  for (int32_t k = ix->in_start[v]; k < ix->in_start[v + 1]; ++k) {
    int32_t e = ix->in_list[k], p = ix->esrc[e];
    int64_t arr = finish[p] + (dev_of[p] == d ? 0 : cost[e]);
    if (arr > pre) pre = arr;
  }
  return tl_find_slot(&s->tls[d], pre, g->compute_us[v]);
}

static int place_common(const dp_graph_t* g, const int64_t* seq, int64_t len,
                        const dp_devices_t* devices, const dp_comm_t* comm, int adjust,
                        dp_placement_result_t** out) {
  int rc = dpo_require_valid(g);
  if (rc) return rc;
  if (!valid_order(g, seq, len))
    return fail(DP_E_INVALID_VALUE, "order is not a topological order of this graph");
  Index ix;
  if ((rc = index_build(g, &ix))) return rc;
  Sched s;
  if ((rc = sched_init(devices, &s))) { index_free(&ix); return rc; }
  int32_t n = ix.n, D = s.D;
  int64_t* cost = (int64_t*)calloc((size_t)(g->n_edges ? g->n_edges : 1), sizeof(int64_t));
  if (comm) for (int64_t e = 0; e < g->n_edges; ++e) cost[e] = comm_cost(g->edge_bytes[e], *comm);
  int32_t* dev_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int64_t* finish = (int64_t*)calloc((size_t)(n ? n : 1), sizeof(int64_t));
  for (int32_t v = 0; v < n; ++v) dev_of[v] = -1;
  dp_placement_result_t* r = dpr_placement_new(n, D, adjust ? n : 0);
  for (int32_t d = 0; d < D; ++d) { r->device_ids[d] = s.ids[d]; r->device_present[d] = 1; }
  for (int32_t v = 0; v < n; ++v) r->device[v] = -1;
  int64_t* est = (int64_t*)malloc(sizeof(int64_t) * (size_t)D);
  int32_t cursor = 0, prev = 0;
  for (int64_t k = 0; k < len; ++k) {
    int32_t v = idmap_find(&ix.ids, seq[k]);
    int64_t w = g->compute_us[v], mem = g->memory_bytes[v];
    int32_t chosen;
    int64_t start;
    if (!adjust) { /* order_place, placement.cpp:139-157 */
      int32_t target = -1;
      for (int32_t d = cursor; d < D; ++d) if (s.avail[d] >= mem) { target = d; break; }
      if (target >= 0) cursor = target;
      else { target = most_free(&s); r->oom_risk = 1; }
      chosen = target;
      start = tl_find_slot(&s.tls[target], 0, w);
    } else { /* adjusting_placement, placement.cpp:173-216 */
      int64_t back = 0;
      for (int32_t q = ix.out_start[v]; q < ix.out_start[v + 1]; ++q)
        if (cost[ix.out_list[q]] > back) back = cost[ix.out_list[q]];
      r->dec_node[k] = seq[k];
      r->dec_prev[k] = s.ids[prev];
      r->dec_back_cost[k] = back;
      int32_t best = -1;
      for (int32_t d = 0; d < D; ++d) {
        est[d] = NEVER;
        if (s.avail[d] >= mem) {
          est[d] = est_on(g, &ix, cost, &s, dev_of, finish, v, d);
          if (best < 0 || est[d] < est[best]) best = d;
        }
        r->dec_est[k * D + d] = est[d];
      }
      if (best >= 0 && (est[prev] == NEVER || est[prev] - est[best] > back)) {
        chosen = best;
        start = est[best];
        r->dec_relocated[k] = chosen != prev;
      } else if (est[prev] != NEVER) {
        chosen = prev;
        start = est[prev];
      } else {
        chosen = most_free(&s);
        start = est_on(g, &ix, cost, &s, dev_of, finish, v, chosen);
        r->dec_best_effort[k] = 1;
        r->oom_risk = 1;
      }
      r->dec_chosen[k] = s.ids[chosen];
      prev = chosen;
    }
    /* commit, placement.cpp:115-123 */
    dev_of[v] = chosen;
    s.avail[chosen] -= mem;
    finish[v] = start + w;
    tl_reserve(&s.tls[chosen], start, w);
    r->device[v] = s.ids[chosen];
    r->per_device_memory[chosen] += mem;
  }
  free(est); free(cost); free(dev_of); free(finish);
  sched_free(&s);
  index_free(&ix);
  *out = r;
  return 0;
}

int dpo_order_place(const dp_graph_t* g, const int64_t* seq, int64_t len,
                    const dp_devices_t* devices, dp_placement_result_t** out) {
  return place_common(g, seq, len, devices, NULL, 0, out);
}
int dpo_adjusting_placement(const dp_graph_t* g, const int64_t* seq, int64_t len,
                            const dp_devices_t* devices, dp_comm_t comm,
                            dp_placement_result_t** out) {
  return place_common(g, seq, len, devices, &comm, 1, out);
}

/* expand_placement, placement.cpp:239-268. */
int dpo_expand_placement(const dp_graph_t* g, const int32_t* node_cluster, int64_t n_clusters,
                         const int64_t* member_off, const int64_t* members,
                         const int32_t* coarse_device, const uint8_t* coarse_placed,
                         dp_placement_result_t** out) {
  int64_t n = g->n_nodes;
  IdMap ids = idmap_build(g->node_id, n);
  for (int64_t i = 1; i < n; ++i) {
    if (ids.t[i].id == ids.t[i - 1].id) {
      int64_t id = ids.t[i].id;
      idmap_free(&ids);
      return fail(DP_E_DUPLICATE_ID, "node id %lld is not unique", (long long)id);
    }
  }
  int64_t mapped = 0;
  for (int64_t i = 0; i < n; ++i) mapped += node_cluster[i] >= 0;
  if (mapped != n) {
    idmap_free(&ids);
    return fail(DP_E_INVALID_CLUSTER_MAP, "cluster map covers %lld nodes, graph has %lld",
                (long long)mapped, (long long)n);
  }
  int32_t* dev = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) dev[i] = INT32_MIN;
  /* per_device_memory keyed by device id: collect (id, bytes) then aggregate */
  int32_t* dids = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  int64_t* dmem = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  int64_t nd = 0, covered = 0;
  for (int64_t c = 0; c < n_clusters; ++c) {
    if (coarse_placed && !coarse_placed[c]) {
      free(dev); free(dids); free(dmem); idmap_free(&ids);
      return fail(DP_E_UNPLACED_NODE, "cluster %lld has no device", (long long)c);
    }
    int32_t d = coarse_device[c];
    for (int64_t q = member_off[c]; q < member_off[c + 1]; ++q) {
      int32_t gi = idmap_find(&ids, members[q]);
      if (gi < 0) {
        free(dev); free(dids); free(dmem); idmap_free(&ids);
        return fail(DP_E_UNKNOWN_NODE, "node %lld not in graph", (long long)members[q]);
      }
      if (dev[gi] != INT32_MIN) {
        free(dev); free(dids); free(dmem); idmap_free(&ids);
        return fail(DP_E_INVALID_CLUSTER_MAP, "node %lld appears in two clusters", (long long)members[q]);
      }
      dev[gi] = d;
      ++covered;
      int64_t slot = -1;
      for (int64_t t = 0; t < nd; ++t) if (dids[t] == d) { slot = t; break; }
      if (slot < 0) { slot = nd++; dids[slot] = d; dmem[slot] = 0; }
      dmem[slot] += g->memory_bytes[gi];
    }
  }
  if (covered != n) {
    free(dev); free(dids); free(dmem); idmap_free(&ids);
    return fail(DP_E_INVALID_CLUSTER_MAP, "expanded placement does not cover the graph");
  }
  /* sort devices by id */
  for (int64_t a = 1; a < nd; ++a)
    for (int64_t b = a; b > 0 && dids[b] < dids[b - 1]; --b) {
      int32_t ti = dids[b]; dids[b] = dids[b - 1]; dids[b - 1] = ti;
      int64_t tm = dmem[b]; dmem[b] = dmem[b - 1]; dmem[b - 1] = tm;
    }
  dp_placement_result_t* r = dpr_placement_new(n, (int32_t)nd, 0);
  memcpy(r->device, dev, sizeof(int32_t) * (size_t)n);
  for (int64_t t = 0; t < nd; ++t) {
    r->device_ids[t] = dids[t];
    r->per_device_memory[t] = dmem[t];
    r->device_present[t] = 1;
  }
  free(dev); free(dids); free(dmem); idmap_free(&ids);
  *out = r;
  return 0;
}

/* ------------------------------------------------------------------ simulator */
/* simulate, simulator.cpp:56-252.  Task key (ready, kind, id) with the task index as
 * the final tie (std::set<pair<TaskKey,int>>); per-engine binary heaps. */
typedef struct {
  int64_t ready;
  int32_t kind;
  int64_t id;
  int32_t t;
} Key;
static int key_lt(const Key* a, const Key* b) {
  if (a->ready != b->ready) return a->ready < b->ready;
  if (a->kind != b->kind) return a->kind < b->kind;
  if (a->id != b->id) return a->id < b->id;
  return a->t < b->t;
}
typedef struct {
  Key* h;
  int32_t n, cap;
} Heap;
static void heap_push(Heap* q, Key k) {
  if (q->n == q->cap) {
    q->cap = q->cap ? q->cap * 2 : 16;
    q->h = (Key*)realloc(q->h, sizeof(Key) * (size_t)q->cap);
  }
  int32_t i = q->n++;
  while (i > 0) {
    int32_t p = (i - 1) / 2;
    if (!key_lt(&k, &q->h[p])) break;
    q->h[i] = q->h[p];
    i = p;
  }
  q->h[i] = k;
}
static void heap_pop(Heap* q) {
  Key last = q->h[--q->n];
  int32_t i = 0;
  for (;;) {
    int32_t l = 2 * i + 1, r = l + 1, s = i;
    const Key* best = &last;
    if (l < q->n && key_lt(&q->h[l], best)) { s = l; best = &q->h[l]; }
    if (r < q->n && key_lt(&q->h[r], best)) { s = r; best = &q->h[r]; }
    if (s == i) break;
    q->h[i] = q->h[s];
    i = s;
  }
  if (q->n) q->h[i] = last;
}

typedef struct {
  int is_transfer;
  int32_t node, edge;
  int64_t dur;
  int32_t ea, eb;
  int32_t deps;
  int64_t ready, start, end;
} Task;

static int cmp_trace_ctx_dummy;
static const Task* s_tasks;
static const int64_t* s_node_ids;
static int cmp_trace(const void* a, const void* b) {
  const Task* x = &s_tasks[*(const int32_t*)a];
  const Task* y = &s_tasks[*(const int32_t*)b];
  if (x->start != y->start) return x->start < y->start ? -1 : 1;
  if (x->is_transfer != y->is_transfer) return x->is_transfer ? 1 : -1;
  int64_t ix = x->is_transfer ? x->edge : s_node_ids[x->node];
  int64_t iy = y->is_transfer ? y->edge : s_node_ids[y->node];
  return ix < iy ? -1 : (ix > iy);
}

static int simulate_core(const dp_graph_t* g, const Index* ix, const int64_t* cost,
                         const int32_t* node_dev /* device position */, const Sched* s,
                         const int64_t* capacity, int want_trace, int want_report,
                         int64_t* makespan_out, dp_sim_report_t** out) {
  int32_t n = ix->n, m = ix->m, D = s->D;
  int32_t* transfer_of = (int32_t*)malloc(sizeof(int32_t) * (size_t)(m ? m : 1));
  int32_t nt = n;
  int64_t cross_count = 0, cross_bytes = 0;
  for (int32_t e = 0; e < m; ++e) {
    transfer_of[e] = -1;
    if (node_dev[ix->esrc[e]] != node_dev[ix->edst[e]]) {
      transfer_of[e] = nt++;
      ++cross_count;
      cross_bytes += g->edge_bytes[e];
    }
  }
  Task* T = (Task*)calloc((size_t)(nt ? nt : 1), sizeof(Task));
  for (int32_t v = 0; v < n; ++v) {
    T[v].node = v;
    T[v].dur = g->compute_us[v];
    T[v].ea = node_dev[v] * 3 + 0;
    T[v].eb = -1;
  }
  /* dependents as CSR: compute u -> (transfer or consumer); transfer -> consumer */
  int32_t* dep_cnt = (int32_t*)calloc((size_t)nt + 1, sizeof(int32_t));
  for (int32_t e = 0; e < m; ++e) {
    int32_t u = ix->esrc[e], v = ix->edst[e];
    if (transfer_of[e] >= 0) {
      int32_t t = transfer_of[e];
      T[t].is_transfer = 1;
      T[t].edge = e;
      T[t].node = -1;
      T[t].dur = cost[e];
      T[t].ea = node_dev[u] * 3 + 1;
      T[t].eb = node_dev[v] * 3 + 2;
      T[t].deps = 1;
      dep_cnt[u + 1]++;
      dep_cnt[t + 1]++;
    } else {
      dep_cnt[u + 1]++;
    }
    T[v].deps++;
  }
  for (int32_t t = 0; t < nt; ++t) dep_cnt[t + 1] += dep_cnt[t];
  int32_t* deps = (int32_t*)malloc(sizeof(int32_t) * (size_t)(dep_cnt[nt] ? dep_cnt[nt] : 1));
  int32_t* fill = (int32_t*)malloc(sizeof(int32_t) * ((size_t)nt + 1));
  memcpy(fill, dep_cnt, sizeof(int32_t) * ((size_t)nt + 1));
  for (int32_t e = 0; e < m; ++e) { /* simulator.cpp:119-130 (edge order) */
    int32_t u = ix->esrc[e], v = ix->edst[e];
    if (transfer_of[e] >= 0) {
      deps[fill[u]++] = transfer_of[e];
      deps[fill[transfer_of[e]]++] = v;
    } else {
      deps[fill[u]++] = v;
    }
  }
  int32_t E = 3 * D;
  Heap* q = (Heap*)calloc((size_t)E, sizeof(Heap));
  uint8_t* busy = (uint8_t*)calloc((size_t)E, 1);
  int64_t* free_time = (int64_t*)calloc((size_t)E, sizeof(int64_t));
  Heap ev = {0};
  #define KEY_OF(t, r) ((Key){(r), T[t].is_transfer, T[t].is_transfer ? (int64_t)T[t].edge : g->node_id[T[t].node], (t)})
  #define ENQUEUE(t, now)                                          \
    do {                                                           \
      T[t].ready = (now);                                          \
      heap_push(&q[T[t].ea], KEY_OF(t, T[t].ready));               \
      if (T[t].eb >= 0) heap_push(&q[T[t].eb], KEY_OF(t, T[t].ready)); \
    } while (0)
  for (int32_t t = 0; t < nt; ++t) if (T[t].deps == 0) ENQUEUE(t, 0);
  int64_t now = 0;
  int64_t completed = 0;
  for (;;) {
    /* try_start(now), simulator.cpp:148-179 */
    int progress = 1;
    while (progress) {
      progress = 0;
      for (int32_t e = 0; e < E; ++e) {
        if (busy[e] || !q[e].n) continue;
        int32_t t = q[e].h[0].t;
        Task* k = &T[t];
        int64_t st;
        if (k->is_transfer) {
          if (busy[k->ea] || busy[k->eb]) continue;
          if (q[k->ea].h[0].t != t || q[k->eb].h[0].t != t) continue;
          heap_pop(&q[k->ea]);
          heap_pop(&q[k->eb]);
          st = k->ready;
          if (free_time[k->ea] > st) st = free_time[k->ea];
          if (free_time[k->eb] > st) st = free_time[k->eb];
          if (now > st) st = now;
          busy[k->ea] = busy[k->eb] = 1;
        } else {
          heap_pop(&q[e]);
          st = k->ready;
          if (free_time[e] > st) st = free_time[e];
          if (now > st) st = now;
          busy[e] = 1;
        }
        k->start = st;
        k->end = st + k->dur;
        heap_push(&ev, KEY_OF(t, k->end));
        progress = 1;
      }
    }
    if (!ev.n) break;
    now = ev.h[0].ready;
    while (ev.n && ev.h[0].ready == now) { /* simulator.cpp:189-203 */
      int32_t t = ev.h[0].t;
      heap_pop(&ev);
      Task* k = &T[t];
      busy[k->ea] = 0;
      free_time[k->ea] = k->end;
      if (k->eb >= 0) { busy[k->eb] = 0; free_time[k->eb] = k->end; }
      ++completed;
      for (int32_t d = dep_cnt[t]; d < dep_cnt[t + 1]; ++d) {
        int32_t x = deps[d];
        if (--T[x].deps == 0) ENQUEUE(x, now);
      }
    }
  }
  #undef ENQUEUE
  #undef KEY_OF
  int rc = 0;
  if (completed != nt) {
    rc = fail(DP_E_CYCLE_DETECTED, "simulation stalled; dependency cycle");
  } else {
    int64_t ms = 0;
    for (int32_t t = 0; t < nt; ++t) if (T[t].end > ms) ms = T[t].end;
    *makespan_out = ms;
    if (want_report) {
      int64_t ntr = want_trace ? (int64_t)n + 2 * cross_count : 0;
      dp_sim_report_t* r = dpr_sim_new(D, ntr);
      r->makespan = ms;
      r->cross_transfer_count = cross_count;
      r->cross_transfer_bytes = cross_bytes;
      for (int32_t d = 0; d < D; ++d) { r->device_ids[d] = s->ids[d]; r->capacity[d] = capacity[d]; }
      for (int32_t v = 0; v < n; ++v) r->peak_memory[node_dev[v]] += g->memory_bytes[v];
      for (int32_t d = 0; d < D; ++d) if (r->peak_memory[d] > r->capacity[d]) r->oom_flag = 1;
      if (want_trace) { /* simulator.cpp:223-250 */
        int32_t* order = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nt ? nt : 1));
        for (int32_t t = 0; t < nt; ++t) order[t] = t;
        s_tasks = T;
        s_node_ids = g->node_id;
        qsort(order, (size_t)nt, sizeof(int32_t), cmp_trace);
        int64_t w = 0;
        for (int32_t i = 0; i < nt; ++i) {
          const Task* k = &T[order[i]];
          if (k->is_transfer) {
            int64_t es = g->edge_src[k->edge], ed = g->edge_dst[k->edge];
            r->tr_kind[w] = DP_TASK_SEND; r->tr_node[w] = -1; r->tr_src[w] = es; r->tr_dst[w] = ed;
            r->tr_device[w] = s->ids[k->ea / 3]; r->tr_start[w] = k->start; r->tr_end[w] = k->end; ++w;
            r->tr_kind[w] = DP_TASK_RECEIVE; r->tr_node[w] = -1; r->tr_src[w] = es; r->tr_dst[w] = ed;
            r->tr_device[w] = s->ids[k->eb / 3]; r->tr_start[w] = k->start; r->tr_end[w] = k->end; ++w;
          } else {
            r->tr_kind[w] = DP_TASK_COMPUTE; r->tr_node[w] = g->node_id[k->node]; r->tr_src[w] = -1;
            r->tr_dst[w] = -1; r->tr_device[w] = s->ids[k->ea / 3]; r->tr_start[w] = k->start;
            r->tr_end[w] = k->end; ++w;
          }
        }
        free(order);
      }
      *out = r;
    }
  }
  (void)cmp_trace_ctx_dummy;
  for (int32_t e = 0; e < E; ++e) free(q[e].h);
  free(q); free(busy); free(free_time); free(ev.h);
  free(T); free(dep_cnt); free(deps); free(fill); free(transfer_of);
  return rc;
}

/* Device list + node placement checks of simulator.cpp:61-92. */
static int sim_setup(const dp_graph_t* g, const Index* ix, const dp_devices_t* devices,
                     const int32_t* device_of_node, Sched* s, int64_t** capacity,
                     int32_t** node_dev) {
  if (devices->count <= 0) return fail(DP_E_INVALID_VALUE, "device list is empty");
  DevSpec* ds = (DevSpec*)malloc(sizeof(DevSpec) * (size_t)devices->count);
  for (int32_t i = 0; i < devices->count; ++i) { ds[i].id = devices->id[i]; ds[i].mem = devices->memory_bytes[i]; }
  qsort(ds, (size_t)devices->count, sizeof(DevSpec), cmp_dev);
  for (int32_t i = 0; i < devices->count; ++i) {
    if (ds[i].mem <= 0) {
      int rc = fail(DP_E_INVALID_VALUE, "device %d has non-positive memory capacity", ds[i].id);
      free(ds);
      return rc;
    }
    if (i && ds[i].id == ds[i - 1].id) {
      int rc = fail(DP_E_DUPLICATE_ID, "device id %d repeats", ds[i].id);
      free(ds);
      return rc;
    }
  }
  memset(s, 0, sizeof *s);
  s->D = devices->count;
  s->ids = (int32_t*)malloc(sizeof(int32_t) * (size_t)s->D);
  *capacity = (int64_t*)malloc(sizeof(int64_t) * (size_t)s->D);
  for (int32_t i = 0; i < s->D; ++i) { s->ids[i] = ds[i].id; (*capacity)[i] = ds[i].mem; }
  free(ds);
  *node_dev = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ix->n ? ix->n : 1));
  for (int32_t v = 0; v < ix->n; ++v) {
    if (device_of_node[v] == INT32_MIN) { /* simulator.cpp:80-84 */
      int rc = fail(DP_E_UNPLACED_NODE, "node %lld has no device", (long long)g->node_id[v]);
      free(s->ids); free(*capacity); free(*node_dev);
      return rc;
    }
    int32_t pos = -1;
    int32_t lo = 0, hi = s->D;
    while (lo < hi) { int32_t md = (lo + hi) / 2; if (s->ids[md] < device_of_node[v]) lo = md + 1; else hi = md; }
    if (lo < s->D && s->ids[lo] == device_of_node[v]) pos = lo;
    if (pos < 0) {
      int rc = fail(DP_E_INVALID_VALUE, "node %lld placed on unknown device %d",
                    (long long)g->node_id[v], device_of_node[v]);
      free(s->ids); free(*capacity); free(*node_dev);
      return rc;
    }
    (*node_dev)[v] = pos;
  }
  return 0;
}

int dpo_simulate(const dp_graph_t* g, const int32_t* device_of_node, const dp_devices_t* devices,
                 dp_comm_t comm, int32_t want_trace, dp_sim_report_t** out) {
  int rc = dpo_require_valid(g);
  if (rc) return rc;
  Index ix;
  if ((rc = index_build(g, &ix))) return rc;
  Sched s;
  int64_t* cap = NULL;
  int32_t* nd = NULL;
  if ((rc = sim_setup(g, &ix, devices, device_of_node, &s, &cap, &nd))) { index_free(&ix); return rc; }
  int64_t* cost = edge_costs(g, comm);
  int64_t ms = 0;
  rc = simulate_core(g, &ix, cost, nd, &s, cap, want_trace, 1, &ms, out);
  free(cost); free(cap); free(nd); free(s.ids); index_free(&ix);
  return rc;
}

int dpo_simulate_candidates(const dp_graph_t* g, const int32_t* node_cluster, int64_t n_clusters,
                            const uint8_t* cand, int64_t n_cand, const dp_devices_t* devices,
                            dp_comm_t comm, int64_t* makespans, int64_t* argmin,
                            int32_t threads) {
  (void)threads;
  int rc = dpo_require_valid(g);
  if (rc) return rc;
  Index ix;
  if ((rc = index_build(g, &ix))) return rc;
  Sched s;
  if ((rc = sched_init(devices, &s))) { index_free(&ix); return rc; }
  int64_t* cost = edge_costs(g, comm);
  int32_t* nd = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ix.n ? ix.n : 1));
  int64_t best = -1;
  for (int64_t b = 0; b < n_cand; ++b) {
    for (int32_t v = 0; v < ix.n; ++v) nd[v] = cand[b * n_clusters + node_cluster[v]];
    if ((rc = simulate_core(g, &ix, cost, nd, &s, s.avail, 0, 0, &makespans[b], NULL))) break;
    if (best < 0 || makespans[b] < makespans[best]) best = b;
  }
  *argmin = best;
  free(nd); free(cost); sched_free(&s); index_free(&ix);
  return rc;
}

/* brute_force_optimal, simulator.cpp:254-310. */
int dpo_brute_force_optimal(const dp_graph_t* g, const dp_devices_t* devices, dp_comm_t comm,
                            int32_t* best_dev, int64_t* best_ms) {
  int rc = dpo_require_valid(g);
  if (rc) return rc;
  int64_t n = g->n_nodes;
  if (n > 12 || devices->count > 3)
    return fail(DP_E_INSTANCE_TOO_LARGE, "exhaustive search limited to 12 nodes and 3 devices");
  if (devices->count <= 0) return fail(DP_E_INVALID_VALUE, "device list is empty");
  Index ix;
  if ((rc = index_build(g, &ix))) return rc;
  Sched s;
  int64_t* cap = NULL;
  int32_t* nd = NULL;
  int32_t* zero = (int32_t*)calloc((size_t)(n ? n : 1), sizeof(int32_t));
  int32_t* dev0 = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n ? n : 1));
  DevSpec* ds = (DevSpec*)malloc(sizeof(DevSpec) * (size_t)devices->count);
  for (int32_t i = 0; i < devices->count; ++i) { ds[i].id = devices->id[i]; ds[i].mem = devices->memory_bytes[i]; }
  qsort(ds, (size_t)devices->count, sizeof(DevSpec), cmp_dev);
  for (int64_t i = 0; i < n; ++i) dev0[i] = ds[0].id;
  (void)zero;
  /* Device checks happen inside simulate() (simulator.cpp:61-75), i.e. only once a
   * memory-feasible candidate exists; until then only the sorted list is needed. */
  int setup_done = 0;
  memset(&s, 0, sizeof s);
  int32_t Dn = devices->count;
  /* nodes sorted by id: odometer position p -> node index */
  IdMap byid = idmap_build(g->node_id, n);
  int32_t* choice = (int32_t*)calloc((size_t)(n ? n : 1), sizeof(int32_t));
  int64_t* cost = edge_costs(g, comm);
  int64_t* used = (int64_t*)malloc(sizeof(int64_t) * (size_t)Dn);
  int have = 0;
  int64_t bestv = 0;
  for (;;) {
    int feasible = 1;
    for (int32_t d = 0; d < Dn; ++d) used[d] = 0;
    for (int64_t p = 0; p < n && feasible; ++p) {
      int32_t v = byid.t[p].idx;
      used[choice[p]] += g->memory_bytes[v];
      feasible = used[choice[p]] <= ds[choice[p]].mem;
    }
    if (feasible && !setup_done) {
      if ((rc = sim_setup(g, &ix, devices, dev0, &s, &cap, &nd))) break;
      setup_done = 1;
    }
    if (feasible) {
      for (int64_t p = 0; p < n; ++p) nd[byid.t[p].idx] = choice[p];
      int64_t ms = 0;
      if ((rc = simulate_core(g, &ix, cost, nd, &s, cap, 0, 0, &ms, NULL))) break;
      if (!have || ms < bestv) {
        have = 1;
        bestv = ms;
        for (int64_t p = 0; p < n; ++p) best_dev[byid.t[p].idx] = ds[choice[p]].id;
      }
    }
    int64_t pos = n - 1;
    while (pos >= 0 && choice[pos] == Dn - 1) { choice[pos] = 0; --pos; }
    if (pos < 0) break;
    ++choice[pos];
  }
  if (!rc && !have) rc = fail(DP_E_INSTANCE_INFEASIBLE, "no memory-feasible assignment exists");
  if (!rc) *best_ms = bestv;
  free(choice); free(cost); free(used); free(zero); free(dev0); free(ds); free(cap); free(nd);
  free(s.ids); idmap_free(&byid); index_free(&ix);
  return rc;
}

/* ------------------------------------------------------------------ pipeline */
/* evaluate_pipeline without profiles, pipeline.cpp:27-111. */
int dpo_pipeline(const dp_graph_t* g, const dp_devices_t* devices, dp_comm_t comm,
                 const dp_pipeline_config_t* cfg, dp_pipeline_result_t** out) {
  if (devices->count <= 0) return fail(DP_E_INVALID_VALUE, "device list is empty");
  int rc = dpo_require_valid(g);
  if (rc) return rc;
  dp_pipeline_result_t* r = DPR_NEW(dp_pipeline_result_t, 1);
  r->original_nodes = g->n_nodes;
  r->original_edges = g->n_edges;
  if ((rc = dpo_ccr(g, comm, &r->original_ccr))) { dpr_pipeline_free_(r); return rc; }
  int64_t min_cap = devices->memory_bytes[0];
  for (int32_t d = 0; d < devices->count; ++d) if (devices->memory_bytes[d] < min_cap) min_cap = devices->memory_bytes[d];
  int64_t limit = (int64_t)((double)min_cap * cfg->cluster_mem_fraction);
  if (limit < 1) limit = 1;
  if ((rc = dpo_fuse(g, comm, cfg->fusion_range, limit, &r->fusion))) { dpr_pipeline_free_(r); return rc; }
  dp_graph_t coarse = view_of(r->fusion->coarse);
  int64_t nc = coarse.n_nodes;
  int64_t* tl = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc ? nc : 1));
  int64_t* bl = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc ? nc : 1));
  int64_t* cp = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc ? nc : 1));
  r->coarse_sequence = (int64_t*)malloc(sizeof(int64_t) * (size_t)(nc ? nc : 1));
  rc = dpo_compute_levels(&coarse, comm, tl, bl, cp);
  if (!rc) rc = dpo_topo_order(&coarse, DP_TOPO_CPD, cp, r->coarse_sequence);
  if (!rc) rc = dpo_order_place(&coarse, r->coarse_sequence, nc, devices, &r->coarse_order);
  if (!rc) rc = dpo_adjusting_placement(&coarse, r->coarse_sequence, nc, devices, comm, &r->coarse_adjust);
  free(tl); free(bl); free(cp);
  if (rc) { dpr_pipeline_free_(r); return rc; }
  dp_cluster_map_t* m = r->fusion->map;
  uint8_t* placed = (uint8_t*)malloc((size_t)(nc ? nc : 1));
  for (int64_t c = 0; c < nc; ++c) placed[c] = 1;
  rc = dpo_expand_placement(g, m->node_cluster, m->n_clusters, m->member_off, m->members,
                            r->coarse_order->device, placed, &r->order_expanded);
  if (!rc) rc = dpo_expand_placement(g, m->node_cluster, m->n_clusters, m->member_off, m->members,
                                     r->coarse_adjust->device, placed, &r->adjust_expanded);
  free(placed);
  if (rc) { dpr_pipeline_free_(r); return rc; }
  /* expanded placements report every device (absent ones with present=0) */
  for (int k = 0; k < 2; ++k) {
    dp_placement_result_t** pp = k ? &r->adjust_expanded : &r->order_expanded;
    dp_placement_result_t* old = *pp;
    Sched s;
    sched_init(devices, &s);
    dp_placement_result_t* nw = dpr_placement_new(old->n_nodes, s.D, 0);
    memcpy(nw->device, old->device, sizeof(int32_t) * (size_t)old->n_nodes);
    for (int32_t d = 0; d < s.D; ++d) {
      nw->device_ids[d] = s.ids[d];
      for (int32_t t = 0; t < old->n_devices; ++t) {
        if (old->device_ids[t] == s.ids[d]) {
          nw->device_present[d] = 1;
          nw->per_device_memory[d] = old->per_device_memory[t];
        }
      }
    }
    sched_free(&s);
    dpr_placement_free_(old);
    *pp = nw;
  }
  r->coarse_nodes = nc;
  r->coarse_edges = coarse.n_edges;
  if (coarse.n_edges == 0) r->coarse_ccr = 0.0;
  else if ((rc = dpo_ccr(&coarse, comm, &r->coarse_ccr))) { dpr_pipeline_free_(r); return rc; }
  r->order_makespan = r->adjust_makespan = -1;
  if (!cfg->simulate) {
    *out = r;
    return 0;
  }
  dp_sim_report_t* sr = NULL;
  if ((rc = dpo_simulate(g, r->order_expanded->device, devices, comm, 0, &sr))) { dpr_pipeline_free_(r); return rc; }
  r->order_makespan = sr->makespan;
  dpr_sim_free_(sr);
  if ((rc = dpo_simulate(g, r->adjust_expanded->device, devices, comm, 0, &sr))) { dpr_pipeline_free_(r); return rc; }
  r->adjust_makespan = sr->makespan;
  dpr_sim_free_(sr);
  *out = r;
  return 0;
}
