"""Pure-Python model of the tree peel (paper_2208_00184_b200/csrc/fixpoint.cu) for small
graphs: the breadth-first order s0 built level by level, the preorder of its freeing
forest T0, the proof T(preorder(T0)) = T0, and the general fixed-point rounds
s <- preorder(T(s)) when the proof fails.  Test infrastructure: the CPU suite checks the
model against the oracle's peel (ordering.cpp:40-114) on seeded families, which pins the
algorithm the kernel implements; the GPU suite checks the kernel itself.
"""
from __future__ import annotations

import numpy as np


def tree_peel(n, src, dst, rank, max_rounds=10_000):
    """Stack-peel order (node indices) of the DAG with edges src[k] -> dst[k] whose
    comparator rank (0 = best) orders freed children and sources.  Returns
    (order, proof_held_first, rounds)."""
    outs = [[] for _ in range(n)]
    ins = [[] for _ in range(n)]
    for u, v in zip(src, dst):
        outs[u].append(v)
        ins[v].append(u)
    for r in outs:
        r.sort(key=lambda c: rank[c])
    roots = sorted((v for v in range(n) if not ins[v]), key=lambda v: rank[v])
    # 1: breadth-first order s0 with the freeing forest (best = s0 position of the parent)
    indeg = [len(ins[v]) for v in range(n)]
    best = [-1] * n
    seq0 = list(roots)
    levels = [(0, len(roots))]
    lb, le = 0, len(roots)
    while lb < le:
        for i in range(lb, le):
            for c in outs[seq0[i]]:
                best[c] = max(best[c], i)
                indeg[c] -= 1
        for i in range(lb, le):
            for c in outs[seq0[i]]:
                if best[c] == i and indeg[c] == 0:
                    seq0.append(c)
        lb, le = le, len(seq0)
        if le > lb:
            levels.append((lb, le))
    assert len(seq0) == n, "not a DAG"

    def preorder(is_child):
        size = [1] * n
        for b, e in reversed(levels):
            for i in range(b, e):
                v = seq0[i]
                size[v] = 1 + sum(size[c] for c in outs[v] if is_child(c, v, i))
        pre = [0] * n
        acc = 0
        for v in roots:
            pre[v] = acc
            acc += size[v]
        for b, e in levels:
            for i in range(b, e):
                v = seq0[i]
                a = pre[v] + 1
                for c in outs[v]:
                    if is_child(c, v, i):
                        pre[c] = a
                        a += size[c]
        return pre

    pos = preorder(lambda c, v, i: best[c] == i)
    ok = all(max(pos[u] for u in ins[v]) == pos[seq0[best[v]]] for v in range(n) if ins[v])
    rounds = 1
    if not ok:
        for _ in range(max_rounds):
            rounds += 1
            par = [max(ins[v], key=lambda u: pos[u]) if ins[v] else -1 for v in range(n)]
            nxt = preorder(lambda c, v, i: par[c] == v)
            if nxt == pos:
                break
            pos = nxt
        else:
            raise RuntimeError("no convergence within the round budget")
    order = [0] * n
    for v in range(n):
        order[pos[v]] = v
    return order, ok, rounds


def ranks_cpd(cpath, ids):
    """rank of each node index under (cpath desc, id asc) — cpd_topo's comparators."""
    o = np.lexsort((ids, -np.asarray(cpath)))
    r = np.empty(len(o), np.int64)
    r[o] = np.arange(len(o))
    return r


def ranks_dfs(ids):
    o = np.argsort(ids, kind="stable")
    r = np.empty(len(o), np.int64)
    r[o] = np.arange(len(o))
    return r
