"""ctypes mirror of include/dagplace_b200.h and a Python surface that reads like the
reference's C++ API (namespace dagplace, /root/reference/proj/include/dagplace/*.hpp).

`Backend` drives any library exporting the flat signature set of the header: the
product (libdagplace_b200.so, prefix ``dp_``, needs a dp_ctx_t) and — in tests only —
the CPU checkers (oracle/dp_oracle.h, prefixes ``dpo_`` / ``dpr_``).  Results come
back as numpy arrays / small dataclasses so parity tests can compare them directly.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

I64P = C.POINTER(C.c_int64)
I32P = C.POINTER(C.c_int32)
U8P = C.POINTER(C.c_uint8)

ERROR_KINDS = [
    "CycleDetected", "DanglingEdge", "DuplicateId", "DuplicateEdge", "InvalidValue",
    "ZeroComputeTime", "NoSuchEdge", "NodeExceedsClusterLimit", "GroupExceedsClusterLimit",
    "InfeasiblePartition", "InvalidClusterMap", "InsufficientSamples", "UnknownNode",
    "NodeUniverseMismatch", "UnplacedNode", "InstanceTooLarge", "InstanceInfeasible",
    "UnreachableTargetCcr", "ParseError",
]
TOPO_M, TOPO_DFS, TOPO_CPD = 0, 1, 2
UNPLACED = np.iinfo(np.int32).min
NEVER = np.iinfo(np.int64).max


class DagError(RuntimeError):
    """dagplace::DagError (error.hpp:37-47): `kind` is the ErrorKind name, str() is what()."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code
        self.kind = ERROR_KINDS[code - 1] if 1 <= code <= len(ERROR_KINDS) else f"abi:{code}"


class GraphC(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_edges", C.c_int64), ("node_id", I64P),
                ("compute_us", I64P), ("memory_bytes", I64P), ("group", I32P),
                ("edge_src", I64P), ("edge_dst", I64P), ("edge_bytes", I64P)]


class CommC(C.Structure):
    _fields_ = [("k_us_per_byte", C.c_double), ("b_us", C.c_double)]


class DevicesC(C.Structure):
    _fields_ = [("count", C.c_int32), ("id", I32P), ("memory_bytes", I64P)]


class ViolationsC(C.Structure):
    _fields_ = [("count", C.c_int64), ("kind", I32P), ("node_off", I64P), ("nodes", I64P),
                ("msg_off", I64P), ("msg", C.c_char_p)]


class GraphOutC(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("n_edges", C.c_int64), ("node_id", I64P),
                ("compute_us", I64P), ("memory_bytes", I64P), ("group", I32P),
                ("edge_src", I64P), ("edge_dst", I64P), ("edge_bytes", I64P)]


class ClusterMapC(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("node_cluster", I32P), ("n_clusters", C.c_int64),
                ("member_off", I64P), ("members", I64P), ("total_compute", I64P),
                ("total_memory", I64P), ("n_breakpoints", C.c_int64), ("breakpoints", I32P)]


class ContractionC(C.Structure):
    _fields_ = [("contracted", C.POINTER(GraphOutC)), ("member_off", I64P), ("members", I64P)]


class FusionC(C.Structure):
    _fields_ = [("coarse", C.POINTER(GraphOutC)), ("map", C.POINTER(ClusterMapC))]


class PlacementC(C.Structure):
    _fields_ = [("n_nodes", C.c_int64), ("device", I32P), ("n_devices", C.c_int32),
                ("device_ids", I32P), ("per_device_memory", I64P), ("device_present", U8P),
                ("oom_risk", C.c_int32), ("n_decisions", C.c_int64), ("dec_node", I64P),
                ("dec_prev", I32P), ("dec_back_cost", I64P), ("dec_est", I64P),
                ("dec_chosen", I32P), ("dec_relocated", U8P), ("dec_best_effort", U8P)]


class SimC(C.Structure):
    _fields_ = [("makespan", C.c_int64), ("cross_transfer_count", C.c_int64),
                ("cross_transfer_bytes", C.c_int64), ("oom_flag", C.c_int32),
                ("n_devices", C.c_int32), ("device_ids", I32P), ("peak_memory", I64P),
                ("capacity", I64P), ("n_trace", C.c_int64), ("tr_kind", I32P),
                ("tr_node", I64P), ("tr_src", I64P), ("tr_dst", I64P), ("tr_device", I32P),
                ("tr_start", I64P), ("tr_end", I64P)]


class PipelineCfgC(C.Structure):
    _fields_ = [("fusion_range", C.c_int32), ("cluster_mem_fraction", C.c_double),
                ("strategy", C.c_int32), ("simulate", C.c_int32)]


class PipelineC(C.Structure):
    _fields_ = [("original_nodes", C.c_int64), ("original_edges", C.c_int64),
                ("original_ccr", C.c_double), ("coarse_nodes", C.c_int64),
                ("coarse_edges", C.c_int64), ("coarse_ccr", C.c_double),
                ("fusion", C.POINTER(FusionC)), ("coarse_order", C.POINTER(PlacementC)),
                ("coarse_adjust", C.POINTER(PlacementC)),
                ("order_expanded", C.POINTER(PlacementC)),
                ("adjust_expanded", C.POINTER(PlacementC)), ("coarse_sequence", I64P),
                ("order_makespan", C.c_int64), ("adjust_makespan", C.c_int64),
                ("generation_ms", C.c_double), ("order_sim", C.c_void_p), ("adjust_sim", C.c_void_p)]


# ----------------------------------------------------------------- python-side types
@dataclass
class Graph:
    """ComputationGraph (graph.hpp:42-45) as SoA numpy arrays."""

    node_id: np.ndarray
    compute_us: np.ndarray
    memory_bytes: np.ndarray
    edge_src: np.ndarray
    edge_dst: np.ndarray
    edge_bytes: np.ndarray
    group: Optional[np.ndarray] = None

    def __post_init__(self):
        for f in ("node_id", "compute_us", "memory_bytes", "edge_src", "edge_dst", "edge_bytes"):
            setattr(self, f, np.ascontiguousarray(getattr(self, f), dtype=np.int64))
        if self.group is not None:
            self.group = np.ascontiguousarray(self.group, dtype=np.int32)

    @property
    def n(self) -> int:
        return int(self.node_id.shape[0])

    @property
    def m(self) -> int:
        return int(self.edge_src.shape[0])

    @staticmethod
    def make(nodes, edges, groups=None) -> "Graph":
        """make_graph (tests/support/test_util.hpp:32-42): nodes (id, compute[, memory=1])."""
        ids = [n[0] for n in nodes]
        comp = [n[1] for n in nodes]
        mem = [n[2] if len(n) > 2 else 1 for n in nodes]
        return Graph(np.array(ids, np.int64), np.array(comp, np.int64), np.array(mem, np.int64),
                     np.array([e[0] for e in edges], np.int64),
                     np.array([e[1] for e in edges], np.int64),
                     np.array([e[2] for e in edges], np.int64),
                     None if groups is None else np.array(groups, np.int32))

    def c(self) -> GraphC:
        g = GraphC()
        g.n_nodes, g.n_edges = self.n, self.m
        g.node_id = _p64(self.node_id)
        g.compute_us = _p64(self.compute_us)
        g.memory_bytes = _p64(self.memory_bytes)
        g.group = self.group.ctypes.data_as(I32P) if self.group is not None else None
        g.edge_src = _p64(self.edge_src)
        g.edge_dst = _p64(self.edge_dst)
        g.edge_bytes = _p64(self.edge_bytes)
        g._keep = self  # noqa: SLF001 — keep arrays alive
        return g


@dataclass
class Violation:
    kind: str
    message: str
    nodes: list


@dataclass
class ClusterMap:
    node_cluster: np.ndarray  # by node index
    members: list             # list of np arrays of ids, cluster order
    total_compute: np.ndarray
    total_memory: np.ndarray
    breakpoints: np.ndarray

    @property
    def n_clusters(self) -> int:
        return len(self.members)

    def member_arrays(self):
        off = np.zeros(len(self.members) + 1, np.int64)
        off[1:] = np.cumsum([len(m) for m in self.members])
        flat = np.concatenate(self.members).astype(np.int64) if self.members else np.zeros(0, np.int64)
        return off, flat


@dataclass
class Placement:
    device: np.ndarray                 # device id by node index (UNPLACED if absent)
    device_ids: np.ndarray             # sorted device ids
    per_device_memory: np.ndarray
    device_present: np.ndarray
    oom_risk: bool = False
    decisions: Optional[dict] = None   # adjusting_placement decision log (arrays)


@dataclass
class SimReport:
    makespan: int
    cross_transfer_count: int
    cross_transfer_bytes: int
    oom_flag: bool
    device_ids: np.ndarray
    peak_memory: np.ndarray
    capacity: np.ndarray
    trace: Optional[dict] = None


@dataclass
class PipelineReport:
    original_nodes: int
    original_edges: int
    original_ccr: float
    coarse_nodes: int
    coarse_edges: int
    coarse_ccr: float
    coarse: Graph
    map: ClusterMap
    coarse_sequence: np.ndarray
    coarse_order: Placement
    coarse_adjust: Placement
    order_expanded: Placement
    adjust_expanded: Placement
    order_makespan: int
    adjust_makespan: int
    generation_ms: float = 0.0
    extra: dict = field(default_factory=dict)


def _p64(a: np.ndarray):
    return a.ctypes.data_as(I64P)


def _arr(ptr, n, dtype):
    if n == 0 or not ptr:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def comm_c(comm) -> CommC:
    k, b = comm
    return CommC(float(k), float(b))


def devices_c(devices):
    """devices: list of (id, memory_bytes)."""
    ids = np.ascontiguousarray([d[0] for d in devices], dtype=np.int32)
    mem = np.ascontiguousarray([d[1] for d in devices], dtype=np.int64)
    d = DevicesC(len(devices), ids.ctypes.data_as(I32P), mem.ctypes.data_as(I64P))
    d._keep = (ids, mem)
    return d


def graph_from_out(o: GraphOutC) -> Graph:
    return Graph(_arr(o.node_id, o.n_nodes, np.int64), _arr(o.compute_us, o.n_nodes, np.int64),
                 _arr(o.memory_bytes, o.n_nodes, np.int64), _arr(o.edge_src, o.n_edges, np.int64),
                 _arr(o.edge_dst, o.n_edges, np.int64), _arr(o.edge_bytes, o.n_edges, np.int64),
                 _arr(o.group, o.n_nodes, np.int32))


def cluster_map_from(c: ClusterMapC) -> ClusterMap:
    off = _arr(c.member_off, c.n_clusters + 1, np.int64)
    flat = _arr(c.members, int(off[-1]) if len(off) else 0, np.int64)
    members = [flat[off[i]:off[i + 1]] for i in range(c.n_clusters)]
    return ClusterMap(_arr(c.node_cluster, c.n_nodes, np.int32), members,
                      _arr(c.total_compute, c.n_clusters, np.int64),
                      _arr(c.total_memory, c.n_clusters, np.int64),
                      _arr(c.breakpoints, c.n_breakpoints, np.int32))


def placement_from(p: PlacementC) -> Placement:
    nd, k = p.n_devices, p.n_decisions
    dec = None
    if k:
        dec = dict(node=_arr(p.dec_node, k, np.int64), prev=_arr(p.dec_prev, k, np.int32),
                   back_cost=_arr(p.dec_back_cost, k, np.int64),
                   est=_arr(p.dec_est, k * nd, np.int64).reshape(k, nd),
                   chosen=_arr(p.dec_chosen, k, np.int32),
                   relocated=_arr(p.dec_relocated, k, np.uint8),
                   best_effort=_arr(p.dec_best_effort, k, np.uint8))
    return Placement(_arr(p.device, p.n_nodes, np.int32), _arr(p.device_ids, nd, np.int32),
                     _arr(p.per_device_memory, nd, np.int64),
                     _arr(p.device_present, nd, np.uint8), bool(p.oom_risk), dec)


def sim_from(r: SimC) -> SimReport:
    nt = r.n_trace
    trace = None
    if nt:
        trace = dict(kind=_arr(r.tr_kind, nt, np.int32), node=_arr(r.tr_node, nt, np.int64),
                     src=_arr(r.tr_src, nt, np.int64), dst=_arr(r.tr_dst, nt, np.int64),
                     device=_arr(r.tr_device, nt, np.int32), start=_arr(r.tr_start, nt, np.int64),
                     end=_arr(r.tr_end, nt, np.int64))
    d = r.n_devices
    return SimReport(int(r.makespan), int(r.cross_transfer_count), int(r.cross_transfer_bytes),
                     bool(r.oom_flag), _arr(r.device_ids, d, np.int32), _arr(r.peak_memory, d, np.int64),
                     _arr(r.capacity, d, np.int64), trace)


_SIGS = {
    "comm_time": (C.c_int64, CommC, I64P),
    "ccr": (C.POINTER(GraphC), CommC, C.POINTER(C.c_double)),
    "validate": (C.POINTER(GraphC), C.POINTER(C.POINTER(ViolationsC))),
    "require_valid": (C.POINTER(GraphC),),
    "graph_index": (C.POINTER(GraphC), I32P, I32P, I32P, I32P, I32P, I32P),
    "compute_levels": (C.POINTER(GraphC), CommC, I64P, I64P, I64P),
    "topo_order": (C.POINTER(GraphC), C.c_int32, I64P, I64P),
    "is_valid_topo_order": (C.POINTER(GraphC), I64P, C.c_int64, I32P),
    "merge_is_safe": (C.POINTER(GraphC), C.c_int64, C.c_int64, I32P),
    "optimal_breakpoints": (C.POINTER(GraphC), I64P, C.c_int64, CommC, C.c_int32, C.c_int64,
                            C.POINTER(C.POINTER(ClusterMapC))),
    "build_coarse_graph": (C.POINTER(GraphC), I64P, C.c_int64, I64P, I32P, C.c_int64, C.c_int64,
                           I32P, I64P, I64P, C.POINTER(C.POINTER(GraphOutC))),
    "contract_colocation_groups": (C.POINTER(GraphC), C.POINTER(C.POINTER(ContractionC))),
    "fuse": (C.POINTER(GraphC), CommC, C.c_int32, C.c_int64, C.POINTER(C.POINTER(FusionC))),
    "order_place": (C.POINTER(GraphC), I64P, C.c_int64, C.POINTER(DevicesC),
                    C.POINTER(C.POINTER(PlacementC))),
    "adjusting_placement": (C.POINTER(GraphC), I64P, C.c_int64, C.POINTER(DevicesC), CommC,
                            C.POINTER(C.POINTER(PlacementC))),
    "expand_placement": (C.POINTER(GraphC), I32P, C.c_int64, I64P, I64P, I32P, U8P,
                         C.POINTER(C.POINTER(PlacementC))),
    "simulate": (C.POINTER(GraphC), I32P, C.POINTER(DevicesC), CommC, C.c_int32,
                 C.POINTER(C.POINTER(SimC))),
    "brute_force_optimal": (C.POINTER(GraphC), C.POINTER(DevicesC), CommC, I32P, I64P),
    "pipeline": (C.POINTER(GraphC), C.POINTER(DevicesC), CommC, C.POINTER(PipelineCfgC),
                 C.POINTER(C.POINTER(PipelineC))),
}

# free-function names: product header vs oracle headers
_FREES_DP = dict(violations="dp_violation_list_free", cluster_map="dp_cluster_map_free",
                 graph_out="dp_graph_out_free", contraction="dp_contraction_free",
                 fusion="dp_fusion_result_free", placement="dp_placement_result_free",
                 sim="dp_sim_report_free", pipeline="dp_pipeline_result_free")


class Backend:
    """Python mirror of the dagplace API over one flat-ABI library."""

    def __init__(self, lib: C.CDLL, prefix: str, ctx=None, name: str = ""):
        self.lib, self.prefix, self.ctx = lib, prefix, ctx
        self.name = name or prefix
        self._fn = {}
        for k, argt in _SIGS.items():
            f = getattr(lib, prefix + k)
            f.restype = C.c_int
            f.argtypes = ((C.c_void_p,) if ctx is not None else ()) + argt
            self._fn[k] = f
        cand = getattr(lib, prefix + "simulate_candidates")
        cand.restype = C.c_int
        base = (C.POINTER(GraphC), I32P, C.c_int64, U8P, C.c_int64, C.POINTER(DevicesC), CommC,
                I64P, I64P)
        cand.argtypes = ((C.c_void_p,) + base) if ctx is not None else base + (C.c_int32,)
        self._fn["simulate_candidates"] = cand
        if prefix == "dp_":
            self._free = {k: getattr(lib, v) for k, v in _FREES_DP.items()}
            err = lib.dp_last_error_message
        else:
            names = dict(violations="free_violations", cluster_map="free_cluster_map",
                         graph_out="free_graph_out", contraction="free_contraction",
                         fusion="free_fusion", placement="free_placement", sim="free_sim_report",
                         pipeline="free_pipeline")
            self._free = {k: getattr(lib, prefix + v) for k, v in names.items()}
            err = getattr(lib, prefix + "last_error_message")
        err.restype = C.c_char_p
        self._err = err
        for f in self._free.values():
            f.restype = None

    # ---------------------------------------------------------------- plumbing
    def _call(self, name, *args):
        f = self._fn[name]
        rc = f(self.ctx, *args) if self.ctx is not None else f(*args)
        if rc != 0:
            raise DagError(rc, (self._err() or b"").decode())
        return rc

    # ---------------------------------------------------------------- graph core
    def comm_time(self, nbytes: int, comm) -> int:
        out = C.c_int64()
        f = self._fn["comm_time"]
        rc = f(self.ctx, nbytes, comm_c(comm), C.byref(out)) if self.ctx is not None else \
            f(nbytes, comm_c(comm), C.byref(out))
        if rc:
            raise DagError(rc, (self._err() or b"").decode())
        return out.value

    def ccr(self, g: Graph, comm) -> float:
        out = C.c_double()
        self._call("ccr", C.byref(g.c()), comm_c(comm), C.byref(out))
        return out.value

    def validate(self, g: Graph):
        p = C.POINTER(ViolationsC)()
        self._call("validate", C.byref(g.c()), C.byref(p))
        v = p.contents
        k = v.count
        kinds = _arr(v.kind, k, np.int32)
        noff = _arr(v.node_off, k + 1, np.int64)
        moff = _arr(v.msg_off, k + 1, np.int64)
        nodes = _arr(v.nodes, int(noff[-1]) if k else 0, np.int64)
        raw = C.string_at(v.msg, int(moff[-1])) if k and moff[-1] else b""
        out = [Violation(ERROR_KINDS[kinds[i] - 1], raw[moff[i]:moff[i + 1]].decode(),
                         nodes[noff[i]:noff[i + 1]].tolist()) for i in range(k)]
        self._free["violations"](p)
        return out

    def require_valid(self, g: Graph) -> None:
        self._call("require_valid", C.byref(g.c()))

    def graph_index(self, g: Graph):
        n, m = g.n, g.m
        es, ed = np.zeros(m, np.int32), np.zeros(m, np.int32)
        os_, ol = np.zeros(n + 1, np.int32), np.zeros(m, np.int32)
        is_, il = np.zeros(n + 1, np.int32), np.zeros(m, np.int32)
        ptr = lambda a: a.ctypes.data_as(I32P)  # noqa: E731
        self._call("graph_index", C.byref(g.c()), ptr(es), ptr(ed), ptr(os_), ptr(ol), ptr(is_), ptr(il))
        return dict(edge_src=es, edge_dst=ed, out_start=os_, out_list=ol, in_start=is_, in_list=il)

    def compute_levels(self, g: Graph, comm):
        t, b, c = (np.zeros(g.n, np.int64) for _ in range(3))
        self._call("compute_levels", C.byref(g.c()), comm_c(comm), _p64(t), _p64(b), _p64(c))
        return t, b, c

    # ---------------------------------------------------------------- ordering
    def topo_order(self, g: Graph, policy: int, cpath: Optional[np.ndarray] = None) -> np.ndarray:
        seq = np.zeros(g.n, np.int64)
        cp = None
        if cpath is not None:
            cp = np.ascontiguousarray(cpath, dtype=np.int64)
        self._call("topo_order", C.byref(g.c()), policy, _p64(cp) if cp is not None else None, _p64(seq))
        return seq

    def m_topo(self, g):
        return self.topo_order(g, TOPO_M)

    def dfs_topo(self, g):
        return self.topo_order(g, TOPO_DFS)

    def cpd_topo(self, g, cpath):
        return self.topo_order(g, TOPO_CPD, cpath)

    def is_valid_topo_order(self, g: Graph, seq) -> bool:
        s = np.ascontiguousarray(seq, dtype=np.int64)
        out = C.c_int32()
        self._call("is_valid_topo_order", C.byref(g.c()), _p64(s), len(s), C.byref(out))
        return bool(out.value)

    # ---------------------------------------------------------------- fusion
    def merge_is_safe(self, g: Graph, u: int, v: int) -> bool:
        out = C.c_int32()
        self._call("merge_is_safe", C.byref(g.c()), u, v, C.byref(out))
        return bool(out.value)

    def optimal_breakpoints(self, g: Graph, seq, comm, rng: int, limit: int) -> ClusterMap:
        s = np.ascontiguousarray(seq, dtype=np.int64)
        p = C.POINTER(ClusterMapC)()
        self._call("optimal_breakpoints", C.byref(g.c()), _p64(s), len(s), comm_c(comm), rng, limit,
                   C.byref(p))
        out = cluster_map_from(p.contents)
        self._free["cluster_map"](p)
        return out

    def build_coarse_graph(self, g: Graph, seq, node_ids, node_cluster, members, cluster_ids=None) -> Graph:
        s = np.ascontiguousarray(seq, dtype=np.int64)
        ids = np.ascontiguousarray(node_ids, dtype=np.int64)
        cl = np.ascontiguousarray(node_cluster, dtype=np.int32)
        k = len(members)
        cid = np.ascontiguousarray(np.arange(k) if cluster_ids is None else cluster_ids, dtype=np.int32)
        off = np.zeros(k + 1, np.int64)
        off[1:] = np.cumsum([len(m) for m in members])
        flat = np.ascontiguousarray(np.concatenate(members) if k else np.zeros(0), dtype=np.int64)
        p = C.POINTER(GraphOutC)()
        self._call("build_coarse_graph", C.byref(g.c()), _p64(s), len(s), _p64(ids),
                   cl.ctypes.data_as(I32P), len(ids), k, cid.ctypes.data_as(I32P), _p64(off),
                   _p64(flat), C.byref(p))
        out = graph_from_out(p.contents)
        self._free["graph_out"](p)
        return out

    def contract_colocation_groups(self, g: Graph):
        p = C.POINTER(ContractionC)()
        self._call("contract_colocation_groups", C.byref(g.c()), C.byref(p))
        c = p.contents
        gg = graph_from_out(c.contracted.contents)
        off = _arr(c.member_off, gg.n + 1, np.int64)
        flat = _arr(c.members, int(off[-1]), np.int64)
        members = [flat[off[i]:off[i + 1]] for i in range(gg.n)]
        self._free["contraction"](p)
        return gg, members

    def fuse(self, g: Graph, comm, rng: int, limit: int):
        p = C.POINTER(FusionC)()
        self._call("fuse", C.byref(g.c()), comm_c(comm), rng, limit, C.byref(p))
        f = p.contents
        out = (graph_from_out(f.coarse.contents), cluster_map_from(f.map.contents))
        self._free["fusion"](p)
        return out

    # ---------------------------------------------------------------- placement
    def order_place(self, g: Graph, seq, devices) -> Placement:
        s = np.ascontiguousarray(seq, dtype=np.int64)
        p = C.POINTER(PlacementC)()
        self._call("order_place", C.byref(g.c()), _p64(s), len(s), C.byref(devices_c(devices)), C.byref(p))
        out = placement_from(p.contents)
        self._free["placement"](p)
        return out

    def adjusting_placement(self, g: Graph, seq, devices, comm) -> Placement:
        s = np.ascontiguousarray(seq, dtype=np.int64)
        p = C.POINTER(PlacementC)()
        self._call("adjusting_placement", C.byref(g.c()), _p64(s), len(s), C.byref(devices_c(devices)),
                   comm_c(comm), C.byref(p))
        out = placement_from(p.contents)
        self._free["placement"](p)
        return out

    def expand_placement(self, g: Graph, cmap: ClusterMap, coarse_device, coarse_placed=None) -> Placement:
        off, flat = cmap.member_arrays()
        nc = np.ascontiguousarray(cmap.node_cluster, dtype=np.int32)
        cd = np.ascontiguousarray(coarse_device, dtype=np.int32)
        cp = None if coarse_placed is None else np.ascontiguousarray(coarse_placed, dtype=np.uint8)
        p = C.POINTER(PlacementC)()
        self._call("expand_placement", C.byref(g.c()), nc.ctypes.data_as(I32P), cmap.n_clusters,
                   _p64(off), _p64(flat), cd.ctypes.data_as(I32P),
                   cp.ctypes.data_as(U8P) if cp is not None else None, C.byref(p))
        out = placement_from(p.contents)
        self._free["placement"](p)
        return out

    # ---------------------------------------------------------------- simulator
    def simulate(self, g: Graph, device_of_node, devices, comm, trace: bool = False) -> SimReport:
        d = np.ascontiguousarray(device_of_node, dtype=np.int32)
        p = C.POINTER(SimC)()
        self._call("simulate", C.byref(g.c()), d.ctypes.data_as(I32P), C.byref(devices_c(devices)),
                   comm_c(comm), int(trace), C.byref(p))
        out = sim_from(p.contents)
        self._free["sim"](p)
        return out

    def simulate_candidates(self, g: Graph, node_cluster, n_clusters: int, cand_dev_pos, devices,
                            comm, threads: int = 1):
        nc = np.ascontiguousarray(node_cluster, dtype=np.int32)
        cand = np.ascontiguousarray(cand_dev_pos, dtype=np.uint8)
        b = cand.size // max(1, n_clusters)
        ms = np.zeros(b, np.int64)
        am = C.c_int64(-1)
        args = [C.byref(g.c()), nc.ctypes.data_as(I32P), n_clusters, cand.ctypes.data_as(U8P), b,
                C.byref(devices_c(devices)), comm_c(comm), _p64(ms), C.byref(am)]
        f = self._fn["simulate_candidates"]
        rc = f(self.ctx, *args) if self.ctx is not None else f(*args, threads)
        if rc:
            raise DagError(rc, (self._err() or b"").decode())
        return ms, am.value

    def brute_force_optimal(self, g: Graph, devices, comm):
        best = np.zeros(g.n, np.int32)
        ms = C.c_int64()
        self._call("brute_force_optimal", C.byref(g.c()), C.byref(devices_c(devices)), comm_c(comm),
                   best.ctypes.data_as(I32P), C.byref(ms))
        return best, ms.value

    # ---------------------------------------------------------------- pipeline
    def evaluate_pipeline(self, g: Graph, devices, comm, fusion_range=200, cluster_mem_fraction=0.25,
                          strategy=1, simulate=True) -> PipelineReport:
        cfg = PipelineCfgC(fusion_range, cluster_mem_fraction, strategy, int(simulate))
        p = C.POINTER(PipelineC)()
        self._call("pipeline", C.byref(g.c()), C.byref(devices_c(devices)), comm_c(comm), C.byref(cfg),
                   C.byref(p))
        return self._report(p)

    def evaluate_pipeline_batch(self, graphs, devices, comm, fusion_range=200, cluster_mem_fraction=0.25,
                                strategy=1, simulate=True) -> list:
        """evaluate_pipeline over independent graphs in one call (dp_pipeline_batch; the
        product only: the reference evaluates one graph per call)."""
        if self.prefix != "dp_":
            return [self.evaluate_pipeline(g, devices, comm, fusion_range, cluster_mem_fraction, strategy, simulate)
                    for g in graphs]
        cfg = PipelineCfgC(fusion_range, cluster_mem_fraction, strategy, int(simulate))
        gcs = [g.c() for g in graphs]
        arr = (C.POINTER(GraphC) * max(1, len(gcs)))(*[C.pointer(x) for x in gcs])
        outs = (C.POINTER(PipelineC) * max(1, len(gcs)))()
        f = self.lib.dp_pipeline_batch
        f.restype = C.c_int
        f.argtypes = [C.c_void_p, C.c_int32, C.POINTER(C.POINTER(GraphC)), C.POINTER(DevicesC), CommC,
                      C.POINTER(PipelineCfgC), C.POINTER(C.POINTER(PipelineC))]
        rc = f(self.ctx, len(gcs), arr, C.byref(devices_c(devices)), comm_c(comm), C.byref(cfg), outs)
        if rc != 0:
            raise DagError(rc, (self._err() or b"").decode(errors="replace"))
        return [self._report(outs[i]) for i in range(len(gcs))]

    def _report(self, p) -> PipelineReport:
        r = p.contents
        rep = PipelineReport(int(r.original_nodes), int(r.original_edges), float(r.original_ccr),
                             int(r.coarse_nodes), int(r.coarse_edges), float(r.coarse_ccr),
                             graph_from_out(r.fusion.contents.coarse.contents),
                             cluster_map_from(r.fusion.contents.map.contents),
                             _arr(r.coarse_sequence, r.coarse_nodes, np.int64),
                             placement_from(r.coarse_order.contents),
                             placement_from(r.coarse_adjust.contents),
                             placement_from(r.order_expanded.contents),
                             placement_from(r.adjust_expanded.contents),
                             int(r.order_makespan), int(r.adjust_makespan), float(r.generation_ms))
        self._free["pipeline"](p)
        return rep


def graph_from_json(lib: C.CDLL, text, prefix: str = "dp_") -> Graph:
    """graph_from_json (json_io.cpp:43-74) through `prefix`graph_from_json: the product's
    SoA loader (dp_, host code, no GPU needed) or the reference shim (dpr_, tests only)."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    f = getattr(lib, prefix + "graph_from_json")
    f.restype = C.c_int
    f.argtypes = [C.c_char_p, C.c_int64, C.POINTER(C.POINTER(GraphOutC))]
    out = C.POINTER(GraphOutC)()
    rc = f(data, len(data), C.byref(out))
    err = getattr(lib, prefix + "last_error_message")
    err.restype = C.c_char_p
    if rc:
        raise DagError(rc, (err() or b"").decode(errors="replace"))
    o = out.contents
    n, m = o.n_nodes, o.n_edges

    def arr(ptr, k, dt):
        return np.ctypeslib.as_array(ptr, shape=(k,)).astype(dt, copy=True) if k else np.zeros(0, dt)
    g = Graph(arr(o.node_id, n, np.int64), arr(o.compute_us, n, np.int64), arr(o.memory_bytes, n, np.int64),
              arr(o.edge_src, m, np.int64), arr(o.edge_dst, m, np.int64), arr(o.edge_bytes, m, np.int64),
              arr(o.group, n, np.int32))
    free = getattr(lib, "dp_graph_out_free" if prefix == "dp_" else prefix + "free_graph_out")
    free.restype = None
    free.argtypes = [C.POINTER(GraphOutC)]
    free(out)
    return g


def devices_from_json(lib: C.CDLL, text, prefix: str = "dp_"):
    """devices_from_json (json_io.cpp:93-117) -> ([(id, memory_bytes)], (k, b))."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    f = getattr(lib, prefix + "devices_from_json")
    f.restype = C.c_int
    f.argtypes = [C.c_char_p, C.c_int64, I32P, I32P, I64P, C.c_int32, C.POINTER(CommC)]
    cap = 4096
    ids = np.zeros(cap, np.int32)
    mem = np.zeros(cap, np.int64)
    cnt = C.c_int32()
    comm = CommC()
    rc = f(data, len(data), C.byref(cnt), ids.ctypes.data_as(I32P), mem.ctypes.data_as(I64P), cap, C.byref(comm))
    err = getattr(lib, prefix + "last_error_message")
    err.restype = C.c_char_p
    if rc:
        raise DagError(rc, (err() or b"").decode(errors="replace"))
    k = min(cnt.value, cap)
    return [(int(ids[i]), int(mem[i])) for i in range(k)], (comm.k_us_per_byte, comm.b_us)


# ---------------------------------------------------------------- Standard Evaluation
class ProfilesC(C.Structure):
    _fields_ = [("n_batches", C.c_int32), ("batch_size", I64P), ("node_off", I64P), ("node_id", I64P),
                ("memory_bytes", I64P), ("compute_us", I64P)]


class NodeModelsC(C.Structure):
    _fields_ = [("n", C.c_int64), ("node_id", I64P), ("fit", C.POINTER(C.c_double))]


class DeviationC(C.Structure):
    _fields_ = [("n_memory", C.c_int64), ("memory_id", I64P), ("memory_dev", C.POINTER(C.c_double)),
                ("n_time", C.c_int64), ("time_id", I64P), ("time_dev", C.POINTER(C.c_double)),
                ("mean_memory", C.c_double), ("mean_time", C.c_double),
                ("n_zero_memory", C.c_int64), ("zero_memory", I64P),
                ("n_zero_time", C.c_int64), ("zero_time", I64P)]


@dataclass
class Profiles:
    """ProfileSet (estimation.hpp:25-28): batches of (node_id, memory_bytes, compute_us)."""
    batch_size: np.ndarray
    node_off: np.ndarray
    node_id: np.ndarray
    memory_bytes: np.ndarray
    compute_us: np.ndarray

    def c(self) -> ProfilesC:
        for f in ("batch_size", "node_off", "node_id", "memory_bytes", "compute_us"):
            setattr(self, f, np.ascontiguousarray(getattr(self, f), dtype=np.int64))
        return ProfilesC(len(self.batch_size), self.batch_size.ctypes.data_as(I64P),
                         self.node_off.ctypes.data_as(I64P), self.node_id.ctypes.data_as(I64P),
                         self.memory_bytes.ctypes.data_as(I64P), self.compute_us.ctypes.data_as(I64P))


class Estimation:
    """Standard Evaluation entry points of one library: the product (dp_, GPU context
    required) or the reference shim (dpr_, tests only)."""

    def __init__(self, lib: C.CDLL, prefix: str, ctx=None):
        self.lib, self.prefix, self.ctx = lib, prefix, ctx
        pre = (C.c_void_p,) if ctx is not None else ()
        self.f_fit = self._f("fit_node_models", pre + (C.POINTER(ProfilesC), C.POINTER(C.POINTER(NodeModelsC))))
        self.f_est = self._f("estimate_graph", pre + (C.POINTER(GraphC), C.POINTER(NodeModelsC), C.c_int64, C.c_int64,
                                                      C.c_int64, I64P, I64P, C.POINTER(C.c_double),
                                                      C.POINTER(C.POINTER(GraphOutC))))
        self.f_comm = self._f("fit_comm_model", pre + (C.c_int64, I64P, C.POINTER(C.c_double), C.POINTER(CommC)))
        self.f_dev = self._f("deviation_report", pre + (C.POINTER(GraphC), C.POINTER(GraphC),
                                                        C.POINTER(C.POINTER(DeviationC))))
        self.f_free_models = getattr(lib, prefix + "node_models_free")
        self.f_free_dev = getattr(lib, prefix + "deviation_free")
        self.f_free_graph = getattr(lib, "dp_graph_out_free" if prefix == "dp_" else prefix + "free_graph_out")
        for f in (self.f_free_models, self.f_free_dev, self.f_free_graph):
            f.restype = None
        err = getattr(lib, prefix + "last_error_message")
        err.restype = C.c_char_p
        self._err = err

    def _f(self, name, argt):
        f = getattr(self.lib, self.prefix + name)
        f.restype = C.c_int
        f.argtypes = list(argt)
        return f

    def _call(self, f, *a):
        rc = f(self.ctx, *a) if self.ctx is not None else f(*a)
        if rc:
            raise DagError(rc, (self._err() or b"").decode(errors="replace"))

    def fit_node_models(self, prof: Profiles):
        """-> (node_id ascending, fit[n, 6])"""
        out = C.POINTER(NodeModelsC)()
        pc = prof.c()
        self._call(self.f_fit, C.byref(pc), C.byref(out))
        o = out.contents
        ids = np.ctypeslib.as_array(o.node_id, shape=(o.n,)).copy() if o.n else np.zeros(0, np.int64)
        fit = np.ctypeslib.as_array(o.fit, shape=(o.n * 6,)).reshape(o.n, 6).copy() if o.n else np.zeros((0, 6))
        self.f_free_models(out)
        return ids, fit

    def estimate_graph(self, g: Graph, models, target_batch: int, reference_batch: int, overrides=()) -> Graph:
        ids, fit = models
        ids = np.ascontiguousarray(ids, np.int64)
        fit = np.ascontiguousarray(fit, np.float64).reshape(-1)
        mc = NodeModelsC(len(ids), ids.ctypes.data_as(I64P), fit.ctypes.data_as(C.POINTER(C.c_double)))
        osrc = np.array([o[0] for o in overrides], np.int64)
        odst = np.array([o[1] for o in overrides], np.int64)
        ofac = np.array([o[2] for o in overrides], np.float64)
        out = C.POINTER(GraphOutC)()
        gc = g.c()
        self._call(self.f_est, C.byref(gc), C.byref(mc), target_batch, reference_batch, len(osrc),
                   osrc.ctypes.data_as(I64P), odst.ctypes.data_as(I64P), ofac.ctypes.data_as(C.POINTER(C.c_double)),
                   C.byref(out))
        o = out.contents
        n, m = o.n_nodes, o.n_edges

        def arr(ptr, k, dt):
            return np.ctypeslib.as_array(ptr, shape=(k,)).astype(dt, copy=True) if k else np.zeros(0, dt)
        r = Graph(arr(o.node_id, n, np.int64), arr(o.compute_us, n, np.int64), arr(o.memory_bytes, n, np.int64),
                  arr(o.edge_src, m, np.int64), arr(o.edge_dst, m, np.int64), arr(o.edge_bytes, m, np.int64))
        self.f_free_graph(out)
        return r

    def fit_comm_model(self, samples):
        b = np.array([x[0] for x in samples], np.int64)
        u = np.array([x[1] for x in samples], np.float64)
        out = CommC()
        self._call(self.f_comm, len(b), b.ctypes.data_as(I64P), u.ctypes.data_as(C.POINTER(C.c_double)),
                   C.byref(out))
        return out.k_us_per_byte, out.b_us

    def deviation_report(self, est: Graph, meas: Graph):
        out = C.POINTER(DeviationC)()
        a, b = est.c(), meas.c()
        self._call(self.f_dev, C.byref(a), C.byref(b), C.byref(out))
        o = out.contents

        def arr(ptr, k, dt):
            return np.ctypeslib.as_array(ptr, shape=(k,)).astype(dt, copy=True) if k else np.zeros(0, dt)
        r = dict(memory=(arr(o.memory_id, o.n_memory, np.int64), arr(o.memory_dev, o.n_memory, np.float64)),
                 time=(arr(o.time_id, o.n_time, np.int64), arr(o.time_dev, o.n_time, np.float64)),
                 mean_memory=o.mean_memory, mean_time=o.mean_time,
                 zero_memory=arr(o.zero_memory, o.n_zero_memory, np.int64),
                 zero_time=arr(o.zero_time, o.n_zero_time, np.int64))
        self.f_free_dev(out)
        return r
