"""Python bindings of the C++ API (paper_2208_00184_b200.dagplace, host/py_dagplace.cpp):
the module exposes every function the reference headers declare on the path
(include/dagplace/{graph,ordering,fusion,placement,simulator,estimation,pipeline}.hpp) and
maps DagError with the reference's kind and message.  The GPU tests run the bound C++ API
(the B200 drop-in underneath) against the unmodified reference compiled by oracle/Makefile
(`ref` fixture) on the same inputs, bit for bit."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_HEADERS = "/root/reference/proj/include/dagplace"

FUNCTIONS = ["validate", "require_valid", "comm_time", "ccr", "compute_levels", "m_topo", "dfs_topo", "cpd_topo",
             "is_valid_topo_order", "merge_is_safe", "optimal_breakpoints", "build_coarse_graph",
             "contract_colocation_groups", "fuse", "order_place", "adjusting_placement", "compute_est",
             "expand_placement", "simulate", "brute_force_optimal", "fit_node_models", "estimate_graph",
             "fit_comm_model", "sequential_eval_placement", "deviation_report", "evaluate_pipeline",
             "topo_policy_from_string", "place_strategy_from_string", "to_string"]


def _mod():
    from paper_2208_00184_b200 import dagplace
    return dagplace


def test_module_surface():
    d = _mod()
    missing = [f for f in FUNCTIONS if not hasattr(d, f)]
    assert not missing, missing
    for t in ("ComputationGraph", "OpNode", "TensorEdge", "CommModel", "DeviceSpec", "LevelTable", "TopoOrder",
              "ClusterMap", "FusionResult", "Placement", "PlacementResult", "SimulationReport", "PipelineConfig",
              "PipelineReport", "DagError", "ErrorKind"):
        assert hasattr(d, t), t


@pytest.mark.skipif(not os.path.isdir(REF_HEADERS), reason="reference headers not present")
def test_every_header_function_is_bound():
    """Every free function of the path's headers (except JSON I/O and the generator, out of
    scope) has a binding."""
    d = _mod()
    names = set()
    for h in ("graph", "ordering", "fusion", "placement", "simulator", "estimation", "pipeline"):
        src = open(os.path.join(REF_HEADERS, h + ".hpp")).read()
        for m in re.finditer(r"^[A-Za-z_:<>, ]+?\b([a-z_]+)\(const ", src, re.M):
            names.add(m.group(1))
    missing = sorted(n for n in names if not hasattr(d, n) and not (n == "for_devices" and
                                                                    hasattr(d.SchedulerState, n)))
    assert not missing, missing


def test_dag_error_kind_and_text():
    d = _mod()
    with pytest.raises(d.DagError) as e:
        d.comm_time(-5, d.CommModel(0.001, 10.0))
    assert e.value.kind == d.ErrorKind.InvalidValue
    assert str(e.value).startswith("InvalidValue: ")
    assert d.comm_time(1000, d.CommModel(0.001, 10.0)) == 11


def _graph(d, g):
    return d.ComputationGraph.from_arrays(g.node_id, g.compute_us, g.memory_bytes, g.edge_src, g.edge_dst,
                                          g.edge_bytes)


@pytest.mark.gpu
def test_bound_api_matches_reference(ref):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from cases import GEN, capacity_for, devices
    from graphs import layered
    d = _mod()
    g = layered(61, 12000, 300)
    cg = _graph(d, g)
    cm = d.CommModel(*GEN)
    # levels and CPD order
    lv = d.compute_levels(cg, cm)
    t, b, c = ref.compute_levels(g, GEN)
    assert [lv.at(int(i)).cpath for i in g.node_id[:500]] == c[:500].tolist()
    assert lv.max_cpath() == int(c.max())
    order = d.cpd_topo(cg, lv)
    assert order.sequence == ref.cpd_topo(g, c).tolist()
    assert d.is_valid_topo_order(cg, order)
    # the whole pipeline
    devs = devices(8, capacity_for(g, 8, 1.25))
    want = ref.evaluate_pipeline(g, devs, GEN)
    rep = d.evaluate_pipeline(cg, None, [d.DeviceSpec(i, cap) for i, cap in devs], cm, d.PipelineConfig())
    assert rep.coarse_nodes == want.coarse_nodes and rep.coarse_edges == want.coarse_edges
    assert rep.order_place.makespan_us == want.order_makespan
    assert rep.adjusting.makespan_us == want.adjust_makespan
    assert rep.original_ccr == want.original_ccr
    exp = want.adjust_expanded if rep.chosen_strategy == "adjust" else want.order_expanded
    got = rep.chosen_placement.assignment
    ids = exp.device_ids
    assert all(got[int(v)] == int(ids[exp.device[i]]) for i, v in enumerate(g.node_id))
    assert rep.chosen_strategy == "adjust"  # PipelineConfig() default (pipeline.cpp:95)
    assert rep.chosen_simulation.makespan == want.adjust_makespan
    assert len(rep.fusion.map.clusters) == want.coarse_nodes


@pytest.mark.gpu
def test_bound_api_errors_match_reference(ref):
    d = _mod()
    cg = d.ComputationGraph([d.OpNode(1, "a", 5, 1), d.OpNode(2, "b", 5, 1)],
                            [d.TensorEdge(1, 2, 10), d.TensorEdge(2, 1, 10)])
    with pytest.raises(d.DagError) as e:
        d.compute_levels(cg, d.CommModel(0.001, 10.0))
    assert e.value.kind == d.ErrorKind.CycleDetected
    from paper_2208_00184_b200._abi import Graph
    from compare import outcome
    g = Graph(np.array([1, 2]), np.array([5, 5]), np.array([1, 1]), np.array([1, 2]), np.array([2, 1]),
              np.array([10, 10]))
    o = outcome(ref.compute_levels, g, (0.001, 10.0))
    assert o[0] == "err" and o[2] == str(e.value)
