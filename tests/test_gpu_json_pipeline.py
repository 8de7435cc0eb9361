"""Graph load -> device, end to end: a JSON document
parsed by dp_graph_from_json / dp_devices_from_json straight into the SoA arrays the
device path uploads, then dp_pipeline on the GPU — against the reference's own
graph_from_json / devices_from_json (json_io.cpp:43-117, nlohmann 3.11.3) followed by
evaluate_pipeline (pipeline.cpp:27-111) on the compiled reference.  At full size: the
config #4 document (1M ops, 4M edges) parsed and checked against the golden digests."""
import json
import os

import numpy as np
import pytest

from compare import same_pipeline  # noqa: F401

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def graph_doc(g, names=True, groups=None, shuffle_seed=None, extras=False) -> str:
    """A graph document in the reference's schema (json_io.cpp:43-74)."""
    idx = np.arange(g.n)
    if shuffle_seed is not None:
        np.random.default_rng(shuffle_seed).shuffle(idx)
    nodes = []
    for i in idx.tolist():
        nd = {"id": int(g.node_id[i]), "compute_us": int(g.compute_us[i]), "memory_bytes": int(g.memory_bytes[i])}
        if names:
            nd["name"] = f"op{i}"
        if groups is not None and groups[i] >= 0:
            nd["colocation_group"] = f"g{groups[i]}"
        if extras and i % 5 == 0:
            nd["attrs"] = {"k": [1, 2.5, None]}
        nodes.append(nd)
    edges = [{"src": int(s), "dst": int(d), "tensor_bytes": int(b)}
             for s, d, b in zip(g.edge_src.tolist(), g.edge_dst.tolist(), g.edge_bytes.tolist())]
    return json.dumps({"schema_version": 1, "nodes": nodes, "edges": edges})


def devices_doc(devs, comm) -> str:
    return json.dumps({"devices": [{"id": d, "memory_bytes": c} for d, c in devs],
                       "comm": {"k_us_per_byte": comm[0], "b_us": comm[1]}})


def load_both(gpu, ref, gtext, dtext):
    from paper_2208_00184_b200._abi import devices_from_json, graph_from_json
    a = graph_from_json(gpu.lib, gtext, "dp_")
    b = graph_from_json(ref.lib, gtext, "dpr_")
    da, ca = devices_from_json(gpu.lib, dtext, "dp_")
    db, cb = devices_from_json(ref.lib, dtext, "dpr_")
    for f in ("node_id", "compute_us", "memory_bytes", "edge_src", "edge_dst", "edge_bytes", "group"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert da == db and ca == cb
    return a, b, da, ca


@pytest.mark.parametrize("case", ["layered", "shuffled_groups", "random_extras", "gnmt_like"])
def test_json_to_pipeline(gpu, ref, case):
    from cases import capacity_for, devices
    from graphs import layered, random_dag
    if case == "layered":
        g = layered(41, 6000, 48)
        text = graph_doc(g)
    elif case == "shuffled_groups":
        # co-location groups inside one layer (every 7th node of a layer) keep the DAG acyclic
        g = layered(42, 3000, 30)
        grp = np.where(np.arange(g.n) % 7 == 0, np.arange(g.n) // 30, -1)
        text = graph_doc(g, groups=grp, shuffle_seed=3)
    elif case == "random_extras":
        g = random_dag(43, 400, 0.05)
        text = graph_doc(g, names=False, extras=True, shuffle_seed=5)
    else:
        from paper_2208_00184_b200 import synth
        g = synth.gnmt(8, 500, 2)
        text = graph_doc(g)
    devs = devices(8, capacity_for(g, 8, 1.25), shuffle_seed=1, base_id=10, stride=7)
    a, b, d, comm = load_both(gpu, ref, text, devices_doc(devs, (0.001, 10.0)))
    from compare import outcome, same_outcome
    want = outcome(ref.evaluate_pipeline, b, d, comm)
    assert want[0] == "ok", want
    same_outcome(outcome(gpu.evaluate_pipeline, a, d, comm), want, same_pipeline, f"json {case}")


def test_json_config4_full_size(gpu):
    """The 1M-op config #4 document (~330 MB) through dp_graph_from_json -> dp_pipeline:
    parsed arrays equal the generator's, and the pipeline matches the reference's golden
    digests (tests/golden/configs.json)."""
    import time

    from golden.make_golden import pipeline_digests
    from paper_2208_00184_b200 import synth
    from paper_2208_00184_b200._abi import devices_from_json, graph_from_json
    g, devs = synth.config4(True)
    parts = ['{"schema_version":1,"nodes":[']
    parts.append(",".join(f'{{"id":{i},"name":"op{i}","compute_us":{c},"memory_bytes":{m}}}'
                          for i, c, m in zip(g.node_id.tolist(), g.compute_us.tolist(), g.memory_bytes.tolist())))
    parts.append('],"edges":[')
    parts.append(",".join(f'{{"src":{s},"dst":{d},"tensor_bytes":{b}}}'
                          for s, d, b in zip(g.edge_src.tolist(), g.edge_dst.tolist(), g.edge_bytes.tolist())))
    parts.append("]}")
    text = "".join(parts).encode()
    t = time.perf_counter()
    a = graph_from_json(gpu.lib, text, "dp_")
    parse_s = time.perf_counter() - t
    for f in ("node_id", "compute_us", "memory_bytes", "edge_src", "edge_dst", "edge_bytes"):
        assert np.array_equal(getattr(a, f), getattr(g, f)), f
    d, comm = devices_from_json(gpu.lib, devices_doc(devs, (0.001, 10.0)), "dp_")
    rep = gpu.evaluate_pipeline(a, d, comm, simulate=True)
    gold = json.load(open(os.path.join(HERE, "golden", "configs.json")))["4d"]
    for k, v in pipeline_digests(rep).items():
        assert v == gold[k], k
    print(f"\njson config#4: {len(text) / 1e6:.1f} MB parsed in {parse_s:.2f} s "
          f"({len(text) / 1e6 / parse_s:.0f} MB/s, {g.n / parse_s / 1e6:.2f} M nodes/s)")
    out = os.environ.get("DP_EVIDENCE_DIR")
    if out:
        os.makedirs(out, exist_ok=True)
        json.dump({"bytes": len(text), "nodes": g.n, "edges": g.m, "parse_s": parse_s},
                  open(os.path.join(out, "json_config4_parse.json"), "w"))
