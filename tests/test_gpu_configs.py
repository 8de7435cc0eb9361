"""Bit-exact parity at BASELINE sizes: the GPU pipeline on every BASELINE.json config
against golden digests produced by the UNMODIFIED reference (tests/golden/configs.json,
made by tests/golden/make_golden.py from oracle/_ref) — coarse graph, cluster map, CPD
sequence, both placements with the decision log, both expanded placements and both
simulated makespans — plus size-independent properties at full size."""
import json
import os

import numpy as np
import pytest

from golden.make_golden import graph_digest, pipeline_digests
from golden_configs import build_config

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "configs.json")))


@pytest.mark.parametrize("name", sorted(GOLD))
def test_config_matches_reference(gpu, name):
    g, devs, comm = build_config(name)
    gold = GOLD[name]
    assert graph_digest(g) == gold["graph"], "input generator drifted"
    rep = gpu.evaluate_pipeline(g, devs, comm, simulate=True)
    got = pipeline_digests(rep)
    for k, v in got.items():
        if isinstance(v, float):
            assert v == pytest.approx(gold[k], rel=0, abs=0), k
        else:
            assert v == gold[k], f"{name}.{k}: {v} vs {gold[k]}"


@pytest.mark.parametrize("name", ["4d", "4w"])
def test_full_size_properties(gpu, name):
    """Size-independent checks at 1M ops: the CPD sequence is a topological order, the
    clusters are contiguous runs that partition the nodes within the memory limit, the
    coarse graph is acyclic with bytes conserved over crossing edges."""
    g, devs, comm = build_config(name)
    rep = gpu.evaluate_pipeline(g, devs, comm, simulate=False)
    m = rep.map
    assert sum(len(x) for x in m.members) == g.n
    allm = np.concatenate(m.members)
    assert np.array_equal(np.sort(allm), np.sort(g.node_id))
    cl = m.node_cluster
    cross = cl[g.edge_src] != cl[g.edge_dst]
    assert int(g.edge_bytes[cross].sum()) == int(rep.coarse.edge_bytes.sum())
    assert np.all(rep.coarse.edge_src < rep.coarse.edge_dst)  # contiguous runs of a topo order
    limit = max(1, int(min(c for _, c in devs) * 0.25))
    assert int(m.total_memory.max()) <= limit
    assert gpu.is_valid_topo_order(rep.coarse, rep.coarse_sequence)


def test_config4_batched_matches_reference(gpu):
    """The throughput path at full size: config #4 deep twice in one dp_pipeline_batch call
    (shared-SM peel + DP kernel, batched coarse phase and placement) against the
    reference's golden digests."""
    g, devs, comm = build_config("4d")
    gold = GOLD["4d"]
    for rep in gpu.evaluate_pipeline_batch([g, g], devs, comm, simulate=True):
        got = pipeline_digests(rep)
        for k, v in got.items():
            if isinstance(v, float):
                assert v == pytest.approx(gold[k], rel=0, abs=0), k
            else:
                assert v == gold[k], f"4d batched.{k}: {v} vs {gold[k]}"
