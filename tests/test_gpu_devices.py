"""Placements on many devices: the reference sizes its engines as 3 x devices with no
cap (simulator.cpp:138) and places on any number of devices (placement.cpp:128-218).
simulate, batched candidates and evaluate_pipeline at 16, 32 and 100 devices (engines
strided over a warp's lanes, simulate.cu k_sim_wide) against the oracle restatement and
the compiled reference, bit-exact."""
import numpy as np
import pytest

from cases import GEN, UNIT, capacity_for, devices
from compare import outcome, same, same_outcome, same_pipeline, same_sim
from graphs import layered, random_dag

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d", [11, 16, 32, 100])
def test_simulate_many_devices(gpu, oracle, d):
    for s, g in enumerate((random_dag(300 + d, 120, 0.08), layered(d, 1500, 40))):
        rng = np.random.default_rng(s + d)
        devs = devices(d, capacity_for(g, d, 0.9), shuffle_seed=s, base_id=3, stride=5)
        ids = np.array(sorted(x[0] for x in devs), np.int32)
        place = ids[rng.integers(0, d, g.n)]
        for comm in (UNIT, GEN):
            same_outcome(outcome(gpu.simulate, g, place, devs, comm, True),
                         outcome(oracle.simulate, g, place, devs, comm, True), same_sim,
                         f"simulate d{d} s{s} {comm}")


@pytest.mark.parametrize("d", [16, 32])
def test_simulate_many_devices_vs_reference(gpu, ref, d):
    g = layered(40 + d, 2000, 64)
    rng = np.random.default_rng(d)
    devs = devices(d, capacity_for(g, d, 1.25))
    ids = np.array(sorted(x[0] for x in devs), np.int32)
    place = ids[rng.integers(0, d, g.n)]
    same_sim(gpu.simulate(g, place, devs, GEN, True), ref.simulate(g, place, devs, GEN, True), f"ref d{d}")


@pytest.mark.parametrize("d", [16, 32])
def test_candidates_many_devices(gpu, oracle, d):
    g = layered(8 + d, 2000, 32)
    _, m = oracle.fuse(g, GEN, 200, int(g.memory_bytes.sum()) // 8)
    rng = np.random.default_rng(d)
    cand = rng.integers(0, d, (48, m.n_clusters)).astype(np.uint8)
    devs = [(7 * k + 1, 10 ** 12) for k in range(d)]
    ma, ia = gpu.simulate_candidates(g, m.node_cluster, m.n_clusters, cand, devs, GEN)
    mb, ib = oracle.simulate_candidates(g, m.node_cluster, m.n_clusters, cand, devs, GEN)
    same(ma, mb, "makespans")
    assert ia == ib


@pytest.mark.parametrize("d", [16, 32])
def test_pipeline_many_devices(gpu, oracle, ref, d):
    # evaluate_pipeline simulates both placements after the window (pipeline.cpp:89-90)
    g = layered(90 + d, 6000, 48)
    devs = devices(d, capacity_for(g, d, 1.25))
    a = gpu.evaluate_pipeline(g, devs, GEN)
    same_pipeline(a, oracle.evaluate_pipeline(g, devs, GEN), f"pipeline d{d} oracle")
    same_pipeline(a, ref.evaluate_pipeline(g, devs, GEN), f"pipeline d{d} ref")


def test_too_many_devices_is_an_error(gpu):
    g = layered(1, 200, 8)
    devs = devices(257, capacity_for(g, 257, 2.0))
    place = np.array([x[0] for x in devs][:1] * g.n, np.int32)
    kind = outcome(gpu.simulate, g, place, devs, UNIT)
    assert kind[0] == "err" and kind[1] == "abi:103", kind  # DP_E_UNSUPPORTED
