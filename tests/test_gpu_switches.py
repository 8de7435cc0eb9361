"""Every diagnostic switch of DESIGN.md §9 selects an equivalent path: the whole pipeline
(and a batched call) under each one must still equal the reference's evaluate_pipeline
(oracle/_ref) bit for bit."""
import pytest

from cases import GEN, capacity_for, devices
from compare import same_pipeline
from graphs import layered, shuffled

pytestmark = pytest.mark.gpu

SWITCHES = ["DP_LEVELS_KAHN", "DP_LEVELS_FLOW", "DP_PEEL_V5", "DP_PEEL_DP_SHARED", "DP_PEEL_EXCLUSIVE",
            "DP_PEEL_NO_PREFETCH", "DP_PEEL_FIXPOINT", "DP_PEEL_NO_FIXPOINT", "DP_DP_V3", "DP_DP_V2", "DP_DP_PERSTEP", "DP_PLACE_GLOBAL_META", "DP_SPIN_SYNC"]


@pytest.mark.parametrize("var", SWITCHES)
def test_switch_is_equivalent(gpu, ref, monkeypatch, var):
    monkeypatch.setenv(var, "1")
    gs = [layered(90, 20000, 128), shuffled(layered(91, 6000, 64), 2, relabel=True)]
    devs = devices(8, max(capacity_for(g, 8, 1.25) for g in gs))
    want = [ref.evaluate_pipeline(g, devs, GEN) for g in gs]
    for g, w in zip(gs, want):
        same_pipeline(gpu.evaluate_pipeline(g, devs, GEN), w, var)
    for i, r in enumerate(gpu.evaluate_pipeline_batch(gs, devs, GEN)):
        same_pipeline(r, want[i], f"{var} batch[{i}]")
