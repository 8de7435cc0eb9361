"""N>1 path on CPU: world_size-2 gloo process group running the candidate sharding and
the single MIN all-reduce of bench.py / paper_2208_00184_b200.shard; the makespans come
from the oracle restatement (CPU) so the test runs without a GPU, and the result must
equal the single-process first strict minimum (simulator.cpp:292-294)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, makespans, out):
    import torch.distributed as dist

    from paper_2208_00184_b200.shard import global_argmin, shard_range
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard_range(len(makespans), rank, world)
    ms, idx = global_argmin(np.asarray(makespans[lo:hi]), lo)
    out[rank] = (ms, idx)
    dist.barrier()
    dist.destroy_process_group()


def _run(makespans, world=2):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, list(map(int, makespans)), out), nprocs=world, join=True)
        return dict(out)


def test_sharded_argmin_matches_single_process(oracle):
    from graphs import layered
    g = layered(3, 600, 12)
    _, m = oracle.fuse(g, (0.001, 10.0), 200, int(g.memory_bytes.sum()) // 8)
    rng = np.random.default_rng(5)
    cand = rng.integers(0, 4, (37, m.n_clusters)).astype(np.uint8)
    devs = [(d, 10 ** 12) for d in range(4)]
    makespans, am = oracle.simulate_candidates(g, m.node_cluster, m.n_clusters, cand, devs, (0.001, 10.0))
    res = _run(makespans)
    assert res[0] == res[1] == (int(makespans[am]), am)


def test_tie_goes_to_lowest_index():
    makespans = np.array([9, 5, 7, 5, 5, 8, 5], np.int64)  # minimum 5 at 1, 3, 4, 6
    res = _run(makespans)
    assert res[0] == res[1] == (5, 1)


def test_empty_shard_and_packing():
    from paper_2208_00184_b200.shard import pack, shard_range, unpack
    assert shard_range(3, 1, 4) == (1, 2) and shard_range(3, 3, 4) == (3, 3)
    assert unpack(pack(123456789, 65535)) == (123456789, 65535)
    with pytest.raises(ValueError):
        pack(1, 1 << 20)
    res = _run(np.array([4], np.int64))
    assert res[0] == res[1] == (4, 0)


def _bench_leg_worker(rank, world, port, B, out):
    import time

    import torch.distributed as dist

    import bench
    from cases import GEN
    from graphs import layered
    from oracle.bind import oracle_backend
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ora = oracle_backend()
    g = layered(4, 500, 10)
    _, m = ora.fuse(g, GEN, 200, int(g.memory_bytes.sum()) // 8)
    devs = [(d, 10 ** 12) for d in range(4)]
    all_rows = np.random.default_rng(9).integers(0, 4, (B, m.n_clusters)).astype(np.uint8)

    def timer(fn):
        t = time.perf_counter()
        fn()
        return time.perf_counter() - t

    ms, lo, secs, best = bench.candidates_leg(
        lambda c: ora.simulate_candidates(g, m.node_cluster, m.n_clusters, c, devs, GEN)[0],
        lambda lo_, count: all_rows[lo_:lo_ + count], B, rank, world, timer)
    out[rank] = (lo, [int(x) for x in ms], secs, best)
    dist.barrier()
    dist.destroy_process_group()


def test_bench_candidates_leg_two_ranks(oracle):
    """bench.py's own sharded config-#5 leg (candidates_leg) on a world-size-2 gloo group:
    each rank simulates its half, the MIN all-reduce (shard.global_argmin) returns the
    single-process first strict minimum, the timing is the max over ranks."""
    from cases import GEN
    from graphs import layered
    B = 23
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_bench_leg_worker, args=(2, port, B, out), nprocs=2, join=True)
        res = dict(out)
    g = layered(4, 500, 10)
    _, m = oracle.fuse(g, GEN, 200, int(g.memory_bytes.sum()) // 8)
    rows = np.random.default_rng(9).integers(0, 4, (B, m.n_clusters)).astype(np.uint8)
    want, am = oracle.simulate_candidates(g, m.node_cluster, m.n_clusters, rows, [(d, 10 ** 12) for d in range(4)], GEN)
    got = res[0][1] + res[1][1]
    assert res[0][0] == 0 and res[1][0] == len(res[0][1])
    assert got == [int(x) for x in want]
    assert res[0][3] == res[1][3] == (int(want[am]), am)
    assert res[0][2] == res[1][2]  # max over ranks
