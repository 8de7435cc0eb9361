#!/usr/bin/env python
"""Benchmark of the B200 placement-generation path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--variant deep|wide] [--candidates B]

Workload (config #4 of BASELINE.json): 1M-op synthetic layered DAG
(W=1024 "deep" by default; W=65,536 "wide"), fan-in 2..6, seed 12345, 8 devices,
R=200, cluster limit 0.25 x capacity.  A step is one placement-policy generation:
index + validation + the reference's timed window (pipeline.cpp:67-79: fuse -> coarse
levels + cpd_topo -> order_place + adjusting_placement -> 2x expand_placement) from a
graph resident in HBM.  value = edges/s = N x m / (max over ranks of the mean step
time).  N > 1 runs independent replicas (one graph per GPU, no collective on the
path).  `e2e` = the same metric through the public C-ABI call
dp_pipeline with pinned host buffers (H2D upload + generation + D2H of the report).
A secondary `candidates` object measures config #5 (batched makespan simulation of
candidate placements of a 100k-op DAG, sharded over ranks, one NCCL MIN all-reduce).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

# Each replica runs on its own stream; the default 8 hardware work queues would make
# streams share queues and serialise long kernels of different replicas.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

COMM = (0.001, 10.0)  # generator.hpp:33
METRIC = "placement-gen edges/s (1M-op DAG, 8 devices)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--variant", default="deep", choices=["deep", "wide"])
    p.add_argument("--candidates", type=int, default=8192, help="config #5 batch size for the secondary line")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--stages", action="store_true", help="print per-stage device times to stderr")
    p.add_argument("--stages-under-load", action="store_true",
                   help="print replica 0's per-stage device times during the throughput steps")
    p.add_argument("--ref-sample", type=int, default=250_000,
                   help="ops per reference copy in --impl reference / cpu_baseline (bounded CPU sample)")
    p.add_argument("--replicas", type=int, default=32,
                   help="independent graphs generated concurrently per GPU (one stream + host thread each)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 2 + i and "Active" in s[2 + i]
                          and "Not" not in s[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def pinned_graph(g):
    """Copy a Graph's arrays into page-locked host memory (torch pin_memory)."""
    import torch
    from paper_2208_00184_b200._abi import Graph

    def pin(a):
        t = torch.empty(a.shape, dtype=torch.int64, pin_memory=True)
        arr = t.numpy()
        arr[...] = a
        return arr, t

    keep = []
    arrs = []
    for a in (g.node_id, g.compute_us, g.memory_bytes, g.edge_src, g.edge_dst, g.edge_bytes):
        x, t = pin(a)
        arrs.append(x)
        keep.append(t)
    pg = Graph(*arrs)
    pg._pins = keep  # noqa: SLF001
    return pg


def _new_ctx(lib, device, stream):
    ctx = C.c_void_p()
    rc = lib.dp_ctx_create(device, C.c_void_p(stream), C.byref(ctx))
    if rc:
        raise RuntimeError(lib.dp_last_error_message().decode())
    return ctx


def ncu_traffic(kernel: str, launches: int = 1):
    """dram__bytes_read.sum + dram__bytes_write.sum of `kernel` summed over its first
    `launches` launches, from the newest committed `ncu --set full` summary under profiles/
    (tools/summarize_profiles.py), with the file it came from; (None, None) when no capture
    of that kernel exists."""
    import glob
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*_full.txt")), reverse=True):
        per, cur = [], None
        for line in open(path):
            if line.startswith("## "):
                cur = {} if kernel in line else None
                if cur is not None:
                    per.append(cur)
                continue
            parts = line.split()
            if cur is not None and parts and parts[0] in ("dram__bytes_read.sum", "dram__bytes_write.sum") \
                    and len(parts) >= 3:
                cur[parts[0]] = float(parts[1]) * scale.get(parts[2], 1)
        per = [d for d in per if len(d) == 2][:launches]
        if len(per) == launches:
            return sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in per), os.path.relpath(path, ROOT)
    return None, None


def flush_l2(buf):
    buf.add_(1)  # 256 MiB write > 126 MB L2


def ours(args):
    import torch
    import paper_2208_00184_b200 as pkg
    from paper_2208_00184_b200 import synth
    from paper_2208_00184_b200._abi import PipelineCfgC, comm_c, devices_c
    from paper_2208_00184_b200._native import stage_times

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    be = pkg.device(local, stream.cuda_stream)
    lib = pkg.library()
    ctx = be.ctx
    deep = args.variant == "deep"
    g, devs = synth.config4(deep)
    cfg = PipelineCfgC(200, 0.25, 1, 0)
    res = C.c_void_p()
    gc = g.c()
    dc = devices_c(devs)
    rc = lib.dp_resident_create(ctx, C.byref(gc), C.byref(dc), comm_c(COMM), C.byref(cfg), C.byref(res))
    if rc:
        raise RuntimeError(lib.dp_last_error_message().decode())
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")

    def step():
        rc = lib.dp_resident_generate(res)
        if rc:
            raise RuntimeError(lib.dp_last_error_message().decode())

    # ---- single-graph latency (one placement generation at a time)
    launches0 = lib.dp_ctx_launch_count(ctx)
    for _ in range(args.warmup):
        flush_l2(flush)
        step()
    torch.cuda.synchronize()
    launches_w = lib.dp_ctx_launch_count(ctx)
    per_step_launches = (launches_w - launches0) / max(1, args.warmup)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush_l2(flush)
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    single_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))

    # ---- throughput: R independent graphs per GPU at once (own stream, context and host
    # thread each), like the reference arm's independent graphs on all host cores
    R = max(1, args.replicas)
    reps = []
    for r in range(R):
        st = torch.cuda.Stream()
        rbe = pkg.Backend(lib, "dp_", ctx=_new_ctx(lib, local, st.cuda_stream), name=f"rep{r}")
        rres = C.c_void_p()
        rc = lib.dp_resident_create(rbe.ctx, C.byref(gc), C.byref(dc), comm_c(COMM), C.byref(cfg), C.byref(rres))
        if rc:
            raise RuntimeError(lib.dp_last_error_message().decode())
        reps.append((st, rbe, rres))
    torch.cuda.synchronize()

    # one persistent host thread per replica (created once), released together each step
    errs = []
    go = threading.Barrier(R + 1)
    done = threading.Barrier(R + 1)
    pool_stop = [False]

    def worker(rres):
        while True:
            go.wait()
            if pool_stop[0]:
                return
            rc = lib.dp_resident_generate(rres)
            if rc:
                errs.append(lib.dp_last_error_message().decode())
            done.wait()

    pool = [threading.Thread(target=worker, args=(rr,), daemon=True) for _, _, rr in reps]
    for t_ in pool:
        t_.start()

    def run_all():
        go.wait()
        done.wait()
        if errs:
            raise RuntimeError(errs[0])

    for _ in range(max(2, args.warmup)):
        flush_l2(flush)
        run_all()
    torch.cuda.synchronize()
    master = stream
    evs = []
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = sum(lib.dp_ctx_launch_count(rb.ctx) for _, rb, _ in reps)
    if args.stages_under_load:
        lib.dp_ctx_enable_stage_timing(reps[0][1].ctx, 1)
    with Clocks(local) as clocks:
        t0 = time.perf_counter()
        for i in range(args.steps):
            flush_l2(flush)
            start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            start.record(master)
            for st, _, _ in reps:
                st.wait_event(start)
            run_all()
            for st, _, _ in reps:
                e = torch.cuda.Event()
                e.record(st)
                master.wait_event(e)
            stop.record(master)
            evs.append((start, stop))
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if world > 1:
        torch.distributed.barrier()
    if args.stages_under_load and rank == 0:
        for nm, ms_, _ in stage_times(lib, reps[0][1].ctx):
            print(f"under load (R={R}): stage {nm:18s} {ms_:10.3f} ms", file=sys.stderr)
        lib.dp_ctx_enable_stage_timing(reps[0][1].ctx, 0)
    launches = sum(lib.dp_ctx_launch_count(rb.ctx) for _, rb, _ in reps) - l0
    pool_stop[0] = True
    go.wait()
    for t_ in pool:
        t_.join()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    mean_ms = float(np.mean(step_ms))
    t = torch.tensor([mean_ms], device="cuda")
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    max_ms = float(t.item())
    value = world * R * g.m / (max_ms / 1e3)
    for _, rb, rres in reps:
        lib.dp_resident_destroy(rres)

    # per-stage device times of one extra, separately-timed step (roofline evidence)
    lib.dp_ctx_enable_stage_timing(ctx, 1)
    flush_l2(flush)
    step()
    stages = stage_times(lib, ctx)
    lib.dp_ctx_enable_stage_timing(ctx, 0)
    # the fine graph's levels come first; the coarse graph's (pipeline.cpp:70) second
    seen = set()
    for i, (nm, ms_, by) in enumerate(stages):
        if nm in seen:
            stages[i] = ("coarse " + nm, ms_, by)
        seen.add(nm)
    if args.stages and rank == 0:
        for nm, ms, by in stages:
            print(f"stage {nm:18s} {ms:10.3f} ms  {by / 1e6:10.1f} MB", file=sys.stderr)
    out_dev = np.zeros(g.n, np.int32)
    adj_dev = np.zeros(g.n, np.int32)
    cn, ce = C.c_int64(), C.c_int64()
    lib.dp_resident_fetch(res, out_dev.ctypes.data_as(C.POINTER(C.c_int32)),
                          adj_dev.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(cn), C.byref(ce))
    lib.dp_resident_destroy(res)

    # roofline of the level/relaxation kernel (HBM-bound by design) and of the dominant kernel
    st = {nm: (ms, by) for nm, ms, by in stages}
    gen_ms = st.get("generate", (mean_ms, 0))[0]
    kernels = [(nm, ms, by) for nm, ms, by in stages if nm != "generate"]
    dom = max(kernels, key=lambda x: x[1]) if kernels else ("generate", mean_ms, 0.0)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"

    def roof(nm, ms, by):
        ach = by / (ms / 1e3) / 1e9 if ms > 0 else 0.0
        return {"kernel": nm, "bound": "hbm", "achieved": round(ach, 3), "peak": hbm, "unit": "GB/s",
                "frac": round(ach / hbm, 6), "traffic": None, "ms": round(ms, 4), "algorithmic_bytes": by,
                "peak_source": peak_src}

    lv = st.get("levels")
    roofline = roof(dom[0], dom[1], dom[2])
    roofline["share_of_step"] = round(dom[1] / gen_ms, 4) if gen_ms else None
    roofline["traffic"], roofline["traffic_source"] = ncu_traffic("k_peel_dp")
    roofline["ns_per_node"] = round(dom[1] * 1e6 / g.n, 2)
    levels_roof = roof("levels", lv[0], lv[1]) if lv else None
    if levels_roof:  # the stage is the forward + backward dataflow kernels of the fine graph
        levels_roof["traffic"], levels_roof["traffic_source"] = ncu_traffic("k_levels_flow", 2)

    # e2e through the public C-ABI (dp_pipeline): pinned H2D + generation + D2H of the report
    e2e = None
    if not args.no_e2e:
        # the public C-ABI call (dp_pipeline) with pinned host buffers: H2D upload,
        # generation, D2H of the report; R calls at once like the device-resident step
        pg = pinned_graph(g)
        pgc = pg.c()
        from paper_2208_00184_b200._abi import PipelineC
        pcfg = PipelineCfgC(200, 0.25, 1, 0)
        d2h_box = [0]

        def e2e_all():
            errs = []

            def work(rb):
                p = C.POINTER(PipelineC)()
                rc = lib.dp_pipeline(rb.ctx, C.byref(pgc), C.byref(dc), comm_c(COMM), C.byref(pcfg), C.byref(p))
                if rc:
                    errs.append(lib.dp_last_error_message().decode())
                    return
                r = p.contents
                k, mc, n = r.coarse_nodes, r.coarse_edges, g.n
                # coarse graph, cluster map, two coarse placements (+ decisions), two
                # expanded placements, coarse sequence
                d2h_box[0] = (k * 8 * 3 + mc * 8 * 3) + (n * 4 + n * 8 + k * 8 * 3) + 2 * (k * 4 + 8 * 8) + \
                    k * (8 + 4 + 8 + 8 * 8 + 4 + 2) + 2 * (n * 4 + 8 * 8) + k * 8
                lib.dp_pipeline_result_free(p)
            ths = [threading.Thread(target=work, args=(rb,)) for _, rb, _ in reps]
            for t_ in ths:
                t_.start()
            for t_ in ths:
                t_.join()
            if errs:
                raise RuntimeError(errs[0])

        e2e_all()  # warm-up
        times = []
        for i in range(max(1, min(3, args.steps))):
            flush_l2(flush)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            e2e_all()
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t1)
        e2e_s = float(np.mean(times))
        tt = torch.tensor([e2e_s], device="cuda")
        if world > 1:
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": world * R * g.m / float(tt.item()), "unit": "edges/s", "ms_per_step": float(tt.item()) * 1e3,
               "h2d_bytes_per_step": int(R * 8 * (3 * g.n + 3 * g.m)), "d2h_bytes_per_step": int(R * d2h_box[0]),
               "api": f"dp_pipeline (C-ABI, pinned host buffers), {R} concurrent calls"}
    for _, rb, _ in reps:
        lib.dp_ctx_destroy(rb.ctx)

    cand = candidates(args, be, lib, rank, world) if args.candidates > 0 else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, sample_nodes=args.ref_sample)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": max_ms, "higher_is_better": True, "scaling": "weak",
            "single_graph": {"ms": single_ms, "edges_per_s": g.m / (single_ms / 1e3),
                             "note": "one placement generation at a time (latency)"},
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (SURVEY §8(d) layered recipe, seed 12345)",
            "config": {"workload": f"config#4 {args.variant}: 1M-op layered DAG "
                                   f"(W={'1024' if deep else '65536'}, fan-in 2..6), 8 devices, R=200, "
                                   f"M=0.25*capacity; {R} independent graphs per GPU generated concurrently",
                       "replicas_per_gpu": R,
                       "nodes": g.n, "edges": g.m, "coarse_nodes": cn.value, "coarse_edges": ce.value,
                       "parallelism": f"independent graphs: {R} per GPU x {world} GPU(s)", "l2": "flushed between steps (256 MiB write)"},
            "clocks": clocks.summary(), "e2e": e2e, "gpu_launches": int(launches),
            "gpu_launches_per_step": per_step_launches, "wall_s_timed_region": wall,
            "step_ms_all": [round(x, 3) for x in step_ms],
            "roofline": roofline, "roofline_levels": levels_roof,
            "stages_ms": {nm: round(ms, 3) for nm, ms, _ in stages},
            "cpu_baseline": cpu, "candidates": cand,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def candidates(args, be, lib, rank, world):
    """Config #5: B candidate placements of the 100k-op DAG (cluster reassignments of the
    adjusting placement), makespans on the GPU, shards across ranks, one MIN all-reduce."""
    import torch
    from paper_2208_00184_b200 import synth
    g, devs = synth.config5_graph()
    rep = be.evaluate_pipeline(g, devs, COMM, simulate=False)
    ids = np.array(sorted(d for d, _ in devs))
    base = np.searchsorted(ids, rep.coarse_adjust.device).astype(np.uint8)
    B = args.candidates
    per = (B + world - 1) // world
    lo, hi = rank * per, min(B, (rank + 1) * per)
    cand = synth.candidates(base, len(devs), lo, max(0, hi - lo))
    # warm-up on a slice, then the timed batch
    be.simulate_candidates(g, rep.map.node_cluster, rep.coarse_nodes, cand[:min(len(cand), 64)], devs, COMM)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ms, am = be.simulate_candidates(g, rep.map.node_cluster, rep.coarse_nodes, cand, devs, COMM)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    key = torch.tensor([(int(ms[am]) << 20) | (lo + am) if len(ms) else (1 << 62)], dtype=torch.int64, device="cuda")
    tt = torch.tensor([dt], device="cuda", dtype=torch.float64)
    if world > 1:
        torch.distributed.all_reduce(key, op=torch.distributed.ReduceOp.MIN)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    k = int(key.item())
    return {"metric": "candidate placements/s (config #5: 100k-op DAG, 8 devices)", "value": B / float(tt.item()),
            "unit": "candidates/s", "candidates": B, "coarse_nodes": rep.coarse_nodes, "n_gpus": world,
            "seconds": float(tt.item()), "best_makespan": k >> 20, "best_candidate": k & ((1 << 20) - 1),
            "collective": "NCCL all_reduce MIN over (makespan << 20 | index)" if world > 1 else None}


def cpu_baseline(args, threads=None, sample_nodes=250_000):
    """The UNMODIFIED reference (oracle/_ref, compiled from /root/reference/proj/src)
    timed on this host: `threads` independent copies of a bounded sample of the
    workload (same recipe, first `sample_nodes` ops) run concurrently through the
    reference's own generation window (pipeline.cpp:67-79)."""
    from oracle.bind import reference_available, reference_backend
    from paper_2208_00184_b200 import synth
    from paper_2208_00184_b200._abi import PipelineCfgC, comm_c, devices_c
    if not reference_available():
        return None
    ref = reference_backend()
    threads = threads or min(os.cpu_count() or 1, 16)
    deep = args.variant == "deep"
    g = synth.layered(sample_nodes, 1024 if deep else 65536, 2, 6, 12345)
    cap = synth.capacity_125(g, 8)
    devs = [(d, cap) for d in range(8)]
    wall = (C.c_int64 * threads)()
    tot = C.c_double()
    cfg = PipelineCfgC(200, 0.25, 1, 0)
    rc = ref.pipeline_replicas(C.byref(g.c()), C.byref(devices_c(devs)), comm_c(COMM), C.byref(cfg), threads, wall,
                               C.byref(tot))
    if rc:
        return {"error": ref._err().decode()}
    per_copy = [w / 1e6 for w in wall]
    value = threads * g.m / max(per_copy)
    return {"value": value, "unit": "edges/s", "cores": threads, "kind": "reference",
            "sample": f"{threads} concurrent copies of the first {sample_nodes} ops of the config#4 {args.variant} "
                      f"recipe ({g.m} edges each), reference generation window (pipeline.cpp:67-79)",
            "per_copy_s": [round(x, 3) for x in per_copy], "wall_s": tot.value}


def reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.bind import reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    import torch  # noqa: F401
    steps = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(args, sample_nodes=min(50_000, args.ref_sample) if i < args.warmup else args.ref_sample)
        if i >= args.warmup:
            steps.append(r)
    value = float(np.mean([s["value"] for s in steps]))
    cores = steps[0]["cores"]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "dtype": "int64", "data": "synthetic (SURVEY §8(d) layered recipe, seed 12345)",
            "config": {"workload": f"config#4 {args.variant}: layered DAG, 8 devices, R=200, bounded sample"},
            "ms_per_step": float(np.mean([max(s["per_copy_s"]) for s in steps])) * 1e3,
            "cpu_baseline": {"value": value, "unit": "edges/s", "cores": cores, "kind": "reference",
                             "sample": steps[0]["sample"]},
            "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        reference_arm(a)
    else:
        ours(a)
