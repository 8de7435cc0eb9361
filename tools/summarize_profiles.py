"""Summarise a gpurun session's ncu output into profiles/ (tracked evidence).

    python tools/summarize_profiles.py <tag> [gpurun_out]

Writes profiles/<tag>_launches.txt (per-kernel share of the launch list, from
`ncu --metrics gpu__time_duration.sum`), profiles/<tag>_ncu_full.txt (key counters of
each kernel in the `ncu --set full` capture, incl. dram bytes = roofline `traffic`) and
profiles/<tag>_stalls.txt (hottest SASS instructions of each captured kernel).
"""
from __future__ import annotations

import csv
import glob
import io
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}


def launches(path: str) -> str:
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = defaultdict(lambda: [0, 0.0])
    for x in rows:
        if x["Metric Name"] != "gpu__time_duration.sum":
            continue
        us = float(x["Metric Value"].replace(",", "")) * UNIT.get(x["Metric Unit"], 1.0)
        name = x["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    out = [f"# {len(rows)} launches, {tot / 1e3:.3f} ms total (ncu: cold-cache, serialised; compare shares)",
           f"{'total_ms':>12} {'launches':>8} {'share':>7}  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{v[1] / 1e3:12.3f} {v[0]:8d} {100 * v[1] / tot:6.2f}%  {k}")
    return "\n".join(out) + "\n"


FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
]


def ncu_csv(rep: str, page: str, extra=()) -> list[list[str]]:
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def full(rep: str) -> str:
    r = ncu_csv(rep, "raw")
    h, units = r[0], r[1]
    idx = [h.index(m) for m in FULL_METRICS if m in h]
    out = [f"# {os.path.basename(rep)}: ncu --set full --clock-control none (per launch)"]
    for row in r[2:]:
        out.append(f"## {row[h.index('Kernel Name')]}")
        for i in idx:
            out.append(f"  {h[i]:70s} {row[i]:>16s} {units[i]}")
    return "\n".join(out) + "\n"


def stalls(rep: str, top: int = 25) -> str:
    names = sorted({row[h_i] for r in [ncu_csv(rep, "raw")] for h_i in [r[0].index("Kernel Name")] for row in r[2:]})
    out = []
    for nm in names:
        import re
        mk = re.search(r"\bk_\w+", nm)
        short = mk.group(0) if mk else nm.split("(")[0].split("::")[-1]
        r = ncu_csv(rep, "source", ["-k", f"regex:{short}", "--print-source", "sass"])
        hi = next((i for i, row in enumerate(r) if row and row[0] == "Address"), None)
        if hi is None:
            out.append(f"## {short}: no source page")
            continue
        h = r[hi]
        nxt = next((i for i in range(hi + 1, len(r)) if r[i] and r[i][0] == "Address"), len(r))
        rows = [x for x in r[hi + 1:nxt] if len(x) == len(h) and x[0].startswith("0x")]  # first launch only
        iS, iE = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
        scols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        tot = sum(int(x[iS] or 0) for x in rows)
        out.append(f"## {short}: {tot} stall samples, {sum(int(x[iE] or 0) for x in rows)} warp instructions")
        for i in sorted(sorted(range(len(rows)), key=lambda i: -int(rows[i][iS] or 0))[:top]):
            x = rows[i]
            why = sorted(((int(x[c] or 0), h[c]) for c in scols), reverse=True)[:2]
            out.append(f"  {x[0][-6:]} {x[1].strip()[:56]:56s} {int(x[iS]):8d} {100 * int(x[iS]) / max(1, tot):5.1f}%"
                       f"  exec={x[iE]:>9s}  {', '.join(f'{n}={v}' for v, n in why if v)}")
    return "\n".join(out) + "\n"


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    dst = os.path.join(ROOT, "profiles")
    os.makedirs(dst, exist_ok=True)
    for f in glob.glob(os.path.join(src, "launches*.csv")):
        suffix = os.path.basename(f)[len("launches"):-4]
        open(os.path.join(dst, f"{tag}_launches{suffix}.txt"), "w").write(launches(f))
    for rep in glob.glob(os.path.join(src, "*.ncu-rep")):
        base = os.path.basename(rep)[:-8]
        open(os.path.join(dst, f"{tag}_{base}_full.txt"), "w").write(full(rep))
        open(os.path.join(dst, f"{tag}_{base}_stalls.txt"), "w").write(stalls(rep))
    print("written to", dst)


if __name__ == "__main__":
    main()
