"""Per-CUDA-source-line stall samples of an ncu report (--page source --print-source cuda,sass):
python tools/ncu_lines.py report.ncu-rep [kernel-regex] [top]."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
extra = ["-k", f"regex:{sys.argv[2]}"] if len(sys.argv) > 2 and sys.argv[2] else []
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", *extra],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, h, res = "?", None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        h = r
    elif h and len(r) == len(h) and r[0] not in ("", "Line No"):
        iS = h.index("Warp Stall Sampling (All Samples)")
        sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
        s = int(r[iS]) if r[iS] not in ("-", "") else 0
        if s:
            why = sorted(((int(r[c]) if r[c] not in ("-", "") else 0, h[c][6:]) for c in sc), reverse=True)[:3]
            res.append((s, fname, r[0], r[1].strip(), why))
tot = sum(x[0] for x in res)
print(f"{tot} stall samples")
for s, f, ln, src, why in sorted(res, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {f}:{ln:5s} {src[:70]:70s} {' '.join(f'{n}={v}' for v, n in why if v)}")
