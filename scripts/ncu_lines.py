"""Summarise an ncu --import-source report per source line (instructions, stall samples).

    python scripts/ncu_lines.py <report.ncu-rep> <units-per-launch> [top-N] [--ranges a-b:name,...]

Lines are keyed by file (decode.cu lines plus inlined CUDA headers such as the
__shfl intrinsics).  Per-unit counts are warp-level instructions per meshlet.
"""
import csv
import os
import subprocess
import sys

rep, per = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 45
ranges = None
if "--ranges" in sys.argv:
    ranges = []
    for part in sys.argv[sys.argv.index("--ranges") + 1].split(","):
        ab, name = part.split(":")
        a, b = ab.split("-")
        ranges.append((int(a), int(b), name))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, lines = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = os.path.basename(r[1])
        continue
    if r and r[0] == "Line No":
        hdr = r
        ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr and r and r[0]:
        try:
            lines.append((cur, int(r[0]), r[1][:90], float(r[ie] or 0), float(r[ss] or 0)))
        except ValueError:
            pass
tot = sum(x[3] for x in lines)
tots = sum(x[4] for x in lines) or 1
print(f"total warp-instructions {tot:.0f}  per unit {tot / per:.1f}")
byfile = {}
for f, *_rest in lines:
    byfile[f] = byfile.get(f, 0) + _rest[2]
print("per file:", {k: round(v / per, 1) for k, v in byfile.items()})
if ranges:
    for a, b, name in ranges:
        s = sum(x[3] for x in lines if x[0] == "decode.cu" and a <= x[1] < b)
        print(f"  {name:20s} lines {a}-{b}: {s / per:7.1f}/u")
for l in sorted(lines, key=lambda x: -x[3])[:top]:
    print(f"{l[0][:14]:14s} {l[1]:5d} {l[3] / per:8.1f}/u {100 * l[3] / tot:5.1f}% stall {100 * l[4] / tots:5.1f}%  {l[2]}")
