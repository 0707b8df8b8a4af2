"""Summarise an ncu --import-source report per CUDA source line (instructions, stall samples)."""
import csv
import subprocess
import sys

rep, per = sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[2]
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
lines = []
for r in rows[3:]:
    if r and r[0]:
        try:
            lines.append((int(r[0]), r[1][:95], float(r[ie] or 0), float(r[ss] or 0)))
        except ValueError:
            pass
tot = sum(x[2] for x in lines)
tots = sum(x[3] for x in lines) or 1
print(f"total warp-instructions {tot:.0f}  per unit {tot / per:.1f}")
for l in sorted(lines, key=lambda x: -x[2])[:int(sys.argv[3]) if len(sys.argv) > 3 else 45]:
    print(f"{l[0]:5d} {l[2] / per:8.1f}/u {100 * l[2] / tot:5.1f}% stall {100 * l[3] / tots:5.1f}%  {l[1]}")
