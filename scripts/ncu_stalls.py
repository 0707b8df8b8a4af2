"""Top SASS instructions by one stall reason in an ncu --set full report (source page).

    python scripts/ncu_stalls.py <report.ncu-rep> [stall column, default stall_long_sb] [top-N]

Prints the instruction, its samples of that reason, and the share of all samples.
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
i_src, i_col, i_all = hdr.index("Source"), hdr.index(col), hdr.index("Warp Stall Sampling (All Samples)")
ins = [r for r in rows if r and r[0].startswith("0x") and len(r) == len(hdr)]
tot = sum(float(r[i_all] or 0) for r in ins) or 1
tcol = sum(float(r[i_col] or 0) for r in ins)
print(f"{col}: {100 * tcol / tot:.1f}% of {tot:.0f} samples")
idx = {r[0]: k for k, r in enumerate(ins)}
for r in sorted(ins, key=lambda r: -float(r[i_col] or 0))[:top]:
    k = idx[r[0]]
    prev = ins[k - 1][i_src].strip() if k else ""
    print(f"{100 * float(r[i_col]) / tot:5.2f}%  {k:5d}  {r[i_src].strip()[:60]:60s} <- {prev[:50]}")
