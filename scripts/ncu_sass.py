"""Print the SASS of one source-line range of an ncu --import-source report with per-instruction
warp-level execution counts per unit.   python scripts/ncu_sass.py <rep> <units> <file> <a> <b>"""
import csv
import os
import subprocess
import sys

rep, per, fname, a, b = sys.argv[1], float(sys.argv[2]), sys.argv[3], int(sys.argv[4]), int(sys.argv[5])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, line, src = None, None, None, ""
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        cur = os.path.basename(r[1]); continue
    if r and r[0] == "Line No":
        hdr = r; ie = hdr.index("Instructions Executed"); continue
    if not hdr or not r:
        continue
    if r[0]:
        if not r[0].isdigit():
            continue
        line, src = int(r[0]), r[1]
        if cur == fname and a <= line < b:
            print(f"--- {line}: {src[:100]}")
    elif cur == fname and line is not None and a <= line < b:
        try:
            n = float(r[ie] or 0) / per
        except ValueError:
            continue
        print(f"   {n:7.2f}  {r[3]}")
