"""Executed warp-instructions per unit by SASS opcode (first mnemonic token) of an ncu
--import-source report.   python scripts/ncu_opmix.py <rep> <units> [top]"""
import csv
import subprocess
import sys
from collections import Counter

rep, per = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
cnt = Counter()
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        ie = hdr.index("Instructions Executed")
        src = hdr.index("Source")
        continue
    if hdr and len(r) > ie:
        try:
            n = float(r[ie] or 0)
        except ValueError:
            continue
        toks = r[src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        cnt[op.split(".")[0]] += n
tot = sum(cnt.values())
print(f"total per unit {tot / per:.1f}")
for op, n in cnt.most_common(top):
    print(f"{op:12s} {n / per:8.1f}  {100 * n / tot:5.1f}%")
