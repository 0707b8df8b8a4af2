"""Render scripts/sweep_cfg5.py output (jsonl) as a markdown table.
    python scripts/sweep_table.py gpurun_out/sweep_cfg5.jsonl [label] > profiles/round1_cfg5_sweep.md"""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1])]
labels = sorted({r["label"] for r in rows})
want = sys.argv[2] if len(sys.argv) > 2 else None
print("# cfg5 sweep — meshlet size x grid width (1 x B200)\n")
print("Displaced cube-sphere k=300 (1.08M tris) x 10 instances, pos3+nrm3+uv2, GTS-Reuse, "
      "kernel time per launch (CUDA events, 20 launches after 3 warm-ups). bits/tri = whole blob "
      "(header + directory + records) per real triangle.\n")
for lab in labels:
    if want and lab != want:
        continue
    print(f"## variant `{lab}`\n")
    print("| Ṽ/T̃ | b | bits/tri | restarts/meshlet | Gtri/s | alg. GB/s | error bits |")
    print("|---|---|---|---|---|---|---|")
    for r in rows:
        if r["label"] != lab:
            continue
        print(f"| {r['vmax']}/{r['tmax']} | {r['bits']} | {r['bits_per_tri']:.1f} | {r['restarts_per_meshlet']} | "
              f"{r['gtri_s']:.1f} | {r['alg_gb_s']:.0f} | {r['error_bits']} |")
    print()
