"""Summarise an `ncu --set full` report into profiles/ (text) and profiles/ncu_summary.json.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep <name> <workload> <units-per-launch>

MC_PROFILES_DIR overrides the output directory (profiles/).  The JSON keeps, per workload, the DRAM bytes of one launch of the decode kernel
(`dram__bytes_read.sum + dram__bytes_write.sum`), which bench.py reports as
roofline.traffic.
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__sass_inst_executed_op_tma_ld.sum",
    "smsp__sass_inst_executed_op_global_st.sum", "smsp__sass_inst_executed_op_shared_ld.sum",
    "sm__cycles_elapsed.avg",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main():
    rep, name, workload = sys.argv[1], sys.argv[2], sys.argv[3]
    units = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, unit = rows[0], rows[1]
    lines = [f"# ncu --set full summary: {name} ({workload}), report {os.path.basename(rep)}"]
    res = {}
    for row in rows[2:]:
        kname = row[hdr.index("Kernel Name")]
        lines.append(f"\n## {kname}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"{k:70s} {unit[i]:>14s} {row[i]}")
                try:
                    res[k] = float(row[i].replace(",", "")) * SCALE.get(unit[i], 1.0)
                except ValueError:
                    pass
    dram = res.get("dram__bytes_read.sum", 0) + res.get("dram__bytes_write.sum", 0)
    t = res.get("gpu__time_duration.sum", 0)
    lines.append(f"\nDRAM bytes per launch: {dram:.0f}  ({dram / units:.2f} per unit)")
    if t:
        lines.append(f"DRAM GB/s under ncu (cold, serialised): {dram / t / 1e9:.1f}")
    if "smsp__inst_executed.sum" in res:
        lines.append(f"warp-instructions per unit: {res['smsp__inst_executed.sum'] / units:.1f}")
    outdir = os.environ.get("MC_PROFILES_DIR", os.path.join(ROOT, "profiles"))
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, f"{name}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    js = os.path.join(outdir, "ncu_summary.json")
    data = json.load(open(js)) if os.path.exists(js) else {}
    data[workload] = {"dram_bytes_per_launch": dram, "report": name, "kernel_time_s_ncu": t,
                      "warp_instructions_per_meshlet": res.get("smsp__inst_executed.sum", 0) / units,
                      "issue_active_pct": res.get("smsp__issue_active.avg.pct_of_peak_sustained_active")}
    json.dump(data, open(js, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
