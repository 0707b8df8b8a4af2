"""Compare key metrics of several ncu reports side by side.   python scripts/ncu_compare.py a.ncu-rep b.ncu-rep ..."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__sass_inst_executed_op_global_st.sum", "smsp__sass_inst_executed_op_global_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
STALL = "smsp__pcsamp_warps_issue_stalled_"
cols = []
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    d = {k: (v[i], u[i]) for i, k in enumerate(h)}
    st = {k[len(STALL):]: float(val.replace(",", "")) for k, (val, _) in d.items()
          if k.startswith(STALL) and not k.endswith("not_issued") and val.replace(",", "").replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    cols.append((rep.split("/")[-1], d, {k: 100 * x / tot for k, x in st.items()}))
print(f"{'metric':62s}" + "".join(f"{c[0][-24:]:>26s}" for c in cols))
for k in KEYS:
    print(f"{k:62s}" + "".join(f"{(c[1].get(k, ('-', ''))[0] + ' ' + c[1].get(k, ('', ''))[1])[:25]:>26s}" for c in cols))
allst = sorted({s for c in cols for s in c[2]}, key=lambda s: -max(c[2].get(s, 0) for c in cols))
for s in allst[:14]:
    print(f"{'stall% ' + s:62s}" + "".join(f"{c[2].get(s, 0):26.1f}" for c in cols))
