"""Key counters of one kernel in an ncu report: python tools/ncu_summary.py report.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "launch__registers_per_thread",
        "launch__grid_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
for v in rows[2:]:
    name = v[h.index("Kernel Name")] if "Kernel Name" in h else ""
    print("==", name[:80])
    for a, b, c in zip(h, u, v):
        if a in keys:
            print(f"  {a:70s} {b:8s} {c}")
    st = []
    for a, c in zip(h, v):
        if a.startswith("smsp__average_warps_issue_stalled") and a.endswith("per_issue_active.ratio"):
            try:
                st.append((float(c), a.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    print("  stalls/issue:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:9]))
