"""Brief of one kernel in an ncu report: key counters, top stall reasons, instruction mix by source
function and line.  Usage: python tools/ncu_brief.py REPORT.ncu-rep [kernel-regex] [lines]"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
k = sys.argv[2] if len(sys.argv) > 2 else "k_eval_gen"
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 20
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{k}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, v = rows[0], rows[2]
for w in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "lts__t_bytes.sum",
          "launch__registers_per_thread", "launch__grid_size", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
          "lts__t_sector_hit_rate.pct"]:
    if w in h:
        print(f"  {w:60s} {v[h.index(w)]} {rows[1][h.index(w)]}")
st = []
for i, name in enumerate(h):
    if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
        try:
            st.append((float(v[i]), name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
        except ValueError:
            pass
print("  stalls/issue:", ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "-k", f"regex:{k}"],
                     capture_output=True, text=True).stdout
open("/tmp/_src.csv", "w").write(src)
root = os.path.dirname(os.path.abspath(__file__))
print(subprocess.run([sys.executable, os.path.join(root, "ncu_lines.py"), "/tmp/_src.csv", str(nl), "inst"],
                     capture_output=True, text=True).stdout)
