"""Summaries of a tools/gpu_profiles.sh run for profiles/ (tracked):
  python tools/summarize_profiles.py CFG TAG
reads gpurun_out/{bench,launches,full}_CFG.* and writes profiles/TAG_{bench_CFG.json,
launches_CFG.txt, ncu_full_CFG.txt} and profiles/traffic.json (DRAM bytes per launch of the eval
kernels, from the full capture, used by bench.py's roofline.traffic)."""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

cfg, tag = sys.argv[1], sys.argv[2]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
pr = os.path.join(root, "profiles")

# bench line
line = open(os.path.join(go, f"bench_{cfg}.json")).read().strip().splitlines()[-1]
json.loads(line)
open(os.path.join(pr, f"{tag}_bench_{cfg}.json"), "w").write(line + "\n")

# launch list: per-kernel count / mean / share of the eval+apply time
rows = [r for r in csv.reader(open(os.path.join(go, f"launches_{cfg}.csv"))) if len(r) > 14]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = defaultdict(list)
for r in rows[1:]:
    if r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    v = float(r[vi]) * (1e-3 if r[ui] == "ns" else 1.0)
    agg[r[ki].split("(")[0]].append(v)
# the tabu iteration's kernels: the eval/apply kernels launched about once per iteration (the
# eval API's few e2e launches of k_eval_bin are not part of the step)
nit = max(len(v) for k, v in agg.items() if k == "k_apply") if "k_apply" in agg else 0
step = [k for k in ("k_eval_bin", "k_eval_binrow", "k_eval_gen", "k_eval", "k_apply")
        if k in agg and len(agg[k]) >= max(1, nit // 2)]
tot = sum(sum(agg[k]) / max(1, len(agg[k])) for k in step if k in agg)
out = [f"ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches) "
       f"of `bench.py --config {cfg} --steps 20 --warmup 5`",
       f"{'kernel':28s} {'launches':>8s} {'mean us':>9s} {'share of step':>14s}"]
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    m = sum(v) / len(v)
    share = f"{100 * m / tot:13.1f}%" if k in step else ""
    out.append(f"{k:28s} {len(v):8d} {m:9.2f} {share:>14s}")
open(os.path.join(pr, f"{tag}_launches_{cfg}.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out))

# full capture
rep = os.path.join(go, f"full_{cfg}.ncu-rep")
if not os.path.exists(rep):
    sys.exit(f"no capture {rep}: rerun tools/gpu_profiles.sh")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
H, U = rr[0], rr[1]
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
txt = [f"ncu --set full --clock-control none, one launch each (tools/prof_step.py {cfg}, after 20 iterations)"]
traffic = 0.0
warp_instr = {}
seen = set()
for v in rr[2:]:
    name = v[H.index("Kernel Name")].split("(")[0]
    if name in seen:   # the capture may run into the next iteration: one launch per kernel
        continue
    seen.add(name)
    txt.append(f"== {name}")
    d = {}
    for a, u, c in zip(H, U, v):
        if a in keys:
            txt.append(f"  {a:66s} {u:10s} {c}")
            d[a] = (u, c)
    st = []
    for a, c in zip(H, v):
        if a.startswith("smsp__average_warps_issue_stalled") and a.endswith("per_issue_active.ratio"):
            try:
                st.append((float(c), a[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    txt.append("  stall cycles per issued instruction: " + ", ".join(f"{n} {x:.2f}" for x, n in sorted(st, reverse=True)[:8]))
    if "smsp__inst_executed.sum" in d:
        warp_instr[name] = float(d["smsp__inst_executed.sum"][1])
    if name in ("k_eval_bin", "k_eval_binrow", "k_eval_gen", "k_eval"):
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            u, c = d[k]
            traffic += float(c) * {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0}[u]
open(os.path.join(pr, f"{tag}_ncu_full_{cfg}.txt"), "w").write("\n".join(txt) + "\n")
json.dump({"config": cfg, "dram_bytes_per_launch": traffic, "warp_instructions_per_launch": warp_instr,
           "source": f"profiles/{tag}_ncu_full_{cfg}.txt: dram__bytes_read.sum + dram__bytes_write.sum of "
                     "k_eval_bin + k_eval_binrow + k_eval_gen + k_eval, one launch each"},
          open(os.path.join(pr, "traffic.json"), "w"), indent=1)
print("traffic", traffic)
