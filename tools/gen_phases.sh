#!/bin/bash
# Timing-only variants of k_eval_gen (results wrong on purpose): which phase of gen_tile costs what.
mkdir -p gpurun_out; : > gpurun_out/gen_phases.txt
for v in "" "-DCHAP_GEN_MINB=4"; do
  CHAP_NVCC_FLAGS="$v" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build fail $v" >> gpurun_out/gen_phases.txt; continue; }
  touch paper_2605_05086_b200/csrc/chap.cu
  timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__grid_size,launch__occupancy_limit_shared_mem,launch__occupancy_limit_registers --clock-control none --csv --log-file gpurun_out/gp.csv python tools/prof_step.py 20 5 G > /dev/null 2>&1
  python - "$v" >> gpurun_out/gen_phases.txt <<'PY'
import csv,sys,collections
rows=list(csv.reader(open('gpurun_out/gp.csv'))); hdr=None; ks=collections.defaultdict(list)
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d['Kernel Name'].startswith('k_eval_gen'): ks[d['Metric Name']].append(float(d['Metric Value']))
print(repr(sys.argv[1]), {k: v[-1] for k,v in ks.items()})
PY
done
