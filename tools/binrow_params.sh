#!/bin/bash
# k_eval_binrow ring shapes (entries per consumer thread x stages) on config G: kernel time by ncu.
mkdir -p gpurun_out; : > gpurun_out/binrow_params.txt
for v in "-DCHAP_ROW_PER=4 -DCHAP_ROW_STAGES=3" "-DCHAP_ROW_PER=2 -DCHAP_ROW_STAGES=6" "-DCHAP_ROW_PER=6 -DCHAP_ROW_STAGES=2"; do
  CHAP_NVCC_FLAGS="$v" python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || { echo "build fail $v" >> gpurun_out/binrow_params.txt; continue; }
  touch paper_2605_05086_b200/csrc/chap.cu
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bp.csv python tools/prof_step.py 20 5 G > /dev/null 2>&1
  python - "$v" >> gpurun_out/binrow_params.txt <<'PY'
import csv,sys
rows=list(csv.reader(open('gpurun_out/bp.csv'))); hdr=None; v=[]
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        d=dict(zip(hdr,r))
        if d['Kernel Name'].startswith('k_eval_binrow'): v.append(float(d['Metric Value']))
print(repr(sys.argv[1]), sum(v[-5:])/5 if v else None)
PY
done
