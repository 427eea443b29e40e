#!/bin/bash
# GPU box: parity suite, per-kernel device times (chap_walkers_profile) on G and Gnl, and one ncu
# --set full capture of the top kernel (default k_eval_gen) on config G.
#   tools/quick_check.sh [kernel-regex] [tag]
set -u
mkdir -p gpurun_out
K=${1:-k_eval_gen}
TAG=${2:-q}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
tail -4 gpurun_out/gputest.log
cp paper_2605_05086_b200/libchap.so /tmp/cur.so
for c in G Gnl; do timeout 200 python tools/variant_time.py $c /tmp/cur.so; done 2>&1 | tee gpurun_out/vt_$TAG.log
rm -f gpurun_out/$TAG.ncu-rep
timeout 600 ncu --set full --import-source on --clock-control none -k regex:$K --launch-skip 20 -c 1 -o gpurun_out/$TAG \
  python tools/prof_step.py 20 3 G > gpurun_out/$TAG.log 2>&1
echo ncu=$?
