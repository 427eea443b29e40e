#!/bin/bash
# Run on the GPU box (gpurun): the default bench line, the ncu launch list of the same command
# (cold-cache, serialised per-launch times) and one full ncu capture of the step's kernels.
set -u
mkdir -p gpurun_out
CFG=${1:-G}
timeout 900 python bench.py --config $CFG > gpurun_out/bench_$CFG.json 2> gpurun_out/bench_$CFG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 20 --warmup 5 \
  --no-cpu-baseline --profile-iters 5 --e2e-iters 2 > gpurun_out/launches_$CFG.log 2>&1
rm -f gpurun_out/full_$CFG.ncu-rep   # never summarise a stale capture
# 40 + 3 iterations of 4-5 matching kernels each: skip 120, capture one whole iteration (the capture
# starts at any of its kernels; -c 5 covers an iteration of either size)
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_eval|k_apply' \
  --launch-skip 120 -c 5 -o gpurun_out/full_$CFG python tools/prof_step.py 40 3 $CFG \
  > gpurun_out/full_$CFG.log 2>&1
tail -c 600 gpurun_out/bench_$CFG.json
