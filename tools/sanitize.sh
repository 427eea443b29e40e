#!/bin/bash
# GPU box: compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_run.py (configs T,
# S-small and a mixed instance with every column class; row-wise forced, column-wise forced, walker
# groups). Summaries in gpurun_out/sanitize_*.txt.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for w in T S M; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py $w \
      > gpurun_out/sanitize_${tool}_$w.txt 2>&1
    echo "$tool $w rc=$? $(tail -1 gpurun_out/sanitize_${tool}_$w.txt)"
  done
done
