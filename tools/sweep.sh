#!/bin/bash
# Bench lines for the non-default configurations (run on the GPU box): P (64 walkers), G with walker
# groups, S, and the X scaling sweep; one JSON line each into gpurun_out/sweep.jsonl.
set -u
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
run() { timeout 300 python bench.py --no-cpu-baseline --e2e-iters 2 --profile-iters 20 "$@" 2>>gpurun_out/sweep.err | tail -1 >> gpurun_out/sweep.jsonl; }
run --config P --steps 1000 --warmup 20
run --config G --walkers 8 --steps 200 --warmup 5
run --config G --walkers 32 --steps 50 --warmup 5
run --config S --steps 4000 --warmup 50
for c in X1e5 X1e6 X1e7 X5e7; do run --config $c --steps 500 --warmup 10; done
