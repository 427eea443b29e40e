#!/bin/bash
# Bench lines for the non-default configurations (run on the GPU box): P (64 walkers), G with walker
# groups, S, the X scaling sweep over nonzeros (1e5 .. 5e7, one walker) and over walkers (X1e6, W = 1
# .. 512); one JSON line each into gpurun_out/sweep.jsonl. Step counts keep every timed region >=
# ~0.5 s (short regions read launch and clock-ramp jitter).
set -u
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
run() { timeout 300 python bench.py --no-cpu-baseline --e2e-iters 2 --profile-iters 20 "$@" 2>>gpurun_out/sweep.err | tail -1 >> gpurun_out/sweep.jsonl; }
run --config P --steps 4000 --warmup 50
run --config G --walkers 8 --steps 800 --warmup 10
run --config G --walkers 32 --steps 250 --warmup 5
run --config S --steps 30000 --warmup 200
run --config X1e5 --steps 20000 --warmup 200
run --config X3e5 --steps 20000 --warmup 200
run --config X1e6 --steps 15000 --warmup 200
run --config X3e6 --steps 8000 --warmup 100
run --config X1e7 --steps 4000 --warmup 50
run --config X2e7 --steps 2000 --warmup 30
run --config X5e7 --steps 1000 --warmup 20
for W in 8 64 512; do
  run --config X1e6 --walkers $W --steps $((4000 / (W / 8 + 1) + 100)) --warmup 10
done
