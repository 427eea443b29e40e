set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log
for W in 1 8 32; do timeout 300 python bench.py --config G --walkers $W --steps 300 --warmup 5 --no-cpu-baseline --e2e-iters 1 --profile-iters 10 2>&1 | tail -1 > gpurun_out/g$W.json; python -c "import json,sys; d=json.load(open('gpurun_out/g$W.json')); print($W, d['ms_per_step'], d['value'], d['roofline']['kernel_ms'])"; done
