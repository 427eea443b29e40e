set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log
for W in 32 128; do timeout 300 python bench.py --config G --walkers $W --steps 150 --warmup 5 --no-cpu-baseline --e2e-iters 1 --profile-iters 5 2>&1 | tail -1 > gpurun_out/g$W.json; cat gpurun_out/g$W.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config'].get('walkers'), d['ms_per_step'], d['value'], d.get('kernels_us', d.get('profile')))"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g32_launches.csv python tools/prof_step.py 6 2 G 32 > /dev/null 2>&1; echo ncu=$?
