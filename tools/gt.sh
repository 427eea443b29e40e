set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
tail -25 gpurun_out/gputest.log
timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-iters 2 --profile-iters 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])"
