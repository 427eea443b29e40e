#!/bin/bash
# GPU box: bench ms/step with chap_params overrides (A/B), e.g.
#   tools/ab_params.sh G "" "l2_persist=0" "aspiration=1"
CFG=$1; shift
EXTRA=${EXTRA:-}
mkdir -p gpurun_out
for ps in "$@"; do
  args=""; for kv in $ps; do args="$args --param $kv"; done
  r=$(timeout 300 python bench.py --config $CFG --steps 2000 --warmup 20 --no-cpu-baseline --profile-iters 50 --e2e-iters 2 $EXTRA $args 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.4f ms/step  kernels %s' % (d['ms_per_step'], {k: round(v*1000,1) for k, v in d['roofline']['kernel_ms'].items()}))")
  echo "$CFG [$ps]: $r" | tee -a gpurun_out/ab.log
done
