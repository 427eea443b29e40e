#!/bin/bash
# bench ms/step of alternative libchap builds (swapped in place):
#   tools/env_sweep.sh CFG lib1.so lib2.so ...
CFG=$1; shift
cp paper_2605_05086_b200/libchap.so /tmp/libchap_keep.so
for lib in "$@"; do
  cp "$lib" paper_2605_05086_b200/libchap.so
  r=$(timeout 300 python bench.py --config $CFG --steps 2000 --warmup 20 --no-cpu-baseline --profile-iters 50 --e2e-iters 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f ms/step  kernels %s' % (d['ms_per_step'], {k: round(v*1000,1) for k, v in d['roofline']['kernel_ms'].items()}))")
  echo "$CFG $(basename $lib): $r"
done
cp /tmp/libchap_keep.so paper_2605_05086_b200/libchap.so
