#!/bin/bash
# GPU box: per-kernel device times of the in-tree build and of vlibs/*.so on G and Gnl; then the
# GPU parity suite on the in-tree build.   tools/vt_check.sh [tag]
TAG=${1:-v}
mkdir -p gpurun_out
cp paper_2605_05086_b200/libchap.so /tmp/cur.so
for c in G Gnl; do timeout 300 python tools/variant_time.py $c /tmp/cur.so $(ls vlibs/*.so 2>/dev/null); done 2>&1 | tee gpurun_out/vt_$TAG.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log
