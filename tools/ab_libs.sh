#!/bin/bash
# GPU box: in-graph timing (tools/graph_time.py) of libchap variants, one process per measurement,
# interleaved over R repetitions.   tools/ab_libs.sh CFG R lib1.so lib2.so ...
#   (PARAMS="--param=pdl=1 ..." in the environment: chap_params overrides)
CFG=$1; R=$2; shift 2
for i in $(seq $R); do for v in "$@"; do timeout 300 python tools/graph_time.py $CFG 1000 1 $v $PARAMS; done; done 2>&1 | grep step | sort | tee -a gpurun_out/ab_libs.log
