#!/bin/bash
# ncu --set full (+source) capture of one kernel of the default bench step
# usage: tools/gpu_ncu_face.sh <tag> <kernel regex> [bench args]
TAG=$1; RX=$2; shift 2
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-converge $*"
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$RX" -s 1 -c 1 -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${TAG}_ncu.log
