#!/bin/bash
# Launch list + ncu --set full captures of the default bench's top kernels.
# usage: bash tools/gpu_prof.sh <tag> [regex] [bench args...]
TAG=${1:-prof}; RX=${2:-"k_face|k_recon"}; shift 2
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-converge $*"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k "regex:$RX" -s 2 -c 2 -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
echo "rc=$?"
