#!/bin/bash
mkdir -p gpurun_out/ncu
cap() {  # tag regex bench-args...
  tag=$1; rx=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s 2 -c 1 \
    -o gpurun_out/ncu/$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-converge "$@" \
    > gpurun_out/ncu/$tag.log 2>&1
  echo "$tag rc=$?"
}
cap c2_face "k_face<.bool.0, .bool.0, .bool.0>"
cap c2_roe_mf6 "k_roe_mf<.int.6>"
cap c1_roe_mf5 "k_roe_mf<.int.5>" --workload c1 --n 64
cap c3_face11 "k_face<.bool.1, .bool.1, .bool.0>" --workload c3
