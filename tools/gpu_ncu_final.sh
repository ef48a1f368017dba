#!/bin/bash
# final-tree ncu evidence: the C2 launch list of the bench command and full
# captures of the two kernels changed late in round 2 (pair-batched Jacobi
# sweep) plus the dominant face kernel
mkdir -p gpurun_out/ncu
cap() {  # tag regex bench-args...
  tag=$1; rx=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$rx" -s 2 -c 1 \
    -o gpurun_out/ncu/$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-converge --no-c5 "$@" \
    > gpurun_out/ncu/$tag.log 2>&1
  echo "$tag rc=$?"
}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_c2.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-converge --no-c5 > /dev/null 2>&1
echo "launches c2 rc=$?"
cap c2_assemble_tile "k_assemble_tile"
cap c2_roe_mf6 "k_roe_mf<.int.6>"
cap c2_face "k_face<.bool.0, .bool.0, .bool.0>"
cap c2_recon_weno "k_recon_weno"
