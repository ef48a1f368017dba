#!/bin/bash
# ncu --set full captures of every kernel family (one launch each) + launch lists
mkdir -p gpurun_out/ncu
cap() {  # tag regex bench-args...
  tag=$1; rx=$2; shift 2
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$rx" -s 2 -c 1 \
    -o gpurun_out/ncu/$tag python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-converge "$@" \
    > gpurun_out/ncu/$tag.log 2>&1
  echo "$tag rc=$?"
}
cap c2_recon_weno "k_recon_weno"
cap c2_assemble5 "k_assemble5"
cap c2_roe_mf5 "k_roe_mf<5>"
cap c2_roe_mf6 "k_roe_mf<6>"
cap c2_axpy_dot "k_axpy_dot"
cap c2_dot2 "k_dot2"
cap c2_jac_faces "k_jac_faces"
cap c2_jac_diag "k_jac_diag"
cap c2_face "k_face<0, 0>"
cap c3_recon_hweno "k_recon_hweno" --workload c3
cap c3_face11 "k_face<1, 1>" --workload c3
cap c1_gm_arnoldi "k_gm_arnoldi" --workload c1 --n 16
for w in "c2" "c3" "c1 --n 16"; do
  tag=$(echo $w | tr -d ' -')
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_$tag.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-converge --workload $w > /dev/null 2>&1
  echo "launches $tag rc=$?"
done
