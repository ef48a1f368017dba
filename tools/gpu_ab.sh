#!/bin/bash
# A/B of library variants on the default bench (kernel breakdown), then the parity tests.
# usage: tools/gpu_ab.sh "<pytest -k expr or empty>" tagA=libA.so tagB=libB.so ...  ("base" = in-tree lib)
mkdir -p gpurun_out
K="$1"; shift
for spec in "$@"; do
  tag=${spec%%=*}; lib=${spec#*=}
  if [ "$lib" = "base" ]; then unset GKS_LIB; else export GKS_LIB=$PWD/$lib; fi
  for rep in 1 2; do
    timeout 600 python bench.py --no-cpu-baseline --no-converge --no-c5 --steps 5 ${BENCH_ARGS} > gpurun_out/ab_${tag}_${rep}.json 2> gpurun_out/ab_${tag}_${rep}.err
    python - "$tag" "$rep" <<'PY'
import json,sys
t,r=sys.argv[1],sys.argv[2]
for l in open(f"gpurun_out/ab_{t}_{r}.json"):
    if l.startswith("{"):
        d=json.loads(l); k=d.get("kernels",{})
        print(t, r, "ms/step %.2f"%d["ms_per_step"], " ".join("%s %.4f"%(n,k[n]["ms_per_launch"]) for n in ("face_flux","recon","assemble","reduce_dot","jacobi_sweep") if n in k), flush=True)
PY
  done
done
unset GKS_LIB
if [ -n "$K" ]; then timeout 1200 python -m pytest tests -m gpu -q -x -k "$K" > gpurun_out/pytest_ab.log 2>&1; tail -3 gpurun_out/pytest_ab.log; fi
