#!/bin/bash
# Ma 3 study runs (profiles/r02/ma3/): KFVS first-order start, then high-order switches
mkdir -p gpurun_out/ma3
t() { tag=$1; shift; timeout 900 python tools/ma3_kfvs.py "$@" --out gpurun_out/ma3/$tag.json > gpurun_out/ma3/$tag.log 2>&1; python -c "
import json,sys; d=json.load(open('gpurun_out/ma3/$tag.json')); d.pop('hist_every_50',None); print('$tag', json.dumps(d))" 2>/dev/null || tail -c 400 gpurun_out/ma3/$tag.log; }
t kfvs_only_ma3 --n 6 --kfvs-only --kfvs-steps 6000
t weno_drop6_ma3 --n 6 --scheme weno_gmres --kfvs-steps 3000 --kfvs-drop 6 --steps 2000
for ma in 2.0 1.5; do
  t weno_ma$ma --n 6 --ma $ma --scheme weno_gmres --kfvs-steps 1500 --kfvs-drop 3 --steps 4000
  t hweno_ma$ma --n 6 --ma $ma --scheme hweno_gmres --kfvs-steps 1500 --kfvs-drop 3 --steps 4000
done
