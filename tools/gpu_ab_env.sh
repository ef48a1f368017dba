#!/bin/bash
# A/B of an environment switch on the default bench (kernel breakdown):
#   tools/gpu_ab_env.sh VAR v1 v2 ...      (BENCH_ARGS for other workloads)
var=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    env $var=$v timeout 600 python bench.py --no-cpu-baseline --no-converge --no-c5 --steps 5 ${BENCH_ARGS} 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']
        print('$var=$v', 'ms/step %.2f'%d['ms_per_step'], ' '.join('%s %.4f'%(n,k[n]['ms_per_launch']) for n in ('face_flux','recon','assemble','reduce_dot','jacobi_sweep') if n in k), flush=True)
"
  done
done
