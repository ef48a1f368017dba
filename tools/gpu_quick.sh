#!/bin/bash
# parity suite + a bench line (args forwarded to bench.py)
mkdir -p gpurun_out
TAG=${1:-q}; shift
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py --no-cpu-baseline "$@" > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python - "$TAG" <<'PY'
import json,sys
t=sys.argv[1]
try:
    d=json.load(open(f"gpurun_out/{t}_bench.json"))
    print("value %.4g ms/step %.2f e2e %.4g" % (d["value"], d["ms_per_step"], d["e2e"]["value"]))
    for k,v in d["kernels"].items(): print(k, v)
except Exception as e: print("no bench", e)
PY
